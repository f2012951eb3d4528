# per-kernel device time of late sweeps (profile mode) and the plan stats
mkdir -p gpurun_out
for sw in 0 9 11 12; do
  echo "== sweep $sw"; HSVD_PROFILE_SWEEP=$sw timeout 300 python tools/profile_sweep.py 8192 2>&1 | tail -4
done
HSVD_PLAN_STATS=1 timeout 300 python bench.py --steps 1 --warmup 0 --no-cpu --no-accuracy 2>&1 | grep -i plan | tail -15
