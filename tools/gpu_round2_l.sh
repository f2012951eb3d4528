mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for k in 0 8 10 12; do HSVD_PROFILE_SWEEP=$k python tools/profile_sweep.py 8192 2>&1 | grep kernel; done
