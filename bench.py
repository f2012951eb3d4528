"""bench.py -- HSVD time-to-solution on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--n 8192] [--p n/2] [--mode pointwise|block]

A "step" is one complete HSVD solve (reference drive(), solver.py:179-269)
of the seeded synthetic factor of SURVEY.md §8(d) config 5: n = r = 8192,
G = default_rng(0).standard_normal, J = diag(+1 x p, -1 x (n-p)), p = n/2,
V^{-T} accumulated.  `value` = seconds per solve with G already in HBM
(timed with CUDA events, includes the D2D input copy the reference also
makes, solver.py:188); `e2e` = the same through the public numpy API
(drive(G_numpy, J)) with the host->device copy of G and the device->host
copies of U, V^{-T}, sigma, lambda inside the timed region.

--impl reference times the reference algorithm on the host CPU: the C
restatement in oracle/ (bit-exact with hjsvd, see tests/golden) with every
host thread, on a bounded sample of the same workload, extrapolated to a
full solve with the exact per-sweep rotation/skip counts (oracle/README).

One process per GPU (torchrun).  N>1 shards the block-column slots of one
solve over the N GPUs (paper_1008_1371_b200.sharded, NCCL ring exchange of
one block column per step); the time is the max over ranks and the scaling
is strong (the n=8192 problem is fixed).
"""

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

TELEMETRY_FILE = os.path.join(ROOT, "profiles", "reference_telemetry.json")
METRIC = "HSVD time-to-solution (s) fp64 n={n}"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--n", type=int, default=8192)
    ap.add_argument("--p", type=int, default=None)
    ap.add_argument("--mode", default="block", choices=["pointwise", "block"])
    ap.add_argument("--block-cols", type=int, default=32)
    ap.add_argument("--block-rotation", default="fast", choices=["fast", "dd"])
    ap.add_argument("--inner-ordering", default="full", choices=["oriented", "full"])
    ap.add_argument("--inner-passes", type=int, default=0)
    ap.add_argument("--block-streams", type=int, default=2)
    ap.add_argument("--cpu-sample-s", type=float, default=12.0)
    ap.add_argument("--e2e-steps", type=int, default=1)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-accuracy", action="store_true")
    ap.add_argument("--sharded", action="store_true",
                    help="use the sharded (NCCL) solver even on 1 GPU (checks that path)")
    a = ap.parse_args()
    if a.p is None:
        a.p = a.n // 2
    return a


def make_input(n, p, seed=0):
    from tests.golden.inputs import make_case_input
    G = make_case_input(n, n, seed, "gauss")
    signs = np.array([1] * p + [-1] * (n - p), np.int8)
    return G, signs


# ---------------------------------------------------------------- clocks


class ClockSampler:
    """nvidia-smi sampling DURING the timed region (B200_PROFILING.md)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-i", str(self.index), "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except (OSError, FileNotFoundError):
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm = [float(r[1]) for r in self.rows if len(r) >= 9 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if len(r) >= 9 and r[2].replace(".", "").isdigit()]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            if len(r) < 9:
                continue
            for name, v in zip(names, r[5:9]):
                if v.lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------- FP64 peak


def measure_fp64_peak(dev, n=8192, sustain_s=4.0):
    """The FP64 roofline denominators on THIS box, before the timed region:
    cuBLAS DGEMM n^3 (torch.matmul float64; the library's DMMA GEMM is the
    reference ceiling for k_update / k_gram).  burst = best single call of
    10 after warm-up; sustained = back-to-back calls for >= sustain_s
    seconds (the solve runs for seconds, so its kernels are compared with
    the sustained figure), with nvidia-smi clocks sampled during that loop."""
    import torch
    a = torch.randn(n, n, dtype=torch.float64, device=dev)
    b = torch.randn(n, n, dtype=torch.float64, device=dev)
    for _ in range(3):
        c = a @ b
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(10):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        c = a @ b
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    flop = 2.0 * n ** 3
    clk = ClockSampler(dev.index if dev.index is not None else 0)
    clk.start()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    calls = max(8, int(sustain_s / (best / 1e3)))
    e0.record()
    for _ in range(calls):
        c = a @ b
    e1.record()
    torch.cuda.synchronize()
    clocks = clk.stop()
    sus_ms = e0.elapsed_time(e1)
    del a, b, c
    torch.cuda.empty_cache()
    return {"burst_tflops": flop / (best / 1e3) / 1e12,
            "sustained_tflops": flop * calls / (sus_ms / 1e3) / 1e12,
            "sustained_s": sus_ms / 1e3, "dgemm_n": n, "clocks_sustained": clocks,
            "source": "cuBLAS DGEMM (torch.matmul float64) measured in this bench run"}


# ---------------------------------------------------------------- CPU legs


def cpu_threads():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


XL_GOLDEN = os.path.join(ROOT, "tests", "golden", "golden_xl.json")


def load_measured_reference(n, p):
    """The reference algorithm run to COMPLETION on the build host for this
    input (tests/golden/make_golden_xl.py: the oracle, bit-exact with
    hjsvd): telemetry, wall time and thread count, or None."""
    if not os.path.exists(XL_GOLDEN):
        return None
    with open(XL_GOLDEN) as f:
        for c in json.load(f)["cases"]:
            if c["n"] == n and c["r"] == n and c["p"] == p and c["kind"] == "gauss":
                return c
    return None


def load_reference_telemetry(n, p):
    """Per-sweep (rotations, skips) of the reference on this exact input:
    from the full reference run (golden_xl.json) when there is one, else
    from profiles/reference_telemetry.json (the pointwise GPU mode, which is
    bit-exact with the reference)."""
    c = load_measured_reference(n, p)
    if c is not None:
        return {"sweeps": c["sweeps_used"], "rotations": c["rotations"], "skips": c["skips"],
                "per_sweep": [[t[1], t[2]] for t in c["telemetry"]],
                "source": "full reference run on the build host (tests/golden/golden_xl.json)"}
    if os.path.exists(TELEMETRY_FILE):
        with open(TELEMETRY_FILE) as f:
            data = json.load(f)
        key = f"n{n}_p{p}"
        if key in data:
            return data[key]
    return None


def save_reference_telemetry(n, p, telemetry):
    data = {}
    if os.path.exists(TELEMETRY_FILE):
        with open(TELEMETRY_FILE) as f:
            data = json.load(f)
    data[f"n{n}_p{p}"] = {"sweeps": len(telemetry),
                          "rotations": sum(int(t[1]) for t in telemetry),
                          "skips": sum(int(t[2]) for t in telemetry),
                          "per_sweep": [[int(t[1]), int(t[2])] for t in telemetry],
                          "source": "pointwise GPU mode (bit-exact with hjsvd.drive)"}
    for path in (TELEMETRY_FILE, os.path.join(ROOT, "gpurun_out", "reference_telemetry.json")):
        if os.path.isdir(os.path.dirname(path)):
            with open(path, "w") as f:
                json.dump(data, f, indent=1)


def cpu_reference_estimate(G, signs, p, budget_s, threads, telemetry):
    """Time the reference algorithm (C restatement, oracle/) on the host:
    sample A = modulus steps of sweep 0 on G (nearly all pairs rotate),
    sample B = the same steps on an orthogonal factor (I, every pair skips).
    Each sample is timed at N and 2N steps and the MARGINAL cost of the
    second N steps is used (the first steps pay cold caches and page
    faults: 141 ms per step for 10 steps vs 53 ms marginal at 20->40 on the
    build host).  Per-visit costs c_rot, c_skip then price the exact
    rotation/skip counts of the full solve.  Validated against a full run on
    the build host (profiles/r02_cpu_estimate_validation.json)."""
    from oracle import oracle as O
    n, r = G.shape
    half = r // 2

    def marginal(M, frac):
        # warm marginal step cost from 4 -> 8 steps sizes the sample
        _, t4 = O.sample_steps(M, signs, p, 4, threads)
        _, t8 = O.sample_steps(M, signs, p, 8, threads)
        per = max((t8 - t4) / 4, t8 / 24, 1e-4)  # the 4->8 difference is noisy
        N = int(max(16, min(512, r // 2, frac * budget_s / (3 * per))))
        rot1, ta = O.sample_steps(M, signs, p, N, threads)
        rot2, tb = O.sample_steps(M, signs, p, 2 * N, threads)
        return N, rot2 - rot1, max(tb - ta, 1e-9), ta + tb

    steps_a, rot_a, ta, wa = marginal(G, 0.7)
    Id = np.asfortranarray(np.eye(n, r))
    steps_b, _, tb, wb = marginal(Id, 0.3)
    c_skip = tb / (steps_b * half)
    skip_a = steps_a * half - rot_a
    c_rot = max((ta - skip_a * c_skip) / max(rot_a, 1), c_skip)
    if telemetry is not None:
        rot = telemetry["rotations"]
        skip = telemetry["skips"]
        sweeps = telemetry["sweeps"]
        how = ("exact rotation/skip counts of this input ("
               + telemetry.get("source", "pointwise GPU mode") + ")")
    else:  # no telemetry yet: every visit of 14 sweeps rotates (upper bound)
        sweeps = 14
        rot, skip = sweeps * r * half, 0
        how = "assumed 14 sweeps, every visit rotating (upper bound)"
    est = rot * c_rot + skip * c_skip
    sample = (f"EXTRAPOLATED: oracle C restatement (bit-exact with hjsvd), {threads} threads: "
              f"marginal cost of steps {steps_a}..{2 * steps_a} of sweep 0 on G and "
              f"{steps_b}..{2 * steps_b} all-skip steps on I ({wa + wb:.1f} s sampled) -> "
              f"c_rot={c_rot*1e6:.2f} us, c_skip={c_skip*1e6:.2f} us "
              f"per pair visit; extrapolated with {how}: {rot} rotations + {skip} skips "
              f"over {sweeps} sweeps")
    return est, sample


def measured_full(n, p):
    """The measured full reference solve of this input (build host), reported
    beside the per-run extrapolation."""
    c = load_measured_reference(n, p)
    if c is None:
        return None
    out = {"wall_s": c["wall_s"], "threads": c["threads"], "sweeps": c["sweeps_used"],
           "solver": c["solver"], "host": "build container (8-core x86; not the GPU box)",
           "source": "tests/golden/golden_xl.json"}
    if "hjsvd" in c:
        out["stock_hjsvd"] = c["hjsvd"]
    return out


def run_reference(a, rank, world):
    """--impl reference: CPU time of the reference algorithm, rank 0 only."""
    if rank != 0:
        return
    G, signs = make_input(a.n, a.p)
    threads = cpu_threads()
    tele = load_reference_telemetry(a.n, a.p)
    vals = []
    sample = ""
    for _ in range(a.warmup if a.warmup < 1 else 1):
        cpu_reference_estimate(G, signs, a.p, 2.0, threads, tele)  # warm caches
    budget = max(6.0, min(a.cpu_sample_s, 150.0 / max(a.steps, 1)))
    for _ in range(a.steps):
        v, sample = cpu_reference_estimate(G, signs, a.p, budget, threads, tele)
        vals.append(v)
    v = float(np.mean(vals))
    line = {
        "impl": "reference", "metric": METRIC.format(n=a.n), "value": v, "unit": "s",
        "n_gpus": a.gpus, "steps": a.steps, "warmup": a.warmup,
        "ms_per_step": v * 1e3, "higher_is_better": False, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic: numpy default_rng(0).standard_normal((n,n)), J=diag(+1 x p, -1 x n-p)",
        "config": {"workload": f"n={a.n} p={a.p} full HSVD with V^-T (SURVEY.md §8(d) cfg 5)",
                   "n": a.n, "p": a.p},
        "cpu_baseline": {"value": v, "unit": "s", "cores": threads, "kind": "port",
                         "sample": sample,
                         "measured_full_solve": measured_full(a.n, a.p)},
        "e2e": {"value": v, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- GPU leg


def residuals(Gdev_orig_t, res, signs):
    """||U^T U - I||_F, ||V^T J V - J||_F/||V||^2, ||G - U S V^T||_F/||G||_F
    on the device in fp64 (torch matmul; validation only)."""
    import torch
    Ut = res.U  # (r, n): row c = column c of U
    r = Ut.shape[0]
    eye = torch.eye(r, dtype=torch.float64, device=Ut.device)
    dU = torch.linalg.norm(Ut @ Ut.t() - eye).item()
    out = {"dU": dU}
    if res.Vinv_t is not None:
        s = torch.as_tensor(signs.astype(np.float64), device=Ut.device)
        Vt_cols = res.Vinv_t  # row c = column c of V^{-T}
        V = (s[:, None] * Vt_cols.t() * s[None, :])  # V = J V^{-T} J (n x n, row-major)
        vjv = V.t() @ (s[:, None] * V) - torch.diag(s)
        out["VtJV"] = (torch.linalg.norm(vjv) / torch.linalg.norm(V) ** 2).item()
        US = Ut.t() * res.sigma[None, :]
        recon = US @ V.t()
        G = Gdev_orig_t.t()
        out["recon"] = (torch.linalg.norm(G - recon) / torch.linalg.norm(G)).item()
    return out


def run_ours(a, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    import paper_1008_1371_b200 as H

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    G, signs = make_input(a.n, a.p, seed=0)
    J = H.SignatureVector(signs, a.p)
    cfg = H.SolverConfig(mode=a.mode, block_cols=a.block_cols,
                         block_rotation=a.block_rotation, inner_ordering=a.inner_ordering,
                         inner_passes=a.inner_passes, block_streams=a.block_streams)
    if a.mode == "block" and a.n % (2 * a.block_cols):
        raise SystemExit("block mode needs n to be a multiple of 2*block_cols")
    sharded = world > 1 or a.sharded
    if sharded and a.mode != "block":
        raise SystemExit("--gpus N > 1 shards block mode only")
    G0 = torch.from_numpy(np.ascontiguousarray(G.T)).to(dev)  # (r, n) = col-major G
    Gw = torch.empty_like(G0)
    stream = torch.cuda.current_stream()
    comm = H.ShardComm() if sharded else None

    def solve(c=cfg):
        if sharded:  # every rank holds the full factor, solves its shard
            return H.drive_sharded_device(G0, J, c, comm)
        Gw.copy_(G0)
        return H.drive_device(Gw, J, c)

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # FP64 roofline denominators on this box (before the timed region)
    fp64 = measure_fp64_peak(dev) if a.mode == "block" else {}
    res = None
    for _ in range(a.warmup):
        res = solve()
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    clk = ClockSampler(local_rank)
    clk.start()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    launches = 0
    sweep_ms = []
    for _ in range(a.steps):
        res = solve()
        launches += res.gpu_launches
        sweep_ms.append(res.sweep_gpu_ms)
    res_timed = res
    ev1.record(stream)
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    clocks = clk.stop()
    ms = max_over_ranks(ev0.elapsed_time(ev1))
    ms_per_step = ms / a.steps
    value = ms_per_step / 1e3

    # ---- roofline of the dominant kernel ---------------------------------
    # One extra solve limited to sweep 0 in profile mode: CUDA events around
    # every launch on the library's launching stream (outside the timed run).
    n = r = a.n
    tele = res.telemetry
    pcfg = H.SolverConfig(mode=a.mode, block_cols=a.block_cols,
                          block_rotation=a.block_rotation, inner_ordering=a.inner_ordering,
                          inner_passes=a.inner_passes, max_sweeps=1, profile=True)
    prof = solve(pcfg)
    kp = prof.kernel_profile
    peaks = {}
    if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")):
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    traffic = {}
    if os.path.exists(os.path.join(ROOT, "profiles", "traffic.json")):
        traffic = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))
    if a.mode == "pointwise":
        t0 = prof.telemetry[0]
        # per rotated pair: read+write 2 G columns + 2 V columns; per skip:
        # read 2 G columns
        bytes_per_launch = (t0[1] * (32 * n + 32 * r) + t0[2] * 16 * n) / r
        avg_s = kp["step"]["ms"] / kp["step"]["launches"] / 1e3
        peak = float(peaks.get("hbm_gbs", 6650.0))
        achieved = bytes_per_launch / avg_s / 1e9
        tr = traffic.get(f"pointwise_n{n}")
        roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                    "frac": achieved / peak, "traffic": tr,
                    "kernel": "k_pointwise_step", "launch_avg_ms": avg_s * 1e3,
                    "alg_bytes_per_launch": bytes_per_launch,
                    "peak_source": "MEASURED_PEAKS.json hbm_gbs" if peaks else "fallback 6.65 TB/s"}
        if rank == 0 and a.n >= 1024:
            save_reference_telemetry(a.n, a.p, tele)
    else:
        b2 = 2 * a.block_cols
        nslots = n // b2 // world  # slots per launch on this rank
        fl = {"gram": 2.0 * n * b2 * b2 * nslots,          # A_P = G_P^T G_P per slot
              "update": 2.0 * (n + r) * b2 * b2 * nslots}  # [G_P; V_P] W_P per slot
        dom = max(("gram", "update"), key=lambda k: kp[k]["ms"])
        avg_s = kp[dom]["ms"] / kp[dom]["launches"] / 1e3
        # k_update runs inside a seconds-long solve: sustained denominator
        peak = float(fp64["sustained_tflops"])
        achieved = fl[dom] / avg_s / 1e12
        tot_ms = sum(v["ms"] for v in kp.values())
        solve_tflops = res.sweeps_used * 12.0 * n ** 3 / value / 1e12
        tr = traffic.get(f"{dom}_n{n}_b{a.block_cols}_N{world}",
                         traffic.get(f"{dom}_n{n}_b{a.block_cols}") if world == 1 else None)
        roofline = {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                    "frac": achieved / peak,
                    "traffic": tr["bytes_per_launch"] if isinstance(tr, dict) else tr,
                    "kernel": f"k_{dom}", "launch_avg_ms": avg_s * 1e3,
                    "alg_flop_per_launch": fl[dom],
                    "peak_source": ("sustained cuBLAS DGEMM 8192^3 on this box in this run "
                                    f"({fp64['sustained_s']:.1f} s loop); burst "
                                    f"{fp64['burst_tflops']:.2f} TFLOP/s"),
                    "peak_burst": fp64["burst_tflops"],
                    "frac_burst": achieved / fp64["burst_tflops"],
                    "fp64_peak_measurement": fp64,
                    "kernel_share_sweep0": {k: round(v["ms"] / tot_ms, 4) for k, v in kp.items()},
                    "kernel_ms_sweep0": {k: round(v["ms"], 3) for k, v in kp.items()},
                    "gram_tflops": fl["gram"] / (kp["gram"]["ms"] / kp["gram"]["launches"] / 1e3) / 1e12,
                    "update_tflops": fl["update"] / (kp["update"]["ms"] / kp["update"]["launches"] / 1e3) / 1e12,
                    "solve_alg_tflops": solve_tflops,
                    "solve_frac": solve_tflops / (peak * world),
                    "solve_frac_note": ("algorithmic: 12 n^3 flop per sweep x sweeps / time / "
                                        "(N x peak); late sweeps skip the updates of slots "
                                        "without rotations, so this can exceed 1")}
        if isinstance(tr, dict):
            roofline["traffic_source"] = tr.get("source")

    # ---- end to end through the public API, host buffers -------------------
    # 1 GPU: drive(G_numpy, J) (H2D of G, D2H of U, V^-T, sigma, lam inside).
    # N GPUs: every rank copies the factor in from pinned host memory, solves
    # its shard, and copies its own columns of U, V^-T, sigma, lam out.
    Gpin = torch.from_numpy(np.ascontiguousarray(G.T)).pin_memory() if sharded else None

    def e2e_call():
        if sharded:
            Gd = Gpin.to(dev, non_blocking=True)
            part = H.drive_sharded_device(Gd, J, cfg, comm)
            outs = []
            for t in (part.U_t, part.Vinv_t_t, part.sigma, part.lam):
                h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
                h.copy_(t, non_blocking=True)
                outs.append(h)
            torch.cuda.current_stream().synchronize()
            return sum(t.numel() * 8 for t in outs)  # this rank's columns
        H.drive(G, J, cfg)
        return (n * r + r * r + 2 * r) * 8

    e2e_call()  # untimed warm-up (page-locked host buffers, allocator caches)
    e2e_ms = []
    d2h = 0
    for _ in range(max(a.e2e_steps, 1)):
        torch.cuda.synchronize()
        barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record(stream)
        d2h = e2e_call()
        e1.record(stream)
        torch.cuda.synchronize()
        wall = (time.perf_counter() - t0) * 1e3
        e2e_ms.append(max(e0.elapsed_time(e1), wall))
    e2e_s = max_over_ranks(float(np.mean(e2e_ms)) / 1e3)
    h2d = world * (n * r * 8 + r)  # every rank copies the whole factor in
    if world > 1:  # all ranks' outputs together
        t = torch.tensor([float(d2h)], device=dev)
        dist.all_reduce(t)
        d2h = int(t.item())

    acc = None
    if not a.no_accuracy:
        if sharded:
            full = H.gather_result(solve(), n, r, to_numpy=False)
            full.U = full.U.t()  # back to the (r, n) convention of residuals()
            full.Vinv_t = full.Vinv_t.t()
            acc = residuals(G0, full, signs)
        else:
            res = solve()
            acc = residuals(G0, res, signs)

    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu:
        tel = load_reference_telemetry(a.n, a.p)
        est, sample = cpu_reference_estimate(G, signs, a.p, a.cpu_sample_s,
                                             cpu_threads(), tel)
        cpu = {"value": est, "unit": "s", "cores": cpu_threads(), "kind": "port",
               "sample": sample, "measured_full_solve": measured_full(a.n, a.p)}
    if comm is not None:
        comm.close()

    if rank == 0:
        line = {
            "metric": METRIC.format(n=a.n), "value": value, "unit": "s",
            "n_gpus": world, "steps": a.steps, "warmup": a.warmup,
            "ms_per_step": ms_per_step, "higher_is_better": False,
            "scaling": "strong",
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic: numpy default_rng(0).standard_normal((n,n)), J=diag(+1 x p, -1 x n-p)",
            "config": {"workload": f"n={a.n} p={a.p} full HSVD with V^-T (SURVEY.md §8(d) cfg 5)",
                       "n": a.n, "p": a.p, "mode": a.mode,
                       **({"block_cols": a.block_cols, "block_rotation": a.block_rotation,
                           "inner_ordering": a.inner_ordering,
                           "inner_passes": (a.inner_passes if a.inner_passes > 0 else
                                            "auto: 2 per step in the dense sweeps, 1 in the late ones"),
                           "block_streams": a.block_streams}
                          if a.mode == "block" else {}),
                       "parallelism": (f"{world} GPUs: block-column slots sharded, NCCL ring "
                                       "exchange per step" if sharded else "1 GPU"),
                       "l2": "inputs larger than L2 (G and V^-T are n*n*8 B each)"},
            "sweeps": res_timed.sweeps_used, "stop_reason": res_timed.stop_reason,
            "rotations": res_timed.rotations, "skips": res_timed.skips,
            "accuracy": acc,
            "roofline": roofline,
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_s, "unit": "s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h},
            "gpu_launches": launches,
            "host_phase_ms": res_timed.host_phase_ms,
            "clocks": clocks,
            "sweep_gpu_ms": [round(x, 3) for x in sweep_ms[-1]],
        }
        print(json.dumps(line), flush=True)


def main():
    # NCCL's version banner goes to stdout; keep stdout to the one JSON line
    os.environ.setdefault("NCCL_DEBUG", "WARN")
    a = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if a.impl == "reference":
        run_reference(a, rank, world)
        return
    dist_on = world > 1 or a.sharded
    if dist_on:
        import torch
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29531")
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", rank=rank, world_size=world,
                                device_id=torch.device("cuda", local_rank))
    try:
        run_ours(a, rank, world, local_rank)
    finally:
        if dist_on:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
