"""Benchmark: FD-apply GDOF/s (FP64, 3D) and preconditioned GMRES time-to-1e-8 on B200.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--n 256] [--impl {fdiga,reference}] [--no-gmres]

Headline (BASELINE.json metric, configs[3] at n=256 = the north-star target size):
  value = N / t_apply  [GDOF/s],  N = n^3,  t_apply = device time of one fd_apply (at n = 256: 6 int8-split
  tensor-core mode products, each a digit split + a tcgen05 GEMM, the eigenvalue divide in the split feeding
  the backward mode-3 product), inputs resident in HBM, CUDA events on the library's stream,
  max over ranks.  fp64_native: the same apply on the IEEE-FP64 DMMA path.
  The 134 MB input plus three 134 MB work buffers exceed the 126 MB L2, so no flush is needed.
Secondary (same JSON line):
  e2e       the same metric through fd_apply_host (pinned host buffers; H2D + apply + D2H timed per step)
  roofline  the dominant kernel's roofline: the int8 tensor-core GEMM (oz_gemm_kernel) on the int8-split path
            (n = 256 default), else the FP64 DMMA mode product; per-launch work / its own CUDA-event launch time
            against the DMMA peak measured on this pool (profiles/r01_peaks_fp64.jsonl)
  gmres     preconditioned GMRES(30) time-to-1e-8 on configs[1], [2], [4] (assembled on the device,
            b and x resident), iterations, and the stored-operator matvec HBM roofline on configs[4]
  cpu_baseline  the CPU oracle (numpy mode products) on the host cores, bounded sample
  clocks    NVML SM clock / throttle reasons sampled during the timed FD region
--impl reference: the oracle is the reference arm (no reference implementation exists).
"""
import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "FD-apply GDOF/s (FP64, 3D) & preconditioned GMRES time-to-1e-8 at 1/2/4/8 B200"
FP64_PEAK_FILE = os.path.join(ROOT, "profiles", "r01_peaks_fp64.jsonl")
NCU_SUMMARY = os.path.join(ROOT, "profiles", "r02_ncu_summary.json")


def fp64_peak():
    best = None
    with open(FP64_PEAK_FILE) as fh:
        for line in fh:
            rec = json.loads(line)
            if rec.get("kind") == "dmma_sustained":
                best = rec["tflops"]
    return best


# The paper's own numbers (context only, not a target): BiCGStab + FD iterations / CPU seconds including the
# preconditioner setup, Matlab R2015a on one core of an Intel Xeon i7-5820K at 3.30 GHz.
PAPER_CONTEXT = {
    "hardware": "Matlab R2015a (GeoPDEs, Tensorlab 3.0), one core of an Intel Xeon i7-5820K at 3.30 GHz (P:499)",
    "tolerance": "unstated (Matlab bicgstab default 1e-6, DESIGN.md reading 16); times include the FD setup (P:528)",
    "table2_collocation_quarter_ring_2d": {"h^-1=256,p=3": {"bicgstab_iters": 13.5, "seconds": 0.25},
                                           "h^-1=1024,p=3": {"bicgstab_iters": 13.5, "seconds": 10.18}},
    "table4_collocation_revolved_ring_3d": {"h^-1=64,p=3": {"bicgstab_iters": 19.5, "seconds": 1.04},
                                            "h^-1=64,p=5": {"bicgstab_iters": 22.5, "seconds": 3.12}},
    "comparable_here": "gmres.cfg2 (2D quarter annulus, 256^2 elements, p = 3) and gmres.cfg5 (3D thick ring, "
                       "128^3 elements, p = 5: 2.25M DOFs vs the paper's 3D h^-1 = 64), solved to 1e-8",
}


def int8_peak():
    """Dense int8 tensor-core peak: MEASURED_PEAKS.json's cuBLAS bf16 (burst) x the nominal int8/bf16 ratio
    (4.5 / 2.25 PFLOP/s, B200_PROFILING.md).  Our own tcgen05.mma.kind::i8 issue loop measured 4.55 POP/s
    (tools/tc/mma_rate.cu, profiles/r01_tc_int8_mma_rate.txt)."""
    try:
        return 2.0 * json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["bf16_tflops"], \
            "2 x MEASURED_PEAKS.json bf16_tflops (nominal int8/bf16 ratio)"
    except Exception:
        return 4500.0, "fallback nominal 4.5 POP/s dense int8"


def roofline(path, kern, flops, int8_ops, achieved_fp64, fp64_pk, traffic, ws):
    """The dominant kernel's roofline.  DMMA path: dmma_gemm_kernel, FP64 tensor, 4 N n_l flop per launch.
    int8 path: oz_gemm_kernel, int8 tensor, 2 M N K ops per digit-pair MMA (34 pairs per mode product)."""
    fp64_eq = {"achieved": achieved_fp64, "peak": fp64_pk, "unit": "TFLOP/s", "frac": achieved_fp64 / fp64_pk,
               "what": "whole FD apply: 4 N sum(n_l) FP64 flop / apply time, against the FP64 (DMMA) peak"}
    if path == "int8_split" and kern and "int8_gemm" in kern:
        g = kern["int8_gemm"]
        ach = int8_ops / g["launches_per_apply"] / (g["avg_ms"] * 1e-3) / 1e12
        pk, src = int8_peak()
        return {"bound": "tensor", "achieved": ach, "peak": pk, "unit": "TOP/s (int8)", "frac": ach / pk,
                "traffic": traffic.get("oz_gemm") if isinstance(traffic, dict) else None,
                "kernel": f"oz_gemm_kernel (tcgen05.mma.kind::i8, {g['launches_per_apply']} launches per apply, "
                          f"{100 * g['share']:.0f}% of the apply; the other steps under 'kernels')",
                "int8_ops_per_apply": int8_ops, "avg_launch_ms": g["avg_ms"], "peak_source": src,
                # context: our own back-to-back tcgen05.mma.kind::i8 issue loop (profiles/r01_tc_int8_mma_rate.txt)
                "probe_peak": 4550.0, "frac_of_probe": ach / 4550.0,
                "kernels": kern, "fp64_equivalent": fp64_eq}
    if kern and "dmma" in kern:
        g = kern["dmma"]
        ach = flops / g["launches_per_apply"] / (g["avg_ms"] * 1e-3) / 1e12
    else:
        ach = achieved_fp64
    return {"bound": "tensor", "achieved": ach, "peak": fp64_pk, "unit": "TFLOP/s", "frac": ach / fp64_pk,
            "traffic": (traffic["dmma"] / 6 if isinstance(traffic, dict) and traffic.get("dmma") else None),
            "kernel": "dmma_gemm_kernel (6 launches per apply: 3 forward + 3 backward mode products)"
                      + (", per GPU" if ws > 1 else ""),
            "flops_per_apply": flops,
            "peak_source": "own DMMA.8x8x4 register loop, sustained 3 s (profiles/r01_peaks_fp64.jsonl); "
                           "MEASURED_PEAKS.json has no FP64 entry",
            "kernels": kern, "fp64_equivalent": fp64_eq}


def hbm_peak():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"], "MEASURED_PEAKS.json hbm_gbs"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """NVML sampling of SM clock and throttle reasons while the timed region runs."""

    def __init__(self, index, period=0.01):
        self.index, self.period = index, period
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        self._thr = None

    def __enter__(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            self._nv = nv
            self._h = nv.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = nv.nvmlDeviceGetMaxClockInfo(self._h, nv.NVML_CLOCK_SM)
        except Exception:
            self._nv = None
            return self
        names = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
                 "sw_power_cap": 0x4, "hw_power_brake_slowdown": 0x80}

        def run():
            while not self._stop.is_set():
                try:
                    self.samples.append(self._nv.nvmlDeviceGetClockInfo(self._h, self._nv.NVML_CLOCK_SM))
                    fn = getattr(self._nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                        getattr(self._nv, "nvmlDeviceGetCurrentClocksThrottleReasons")
                    r = fn(self._h)
                    for k, bit in names.items():
                        if r & bit:
                            self.reasons.add(k)
                except Exception:
                    pass
                time.sleep(self.period)
        self._thr = threading.Thread(target=run, daemon=True)
        self._thr.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._thr:
            self._thr.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0}
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def dist_init():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def weak_shape(n, ws):
    """Weak-scaling FD family: N/P fixed at n^3; directions doubled from the last one
    (P = 1, 2, 4, 8 -> (n,n,n), (n,n,2n), (n,2n,2n), (2n,2n,2n)); other P stretch the last axis."""
    if ws & (ws - 1) == 0 and ws <= 8:
        k = ws.bit_length() - 1
        return tuple(n * (2 if l >= 3 - k else 1) for l in range(3))
    return (n, n, n * ws)


def cpu_fd_sample(n, budget_s=12.0, max_reps=20):
    """Oracle FD apply (numpy mode products, all host BLAS threads) on cfg4 factors: GDOF/s."""
    from oracle import fastdiag
    from synth import fd_sweep_factors, fd_sweep_vector
    rng, U, lam = fd_sweep_factors(n)
    f = fastdiag.factors_from_eig(U, lam)
    x = fd_sweep_vector(rng, n ** 3)
    fastdiag.apply(f, x)  # warm-up
    times = []
    t_start = time.perf_counter()
    while len(times) < max_reps and time.perf_counter() - t_start < budget_s:
        t0 = time.perf_counter()
        fastdiag.apply(f, x)
        times.append(time.perf_counter() - t0)
    try:
        from threadpoolctl import threadpool_info
        threads = max([p.get("num_threads", 1) for p in threadpool_info()] + [1])
    except Exception:
        threads = os.cpu_count()
    t = float(np.median(times))
    return dict(value=n ** 3 / t / 1e9, unit="GDOF/s", cores=threads, kind="oracle",
                sample=f"{len(times)} oracle FD applies (numpy mode products) at n={n}, median {t * 1e3:.1f} ms/apply; "
                       f"host has {os.cpu_count()} logical cores", seconds_per_apply=t)


def cpu_fd_sample_1thread(n=128, budget_s=8.0):
    """The oracle FD apply on ONE host thread (threadpoolctl), the closest analogue of the paper's single
    core, at a size whose apply takes about a second."""
    try:
        from threadpoolctl import threadpool_limits
    except Exception:
        return None
    with threadpool_limits(limits=1):
        r = cpu_fd_sample(n, budget_s=budget_s, max_reps=10)
    r["cores"] = 1
    r["sample"] = r["sample"].replace("host has", "1 BLAS thread (threadpoolctl); host has")
    return r


def cpu_gmres_sample(budget_s=45.0):
    """The oracle's FD-preconditioned GMRES(30) (oracle/krylov.py, oracle/fastdiag.py, oracle's sum-factorised
    matvec) on the host cores: full solves for configs[0..2]; configs[4] timed over its first few Arnoldi steps
    (ms per iteration, extrapolated to the GPU's iteration count in `est_total_s`)."""
    from oracle import assembly, fastdiag, krylov
    from synth import get_config, rhs
    out = {}
    t_all = time.perf_counter()
    for cfg in (1, 2, 3, 5):
        c = get_config(cfg)
        t0 = time.perf_counter()
        disc = assembly.Discretisation(c.d, c.p, c.ne, c.geometry, c.geo_params)
        f = fastdiag.setup([disc.M] * c.d, [disc.K] * c.d)
        t_setup = time.perf_counter() - t0
        b = rhs(cfg, disc.N)
        cap = 3 if cfg == 5 else 1000
        t0 = time.perf_counter()
        _, rep = krylov.gmres(disc.matvec, b, precond=lambda v: fastdiag.apply(f, v), max_iters=cap)
        dt = time.perf_counter() - t0
        e = {"N": disc.N, "iters": rep["iters"], "setup_s": t_setup, "solve_s": dt,
             "ms_per_iter": dt / max(1, rep["iters"]) * 1e3}
        if cfg == 5:
            e["note"] = f"first {rep['iters']} Arnoldi steps only (bounded sample)"
        out[f"cfg{cfg}"] = e
        if time.perf_counter() - t_all > budget_s:
            break
    return out


def run_reference(args):
    """The reference arm: the CPU oracle (numpy mode products) on this box's host cores, on the same
    workload as our arm (the n^3 apply at every N), rank 0 only.  Steps are capped so that the run
    stays within ~1 minute of CPU work (a bounded sample; the JSON says how many applies were timed)."""
    ws, rank, _ = dist_init()
    if rank != 0:
        return
    n = args.n
    ns = (n, n, n)
    N = int(np.prod(ns))
    from oracle import fastdiag
    from synth import fd_sweep_factors, fd_sweep_vector
    rng, U, lam = fd_sweep_factors(ns)
    f = fastdiag.factors_from_eig(U, lam)
    x = fd_sweep_vector(rng, N)
    t0 = time.perf_counter()
    fastdiag.apply(f, x)
    t_one = time.perf_counter() - t0
    warm = max(0, min(args.warmup, int(20.0 / max(t_one, 1e-3))) - 1)
    for _ in range(warm):
        fastdiag.apply(f, x)
    steps = max(1, min(args.steps, int(60.0 / max(t_one, 1e-3))))
    t0 = time.perf_counter()
    for _ in range(steps):
        fastdiag.apply(f, x)
    dt = (time.perf_counter() - t0) / steps
    try:
        from threadpoolctl import threadpool_info
        threads = max([p.get("num_threads", 1) for p in threadpool_info()] + [1])
    except Exception:
        threads = os.cpu_count()
    val = N / dt / 1e9
    shape = "x".join(map(str, ns))
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": val, "unit": "GDOF/s", "n_gpus": ws, "steps": steps,
        "warmup": warm + 1, "ms_per_step": dt * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": arm_config(ns, ws),
        "cpu_baseline": {"value": val, "unit": "GDOF/s", "cores": threads, "kind": "oracle",
                         "sample": f"{steps} oracle FD applies at {shape} after {warm + 1} warm-up "
                                   f"(requested --steps {args.steps}; capped at ~60 s of CPU work)"},
        "e2e": {"value": val, "unit": "GDOF/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def arm_config(ns, ws):
    """The workload's config dict, identical for both arms (the driver compares them)."""
    n = ns[0]
    return {"workload": f"cfg4 FD apply P^-1 r, d=3, n={'x'.join(map(str, ns))} (BASELINE.json configs[3]"
                        + (f", slab-sharded over {ws} GPUs)" if ws > 1 else ")"),
            "n": n, "shape": list(ns), "N": int(np.prod(ns)),
            "factors": "U ~ N(0,1), lam ~ U(1,100), W = U^-1, x ~ N(0,1)",
            "l2": "inputs > L2: 134 MB vector + 3 x 134 MB work buffers per GPU vs 126 MB L2" if n >= 256
            else "vector fits in L2 (no flush)",
            "parallelism": f"slab-sharded over {ws} GPUs (NCCL all-to-all in the mode-d pass)" if ws > 1
            else "single GPU"}


def fd_kernels(fd, plan, x, s, reps=5):
    """Per-kernel CUDA-event durations of reps applies (fd_apply_timed): launches per apply, avg ms, share."""
    per = {}
    for _ in range(reps):
        for kind, kms in fd.fd_apply_timed(plan, x, s):
            per.setdefault(kind, []).append(kms)
    tot = sum(sum(v) for v in per.values())
    return {k: {"launches_per_apply": len(v) // reps, "avg_ms": float(np.mean(v)), "share": sum(v) / tot}
            for k, v in per.items()}


def timed(fn, stream, steps, warmup, sync_all=None):
    import torch
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    if sync_all:
        sync_all()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        fn()
    e1.record(stream)
    e1.synchronize()
    torch.cuda.synchronize()
    if sync_all:
        sync_all()
    return e0.elapsed_time(e1) / steps


def gmres_section(ctx, fd, steps, ws=1, rank=0, sharded=False):
    """GMRES(30) time-to-1e-8 on configs[1], [2], [4] (single GPU) or, sharded over ws > 1 ranks, on the
    3D configs [2] and [4] (2D problems run as replicas only).  Device time, max over ranks."""
    import torch
    import torch.distributed as dist
    from synth import get_config, rhs
    out = {}
    dev = torch.device("cuda", torch.cuda.current_device())
    hbm, hbm_src = hbm_peak()

    def gmax(v):
        if ws == 1:
            return v
        t = torch.tensor([v], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    for cfg in ((3, 5) if sharded else (2, 3, 5)):
        c = get_config(cfg)
        A = fd.colloc_assemble(ctx, c.d, c.p, c.ne, c.geometry, c.geo_params)
        M, K = fd.colloc_1d_factors(c.p, c.ne)
        # setup timed three times (the first one in a process also pays cuSOLVER's one-time initialisation)
        setups = []
        for _ in range(3):
            t0 = time.perf_counter()
            P = fd.fd_setup(ctx, [M] * c.d, [K] * c.d)
            setups.append(time.perf_counter() - t0)
            if len(setups) < 3:
                P.close()
        t_setup = float(np.median(setups))
        lo = A.slab[0] * A.n[0] * A.n[1]
        b = torch.from_numpy(rhs(cfg, A.N_global)[lo:lo + A.N].copy()).to(dev)
        x = torch.empty_like(b)
        rep = fd.gmres_solve(ctx, A, P, b, x)  # warm-up (captures the cycle graph)
        times, iters = [], []
        for _ in range(max(3, min(steps, 10))):
            rep = fd.gmres_solve(ctx, A, P, b, x)
            times.append(gmax(rep["t_total_ms"]))
            iters.append(rep["iters"])
        # the paper's own solver on the same system: BiCGStab + FD, half-iteration counts
        brep = fd.bicgstab_solve(ctx, A, P, b, x)  # warm-up (captures the chunk graph)
        btimes = []
        for _ in range(max(3, min(steps, 10))):
            brep = fd.bicgstab_solve(ctx, A, P, b, x)
            btimes.append(gmax(brep["t_total_ms"]))
        bicg = {"time_to_tol_ms": float(np.median(btimes)), "iters": brep["iters"],
                "rel_res_true": brep["rel_res_true"]}
        # per-stage breakdown from one profiled solve (eagerly launched cycles, a CUDA event at every stage
        # change; include/fdiga.h gmres_report.t_*_ms), max over ranks per stage
        prof = fd.gmres_solve(ctx, A, P, b, x, profile=True)
        stages = {k: gmax(prof[k]) for k in ("t_fd_ms", "t_matvec_ms", "t_orth_ms", "t_comm_ms", "t_other_ms")}
        stages["t_total_ms"] = gmax(prof["t_total_ms"])
        stages["note"] = "one profiled solve (eager launches, events at stage changes); fractions apply to time_to_tol_ms"
        t_solve = float(np.median(times))
        entry = {"time_to_tol_ms": t_solve, "iters": int(np.median(iters)),
                 "rel_res_true": rep["rel_res_true"], "n": A.n[0], "N": A.N_global, "fd_setup_ms": t_setup * 1e3,
                 "fd_setup_first_ms": setups[0] * 1e3,
                 "paper_style_total_ms": t_setup * 1e3 + t_solve,
                 "paper_style_note": "setup (1D eigendecompositions, factor upload) + solve, as the paper's times (P:528)",
                 "ms_per_iter": t_solve / max(1, int(np.median(iters))), "ranks": ws,
                 "breakdown": stages, "bicgstab": bicg}
        if c.d == 3:
            # the same solves with the matrix-free sum-factorised operator (NEXT-1, no stored values)
            Amf = fd.colloc_assemble(ctx, c.d, c.p, c.ne, c.geometry, c.geo_params, matrix_free=True)
            fd.gmres_solve(ctx, Amf, P, b, x)
            mt, mi = [], []
            for _ in range(max(3, min(steps, 10))):
                r2 = fd.gmres_solve(ctx, Amf, P, b, x)
                mt.append(gmax(r2["t_total_ms"]))
                mi.append(r2["iters"])
            fd.bicgstab_solve(ctx, Amf, P, b, x)
            bt2 = []
            for _ in range(max(3, min(steps, 10))):
                b2 = fd.bicgstab_solve(ctx, Amf, P, b, x)
                bt2.append(gmax(b2["t_total_ms"]))
            entry["matrix_free"] = {"gmres_time_to_tol_ms": float(np.median(mt)), "gmres_iters": int(np.median(mi)),
                                    "gmres_rel_res_true": r2["rel_res_true"],
                                    "bicgstab_time_to_tol_ms": float(np.median(bt2)), "bicgstab_iters": b2["iters"]}
            if cfg == 5:
                stream = torch.cuda.current_stream()
                xv = torch.randn(A.N, dtype=torch.float64, device=dev)
                yv = torch.empty_like(xv)
                sync = (lambda: dist.barrier()) if ws > 1 else None
                entry["matrix_free"]["matvec_ms"] = gmax(timed(lambda: fd.stencil_matvec(Amf, xv, yv), stream, 20, 3,
                                                               sync))
            Amf.close()
        if cfg == 5:
            # stored-operator matvec roofline (HBM): bytes = 8 nnz + 16 N (this rank's rows)
            stream = torch.cuda.current_stream()
            xv = torch.randn(A.N, dtype=torch.float64, device=dev)
            yv = torch.empty_like(xv)
            sync = (lambda: dist.barrier()) if ws > 1 else None
            ms = gmax(timed(lambda: fd.stencil_matvec(A, xv, yv), stream, 20, 3, sync))
            byts = 8 * A.nnz + 16 * A.N
            entry["matvec"] = {"ms": ms, "nnz": A.nnz, "bytes": byts, "achieved_gbs": byts / ms / 1e6,
                               "peak_gbs": hbm, "peak_source": hbm_src, "frac": byts / ms / 1e6 / hbm,
                               "per": "rank" if ws > 1 else "gpu"}
            fd_flops = P.flops()
            ms_fd = gmax(timed(lambda: fd.fd_apply(P, xv, yv), stream, 20, 3, sync))
            entry["fd_apply"] = {"ms": ms_fd, "tflops": fd_flops / ms_fd / 1e9}
        out[f"cfg{cfg}"] = entry
        P.close()
        A.close()
    # NEXT-3: weighted-quadrature Galerkin systems (synth configs 8, 9), symmetric FD of the Galerkin pencils
    for cfg in ((9,) if sharded else (8, 9)):
        c = get_config(cfg)
        A = fd.wq_assemble(ctx, c.d, c.p, c.ne, c.geometry, c.geo_params)
        M, K = fd.galerkin_1d_factors(c.p, c.ne)
        P = fd.fd_setup(ctx, [M] * c.d, [K] * c.d)
        lo = A.slab[0] * A.n[0] * A.n[1]
        b = torch.from_numpy(rhs(cfg, A.N_global)[lo:lo + A.N].copy()).to(dev)
        x = torch.empty_like(b)
        fd.gmres_solve(ctx, A, P, b, x)
        tg, tb = [], []
        for _ in range(3):
            rg = fd.gmres_solve(ctx, A, P, b, x)
            tg.append(gmax(rg["t_total_ms"]))
            rb = fd.bicgstab_solve(ctx, A, P, b, x)
            tb.append(gmax(rb["t_total_ms"]))
        out[f"cfg{cfg}_wq"] = {"N": A.N_global, "p": c.p, "ne": c.ne, "nnz_stored": A.nnz,
                               "gmres": {"time_to_tol_ms": float(np.median(tg)), "iters": rg["iters"]},
                               "bicgstab": {"time_to_tol_ms": float(np.median(tb)), "iters": rb["iters"]}}
        P.close()
        A.close()
    # NEXT-4: convection-diffusion on the cfg5 geometry (synth configs 6, 7), matrix-free operator, GMRES(30)
    # with the wind-aware FD (collocation analogue of eq:convec_prec_2; complex pairs at cfg 6) and, for
    # comparison, the plain Laplacian FD (eq:convec_prec_1)
    for cfg in (6, 7):
        c = get_config(cfg)
        A = fd.colloc_assemble(ctx, 3, c.p, c.ne, c.geometry, c.geo_params, matrix_free=True, wind=c.wind,
                               wind_params=c.wind_params)
        M, K = fd.colloc_1d_factors(c.p, c.ne)
        H2 = fd.colloc_1d_convection(c.p, c.ne, 2 * c.wind_params[0] / np.pi)
        try:
            Pw = fd.fd_setup(ctx, [M] * 3, [K, K + H2, K], allow_complex_pairs=True, cond_max=1e30)
        except fd.FdigaError as e:  # complex-pair FD is single-rank
            out[f"cfg{cfg}_convection"] = {"skipped": str(e)[:120]}
            A.close()
            continue
        P0 = fd.fd_setup(ctx, [M] * 3, [K] * 3)
        lo = A.slab[0] * A.n[0] * A.n[1]
        b = torch.from_numpy(rhs(cfg, A.N_global)[lo:lo + A.N].copy()).to(dev)
        x = torch.empty_like(b)
        fd.gmres_solve(ctx, A, Pw, b, x, max_iters=300)
        tw = []
        for _ in range(3):
            rw = fd.gmres_solve(ctx, A, Pw, b, x, max_iters=300)
            tw.append(gmax(rw["t_total_ms"]))
        r0 = fd.gmres_solve(ctx, A, P0, b, x, max_iters=300, raise_on_nonconvergence=False)
        out[f"cfg{cfg}_convection"] = {
            "omega": c.wind_params[0], "ne": c.ne, "N": A.N_global,
            "wind_fd": {"time_to_tol_ms": float(np.median(tw)), "iters": rw["iters"], "converged": rw["converged"],
                        "complex_pairs": bool(np.any(Pw.factors(1)[3] != 0))},
            "plain_fd": {"time_ms": gmax(r0["t_total_ms"]), "iters": r0["iters"], "converged": r0["converged"]}}
        Pw.close()
        P0.close()
        A.close()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--n", type=int, default=256)
    ap.add_argument("--impl", default="fdiga", choices=["fdiga", "reference"])
    ap.add_argument("--no-gmres", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-weak", action="store_true")
    ap.add_argument("--no-sweep", action="store_true")
    ap.add_argument("--weak", action="store_true", help="also run the weak-scaling section at N = 1 (tests)")
    ap.add_argument("--sharded", action="store_true",
                    help="at --gpus 1: run the slab-sharded path over a one-rank NCCL communicator (tests the N>1 code)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist
    import paper_1705_04384_b200 as fd
    from synth import fd_sweep_factors, fd_sweep_vector

    ws, rank, local = dist_init()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    uid = None
    if ws == 1 and args.sharded:
        uid = fd.nccl_unique_id()
    if ws > 1:
        # NCCL prints each communicator's rank / nranks at init (the driver checks the communicator size)
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        dist.init_process_group("nccl", init_method="env://", device_id=dev)
        # the library's own NCCL communicator: rank 0 draws the unique id, torch.distributed carries it
        t = torch.zeros(128, dtype=torch.uint8, device=dev)
        if rank == 0:
            t.copy_(torch.tensor(list(fd.nccl_unique_id()), dtype=torch.uint8))
        dist.broadcast(t, 0)
        uid = bytes(t.cpu().tolist())

    def sync_all():
        if ws > 1:
            dist.barrier()

    stream = torch.cuda.current_stream()
    ctx = fd.Context(local, stream=stream.cuda_stream, nranks=ws, rank=rank, nccl_unique_id=uid)
    n = args.n
    # every N applies the same n^3 FD (strong scaling; the driver computes the efficiency from the values);
    # the weak-scaling family of SURVEY.md §8(d) is reported beside it (flop-rate efficiency)
    ns = (n, n, n)
    N = int(np.prod(ns))
    # setup (not timed): W_l = U_l^{-1} on the device (fd_setup_from_eig, M = I), BASELINE.json configs[3]
    rng, U, lam = fd_sweep_factors(ns)
    plan = fd.fd_setup_from_eig(ctx, U, lam)
    if ws == 1:
        x = torch.from_numpy(fd_sweep_vector(rng, N)).to(dev)
    else:  # this rank's slab, N(0,1) drawn on the device (the full vector is never formed)
        g = torch.Generator(device=dev)
        g.manual_seed(4000 + rank)
        x = torch.randn(plan.N, dtype=torch.float64, device=dev, generator=g)
    s = torch.empty_like(x)

    launches0 = ctx.kernel_launches()
    for _ in range(args.warmup):
        fd.fd_apply(plan, x, s)
    torch.cuda.synchronize()
    sync_all()
    launches0 = ctx.kernel_launches()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        torch.cuda.profiler.start()  # ncu --profile-from-start off captures exactly the timed steps
        e0.record(stream)
        for _ in range(args.steps):
            fd.fd_apply(plan, x, s)
        e1.record(stream)
        e1.synchronize()
        torch.cuda.profiler.stop()
    torch.cuda.synchronize()
    sync_all()
    launches = ctx.kernel_launches() - launches0
    ms = e0.elapsed_time(e1) / args.steps
    if ws > 1:
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = N / (ms * 1e-3) / 1e9           # all ranks' DOFs / max-over-ranks time
    flops = plan.flops()                     # whole apply (all ranks)
    peak = fp64_peak()
    achieved = flops / ws / (ms * 1e-3) / 1e12   # per GPU (FP64-equivalent rate of the whole apply)
    path, int8_ops = plan.path()
    # per-kernel durations of the apply (CUDA events after every launch on the ctx stream, single rank):
    # the dominant kernel's roofline is its own algorithmic work / its own average launch time
    # every rank (fd_apply_timed is collective on sharded plans); rank 0's durations are reported
    # (after a pause: the int8 path reaches the 1000 W power cap after ~0.1 s of back-to-back applies and the SM
    # clock drops; the timed region above and these per-kernel durations are the burst regime, `sustained` below
    # the power-capped one)
    time.sleep(0.5)
    kern = fd_kernels(fd, plan, x, s)
    if "split" in kern:  # the digit splits are HBM-bound: 8 N bytes read + 7 N written per launch
        hb, hsrc = hbm_peak()
        sb = 15.0 * N / ws
        kern["split"].update({"bound": "hbm", "algorithmic_bytes_per_launch": sb,
                              "achieved_gbs": sb / (kern["split"]["avg_ms"] * 1e-3) / 1e9, "peak_gbs": hb,
                              "frac": sb / (kern["split"]["avg_ms"] * 1e-3) / 1e9 / hb, "peak_source": hsrc})

    # the same apply with IEEE FP64 dot products only (DMMA mode products, no int8 splitting)
    fp64_native = None
    if path != "dmma":
        plan.set_path("dmma")
        ms64 = timed(lambda: fd.fd_apply(plan, x, s), stream, max(5, min(args.steps, 20)), 3, sync_all)
        if ws > 1:
            t = torch.tensor([ms64], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms64 = float(t.item())
        k64 = fd_kernels(fd, plan, x, s)
        plan.set_path(path)
        d = k64.get("dmma")
        ach = flops / ws / d["launches_per_apply"] / (d["avg_ms"] * 1e-3) / 1e12 if d else None
        fp64_native = {"value": N / (ms64 * 1e-3) / 1e9, "unit": "GDOF/s", "ms_per_apply": ms64, "path": "dmma",
                       "apply_tflops_per_gpu": flops / ws / (ms64 * 1e-3) / 1e12,
                       "roofline": {"bound": "tensor", "achieved": ach, "peak": peak, "unit": "TFLOP/s",
                                    "frac": ach / peak if ach else None, "kernel": "dmma_gemm_kernel (DMMA.8x8x4)",
                                    "peak_source": "own DMMA register loop, sustained (profiles/r01_peaks_fp64.jsonl)"},
                       "kernels": k64}

    # the same apply under sustained load (single GPU): ~0.7 s of back-to-back applies first, then 200 timed ones
    sustained = None
    if ws == 1 and not args.no_sweep:
        with ClockSampler(local) as clk_s:
            for _ in range(600):
                fd.fd_apply(plan, x, s)
            ms_s = timed(lambda: fd.fd_apply(plan, x, s), stream, 200, 0, sync_all)
            k_s = fd_kernels(fd, plan, x, s, reps=3)
        sustained = {"value": N / (ms_s * 1e-3) / 1e9, "unit": "GDOF/s", "ms_per_apply": ms_s, "path": path,
                     "applies_before": 600, "timed_applies": 200, "kernels": k_s, "clocks": clk_s.summary(),
                     "note": "back-to-back applies for ~1 s; the int8 tensor-core path runs into the board's power "
                             "cap (sw_power_cap) and a lower SM clock, the headline `value` is the first "
                             "warmup + steps applies after idle"}
        time.sleep(1.0)

    # e2e: same metric through the C ABI with pinned host buffers (H2D + apply + D2H per step)
    xh = torch.from_numpy(np.random.default_rng(4001 + rank).standard_normal(plan.N)).pin_memory()
    sh = torch.empty(plan.N, dtype=torch.float64).pin_memory()
    xh_np, sh_np = xh.numpy(), sh.numpy()
    e2e_steps = max(3, min(args.steps, 20))
    for _ in range(2):
        fd.fd_apply_host(plan, xh_np, sh_np)
    sync_all()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        fd.fd_apply_host(plan, xh_np, sh_np)
    e2e_sync_ms = (time.perf_counter() - t0) / e2e_steps * 1e3
    # streaming: every step still copies its input in and its result out, but consecutive steps overlap
    # (H2D of step k+1, apply of step k, D2H of step k-1; double-buffered inside the library)
    for _ in range(2):
        fd.fd_apply_host_async(plan, xh_np, sh_np)
    fd.fd_host_sync(plan)
    sync_all()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        fd.fd_apply_host_async(plan, xh_np, sh_np)
    fd.fd_host_sync(plan)
    e2e_ms = (time.perf_counter() - t0) / e2e_steps * 1e3
    e2e_per_rank = [e2e_ms]
    if ws > 1:
        t = torch.zeros(ws, device=dev, dtype=torch.float64)
        t[rank] = e2e_ms
        dist.all_reduce(t)
        e2e_per_rank = [float(v) for v in t.cpu().tolist()]
        e2e_ms = max(e2e_per_rank)

    weak = None
    if (ws > 1 or args.weak) and not args.no_weak:
        # weak-scaling family: N / P fixed at n^3, directions doubled from the last one.
        # Flop-rate efficiency against this GPU's own single-rank n^3 apply (FD work per DOF grows with the
        # factor sizes, so GDOF/s is not comparable across the family)
        wns = weak_shape(n, ws)
        rngw, Uw, lamw = fd_sweep_factors(wns)
        plan_w = fd.fd_setup_from_eig(ctx, Uw, lamw)
        gw = torch.Generator(device=dev)
        gw.manual_seed(5000 + rank)
        xw = torch.randn(plan_w.N, dtype=torch.float64, device=dev, generator=gw)
        sw = torch.empty_like(xw)
        ms_w = timed(lambda: fd.fd_apply(plan_w, xw, sw), stream, max(3, min(args.steps, 10)), 2, sync_all)
        if ws > 1:
            t = torch.tensor([ms_w], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms_w = float(t.item())
        ctx1 = fd.Context(local, stream=stream.cuda_stream)  # single-rank reference on this GPU
        plan_1 = fd.fd_setup_from_eig(ctx1, U, lam)
        x1 = torch.randn(N, dtype=torch.float64, device=dev, generator=gw)
        s1 = torch.empty_like(x1)
        ms_1 = timed(lambda: fd.fd_apply(plan_1, x1, s1), stream, max(3, min(args.steps, 10)), 2)
        tf_1 = plan_1.flops() / ms_1 / 1e9
        tf_w = plan_w.flops() / ws / ms_w / 1e9
        weak = {"shape": list(wns), "N": int(np.prod(wns)), "ms_per_apply": ms_w,
                "GDOF_per_s": float(np.prod(wns)) / ms_w / 1e6, "tflops_per_gpu": tf_w,
                "single_gpu_tflops_n3": tf_1, "flop_rate_efficiency": tf_w / tf_1}
        plan_1.close()
        ctx1.close()
        plan_w.close()
        del x1, s1, xw, sw
    traffic = None  # dram bytes per launch of the dominant kernel, from the committed ncu --set full summary
    if os.path.exists(NCU_SUMMARY):
        try:
            js = json.load(open(NCU_SUMMARY))
            traffic = {"dmma": js.get("fd_apply_dram_bytes_per_apply"), "oz_gemm": js.get("oz_gemm_dram_bytes_per_launch")}
        except Exception:
            traffic = None

    gm = None
    if not args.no_gmres:
        gm = gmres_section(ctx, fd, args.steps, ws, rank, sharded=uid is not None)
    sweep = None
    if ws == 1 and not args.no_sweep:
        # the rest of the configs[3] sweep (n in {128, 256, 512}; 256 is the headline): default path and DMMA
        sweep = {}
        for nn in (128, 512):
            nss = (nn, nn, nn)
            rng2, U2, lam2 = fd_sweep_factors(nss)
            p2 = fd.fd_setup_from_eig(ctx, U2, lam2)
            x2 = torch.from_numpy(fd_sweep_vector(rng2, nn ** 3)).to(dev)
            s2 = torch.empty_like(x2)
            st2 = max(3, min(args.steps, 20 if nn < 512 else 5))
            ms2 = timed(lambda: fd.fd_apply(p2, x2, s2), stream, st2, 2)
            path2 = p2.path()[0]
            e = {"n": nn, "path": path2, "ms_per_apply": ms2, "GDOF_per_s": nn ** 3 / ms2 / 1e6,
                 "apply_tflops": p2.flops() / ms2 / 1e9}
            if path2 != "dmma":
                p2.set_path("dmma")
                ms3 = timed(lambda: fd.fd_apply(p2, x2, s2), stream, st2, 2)
                e["dmma"] = {"ms_per_apply": ms3, "GDOF_per_s": nn ** 3 / ms3 / 1e6, "apply_tflops": p2.flops() / ms3 / 1e9}
            sweep[f"n{nn}"] = e
            p2.close()
            del x2, s2
    cpu = None
    if rank == 0 and not args.no_cpu:
        cpu = cpu_fd_sample(n)
        cpu["one_thread"] = cpu_fd_sample_1thread()
        if not args.no_gmres:
            cpu["gmres"] = cpu_gmres_sample()

    if rank == 0:
        rec = {
            "metric": METRIC, "value": value, "unit": "GDOF/s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": arm_config(ns, ws),
            "arithmetic": ("int8-split tensor-core mode products (exact digit products, one FP64 rounding; the "
                           "accuracy contract of DESIGN.md 5.1) with IEEE FP64 fallback for guard-flagged rows"
                           if path == "int8_split" else "IEEE FP64 (DMMA) mode products"),
            "roofline": roofline(path, kern, flops, int8_ops, achieved, peak, traffic, ws),
            "fp64_native": fp64_native,
            "sustained": sustained,
            "sweep": sweep,
            "comm": {"backend": "nccl" if ws > 1 else None, "nranks": ws},
            "e2e": {"value": N / (e2e_ms * 1e-3) / 1e9, "unit": "GDOF/s", "ms_per_step": e2e_ms,
                    "per_rank_ms": e2e_per_rank,
                    "h2d_bytes_per_step": 8 * N, "d2h_bytes_per_step": 8 * N,
                    "path": "fd_apply_host_async (pinned host buffers; every step H2D + apply + D2H, consecutive "
                            "steps overlapped on two copy streams, wall clock over the steps incl. the final sync)",
                    "sync_call": {"value": N / (e2e_sync_ms * 1e-3) / 1e9, "ms_per_step": e2e_sync_ms,
                                  "path": "fd_apply_host (one blocking call per step)"}},
            "gpu_launches": launches,
            "clocks": clk.summary(),
            "cpu_baseline": cpu,
            "gmres": gm,
            "weak_scaling": weak,
            "paper_context": PAPER_CONTEXT,
        }
        print(json.dumps(rec), flush=True)
    for h in (plan,):
        h.close()
    ctx.close()
    if ws > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
