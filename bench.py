"""Benchmark: TT apply + round (one "op") on one B200 per rank, fp64.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3] [--impl ours|reference]

Prints ONE JSON line (rank 0).  Metric (BASELINE.json "metric"): TT apply+round ops/s, with
the dominant kernel's roofline (FP64 tensor pipe or HBM) and the CPU oracle beside it.

* a step = tk_apply_op + tk_round on the config's seeded input TT (inputs resident in HBM);
* timed with CUDA events on the library's stream, barrier + synchronize on both sides,
  max over ranks; multi-GPU = independent replicas (the path does not shard: DESIGN.md);
* L2: c3/c4 inputs and intermediates are far larger than the 126 MB L2; for c1/c2 a 256 MB
  buffer is written between timed steps (outside the per-step event brackets);
* e2e: the same op through the public binding with HOST inputs: pinned H2D copy of the
  input cores, apply + round, D2H of the rounded cores, all inside the timed region;
* --impl reference: the CPU oracle (oracle/) timed on this host's cores on the same config.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "TT apply+round ops/s"
UNIT = "ops/s"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--config", default=os.environ.get("TTK_BENCH_CONFIG", "c4"))
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--breakdown", action="store_true", help="per-phase times to stderr")
    p.add_argument("--prec", action="store_true",
                   help="c5 / c7 / c8: right-precondition GMRES with the mean-based LSC "
                        "preconditioner (NEXT-3)")
    p.add_argument("--group-space", action="store_true",
                   help="optional exact factor grouping of the space core (SURVEY 8d; reported "
                        "separately, the literal T r growth is the primary line)")
    p.add_argument("--gemm-feed", type=int, default=1, choices=[0, 1],
                   help="operand feed of the heavy DMMA products: 1 = TMA tensor tiles (default), "
                        "0 = cp.async (A/B comparison)")
    p.add_argument("--jacobi-schedule", type=int, default=1, choices=[0, 1],
                   help="block-Jacobi schedule: 1 = dataflow (default), 0 = grid barriers")
    return p.parse_args()


# ----------------------------------------------------------------------------- dist helpers
def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


class Clocks:
    """nvidia-smi sampler during the timed region (the recipe's clocks line)."""

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.lines = []

    def __enter__(self):
        if self.gpu < 0:
            return self
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [v.strip() for v in ln.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                mx = float(f[1])
            except ValueError:
                continue
            for n, v in zip(names, f[3:7]):
                if v.lower() == "active":
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# FP64 tensor-pipe (DMMA) ceiling MEASURED on this pool's B200: tools/ubench/dmma_peak.cu
# (register-only mma.sync m8n8k4 f64 chains, 296 CTAs, >= 16 warps/SM; 37.07-37.15 TF/s at
# 1965 MHz with no throttle reason; profiles/r02/dmma_peak.txt).  tcgen05 has no f64 kind, so
# this is the fp64 tensor roofline of every DMMA GEMM of the rounding.
DMMA_PEAK = {"tflops": 37.15,
             "source": "measured DMMA ubench (tools/ubench/dmma_peak.cu, register-only "
                       "mma.sync m8n8k4 f64, 1965 MHz; profiles/r02/dmma_peak.txt)"}


def dgemm_traffic():
    """Per-launch DRAM bytes (dram__bytes_read.sum + dram__bytes_write.sum) of the dominant
    kernel's heavy launches from one ncu capture of one c4 step (profiles/r02/)."""
    p = os.path.join(ROOT, "profiles", "r02", "dgemm_traffic.json")
    try:
        return json.load(open(p))
    except Exception:
        return None


def algorithmic_round_flops(op, cfg, ranks_out):
    """SURVEY.md 8(d) algorithmic FLOPs of one apply+round on the Gram path: the Gram of the
    grown space core (n_x R1^2), its reconstruction (2 n_x R1 r1'), the Gram of the middle
    unfolding (R1^2 n_xi min(R2, n_t)) and of the time core (R2^2 n_t)."""
    R1, R2 = op.T * cfg.ranks[0], op.T * cfg.ranks[1]
    return (op.n_x * R1 * R1 + 2.0 * op.n_x * R1 * ranks_out[0]
            + R1 * R1 * op.n_xi * min(R2, op.n_t) + R2 * R2 * op.n_t)


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        return json.load(open(p)), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


# ----------------------------------------------------------------------------- oracle arm
def cpu_cores_used():
    try:
        from threadpoolctl import threadpool_info
        return max(int(i.get("num_threads", 1)) for i in threadpool_info()) or 1
    except Exception:
        return os.cpu_count() or 1


def time_oracle_op(op, x, cfg):
    from oracle import tt as otT
    t0 = time.perf_counter()
    y = otT.apply_op(op, x)
    t1 = time.perf_counter()
    otT.round_tt(y, cfg.tol, cfg.rmax)
    t2 = time.perf_counter()
    return t2 - t0, t1 - t0, t2 - t1


# configs whose full oracle op is too long for one --impl reference STEP (c4: ~100 s on 16
# cores): each reference step is then a bounded sample (oracle_sample_step)
SAMPLED = {"c4": (16, 8)}


def _round_input_sample(y, f_inv):
    """The applied TT restricted to its first n_x/f_inv spatial rows and first n_xi/f_inv
    chaos indices: the same rounding algorithm on a proportionally smaller middle and space
    core (every n_x- or n_xi-proportional cost of the oracle round shrinks by f_inv; the
    O(R^3) small SVDs do not)."""
    rows = y[0].shape[0] // f_inv
    nxi = max(1, y[1].shape[1] // f_inv)
    return (np.ascontiguousarray(y[0][:rows]), np.ascontiguousarray(y[1][:, :nxi, :]), y[2])


def oracle_sample_step(op, x, cfg, y_cache, f_inv):
    """One --impl reference step of a SAMPLED config: the full oracle apply (timed), then the
    full rounding algorithm on the 1/f_inv row+chaos sample of its output.  Returns
    (measured seconds, apply seconds, round-sample seconds)."""
    from oracle import tt as otT
    t0 = time.perf_counter()
    y = otT.apply_op(op, x)
    ta = time.perf_counter() - t0
    ys = _round_input_sample(y, f_inv)
    del y
    t0 = time.perf_counter()
    otT.round_tt(ys, cfg.tol, cfg.rmax)
    tr = time.perf_counter() - t0
    return ta + tr, ta, tr


def cpu_baseline(cfg, op, x):
    """The oracle as it stands on ONE full op of the workload (no sampling, no extrapolation:
    ~100 s on 16 cores at c4), plus a single-thread figure on the reference arm's bounded
    sample (1/16 of n_x and n_xi; the time of that sample, not an op rate)."""
    cores = cpu_cores_used()
    dt, ta, tr = time_oracle_op(op, x, cfg)
    out = {"value": 1.0 / dt, "unit": UNIT, "cores": cores, "kind": "oracle",
           "sample": f"1 full {cfg.name} oracle apply ({ta:.1f} s) + round ({tr:.1f} s), "
                     f"NumPy/SciPy OpenBLAS, {cores} threads: {dt:.1f} s/op, measured "
                     f"(not extrapolated)"}
    if cfg.name in SAMPLED:
        try:
            from threadpoolctl import threadpool_limits
            f_inv = SAMPLED[cfg.name][0]
            with threadpool_limits(limits=1):
                t1, a1, r1 = oracle_sample_step(op, x, cfg, None, f_inv)
            out["single_thread"] = {
                "seconds": t1, "cores": 1,
                "sample": f"full {cfg.name} oracle apply ({a1:.1f} s) + round of the first "
                          f"1/{f_inv} of n_x and n_xi ({r1:.1f} s), BLAS limited to 1 thread"}
        except Exception as e:  # pragma: no cover
            out["single_thread"] = {"error": str(e)}
    return out


def run_reference(args, cfg, op, x):
    """--impl reference: the oracle on this host's cores, W warm-up + K timed steps.  Configs
    whose full op fits a step run it in full; c4 (SAMPLED) alternates the 1/16 and 1/8
    row+chaos samples of the round (oracle_sample_step).  Its op time is then EXTRAPOLATED
    with the affine model t_round(f) = a + b f fitted to the two sample sizes of this run
    (t_op = t_apply + t_round(f) + b (1 - f) per step), which ignores the oracle's slowdown on
    the full-size arrays and so OVERSTATES its rate (a measured full op is the main arm's
    cpu_baseline).  ms_per_step is the measured sample time."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    oop = op.oracle_op()
    cores = cpu_cores_used()
    samp = SAMPLED.get(cfg.name)
    meas, ext, what = [], [], ""
    if not samp:
        for _ in range(args.warmup):
            time_oracle_op(oop, x, cfg)
        for _ in range(args.steps):
            dt, _, _ = time_oracle_op(oop, x, cfg)
            meas.append(dt)
        ext = list(meas)
        what = f"1 full {cfg.name} oracle apply+round op per step (measured)"
    else:
        f_lo, f_hi = samp
        for _ in range(args.warmup):
            oracle_sample_step(oop, x, cfg, None, f_hi)
        rec = []
        for k in range(args.steps):
            f_inv = f_lo if k % 2 == 0 else f_hi
            dt, ta, tr = oracle_sample_step(oop, x, cfg, None, f_inv)
            meas.append(dt)
            rec.append((1.0 / f_inv, ta, tr))
        lo = [r for f, _, r in rec if f == 1.0 / f_lo]
        hi = [r for f, _, r in rec if f == 1.0 / f_hi]
        b = 0.0
        if lo and hi:
            b = max(0.0, (statistics.mean(hi) - statistics.mean(lo)) / (1.0 / f_hi - 1.0 / f_lo))
        ext = [ta + tr + b * (1.0 - f) for f, ta, tr in rec]
        what = (f"per step: the full {cfg.name} oracle apply + the oracle round of the first "
                f"1/{f_lo} (even steps) or 1/{f_hi} (odd steps) of n_x and n_xi; op time "
                f"extrapolated as t_apply + t_round(f) + b (1 - f), b = {b:.1f} s fitted to "
                f"the two sample sizes (affine model, overstates the oracle's rate)")
    v = len(ext) / sum(ext)
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * statistics.mean(meas),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": workload_config(cfg, op),
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle",
                         "sample": f"{what}; NumPy/SciPy OpenBLAS, {cores} threads; "
                                   f"measured {statistics.mean(meas):.1f} s per step"},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- multi-rank
def max_over_ranks(value: float, device: str) -> float:
    """All-reduce MAX of a per-rank timing (the slowest replica defines the job time)."""
    import torch
    import torch.distributed as tdist
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
    return float(t.item())


def replica_throughput(world: int, steps: int, max_total_ms: float) -> float:
    """Whole-job ops/s of N independent replicas: every rank ran `steps` ops; the job took the
    max-over-ranks time (weak scaling)."""
    return world * 1000.0 * steps / max_total_ms


# ----------------------------------------------------------------------------- our arm
def workload_config(cfg, op):
    return {"workload": f"{cfg.name}: apply+round", "n_x": op.n_x, "n_xi": op.n_xi, "n_t": op.n_t,
            "terms": op.T, "ranks_in": list(cfg.ranks),
            "ranks_grown": [op.T * cfg.ranks[0], op.T * cfg.ranks[1]], "tol": cfg.tol,
            "rmax": cfg.rmax, "parallelism": "replicas",
            "l2": "inputs+intermediates > L2" if cfg.name in ("c3", "c4") else "256MB flush between steps"}


def run_ours(args, cfg, op, x):
    import torch
    import torch.distributed as tdist

    rank, world, local = dist_env()
    if world > 1:
        tdist.init_process_group("nccl")
    torch.cuda.set_device(local)
    import paper_1906_06785_b200 as ttk
    from paper_1906_06785_b200 import ttk as ttkmod

    stream = torch.cuda.current_stream()
    ctx = ttk.default_context()
    ctx.set_gemm_feed(ARGS_GLOBAL.gemm_feed)
    ctx.set_jacobi_schedule(ARGS_GLOBAL.jacobi_schedule)
    gop = op.gpu_op(ctx)
    groups = gop.group_space(True) if args.group_space else None
    xg = ttk.TT.from_cores(*x)
    T = op.T
    ycap = ttk.TT(op.n_x, op.n_xi, op.n_t, T * xg.r1, T * xg.r2)
    flush = None
    if cfg.name not in ("c3", "c4"):
        flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")

    def step():
        # the fused entry point: apply + round in one call (tk_apply_round)
        return ttk.tt_apply_round(gop, xg, cfg.tol, cfg.rmax, out=ycap)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        tdist.barrier()
    L = ttkmod.lib()
    # timed region: events around the heavy launches only (enable == 2; the full per-kernel
    # record list costs ~2 ms per c4 step on the latency-bound chain) — the complete phase
    # table comes from one extra, untimed, fully profiled step below
    L.tk_ctx_profile(ctx._h, 0 if os.environ.get('TTK_BENCH_NOPROF') else 2)
    launches0 = ctx.launches
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    with Clocks(-1 if os.environ.get('TTK_BENCH_NOCLOCKS') else local) as clk:
        torch.cuda.synchronize()
        for i in range(args.steps):
            if flush is not None:
                flush.fill_(float(i))
            evs[i][0].record(stream)
            y = step()
            evs[i][1].record(stream)
        torch.cuda.synchronize()
    launches = ctx.launches - launches0
    buf = __import__("ctypes").create_string_buffer(1 << 22)
    nrec = L.tk_ctx_profile_dump(ctx._h, buf, len(buf))
    L.tk_ctx_profile(ctx._h, 0)
    step_ms = [a.elapsed_time(b) for a, b in evs]
    total_ms = sum(step_ms)
    if world > 1:
        total_ms = max_over_ranks(total_ms, "cuda")
        tdist.barrier()
    ranks_out = y.ranks
    heavy = {}
    for ln in buf.value.decode().splitlines():
        cat, ms, fl, by = ln.split()[:4]
        kn = {"spmm_multi": "spmm_merged_k", "stoch_apply": "stoch_apply_k",
              "time_apply": "time_apply_k"}.get(
                  cat, "dgemm_tma_kernel" if args.gemm_feed else "dgemm_kernel")
        d = heavy.setdefault(kn, [0, 0.0, 0.0, 0.0])
        d[0] += 1
        d[1] += float(ms)
        d[2] += float(fl)
        d[3] += float(by)
    # one untimed step with every launch recorded: the per-phase table
    L.tk_ctx_profile(ctx._h, 1)
    step()
    torch.cuda.synchronize()
    nrec = L.tk_ctx_profile_dump(ctx._h, buf, len(buf))
    L.tk_ctx_profile(ctx._h, 0)
    full_steps = 1

    # per-phase breakdown and the dominant kernel
    phases = {}
    for ln in buf.value.decode().splitlines():
        cat, ms, fl, by = ln.split()
        d = phases.setdefault(cat, [0, 0.0, 0.0, 0.0])
        d[0] += 1
        d[1] += float(ms)
        d[2] += float(fl)
        d[3] += float(by)
    peaks, peak_kind = load_peaks()
    fp64_peak = DMMA_PEAK["tflops"]
    # group the phase records by KERNEL FUNCTION: every phase tag that is not one of the
    # named kernels below is a launch of the DMMA GEMM (dgemm_kernel + its split-K reduce)
    # (kernel names as in the ncu launch list, profiles/r02/launches_c4_r2*.csv; the heavy DMMA
    # products run the TMA-fed dgemm_tma_kernel, the light ones and the 128 x 80 tile of form_U1
    # the cp.async dgemm_kernel)
    gemm_name = "dgemm_tma_kernel" if args.gemm_feed else "dgemm_kernel"
    named = {"jacobi": "jacobi_flow_k" if args.jacobi_schedule else "jacobi_persistent_k",
             "qr_panel": "qr_panel_reg_k",
             "qr_reflector": "apply_reflector_k", "pchol_panel": "pchol_panel_reg_k",
             "spmm_multi": "spmm_merged_k", "stoch_apply": "stoch_apply_k",
             "time_apply": "time_apply_k"}
    kernels = {}
    for cat, v in phases.items():
        kn = named.get(cat, gemm_name)
        d = kernels.setdefault(kn, [0, 0.0, 0.0, 0.0])
        for i in range(4):
            d[i] += v[i]
    dom = max(kernels.items(), key=lambda kv: kv[1][1]) if kernels else None
    roofline = None
    if dom:
        cat = dom[0]
        # achieved = algorithmic work / average duration of the dominant kernel's launches
        # recorded INSIDE the timed region (the heavy ones: >= 1e8 flops or bytes); the
        # all-launch average of the untimed fully profiled step is reported beside it
        cnt, ms, fl, by = heavy.get(cat, dom[1])
        ms_all = dom[1][1] / full_steps
        avg_ms = ms / cnt
        if fl > 0 and (by <= 0 or fl / by > 6.0):
            ach = fl / cnt / (avg_ms * 1e-3) / 1e12
            alg = algorithmic_round_flops(op, cfg, ranks_out)
            tr = dgemm_traffic() if cfg.name == "c4" and not args.group_space else None
            roofline = {"kernel": cat, "bound": "tensor", "achieved": ach, "peak": fp64_peak,
                        "unit": "TFLOP/s", "frac": ach / fp64_peak,
                        "traffic": tr["dram_bytes_per_launch"] if tr else None,
                        "traffic_capture": tr,
                        "peak_source": DMMA_PEAK["source"],
                        "launches": cnt, "avg_ms": avg_ms, "share_of_step": ms / total_ms,
                        "launches_recorded": "timed region, launches >= 1e8 flops or bytes",
                        "achieved_all_launches": dom[1][2] / (dom[1][1] * 1e-3) / 1e12,
                        "launches_all_per_step": dom[1][0] / full_steps,
                        "share_of_step_all_launches": ms_all / (total_ms / args.steps),
                        # SURVEY 8(d) algorithmic FLOPs of the whole op (Gram path) over the
                        # whole step time: what the method needs vs what the step delivers
                        "algorithmic_flops_per_op": alg,
                        "frac_algorithmic": alg / (total_ms / args.steps * 1e-3) / 1e12 / fp64_peak}
        elif by > 0:
            ach = by / cnt / (avg_ms * 1e-3) / 1e9
            roofline = {"kernel": cat, "bound": "hbm", "achieved": ach, "peak": peaks["hbm_gbs"],
                        "unit": "GB/s", "frac": ach / peaks["hbm_gbs"], "traffic": None,
                        "peak_source": peak_kind, "launches": cnt, "avg_ms": avg_ms,
                        "share_of_step": ms / total_ms}
        else:
            roofline = {"kernel": cat, "bound": "latency", "achieved": None, "peak": None,
                        "unit": None, "frac": None, "traffic": None, "launches": cnt,
                        "avg_ms": avg_ms, "share_of_step": ms / total_ms}
    spmm = phases.get("spmm_multi")
    # inside the step the SpMM shares the GPU with the small-core sweep (side stream), so its
    # bandwidth is measured alone as well: three plain tk_apply_op calls, library events
    spmm_gbs_in_step = spmm[3] / (spmm[1] * 1e-3) / 1e9 if spmm else None
    yapp = ttk.TT(op.n_x, op.n_xi, op.n_t, T * xg.r1, T * xg.r2)
    L.tk_ctx_profile(ctx._h, 1)
    for _ in range(3):
        ttk.tt_apply_op(gop, xg, out=yapp)
    torch.cuda.synchronize()
    del yapp
    buf3 = __import__("ctypes").create_string_buffer(1 << 16)
    L.tk_ctx_profile_dump(ctx._h, buf3, len(buf3))
    L.tk_ctx_profile(ctx._h, 0)
    sp = [ln.split() for ln in buf3.value.decode().splitlines() if ln.startswith("spmm_multi")]
    spmm_gbs = (sum(float(a[3]) for a in sp) / (sum(float(a[1]) for a in sp) * 1e-3) / 1e9
                if sp else spmm_gbs_in_step)

    # the TT axpby of GMRES (a9/a10 rows) on the rounded result: z = a y + b y, a copy stream
    # (16 bytes per U1 entry of z), timed by the library's own per-kernel events
    axpby_gbs = None
    # x and y are distinct TTs of equal ranks (y and a copy of it: no L2 reuse between them)
    y2 = ttk.TT.from_cores(*y.cores_numpy())
    zcap = ttk.TT(op.n_x, op.n_xi, op.n_t, 2 * y.r1, 2 * y.r2)
    ttk.tt_axpby(0.5, y, -0.25, y2, ctx, out=zcap)
    torch.cuda.synchronize()
    L.tk_ctx_profile(ctx._h, 1)
    for _ in range(5):
        ttk.tt_axpby(0.5, y, -0.25, y2, ctx, out=zcap)
    torch.cuda.synchronize()
    buf2 = __import__("ctypes").create_string_buffer(1 << 16)
    L.tk_ctx_profile_dump(ctx._h, buf2, len(buf2))
    L.tk_ctx_profile(ctx._h, 0)
    ax = [ln.split() for ln in buf2.value.decode().splitlines() if ln.startswith("axpby")]
    if ax:
        axpby_gbs = {"value": sum(float(a[3]) for a in ax) / (sum(float(a[1]) for a in ax) * 1e-3) / 1e9,
                     "unit": "GB/s", "peak": peaks["hbm_gbs"], "ranks": [2 * y.r1, 2 * y.r2],
                     "bytes_per_call": float(ax[0][3]), "calls": len(ax)}
        axpby_gbs["frac"] = axpby_gbs["value"] / peaks["hbm_gbs"]
    del zcap, y2

    # e2e through the public API with host buffers: every step copies its input TT from pinned
    # host memory and reads its rounded result back, pipelined the way a user would stream a
    # batch of ops (step i+1's H2D and step i-1's D2H on copy streams overlap step i's compute;
    # double-buffered device TTs, event-ordered reuse)
    e2e = None
    if rank == 0 or world > 1:
        pinned = [torch.from_numpy(np.ascontiguousarray(c)).pin_memory() for c in x]
        h2d = sum(p.numel() * 8 for p in pinned)
        xes = [ttk.TT(op.n_x, op.n_xi, op.n_t, cfg.ranks[0], cfg.ranks[1]) for _ in range(2)]
        yes = [ttk.TT(op.n_x, op.n_xi, op.n_t, T * cfg.ranks[0], T * cfg.ranks[1]) for _ in range(2)]
        # the rounded result's ranks are <= rmax (when set) and <= the grown ranks
        r1o = min(T * cfg.ranks[0], cfg.rmax) if cfg.rmax else T * cfg.ranks[0]
        r2o = min(T * cfg.ranks[1], cfg.rmax) if cfg.rmax else T * cfg.ranks[1]
        outs = [[torch.empty(n, dtype=torch.float64).pin_memory()
                 for n in (op.n_x * r1o, r1o * op.n_xi * r2o, r2o * op.n_t)] for _ in range(2)]
        s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
        ne = max(2, min(args.steps, 6))
        ev = lambda: torch.cuda.Event()  # noqa: E731
        in_done, comp_done, out_done = ([ev() for _ in range(ne)] for _ in range(3))
        d2h = 0

        def gate(s_):
            # copy-window gate; a driver without the needed entry points just runs ungated
            try:
                return gop.ctx.gate_stream(s_)
            except ttk.TkError:
                return False

        def h2d_step(i):
            with torch.cuda.stream(s_in):
                if i >= 1:
                    # copy window: step i's input travels while step i - 1 (the rounding just
                    # submitted) is in its DMMA-bound phase (tk_ctx_gate_stream)
                    gate(s_in)
                if i >= 2:
                    s_in.wait_event(comp_done[i - 2])  # xes[i % 2] free again
                for buf_, src in zip((xes[i % 2].b1, xes[i % 2].b2, xes[i % 2].b3), pinned):
                    buf_[: src.numel()].copy_(src.reshape(-1), non_blocking=True)
                in_done[i].record(s_in)

        # async boundary (tk_ctx_set_async): the calls return at once, the roundings run in
        # stream order on the library's worker, so the host queues the whole pipeline ahead;
        # each step reads back the rank-capacity prefix of the result cores (the ranks are
        # published at tk_sync_ranks; rmax bounds them)
        use_async = gop.ctx.set_async(True)
        # one-time setup of the copy-window gate outside the timed region (its first call loads
        # the library's kernels and synchronises the context once; nothing is pending here, so
        # the streams are not delayed)
        gate(s_in)
        gate(s_out)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(stream)
        s_in.wait_event(e0)
        h2d_step(0)

        def d2h_step(i, ye, gated):
            with torch.cuda.stream(s_out):
                s_out.wait_event(comp_done[i])
                if gated:
                    gate(s_out)  # read back inside the next step's copy window
                n = 0
                srcs = ((ye.b1, op.n_x * r1o), (ye.b2, r1o * op.n_xi * r2o), (ye.b3, r2o * op.n_t)) \
                    if use_async else ((c.reshape(-1), c.numel()) for c in (ye.U1, ye.U2, ye.U3))
                for o, (c, m) in zip(outs[i % 2], srcs):
                    o[:m].copy_(c[:m], non_blocking=True)
                    n += m * 8
                out_done[i].record(s_out)
            return n

        prev = None
        for i in range(ne):
            stream.wait_event(in_done[i])
            if i >= 2:
                stream.wait_event(out_done[i - 2])  # yes[i % 2] read back
            ye = ttk.tt_apply_round(gop, xes[i % 2], cfg.tol, cfg.rmax, out=yes[i % 2])
            comp_done[i].record(stream)
            # step i is submitted: the transfers of its neighbours wait for its copy window
            if i + 1 < ne:
                h2d_step(i + 1)
            if prev is not None:
                d2h = d2h_step(i - 1, prev, True)
            prev = ye
        d2h = d2h_step(ne - 1, prev, False)
        stream.wait_event(out_done[ne - 1])
        e1.record(stream)
        torch.cuda.synchronize()
        e2e_ms = e0.elapsed_time(e1)
        gop.ctx.set_async(False)  # (publishes the queued ranks)
        assert ye.ranks == tuple(ranks_out), (ye.ranks, ranks_out)
        e2e = {"value": world * 1000.0 * ne / e2e_ms, "unit": UNIT,
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "steps": ne,
               "ms_per_step": e2e_ms / ne,
               "pipelined": "H2D of step i+1 and D2H of step i-1 on copy streams overlap step i's "
                            "DMMA-bound phase (tk_ctx_gate_stream)",
               "boundary": "async (tk_ctx_set_async)" if use_async else "synchronous"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(cfg, op.oracle_op(), x)

    if args.breakdown and rank == 0:
        for cat, (cnt, ms, fl, by) in sorted(phases.items(), key=lambda kv: -kv[1][1]):
            tf = fl / (ms * 1e-3) / 1e12 if ms > 0 else 0
            gb = by / (ms * 1e-3) / 1e9 if ms > 0 else 0
            print(f"  {cat:18s} n={cnt:4d} {ms / full_steps:9.3f} ms/step  {tf:7.2f} TF/s  {gb:8.1f} GB/s",
                  file=sys.stderr)
        print(f"  step times ms: {[round(s, 3) for s in step_ms]}", file=sys.stderr)

    if rank == 0:
        ms_per_step = total_ms / args.steps
        line = {
            "metric": METRIC, "value": replica_throughput(world, args.steps, total_ms), "unit": UNIT,
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": dict(workload_config(cfg, op), **(
                {"workload": f"{cfg.name}: apply+round, space factors grouped (optional, exact)",
                 "space_groups": groups} if groups is not None else {})),
            "ranks_out": list(ranks_out),
            "roofline": roofline, "spmm_gbs": spmm_gbs,
            "spmm_frac": spmm_gbs / peaks["hbm_gbs"] if spmm_gbs else None,
            "spmm_frac_of_8tbs_spec": spmm_gbs / 8000.0 if spmm_gbs else None,
            "spmm_gbs_in_step": spmm_gbs_in_step, "axpby_gbs": axpby_gbs,
            "phases_ms_per_step": {k: round(v[1] / full_steps, 4) for k, v in phases.items()},
            "kernels_ms_per_step": {k: round(v[1] / full_steps, 4) for k, v in kernels.items()},
            "phases_note": "one untimed, fully profiled step (every launch bracketed by events)",
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches, "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        tdist.destroy_process_group()


# ----------------------------------------------------------------------------- c5: GMRES cycle
GMRES_METRIC = "low-rank GMRES Krylov steps/s"
GMRES_UNIT = "steps/s"


def gmres_config(cfg, op):
    return {"workload": f"{cfg.name}: one {cfg.gmres_steps}-step low-rank GMRES cycle",
            "n_x": op.n_x, "n_xi": op.n_xi, "n_t": op.n_t, "terms": op.T,
            "rhs_ranks": list(cfg.rhs_ranks), "tol": cfg.tol, "parallelism": "replicas",
            "l2": "256MB flush between cycles"}


def oracle_sample_gmres(op, b, cfg, budget=30.0):
    """Bounded oracle sample of c5: the first k Krylov steps of the oracle cycle, k grown until
    the ~30 s budget is used (later steps cost more: the sample is optimistic for the oracle)."""
    from oracle import gmres as og
    k = 1
    while True:
        t0 = time.perf_counter()
        og.gmres_cycle(op, b, steps=k, tol=cfg.tol)
        dt = time.perf_counter() - t0
        if dt > budget / 3 or k >= cfg.gmres_steps:
            return k / dt, f"oracle cycle truncated to its first {k} of {cfg.gmres_steps} Krylov steps ({dt:.1f} s)"
        k *= 2


def run_gmres(args, cfg, op):
    import torch
    import torch.distributed as tdist
    from synth.tt import make_rhs_tt
    rank, world, local = dist_env()
    if world > 1:
        tdist.init_process_group("nccl")
    torch.cuda.set_device(local)
    import paper_1906_06785_b200 as ttk
    from paper_1906_06785_b200 import ttk as ttkmod
    b = make_rhs_tt(cfg, op.n_xi)
    if args.impl == "reference":
        if rank == 0:
            v, what = oracle_sample_gmres(op.oracle_op(), b, cfg, budget=120.0)
            cores = cpu_cores_used()
            print(json.dumps({
                "impl": "reference", "metric": GMRES_METRIC, "value": v, "unit": GMRES_UNIT,
                "n_gpus": args.gpus, "steps": 1, "warmup": 0, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": gmres_config(cfg, op),
                "cpu_baseline": {"value": v, "unit": GMRES_UNIT, "cores": cores, "kind": "oracle",
                                 "sample": what},
                "e2e": {"value": v, "unit": GMRES_UNIT, "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}}), flush=True)
        return
    stream = torch.cuda.current_stream()
    ctx = ttk.default_context()
    ctx.set_gemm_feed(ARGS_GLOBAL.gemm_feed)
    ctx.set_jacobi_schedule(ARGS_GLOBAL.jacobi_schedule)
    gop = op.gpu_op(ctx)
    bg = ttk.TT.from_cores(*b)
    steps_k = cfg.gmres_steps
    P = None
    if args.prec:  # NEXT-3: flexible GMRES with the mean-based LSC preconditioner
        from synth.operator import mean_blocks
        F0s, Bd = mean_blocks(cfg)
        P = ttk.MeanLSC(F0s, Bd, cfg.tau, op.n_xi, op.n_t, tol=cfg.tol, grid=cfg.grid, ctx=ctx)
        steps_k = 3
    flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")
    for _ in range(args.warmup):
        ttk.gmres_cycle(gop, bg, steps_k, cfg.tol, prec=P)
    torch.cuda.synchronize()
    if world > 1:
        tdist.barrier()
    L = ttkmod.lib()
    # events around the heavy launches only (enable == 2): the per-launch events of the
    # latency-bound chain would slow the cycle itself
    L.tk_ctx_profile(ctx._h, 0 if os.environ.get('TTK_BENCH_NOPROF') else 2)
    launches0 = ctx.launches
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    res = None
    krylov = 0
    with Clocks(-1 if os.environ.get('TTK_BENCH_NOCLOCKS') else local) as clk:
        torch.cuda.synchronize()
        for i in range(args.steps):
            flush.fill_(float(i))
            evs[i][0].record(stream)
            res = ttk.gmres_cycle(gop, bg, steps_k, cfg.tol, prec=P)
            evs[i][1].record(stream)
            krylov += res["steps"]
        torch.cuda.synchronize()
    launches = ctx.launches - launches0
    buf = __import__("ctypes").create_string_buffer(1 << 24)
    L.tk_ctx_profile_dump(ctx._h, buf, len(buf))
    L.tk_ctx_profile(ctx._h, 0)
    total_ms = sum(a.elapsed_time(b_) for a, b_ in evs)
    if world > 1:
        total_ms = max_over_ranks(total_ms, "cuda")
    phases = {}
    for ln in buf.value.decode().splitlines():
        cat, ms, fl, by = ln.split()
        d = phases.setdefault(cat, [0, 0.0])
        d[0] += 1
        d[1] += float(ms)
    # e2e: the right-hand side from pinned host memory each cycle (the history comes back to
    # the host inside the cycle)
    pinned = [torch.from_numpy(np.ascontiguousarray(c)).pin_memory() for c in b]
    h2d = sum(p.numel() * 8 for p in pinned)
    be = ttk.TT(op.n_x, op.n_xi, op.n_t, cfg.rhs_ranks[0], cfg.rhs_ranks[1])
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    for buf_, src in zip((be.b1, be.b2, be.b3), pinned):
        buf_[: src.numel()].copy_(src.reshape(-1), non_blocking=True)
    re_ = ttk.gmres_cycle(gop, be, steps_k, cfg.tol, prec=P)
    e1.record(stream)
    torch.cuda.synchronize()
    e2e = {"value": world * 1000.0 * re_["steps"] / e0.elapsed_time(e1), "unit": GMRES_UNIT,
           "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": 8 * (len(re_["history"]) + 1),
           "steps": 1}
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and P is None:
        v, what = oracle_sample_gmres(op.oracle_op(), b, cfg)
        cores = cpu_cores_used()
        cpu = {"value": v, "unit": GMRES_UNIT, "cores": cores, "kind": "oracle",
               "sample": f"{what}; NumPy/SciPy OpenBLAS, {cores} threads"}
    if args.breakdown and rank == 0:
        for cat, (cnt, ms) in sorted(phases.items(), key=lambda kv: -kv[1][1]):
            print(f"  {cat:18s} n={cnt:5d} {ms / args.steps:10.3f} ms/cycle", file=sys.stderr)
    if rank == 0:
        line = {
            "metric": GMRES_METRIC, "value": world * 1000.0 * krylov / max(total_ms, 1e-9),
            "unit": GMRES_UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": total_ms / args.steps, "ms_per_krylov_step": total_ms / max(krylov, 1),
            "krylov_step_ms_host": [round(t, 2) for t in res["step_ms"].tolist()],
            "residual_history": res["history"].tolist(), "explicit_residual": res["explicit"],
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": gmres_config(cfg, op),
            "phases_ms_per_cycle": {k: round(v[1] / args.steps, 3) for k, v in phases.items()},
            "phases_note": "heavy launches only (>= 1e8 flops or bytes); tools/gmres_profile.py has all",
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches, "clocks": clk.summary(),
            "note": "step = one GMRES cycle (the c5 line; the headline bench line is c4)",
        }
        if P is not None:
            line["config"]["workload"] = (f"{cfg.name}: one {steps_k}-step flexible low-rank GMRES "
                                          "cycle, mean-based LSC preconditioner (NEXT-3)")
            line["note"] = ("NEXT-3 line (not a BASELINE.json config): each Krylov step applies "
                            "P^{-1} (two pressure solves, B(F0+C)B^T, an inner GMRES with M)")
        print(json.dumps(line), flush=True)
    if world > 1:
        tdist.destroy_process_group()


# ----------------------------------------------------------------------------- c7/c8: Picard
def run_picard(args, cfg):
    """NEXT-4 line (not a BASELINE.json config): one full inexact Picard solve (Alg. 1) per step
    on the synthetic stochastic Galerkin Navier-Stokes problem of config c7 / c8."""
    import torch
    import paper_1906_06785_b200 as ttk
    from synth import gpc
    from synth.operator import (build_operator, convection_stencils, mean_blocks,
                                picard_forcing)
    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    op = build_operator(cfg)
    H = gpc.h_matrices(cfg.m, cfg.p)
    D, nv = convection_stencils(cfg.grid)
    f = picard_forcing(cfg, op.n_xi)
    kw = dict(tol_picard=1e-3, maxit=12, tol_gmres=1e-1, eps_gmres=cfg.tol, restart=20,
              max_cycles=5)
    wl = {"workload": f"{cfg.name}: inexact Picard solve (Alg. 1), stochastic Galerkin NS",
          "n_x": op.n_x, "n_xi": op.n_xi, "n_t": op.n_t, "grid": cfg.grid, **kw,
          "prec": "mean-based LSC" if args.prec else "none", "parallelism": "replicas"}
    if args.impl == "reference":
        if rank == 0:
            from oracle.precond import MeanLSC as OLSC
            from oracle.picard import picard as o_picard
            prec = None
            if args.prec:
                F0s, Bd = mean_blocks(cfg)
                prec = OLSC(F0s, Bd, cfg.tau, op.n_xi, op.n_t, tol=cfg.tol).apply
            t0 = time.perf_counter()
            o_picard(op, H, D, nv, f, prec=prec, **kw)
            dt = time.perf_counter() - t0
            v = 1.0 / dt
            print(json.dumps({"impl": "reference", "metric": "Picard solves/s", "value": v,
                              "unit": "solves/s", "n_gpus": args.gpus, "steps": 1, "warmup": 0,
                              "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
                              "dtype": "f64", "data": "synthetic", "config": wl,
                              "cpu_baseline": {"value": v, "unit": "solves/s",
                                               "cores": cpu_cores_used(), "kind": "oracle",
                                               "sample": f"1 full oracle Picard solve ({dt:.1f} s)"},
                              "e2e": {"value": v, "unit": "solves/s", "h2d_bytes_per_step": 0,
                                      "d2h_bytes_per_step": 0}}), flush=True)
        return
    ctx = ttk.default_context()
    ctx.set_gemm_feed(ARGS_GLOBAL.gemm_feed)
    ctx.set_jacobi_schedule(ARGS_GLOBAL.jacobi_schedule)
    g_op = ttk.Operator.from_kronsum(op, ctx)
    conv = ttk.Convection(op.n_x, op.n_xi, op.n_t, D, nv, np.array(H), ctx=ctx)
    P = None
    if args.prec:
        F0s, Bd = mean_blocks(cfg)
        P = ttk.MeanLSC(F0s, Bd, cfg.tau, op.n_xi, op.n_t, tol=cfg.tol, grid=cfg.grid, ctx=ctx)
    fg = ttk.TT.from_cores(*f)
    for _ in range(args.warmup):
        ttk.picard(g_op, conv, fg, prec=P, **kw)
    stream = torch.cuda.current_stream()
    torch.cuda.synchronize()
    launches0 = ctx.launches
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Clocks(local) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            res = ttk.picard(g_op, conv, fg, prec=P, **kw)
        e1.record(stream)
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    cpu = None
    if rank == 0 and not args.no_cpu_baseline and cfg.name == "c7":
        from oracle.picard import picard as o_picard
        t0 = time.perf_counter()
        o_picard(op, H, D, nv, f, **kw)
        dt = time.perf_counter() - t0
        cpu = {"value": 1.0 / dt, "unit": "solves/s", "cores": cpu_cores_used(), "kind": "oracle",
               "sample": f"1 full oracle Picard solve without P ({dt:.1f} s)"}
    fn = float(np.linalg.norm(f[0]) * np.linalg.norm(f[1]) * np.linalg.norm(f[2]))
    if rank == 0:
        print(json.dumps({
            "metric": "Picard solves/s", "value": world * 1000.0 / ms, "unit": "solves/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "picard_iterations": res["iterations"],
            "residuals_rel": (res["residuals"] / fn).tolist(), "ranks": res["ranks"],
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": wl, "cpu_baseline": cpu,
            "gpu_launches": ctx.launches - launches0, "clocks": clk.summary(),
            "note": "NEXT-4 line, not a BASELINE.json config (the headline bench line is c4)"}),
            flush=True)


class Workload:
    """The config's operator: a host descriptor (c1..c5, built by synth) or, for the NEXT-1
    convection config c6, the discretisation + velocity TT from which the LIBRARY builds N(u)
    on the device (tk_op_convection) and the oracle builds its own eq:N_kron operator."""

    def __init__(self, cfg):
        from synth import gpc
        from synth.operator import build_operator, convection_stencils
        from synth.tt import make_velocity_tt
        self.cfg = cfg
        self._oracle = None
        if cfg.operator == "convection":
            self.H = gpc.h_matrices(cfg.m, cfg.p)
            self.D, self.n_v = convection_stencils(cfg.grid)
            self.u = make_velocity_tt(cfg, len(self.H))
            self.host = None
            self.n_x, self.n_xi, self.n_t = cfg.n_x, len(self.H), cfg.n_t
            self.T = cfg.n_terms
        else:
            self.host = build_operator(cfg)
            self.n_x, self.n_xi, self.n_t, self.T = (self.host.n_x, self.host.n_xi,
                                                     self.host.n_t, self.host.T)

    def gpu_op(self, ctx):
        import paper_1906_06785_b200 as ttk
        if self.host is not None:
            return ttk.Operator.from_kronsum(self.host, ctx)
        self._conv = ttk.Convection(self.n_x, self.n_xi, self.n_t, self.D, self.n_v,
                                    np.stack(self.H), ctx)
        self._u_dev = ttk.TT.from_cores(*self.u)
        return self._conv.operator(self._u_dev)   # N(u) built on the device

    def oracle_op(self):
        if self.host is not None:
            return self.host
        if self._oracle is None:
            from oracle.convection import convection_operator
            self._oracle = convection_operator(*self.u, self.H, self.D, self.n_v)
        return self._oracle


ARGS_GLOBAL = None


def main():
    global ARGS_GLOBAL
    args = ARGS_GLOBAL = parse()
    from synth.configs import CONFIGS
    from synth.tt import make_input_tt
    cfg = CONFIGS[args.config]
    if cfg.operator == "picard":
        run_picard(args, cfg)
        return
    op = Workload(cfg)
    if cfg.name == "c5":
        run_gmres(args, cfg, op)
        return
    x = make_input_tt(cfg, op.n_xi)
    if args.impl == "reference":
        run_reference(args, cfg, op, x)
    else:
        run_ours(args, cfg, op, x)


if __name__ == "__main__":
    main()
