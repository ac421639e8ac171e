#!/usr/bin/env python
"""bench.py -- KS matmul on B200 (arXiv 2405.15013 hot path).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload fft] [--impl ours|reference]

Default workload = BASELINE.json configs[1]: the FFT-style butterfly chain,
N = 4096, 12 factors (2^{l-1},2,2,2^{12-l}), global batch B = 8192, FP32, BSF.
One *step* = one pass of the whole hot path over the batch: the 12 KS factor
launches of the chain (K_12 first), inputs resident in HBM.

metric: achieved GB/s with the paper's byte model (read X + nnz(K) + write Y
per factor), summed over the factors, divided
by device time.  Multi-GPU (torchrun): the configuration's global
batch B is partitioned, B_g = ceil(B/G) contiguous rows per rank (one seeded
global X, rows drawn by counter so any shard has the same bytes); no
collective on the compute path; value = all ranks' bytes / max over ranks of
the device time ("scaling": "strong": the total work is fixed).

The same line also carries configs[3] (ViT-S/16 MLP) and configs[4] (GPT-2
medium MLP) chains in FP32 and TF32 ("models"), each with its own roofline
against the bound of its dominant kernel (HBM, the measured FFMA peak for the
FP32 CUDA-core kernels, or the measured TF32 tensor peak), the dense cuBLAS
GEMM and the paper's bmm+permute baseline on the same inputs, and an oracle
check of sampled rows from every rank; and (N = 1) the configs[2] sweep.

Prints ONE JSON line on rank 0; exits 1 (with "value": null) if any oracle
check fails.
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

METRIC = "KS matmul achieved HBM GB/s (% peak) & median speedup vs bmm+permute over sweep"
FALLBACK_HBM_GBS = 6650.0   # B200_PROFILING.md fallback ("of fallback")
MODEL_WORKLOADS = ("vit_up", "vit_down", "gpt2_down", "gpt2_up")


# ----------------------------------------------------------------- helpers --
def parse_args(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", default="fft",
                    choices=["fft", "tiny", "vit_up", "vit_down", "gpt2_down", "gpt2_up"])
    ap.add_argument("--layout", choices=["bsf", "bsl"], default="bsf")
    ap.add_argument("--math", choices=["fp32", "tf32", "f32x3"], default="fp32",
                    help="per-factor math: FP32 CUDA cores (default), TF32 or 3xTF32 on tcgen05")
    ap.add_argument("--no-baselines", action="store_true",
                    help="skip the bmm+permute / dense cuBLAS timing of the same chain")
    ap.add_argument("--batch", type=int, default=None, help="global batch override")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-sweep", action="store_true", help="skip the configs[2] sweep vs bmm+permute")
    ap.add_argument("--no-models", action="store_true", help="skip the configs[3]/[4] model chains")
    ap.add_argument("--no-verify", action="store_true", help="skip the oracle check of sampled rows")
    ap.add_argument("--sweep-reps", type=int, default=10)
    return ap.parse_args(argv)


def workload(name: str):
    from ksgen import configs
    if name == "fft":
        return dict(name=f"fft_chain_N4096_L{configs.FFT_L}", patterns=configs.dyadic_patterns(configs.FFT_L),
                    batch=configs.FFT_BATCH, cfg_index=1)
    if name == "tiny":
        return dict(name="tiny_(2,4,4,2)", patterns=[configs.TINY_PATTERNS[0]], batch=configs.TINY_BATCH, cfg_index=0)
    table = {"vit_up": (configs.VIT_UP, configs.VIT_BATCH, 3), "vit_down": (configs.VIT_DOWN, configs.VIT_BATCH, 3),
             "gpt2_down": (configs.GPT2_DOWN, configs.GPT2_BATCH, 4), "gpt2_up": (configs.GPT2_UP, configs.GPT2_BATCH, 4)}
    pats, B, idx = table[name]
    return dict(name=name, patterns=pats, batch=B, cfg_index=idx)


def model_bytes(p, B):
    a, b, c, d = p
    return 4 * (B * a * c * d + a * b * c * d + B * a * b * d)


def model_flops(p, B):
    a, b, c, d = p
    return 2 * B * a * b * c * d


def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            return json.load(f), "measured"
    except Exception:
        return {"hbm_gbs": FALLBACK_HBM_GBS}, "fallback"


def ncu_traffic(workload_name, layout):
    """dram bytes per launch of the dominant kernel from the committed ncu
    capture (profiles/), or None."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            t = json.load(f)
        return t.get(f"{workload_name}:{layout}")
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled in the background."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self.proc = None
        self._t = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        self._t = threading.Thread(target=self._read, daemon=True)
        self._t.start()

    def _read(self):
        for line in self.proc.stdout:
            self.samples.append((time.time(), line.strip()))

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self, t0, t1):
        rows = [s for (t, s) in self.samples if t0 - 0.05 <= t <= t1 + 0.05] or \
               [s for (_, s) in self.samples[-5:]]
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            f = [x.strip() for x in r.split(",")]
            if len(f) < 6:
                continue
            try:
                sm.append(float(f[0]))
                mx = float(f[1])
            except ValueError:
                continue
            for n, v in zip(names, f[2:6]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def iqr(ts):
    if len(ts) < 4:
        return 0.0
    q = statistics.quantiles(ts, n=4)
    return q[2] - q[0]


# ------------------------------------------------------------- multi-GPU ----
class Ctx:
    """Process / device context of one rank."""

    def __init__(self):
        import torch
        import torch.distributed as tdist
        from paper_2405_15013_b200 import dist as kdist
        self.rank, self.world, self.local = kdist.env_rank_world()
        if self.world > 1 and not tdist.is_initialized():
            tdist.init_process_group("nccl", device_id=torch.device("cuda", self.local))
        torch.cuda.set_device(self.local)
        self.dev = torch.device("cuda", self.local)
        self.stream = torch.cuda.current_stream()
        props = torch.cuda.get_device_properties(self.dev)
        self.flush = torch.empty(2 * props.L2_cache_size, dtype=torch.uint8, device=self.dev)
        self.kdist = kdist

    def barrier(self):
        import torch.distributed as tdist
        if self.world > 1:
            tdist.barrier()

    def close(self):
        import torch.distributed as tdist
        if self.world > 1 and tdist.is_initialized():
            tdist.barrier()
            tdist.destroy_process_group()


def shard_input(B_global, N, rank, world, layout):
    """This rank's rows [lo, hi) of the one seeded global X (counter-based
    rows: identical bytes whatever the world size), in the requested layout."""
    import numpy as np
    import ksgen
    from paper_2405_15013_b200.dist import shard_bounds
    lo, hi = shard_bounds(B_global, world, rank)
    X = ksgen.x_rows_normal(np.arange(lo, hi), N, seed=0)
    return lo, hi, X, (X if layout == "bsf" else ksgen.to_bsl(X))


def verify_sharded(Y_local, lo, hi, layout, ref_fn, tol, err_fn, check=True):
    """Sampled rows of every rank's result shard, gathered to all ranks
    (dist.gather_samples) and, where check is set (rank 0), compared with
    ref_fn(global rows) (the oracle).  Returns the verify record (ok, error,
    rows, ranks), or None where check is not set."""
    from paper_2405_15013_b200 import dist as kdist
    rows = kdist.sample_rows(lo, hi)
    loc = [int(r - lo) for r in rows if r >= 0]
    if loc:
        vals = Y_local[loc] if layout == "bsf" else Y_local[:, loc].t()
        if len(loc) < len(rows):
            vals = vals[:1].expand(len(rows), -1)
    else:
        import torch
        M = Y_local.shape[1] if layout == "bsf" else Y_local.shape[0]
        vals = torch.zeros((len(rows), M), dtype=Y_local.dtype, device=Y_local.device)
    rows_all, vals_all = kdist.gather_samples(rows, vals.float().contiguous())
    if not check:
        return None
    rec = kdist.check_samples(rows_all, vals_all, ref_fn, err_fn)
    world = len(rows_all) // len(rows)
    rec.update({"ranks": world, "tolerance": tol, "ok": bool(rec["max_normwise_err"] <= tol)})
    return rec


def oracle_ref(pats, K4s, N):
    """ref_fn for verify_sharded: the FP64 oracle chain on the global rows
    (regenerated by counter from the same seed)."""
    import ksgen
    import oracle

    def ref(rows):
        return oracle.chain(pats, K4s, ksgen.x_rows_normal(rows, N, seed=0))
    return ref


# ------------------------------------------------------------- rooflines ----
def measure_peaks(ctx):
    """HBM (MEASURED_PEAKS.json), FP32 FFMA (ks_peak_ffma: an FFMA loop on this
    device) and TF32 tensor (torch.matmul 8192^3 with allow_tf32, cuBLAS, best of
    5) peaks.  FFMA / TF32 are measured live, rank 0's device."""
    import torch
    import paper_2405_15013_b200 as ksb
    peaks, src = measured_peaks()
    out = {"hbm_gbs": float(peaks.get("hbm_gbs", FALLBACK_HBM_GBS)), "hbm_source": src}
    out["ffma_tflops"] = round(ksb.peak_ffma_tflops(), 2)
    out["ffma_source"] = "measured: ks_peak_ffma (FFMA loop, 8 chains/thread, 1024 threads/SM)"
    n = 8192
    a = torch.randn(n, n, device=ctx.dev)
    b = torch.randn(n, n, device=ctx.dev)
    old = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = True
    for _ in range(2):
        a @ b
    best = 1e30
    for _ in range(5):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        a @ b
        e.record()
        e.synchronize()
        best = min(best, s.elapsed_time(e))
    torch.backends.cuda.matmul.allow_tf32 = old
    out["tf32_tflops"] = round(2 * n ** 3 / (best * 1e-3) / 1e12, 1)
    out["tf32_source"] = "measured: cuBLAS TF32 GEMM 8192^3 (torch.matmul, allow_tf32), best of 5"
    del a, b
    return out


def roofline_record(fam, bytes_per_launch, flops_per_launch, avg_ms, peaks):
    """Bound of the dominant kernel family: HBM, or its compute pipe (FFMA for
    the CUDA-core families, the TF32 tensor pipe for tcgen05) -- whichever
    takes longer at its measured peak; achieved and peak in that unit."""
    hbm = peaks["hbm_gbs"]
    t_mem = bytes_per_launch / (hbm * 1e9)
    if fam == "tf32":
        cpeak, bound_c = peaks["tf32_tflops"], "tensor"
    else:
        cpeak, bound_c = peaks["ffma_tflops"], "alu"
    t_cmp = flops_per_launch / (cpeak * 1e12)
    sec = avg_ms * 1e-3
    if t_mem >= t_cmp:
        ach = bytes_per_launch / sec / 1e9
        return {"bound": "hbm", "kernel": fam, "achieved": round(ach, 1), "peak": hbm, "unit": "GB/s",
                "frac": round(ach / hbm, 4), "peak_source": peaks["hbm_source"],
                "algorithmic_bytes_per_launch": int(bytes_per_launch),
                "algorithmic_flops_per_launch": int(flops_per_launch), "avg_launch_us": round(avg_ms * 1e3, 3),
                "hbm_gbs_achieved": round(ach, 1)}
    ach = flops_per_launch / sec / 1e12
    return {"bound": bound_c, "kernel": fam, "achieved": round(ach, 2), "peak": cpeak, "unit": "TFLOP/s",
            "frac": round(ach / cpeak, 4),
            "peak_source": peaks["tf32_source"] if fam == "tf32" else peaks["ffma_source"],
            "algorithmic_bytes_per_launch": int(bytes_per_launch),
            "algorithmic_flops_per_launch": int(flops_per_launch), "avg_launch_us": round(avg_ms * 1e3, 3),
            "hbm_gbs_achieved": round(bytes_per_launch / sec / 1e9, 1)}


def traced_families(ksb, pats, B, step_fn, ctx, K):
    """Per-launch CUDA events (library trace, on the launching stream) over K
    flushed steps -> per family: launches, total ms, bytes, flops."""
    ksb.trace_enable(True)
    for s in range(K):
        ctx.flush.fill_(s & 0xFF)
        step_fn()
    import torch
    torch.cuda.synchronize()
    k_ms, k_fam, k_bytes = ksb.trace_read()
    ksb.trace_enable(False)
    order = list(reversed(pats))             # application order, K_L first
    fam = {}
    for i, (ms_, f_, b_) in enumerate(zip(k_ms, k_fam, k_bytes)):
        p = order[i % len(order)]
        r = fam.setdefault(f_, {"n": 0, "ms": 0.0, "bytes": 0.0, "flops": 0.0})
        r["n"] += 1
        r["ms"] += float(ms_)
        r["bytes"] += float(b_)
        r["flops"] += model_flops(p, B)
    return fam


def time_steps(fn, ctx, K):
    """K steps, L2 flushed before each (untimed), one CUDA event pair per
    step on the launching stream -> list of ms."""
    import torch
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    for s in range(K):
        ctx.flush.fill_(s & 0xFF)
        ev[s][0].record(ctx.stream)
        fn()
        ev[s][1].record(ctx.stream)
    torch.cuda.synchronize()
    return [a.elapsed_time(b) for a, b in ev]


# --------------------------------------------------------------- our arm ----
def run_ours(args):
    import numpy as np
    import torch

    import ksgen
    import paper_2405_15013_b200 as ksb

    ctx = Ctx()
    ksb.load_library()
    kd = ctx.kdist
    wl = workload(args.workload)
    pats = wl["patterns"]
    Bg = args.batch or wl["batch"]
    L = len(pats)
    lay = args.layout
    K4s = [ksgen.k4_uniform(*p, seed=1000 + l) for l, p in enumerate(pats, 1)]
    facs = [ksb.Factor(*p, k) for p, k in zip(pats, K4s)]
    math_id = {"fp32": None, "tf32": ksb.MATH_TF32, "f32x3": ksb.MATH_F32X3}[args.math]
    if math_id is not None:
        for f in facs:
            f.set_math(math_id)
    tol = 5e-3 if args.math == "tf32" else 1e-5          # north star: 1e-5 FP32, 5e-3 TF32 (normwise, R9)
    dims = [pats[-1][0] * pats[-1][2] * pats[-1][3]] + [p[0] * p[1] * p[3] for p in reversed(pats)]
    lo, hi, X_host, X_host_l = shard_input(Bg, dims[0], ctx.rank, ctx.world, lay)
    B = hi - lo
    X = torch.from_numpy(X_host_l).to(ctx.dev)
    shape = (lambda n: (B, n)) if lay == "bsf" else (lambda n: (n, B))
    Y = torch.empty(shape(dims[-1]), device=ctx.dev)

    # The metric's byte model counts every factor's X/K/Y traffic, so
    # the headline leg runs the chain one fused KS kernel per factor; the fused
    # multi-factor chain (NEXT-1) is timed separately below ("fused_chain").
    ksb.set_chain_fusion(False)

    def step():
        """One pass of the hot path: the whole chain through the C ABI (ks_chain_ex)."""
        ksb.chain(facs, X, Y, layout=lay)

    for _ in range(max(args.warmup, 0)):
        step()
    torch.cuda.synchronize()

    K = args.steps
    sampler = ClockSampler(ctx.local)
    sampler.start()
    time.sleep(0.3)
    ctx.barrier()
    torch.cuda.synchronize()
    # Pass 1 (the headline): K steps, one event pair per step, no per-launch
    # instrumentation -- an event record between two launches costs ~5 us of
    # device time per launch and breaks the programmatic-dependent-launch overlap.
    l0 = ksb.launch_count()
    t0 = time.time()
    step_ms = time_steps(step, ctx, K)
    t1 = time.time()
    launches = ksb.launch_count() - l0
    # Pass 2 (the roofline): the same K steps with library-side CUDA events
    # around every launch on the launching stream -> per-launch time per family.
    fam = traced_families(ksb, pats, B, step, ctx, K)
    t2 = time.time()
    ctx.barrier()
    time.sleep(0.1)
    sampler.stop()
    clocks = sampler.summary(t0, t2)

    tot_ms = sum(step_ms)
    tot_ms_max = kd.max_over_ranks(tot_ms, ctx.dev)
    step_bytes = sum(model_bytes(p, B) for p in pats)
    all_bytes = kd.sum_over_ranks(step_bytes, ctx.dev)
    value = K * all_bytes / (tot_ms_max * 1e-3) / 1e9
    plans = [facs[l].plan(B, lay) for l in range(L - 1, -1, -1)]
    dom = max(fam, key=lambda f: fam[f]["ms"])
    d_ = fam[dom]
    traced_avg_ms = d_["ms"] / d_["n"]
    if d_["n"] == sum(r["n"] for r in fam.values()) and launches == d_["n"]:
        # every launch of the step is the dominant family: its average launch
        # duration is the event-timed step (pass 1, no per-launch instrumentation)
        # divided by the launches (per-launch event pairs add ~5 us each)
        avg_launch_ms = (tot_ms / K) / (launches / K)
        timing = ("pass-1 step time (CUDA events on the launching stream) / launches per step: "
                  "every launch of the step is this family")
    else:
        avg_launch_ms = traced_avg_ms
        timing = "per-launch CUDA events in a second pass of the same K steps"
    peaks = measure_peaks(ctx)
    roof = roofline_record(dom, d_["bytes"] / d_["n"], d_["flops"] / d_["n"], avg_launch_ms, peaks)
    roof.update({"traffic": ncu_traffic(wl["name"], lay), "traced_avg_launch_us": round(traced_avg_ms * 1e3, 3),
                 "share_of_step": round(d_["ms"] / sum(r["ms"] for r in fam.values()), 4), "timing": timing})

    # The same per-factor chain replayed from a CUDA graph (ks_chain_graph, a-7).
    graph = ksb.ChainGraph(facs, X, Y, layout=lay)
    for _ in range(3):
        graph.launch()
    torch.cuda.synchronize()
    ctx.barrier()
    g_ms = kd.max_over_ranks(sum(time_steps(graph.launch, ctx, K)), ctx.dev) / K
    cuda_graph = {"ms_per_step": round(g_ms, 5), "kernels_per_replay": graph.kernels,
                  "gbs": round(all_bytes / (g_ms * 1e-3) / 1e9, 2),
                  "vs_stream_launches": round((tot_ms_max / K) / g_ms, 4),
                  "note": "same launches captured once (ks_chain_graph) and replayed with one cudaGraphLaunch"}
    graph.free()

    # NEXT-1: the same chain as ONE fused launch (rows stay on chip across
    # factors).  Compulsory traffic: X + Y + every K once -> its own roofline.
    fused = None
    ksb.set_chain_fusion(True)
    if ksb.chain_fusion_eligible(facs, B, lay):
        Yf = torch.empty_like(Y)
        for _ in range(3):
            ksb.chain(facs, X, Yf, layout=lay)
        torch.cuda.synchronize()
        if not torch.equal(Yf, Y):
            raise RuntimeError("fused chain differs from the per-factor chain")
        ctx.barrier()
        fts = time_steps(lambda: ksb.chain(facs, X, Yf, layout=lay), ctx, K)
        f_ms = kd.max_over_ranks(float(np.median(fts)), ctx.dev)
        hbm_bytes = 4 * (B * dims[0] + sum(p[0] * p[1] * p[2] * p[3] for p in pats) + B * dims[-1])
        all_hbm = kd.sum_over_ranks(hbm_bytes, ctx.dev)
        fused = {"ms_per_chain": round(f_ms, 5), "iqr_ms": round(iqr(fts), 5), "launches_per_chain": 1,
                 "hbm_bytes_per_chain": int(all_hbm),
                 "effective_hbm_gbs": round(all_hbm / (f_ms * 1e-3) / 1e9, 1),
                 "model_gbs_equivalent": round(all_bytes / (f_ms * 1e-3) / 1e9, 1),
                 "roofline": {"bound": "hbm", "achieved": round(hbm_bytes / (f_ms * 1e-3) / 1e9, 1),
                              "peak": peaks["hbm_gbs"], "unit": "GB/s",
                              "frac": round(hbm_bytes / (f_ms * 1e-3) / 1e9 / peaks["hbm_gbs"], 4),
                              "note": "compulsory traffic X + Y + nnz(K) of the whole chain"},
                 "speedup_vs_per_factor_chain": round((tot_ms_max / K) / f_ms, 3),
                 "bit_identical_to_per_factor": True,
                 "note": "NEXT-1 fused multi-factor chain (SURVEY §8f); median of K flushed steps"}
    ksb.set_chain_fusion(False)

    # e2e through the C ABI with HOST buffers (pinned), copies inside the region
    e2e = None
    if not args.no_e2e:
        Xh = torch.from_numpy(X_host_l).pin_memory()
        Yh = torch.empty(shape(dims[-1]), dtype=torch.float32).pin_memory()
        ke = max(3, min(K, 20))
        for _ in range(2):
            ksb.chain_host(facs, Xh, Yh, layout=lay)
        torch.cuda.synchronize()
        ctx.barrier()
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(ke)]
        for s in range(ke):
            evs[s][0].record(ctx.stream)
            ksb.chain_host(facs, Xh, Yh, layout=lay)
            evs[s][1].record(ctx.stream)
        torch.cuda.synchronize()
        e_ms = kd.max_over_ranks(sum(a.elapsed_time(b) for a, b in evs), ctx.dev)
        e2e = {"value": round(ke * all_bytes / (e_ms * 1e-3) / 1e9, 2),
               "unit": "GB/s", "h2d_bytes_per_step": int(Xh.numel() * 4),
               "d2h_bytes_per_step": int(Yh.numel() * 4), "api": "ks_chain_host", "steps": ke}
        step()
        torch.cuda.synchronize()
        if not torch.equal(Yh, Y.cpu()):
            raise RuntimeError("e2e result differs from device-resident result")

    verify = None
    if not args.no_verify:
        import oracle
        verify = verify_sharded(Y, lo, hi, lay, oracle_ref(pats, K4s, dims[0]), tol, oracle.normwise_error,
                                check=ctx.rank == 0)

    models = None
    if not args.no_models and args.workload == "fft":
        models = run_models(ctx, args, peaks)

    line = None
    if ctx.rank == 0:
        ok = (verify is None or verify["ok"]) and all(
            (m.get("verify") or {}).get("ok", True) for m in (models or {}).values() if isinstance(m, dict))
        line = {
            "metric": METRIC, "value": round(value, 2) if ok else None, "unit": "GB/s", "n_gpus": ctx.world,
            "steps": K, "warmup": args.warmup, "ms_per_step": round(tot_ms_max / K, 5),
            "iqr_ms_per_step": round(iqr(step_ms), 5),
            "higher_is_better": True, "scaling": "strong",
            "scaling_note": "the configuration's global batch is partitioned over the ranks (SURVEY §8e, B_g = "
                            "ceil(B/G)); value = all ranks' byte-model bytes / max-over-ranks device time",
            "vs_baseline": None,
            "dtype": {"fp32": "f32", "tf32": "tf32 (fp32 accumulate)", "f32x3": "3xtf32 (fp32-accurate)"}[args.math],
            "data": "synthetic (X ~ N(0,1) rows by counter, K ~ U[-1/sqrt(c),1/sqrt(c)], PAPER.md:1220), seeded",
            "config": {"workload": wl["name"], "baseline_config_index": wl["cfg_index"],
                       "patterns": [list(p) for p in pats], "global_batch": Bg,
                       "batch_per_gpu": int(hi - lo), "batch_shards": ctx.world,
                       "layout": lay, "math": args.math,
                       "parallelism": f"batch-partitioned x{ctx.world}, no collective on the compute path",
                       "l2": "flushed between timed steps (2x L2 write, untimed)",
                       "bytes_per_step_all_ranks": int(all_bytes)},
            "hbm_frac_of_" + peaks["hbm_source"]: round(value / ctx.world / peaks["hbm_gbs"], 4),
            "roofline": roof,
            "peaks": peaks,
            "gpu_launches": int(launches),
            "launches_per_step": launches / K,
            "kernel_ms_per_step": round(sum(r["ms"] for r in fam.values()) / K, 5),
            "fused_chain": fused,
            "cuda_graph": cuda_graph,
            "clocks": clocks,
            "e2e": e2e,
            "plans": plans,
            "verify": verify,
        }
        if models is not None:
            line["models"] = models
    if not args.no_baselines and ctx.rank == 0:
        line["baselines"] = chain_baselines(pats, K4s, X, lay, args.math, ctx, tot_ms_max / K)
    if not args.no_cpu_baseline and ctx.world == 1:
        line["cpu_baseline"] = cpu_baseline(pats, K4s, B, dims[0], budget_s=15.0)
    if not args.no_sweep and ctx.world == 1:
        line["sweep"] = run_sweeps(ctx, peaks, args.sweep_reps)
    ctx.close()
    return line


def run_models(ctx, args, peaks):
    """configs[3] / configs[4]: the ViT-S/16 and GPT-2 medium MLP KSLinear chains
    (BSF, the paper's end-to-end layout), FP32 and TF32, on this
    rank's shard of the configuration's batch."""
    out = {}
    for name in MODEL_WORKLOADS:
        for math in ("fp32", "tf32"):
            out[f"{name}:{math}"] = run_model_entry(ctx, name, math, args, peaks)
    return out


def run_model_entry(ctx, name, math, args, peaks):
    import torch

    import ksgen
    import paper_2405_15013_b200 as ksb
    kd = ctx.kdist
    wl = workload(name)
    pats = wl["patterns"]
    Bg = wl["batch"]
    K4s = [ksgen.k4_uniform(*p, seed=1000 + l) for l, p in enumerate(pats, 1)]
    facs = [ksb.Factor(*p, k) for p, k in zip(pats, K4s)]
    if math == "tf32":
        for f in facs:
            f.set_math(ksb.MATH_TF32)
    N = ksgen.configs.chain_dims(pats)[0]
    lo, hi, X_host, _ = shard_input(Bg, N, ctx.rank, ctx.world, "bsf")
    B = hi - lo
    X = torch.from_numpy(X_host).to(ctx.dev)
    Y = torch.empty((B, facs[0].M), device=ctx.dev)

    def step():
        ksb.chain(facs, X, Y, layout="bsf")

    for _ in range(3):
        step()
    torch.cuda.synchronize()
    K = max(10, min(args.steps, 20))
    ctx.barrier()
    ts = time_steps(step, ctx, K)
    ms = kd.max_over_ranks(statistics.median(ts), ctx.dev)
    fam = traced_families(ksb, pats, B, step, ctx, 3)
    dom = max(fam, key=lambda f: fam[f]["ms"])
    d_ = fam[dom]
    roof = roofline_record(dom, d_["bytes"] / d_["n"], d_["flops"] / d_["n"], d_["ms"] / d_["n"], peaks)
    roof["share_of_step"] = round(d_["ms"] / sum(r["ms"] for r in fam.values()), 4)
    step_bytes = sum(model_bytes(p, B) for p in pats)
    step_flops = sum(model_flops(p, B) for p in pats)
    all_bytes = kd.sum_over_ranks(step_bytes, ctx.dev)
    all_flops = kd.sum_over_ranks(step_flops, ctx.dev)
    rec = {"patterns": [list(p) for p in pats], "global_batch": Bg, "batch_per_gpu": B,
           "ms_per_chain": round(ms, 5), "iqr_ms": round(iqr(ts), 5),
           "gbs": round(all_bytes / (ms * 1e-3) / 1e9, 1), "tflops": round(all_flops / (ms * 1e-3) / 1e12, 2),
           "plans": [f.plan(B, "bsf") for f in reversed(facs)],
           "kernel_families_ms": {k: round(v["ms"] / 3, 5) for k, v in fam.items()},
           "roofline": roof}
    if not args.no_baselines:
        rec["baselines"] = chain_baselines(pats, K4s, X, "bsf", math, ctx, ms, reps=5)
    if not args.no_verify:
        import oracle
        tol = 5e-3 if math == "tf32" else 1e-5
        rec["verify"] = verify_sharded(Y, lo, hi, "bsf", oracle_ref(pats, K4s, N), tol, oracle.normwise_error,
                                       check=ctx.rank == 0)
    for f in facs:
        f.free()
    del X, Y
    torch.cuda.empty_cache()
    return rec


def run_sweeps(ctx, peaks, reps):
    """configs[2]: medians vs bmm+permute in FP32, TF32 (north star) and the
    FP32-accurate 3xTF32 / BF16 modes; FP32 judged against the measured FFMA
    peak, TF32 against HBM."""
    from bench_sweep import run_sweep
    sw = {}
    for math in ("fp32", "tf32", "f32x3", "bf16"):
        r = run_sweep(ctx.dev, reps=reps, math=math)
        rows = r.pop("rows")
        if math == "fp32":
            fr = [max(x["bsf_ks_tflops"], x["bsl_ks_tflops"]) / peaks["ffma_tflops"] for x in rows]
            r["median_frac_of_ffma_peak_bsf"] = round(statistics.median(
                x["bsf_ks_tflops"] / peaks["ffma_tflops"] for x in rows), 4)
            r["median_frac_of_ffma_peak_bsl"] = round(statistics.median(
                x["bsl_ks_tflops"] / peaks["ffma_tflops"] for x in rows), 4)
            r["median_frac_of_ffma_peak_best_layout"] = round(statistics.median(fr), 4)
        if math == "tf32":
            r["median_frac_of_hbm_bsf"] = round(statistics.median(x["bsf_ks_gbs"] for x in rows) / peaks["hbm_gbs"], 4)
            r["median_frac_of_hbm_bsl"] = round(statistics.median(x["bsl_ks_gbs"] for x in rows) / peaks["hbm_gbs"], 4)
        r["median_iqr_over_median"] = round(statistics.median(
            max(x.get("bsf_ks_iqr_ms", 0) / x["bsf_ks_ms"], x.get("bsl_ks_iqr_ms", 0) / x["bsl_ks_ms"])
            for x in rows), 4)
        sw[math] = r
    return sw


def cpu_baseline(pats, K4s, B, N, budget_s=15.0):
    """The oracle as it stands, on this host's cores, on a bounded row sample
    (rows doubled until one timed run takes >= budget/3 seconds)."""
    import numpy as np
    import ksgen
    import oracle
    threads = oracle.default_threads()
    X0 = ksgen.x_rows_normal([0], N, seed=0)
    oracle.chain(pats, K4s, X0, threads=threads)      # warm (page-in, build)
    R = 1
    while True:
        Xs = ksgen.x_rows_normal(np.arange(R), N, seed=0)
        t = time.time()
        oracle.chain(pats, K4s, Xs, threads=threads)
        dt = time.time() - t
        if dt >= budget_s / 3 or R >= B or dt * 2.2 > budget_s:
            break
        R = min(B, R * 2)
    byts = sum(model_bytes(p, R) for p in pats)
    return {"value": round(byts / dt / 1e9, 6), "unit": "GB/s", "cores": threads, "kind": "oracle",
            "sample": f"{R} of {B} batch rows of the workload, FP64 naive dense triple loop (oracle/ks_oracle.c)",
            "seconds": round(dt, 3)}


def chain_baselines(pats, K4s, X, lay, math, ctx, ks_ms, reps=10):
    """The same chain through the paper's bmm+permute listing (App. A,
    PAPER.md:813-832, one bmm + two permutation copies per factor) and through
    one dense cuBLAS GEMM with the collapsed product W = K_1...K_L (PAPER.md:
    892-897), same inputs, L2 flushed before every rep, median.
    Timing only: the library never calls these."""
    import numpy as np
    import torch
    from bench_sweep import bmm_bsf, bmm_bsl
    torch.backends.cuda.matmul.allow_tf32 = (math == "tf32")   # f32x3 vs true-FP32 baselines
    Kbs = [torch.from_numpy(k.transpose(0, 3, 1, 2).reshape(p[0] * p[3], p[1], p[2]).copy()).to(ctx.dev)
           for p, k in zip(pats, K4s)]
    bfn = bmm_bsf if lay == "bsf" else bmm_bsl

    def bmm_chain():
        Z = X
        for p, Kb in zip(reversed(pats), reversed(Kbs)):
            Z = bfn(Z, Kb, *p)
        return Z

    def dense_of(p, k):
        a, b, c, d = p
        D = np.zeros((a * b * d, a * c * d), dtype=np.float64)
        for i in range(a):
            for j in range(d):
                D[np.ix_(i * b * d + np.arange(b) * d + j, i * c * d + np.arange(c) * d + j)] = k[i, :, :, j]
        return D
    W = torch.from_numpy(dense_of(pats[0], K4s[0])).to(ctx.dev)
    for p, k in zip(pats[1:], K4s[1:]):
        W = W @ torch.from_numpy(dense_of(p, k)).to(ctx.dev)          # FP64 product on the device
    Wt = W.float().contiguous()
    del W

    def dense():
        return X @ Wt.t() if lay == "bsf" else Wt @ X

    def timeit(fn):
        for _ in range(3):
            fn()
        ts = time_steps(fn, ctx, reps)
        return float(np.median(ts))
    t_bmm, t_dense = timeit(bmm_chain), timeit(dense)
    torch.backends.cuda.matmul.allow_tf32 = False
    return {"bmm_permute_ms": round(t_bmm, 5), "dense_cublas_ms": round(t_dense, 5),
            "speedup_vs_bmm_permute": round(t_bmm / ks_ms, 4), "speedup_vs_dense": round(t_dense / ks_ms, 4),
            "allow_tf32": math == "tf32",
            "note": f"same chain, same inputs: paper's bmm+permute listing per factor (App. A) and one dense "
                    f"cuBLAS GEMM with W = K_1...K_L; median of {reps} L2-flushed reps"}


# --------------------------------------------------------- reference arm ----
def run_reference(args):
    """The CPU oracle timed as the reference arm (this tier has no reference code)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return None
    import numpy as np
    import ksgen
    import oracle
    wl = workload(args.workload)
    pats = wl["patterns"]
    B = args.batch or wl["batch"]
    K4s = [ksgen.k4_uniform(*p, seed=1000 + l) for l, p in enumerate(pats, 1)]
    N = pats[-1][0] * pats[-1][2] * pats[-1][3]
    threads = oracle.default_threads()
    budget = 150.0
    steps, warm = max(args.steps, 1), max(args.warmup, 0)
    # rows per step: fill the threads once if the budget allows, else 1
    t = time.time()
    X1 = ksgen.x_rows_normal([0], N, seed=0)
    oracle.chain(pats, K4s, X1, threads=threads)
    t1 = max(time.time() - t, 1e-4)
    R = max(1, min(threads, int(budget / (steps + warm) / t1)))
    Xs = ksgen.x_rows_normal(np.arange(R), N, seed=0)
    for _ in range(warm):
        oracle.chain(pats, K4s, Xs, threads=threads)
    t = time.time()
    for _ in range(steps):
        oracle.chain(pats, K4s, Xs, threads=threads)
    dt = time.time() - t
    byts = sum(model_bytes(p, R) for p in pats)
    v = steps * byts / dt / 1e9
    return {"impl": "reference", "metric": METRIC, "value": round(v, 6), "unit": "GB/s", "n_gpus": args.gpus,
            "steps": steps, "warmup": warm, "ms_per_step": round(dt / steps * 1e3, 3),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic, seeded", "config": {"workload": wl["name"], "baseline_config_index": wl["cfg_index"],
                                                     "global_batch": B, "batch_per_step": R, "layout": "bsf"},
            "cpu_baseline": {"value": round(v, 6), "unit": "GB/s", "cores": threads, "kind": "oracle",
                             "sample": f"{R} of {B} batch rows per step"},
            "e2e": {"value": round(v, 6), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def main(argv=None):
    args = parse_args(argv)
    line = run_reference(args) if args.impl == "reference" else run_ours(args)
    if line is not None:
        print(json.dumps(line), flush=True)
        if line.get("impl") != "reference" and line.get("value") is None:
            sys.exit(1)          # an oracle check failed: the record carries no value


if __name__ == "__main__":
    main()
