#!/usr/bin/env python
"""bench.py -- KS matmul on B200 (arXiv 2405.15013 hot path).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload fft] [--impl ours|reference]

Default workload = BASELINE.json configs[1]: the FFT-style butterfly chain,
N = 4096, 12 factors (2^{l-1},2,2,2^{12-l}), B = 8192 per GPU, FP32, BSF.
One *step* = one pass of the whole hot path over one batch: the 12 fused
factor launches of the chain (K_12 first), inputs resident in HBM.

metric: achieved GB/s with the paper's byte model (read X + nnz(K) + write Y
per factor), summed over the factors, divided
by device time.  Multi-GPU (torchrun): the batch is partitioned (weak scaling,
each rank runs its own B), no collective on the compute path, value = all
ranks' bytes / max over ranks of the device time.

Prints ONE JSON line on rank 0.
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
    ap.add_argument("--batch", type=int, default=None, help="per-GPU batch override")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-sweep", action="store_true", help="skip the configs[2] sweep vs bmm+permute")
    ap.add_argument("--no-verify", action="store_true", help="skip the oracle check of sampled rows")
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
        self.window = None
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


# --------------------------------------------------------------- our arm ----
def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    import ksgen
    import paper_2405_15013_b200 as ksb

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    ksb.load_library()

    wl = workload(args.workload)
    pats = wl["patterns"]
    B = args.batch or wl["batch"]
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
    X_host = ksgen.x_normal(B, dims[0], seed=rank)
    X_host_l = X_host if lay == "bsf" else ksgen.to_bsl(X_host)
    X = torch.from_numpy(X_host_l).to(dev)
    shape = (lambda n: (B, n)) if lay == "bsf" else (lambda n: (n, B))
    bufs = [torch.empty(shape(max(dims[1:-1] or [1])), device=dev) for _ in range(2)]
    Y = torch.empty(shape(dims[-1]), device=dev)
    stream = torch.cuda.current_stream()
    props = torch.cuda.get_device_properties(dev)
    flush = torch.empty(2 * props.L2_cache_size, dtype=torch.uint8, device=dev)

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
    ev_step = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.3)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    # Pass 1 (the headline): K steps, one event pair per step, no per-launch
    # instrumentation -- an event record between two launches costs ~5 us of
    # device time per launch (measured: 611 vs 545 us per FFT chain) and breaks
    # the programmatic-dependent-launch overlap of consecutive factors.
    l0 = ksb.launch_count()
    t0 = time.time()
    for s in range(K):
        flush.fill_(s & 0xFF)                 # evict L2 between timed steps (not timed)
        ev_step[s][0].record(stream)
        step()
        ev_step[s][1].record(stream)
    torch.cuda.synchronize()
    t1 = time.time()
    launches = ksb.launch_count() - l0
    # Pass 2 (the roofline): the same K steps with library-side CUDA events around
    # every launch on the launching stream -> per-launch device time per family.
    ksb.trace_enable(True)
    ev_tr = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    for s in range(K):
        flush.fill_(s & 0xFF)
        ev_tr[s][0].record(stream)
        step()
        ev_tr[s][1].record(stream)
    torch.cuda.synchronize()
    t2 = time.time()
    k_ms, k_fam, k_bytes = ksb.trace_read()
    ksb.trace_enable(False)
    if world > 1:
        dist.barrier()
    time.sleep(0.1)
    sampler.stop()
    clocks = sampler.summary(t0, t2)

    step_ms = [a.elapsed_time(b) for a, b in ev_step]
    tot_ms = sum(step_ms)
    tr_ms = sum(a.elapsed_time(b) for a, b in ev_tr)
    plans = [facs[l].plan(B, lay) for l in range(L - 1, -1, -1)]
    fam_time, fam_bytes, fam_n = {}, {}, {}
    for ms_, f_, b_ in zip(k_ms, k_fam, k_bytes):
        fam_time[f_] = fam_time.get(f_, 0.0) + float(ms_)
        fam_bytes[f_] = fam_bytes.get(f_, 0.0) + float(b_)
        fam_n[f_] = fam_n.get(f_, 0) + 1
    dom = max(fam_time, key=fam_time.get)

    tot_t = torch.tensor([tot_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(tot_t, op=dist.ReduceOp.MAX)
    tot_ms_max = float(tot_t.item())
    step_bytes = sum(model_bytes(p, B) for p in pats)
    value = world * K * step_bytes / (tot_ms_max * 1e-3) / 1e9

    # The same per-factor chain replayed from a CUDA graph (ks_chain_graph,
    # SURVEY §8a a-7): one cudaGraphLaunch per step instead of L host launches.
    cuda_graph = None
    graph = ksb.ChainGraph(facs, X, Y, layout=lay)
    for _ in range(3):
        graph.launch()
    torch.cuda.synchronize()
    evg = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    if world > 1:
        dist.barrier()
    for s in range(K):
        flush.fill_(s & 0xFF)
        evg[s][0].record(stream)
        graph.launch()
        evg[s][1].record(stream)
    torch.cuda.synchronize()
    g_ms = torch.tensor([sum(a.elapsed_time(b) for a, b in evg)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(g_ms, op=dist.ReduceOp.MAX)
    g_ms = float(g_ms.item()) / K
    cuda_graph = {"ms_per_step": round(g_ms, 5), "kernels_per_replay": graph.kernels,
                  "gbs": round(world * step_bytes / (g_ms * 1e-3) / 1e9, 2),
                  "vs_stream_launches": round((tot_ms_max / K) / g_ms, 4),
                  "note": "same launches captured once (ks_chain_graph) and replayed with one cudaGraphLaunch"}
    graph.free()

    # NEXT-1: the same chain as ONE fused launch (rows stay in shared memory
    # across factors).  Traffic it must move: X + Y + every K once.
    fused = None
    ksb.set_chain_fusion(True)
    if ksb.chain_fusion_eligible(facs, B, lay):
        Yf = torch.empty_like(Y)
        for _ in range(3):
            ksb.chain(facs, X, Yf, layout=lay)
        torch.cuda.synchronize()
        if not torch.equal(Yf, Y):
            raise RuntimeError("fused chain differs from the per-factor chain")
        kf = K
        evf = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(kf)]
        if world > 1:
            dist.barrier()
        for s in range(kf):
            flush.fill_(s & 0xFF)
            evf[s][0].record(stream)
            ksb.chain(facs, X, Yf, layout=lay)
            evf[s][1].record(stream)
        torch.cuda.synchronize()
        f_ms = float(np.median([a.elapsed_time(b) for a, b in evf]))
        f_max = torch.tensor([f_ms], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(f_max, op=dist.ReduceOp.MAX)
        f_ms = float(f_max.item())
        hbm_bytes = 4 * (B * dims[0] + sum(p[0] * p[1] * p[2] * p[3] for p in pats) + B * dims[-1])
        fused = {"ms_per_chain": round(f_ms, 5), "launches_per_chain": 1,
                 "hbm_bytes_per_chain": hbm_bytes,
                 "effective_hbm_gbs": round(hbm_bytes / (f_ms * 1e-3) / 1e9, 1),
                 "model_gbs_equivalent": round(step_bytes / (f_ms * 1e-3) / 1e9, 1),
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
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(ke)]
        if world > 1:
            dist.barrier()
        for s in range(ke):
            evs[s][0].record(stream)
            ksb.chain_host(facs, Xh, Yh, layout=lay)
            evs[s][1].record(stream)
        torch.cuda.synchronize()
        e_ms = torch.tensor([sum(a.elapsed_time(b) for a, b in evs)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(e_ms, op=dist.ReduceOp.MAX)
        e2e = {"value": round(world * ke * step_bytes / (float(e_ms.item()) * 1e-3) / 1e9, 2),
               "unit": "GB/s", "h2d_bytes_per_step": int(Xh.numel() * 4),
               "d2h_bytes_per_step": int(Yh.numel() * 4), "api": "ks_chain_host", "steps": ke}
        # the e2e result must equal the device-resident one
        step()
        torch.cuda.synchronize()
        if not torch.equal(Yh, Y.cpu()):
            raise RuntimeError("e2e result differs from device-resident result")

    # verification (outside the timed region): sampled rows of every rank's Y,
    # gathered to all ranks over NCCL, checked on rank 0 against the oracle
    vrows = np.array(sorted({0, 1, B // 2, B - 1}))
    Yc = Y.cpu().numpy()
    samp = torch.from_numpy(np.ascontiguousarray(Yc[vrows] if lay == "bsf" else Yc[:, vrows].T)).to(dev)
    parts = [samp]
    if world > 1:
        parts = [torch.empty_like(samp) for _ in range(world)]
        dist.all_gather(parts, samp)

    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return None
    verify = None
    if not args.no_verify:
        import oracle
        errs = []
        for r, part in enumerate(parts):
            Xr = X_host if r == rank else ksgen.x_normal(B, dims[0], seed=r)
            ref = oracle.chain(pats, K4s, Xr, rows=vrows)
            errs.append(oracle.normwise_error(part.cpu().numpy(), ref))
        verify = {"rows_per_rank": len(vrows), "ranks": world, "max_normwise_err": max(errs),
                  "tolerance": tol, "ok": bool(max(errs) <= tol)}

    peaks, src = measured_peaks()
    peak = float(peaks.get("hbm_gbs", FALLBACK_HBM_GBS))
    traced_avg_ms = fam_time[dom] / fam_n[dom]
    bytes_per_launch = fam_bytes[dom] / fam_n[dom]
    if fam_n[dom] == sum(fam_n.values()) and launches == fam_n[dom]:
        # every launch of the step is the dominant family: its average launch
        # duration is the event-timed step (pass 1, no per-launch instrumentation)
        # divided by the launches -- per-launch event pairs add ~5 us each and
        # serialise the programmatic-dependent-launch overlap
        avg_launch_ms = (tot_ms_max / K) / (launches / K)
        timing = ("pass-1 step time (CUDA events on the launching stream, max over ranks) / launches per step: "
                  "every launch of the step is this family")
    else:
        avg_launch_ms = traced_avg_ms
        timing = ("per-launch CUDA events in a second pass of the same K steps (pass 1, the headline, has no "
                  "per-launch events)")
    achieved = bytes_per_launch / (avg_launch_ms * 1e-3) / 1e9
    line = {
        "metric": METRIC, "value": round(value, 2), "unit": "GB/s", "n_gpus": world,
        "steps": K, "warmup": args.warmup, "ms_per_step": round(tot_ms_max / K, 5),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": {"fp32": "f32", "tf32": "tf32 (fp32 accumulate)", "f32x3": "3xtf32 (fp32-accurate)"}[args.math],
        "data": "synthetic (X ~ N(0,1), K ~ U[-1/sqrt(c),1/sqrt(c)], PAPER.md:1220), seeded",
        "config": {"workload": wl["name"], "baseline_config_index": wl["cfg_index"],
                   "patterns": [list(p) for p in pats], "batch_per_gpu": B, "global_batch": B * world,
                   "layout": lay, "math": args.math, "parallelism": f"batch-partitioned x{world}, no collective",
                   "l2": "flushed between timed steps (2x L2 write, untimed)",
                   "bytes_per_step_per_gpu": step_bytes},
        "hbm_frac_of_" + src: round(value / world / peak, 4),
        "roofline": {"bound": "hbm", "kernel": dom, "achieved": round(achieved, 1), "peak": peak,
                     "peak_source": src, "unit": "GB/s", "frac": round(achieved / peak, 4),
                     "traffic": ncu_traffic(wl["name"], lay),
                     "algorithmic_bytes_per_launch": int(bytes_per_launch),
                     "avg_launch_us": round(avg_launch_ms * 1e3, 3),
                     "traced_avg_launch_us": round(traced_avg_ms * 1e3, 3),
                     "share_of_step": round(fam_time[dom] / tr_ms, 4),
                     "timing": timing},
        "gpu_launches": int(launches),
        "launches_per_step": launches / K,
        "kernel_ms_per_step": round(sum(fam_time.values()) / K, 5),
        "ms_per_step_traced": round(tr_ms / K, 5),
        "fused_chain": fused,
        "cuda_graph": cuda_graph,
        "clocks": clocks,
        "e2e": e2e,
        "plans": plans,
    }
    line["verify"] = verify
    if not args.no_baselines:
        line["baselines"] = chain_baselines(pats, K4s, X, lay, args.math, flush, stream, tot_ms_max / K, dev)
    if not args.no_cpu_baseline and world == 1:
        line["cpu_baseline"] = cpu_baseline(pats, K4s, X_host, B, budget_s=15.0)
    if not args.no_sweep and world == 1:
        # second half of the metric: configs[2] median speedup vs bmm+permute
        from bench_sweep import run_sweep
        sw = {}
        for math in ("fp32", "f32x3", "tf32", "bf16"):
            r = run_sweep(dev, reps=5, math=math)
            r.pop("rows")
            sw[math] = r
        line["sweep"] = sw
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return line


def cpu_baseline(pats, K4s, X_host, B, budget_s=15.0):
    """The oracle as it stands, on this host's cores, on a bounded row sample
    (rows doubled until one timed run takes >= budget/3 seconds)."""
    import oracle
    import numpy as np
    threads = oracle.default_threads()
    oracle.chain(pats, K4s, X_host, rows=[0], threads=threads)      # warm (page-in, build)
    R = 1
    while True:
        t = time.time()
        oracle.chain(pats, K4s, X_host, rows=np.arange(R), threads=threads)
        dt = time.time() - t
        if dt >= budget_s / 3 or R >= B or dt * 2.2 > budget_s:
            break
        R = min(B, R * 2)
    byts = sum(model_bytes(p, R) for p in pats)
    return {"value": round(byts / dt / 1e9, 6), "unit": "GB/s", "cores": threads, "kind": "oracle",
            "sample": f"{R} of {B} batch rows of the workload, FP64 naive dense triple loop (oracle/ks_oracle.c)",
            "seconds": round(dt, 3)}


def chain_baselines(pats, K4s, X, lay, math, flush, stream, ks_ms, dev, reps=10):
    """The same chain through the paper's bmm+permute listing (App. A,
    PAPER.md:813-832, one bmm + two permutation copies per factor) and through
    one dense cuBLAS GEMM with the collapsed product W = K_1...K_L (PAPER.md:
    892-897), same inputs, L2 flushed before every rep, median.
    Timing only: the library never calls these."""
    import numpy as np
    import torch
    from bench_sweep import bmm_bsf, bmm_bsl
    torch.backends.cuda.matmul.allow_tf32 = (math == "tf32")   # f32x3 vs true-FP32 baselines
    Kbs = [torch.from_numpy(k.transpose(0, 3, 1, 2).reshape(p[0] * p[3], p[1], p[2]).copy()).to(dev)
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
    W = torch.from_numpy(dense_of(pats[0], K4s[0])).to(dev)
    for p, k in zip(pats[1:], K4s[1:]):
        W = W @ torch.from_numpy(dense_of(p, k)).to(dev)          # FP64 product on the device
    Wt = W.float().contiguous()
    del W

    def dense():
        return X @ Wt.t() if lay == "bsf" else Wt @ X

    def timeit(fn):
        for _ in range(3):
            fn()
        ts = []
        for r in range(reps):
            flush.fill_(r & 0xFF)
            s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s0.record(stream)
            fn()
            s1.record(stream)
            s1.synchronize()
            ts.append(s0.elapsed_time(s1))
        return float(np.median(ts))
    t_bmm, t_dense = timeit(bmm_chain), timeit(dense)
    torch.backends.cuda.matmul.allow_tf32 = False
    return {"bmm_permute_ms": round(t_bmm, 5), "dense_cublas_ms": round(t_dense, 5),
            "speedup_vs_bmm_permute": round(t_bmm / ks_ms, 4), "speedup_vs_dense": round(t_dense / ks_ms, 4),
            "allow_tf32": math == "tf32",
            "note": "same chain, same inputs: paper's bmm+permute listing per factor (App. A) and one dense "
                    "cuBLAS GEMM with W = K_1...K_L; median of 10 L2-flushed reps"}


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
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic, seeded", "config": {"workload": wl["name"], "baseline_config_index": wl["cfg_index"],
                                                     "batch_per_step": R, "layout": "bsf"},
            "cpu_baseline": {"value": round(v, 6), "unit": "GB/s", "cores": threads, "kind": "oracle",
                             "sample": f"{R} of {B} batch rows per step"},
            "e2e": {"value": round(v, 6), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def main(argv=None):
    args = parse_args(argv)
    line = run_reference(args) if args.impl == "reference" else run_ours(args)
    if line is not None:
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
