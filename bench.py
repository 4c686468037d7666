#!/usr/bin/env python
"""Benchmark of the q-adic transform pipeline on B200 (one JSON line).

Headline workload (BASELINE.json configs[1], "C2"): batched REDQ of 2^26 fp64
words (7 digits at q = 2^7, p = 5, float_premul + window-4 correction table)
per GPU per step -> 7 residues/word as uint8.  Multi-GPU: one process per GPU,
each rank reduces its own 2^26-word shard of the seeded stream (weak scaling,
no data-path collective); time = max over ranks.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

value     residues/s over all ranks, inputs resident in HBM (CUDA events on
          the launching stream, K back-to-back steps, barrier + sync around)
e2e       same metric through the C-ABI host entry point
          (qpk_redq_residues_f64_host): pinned host words in, H2D + kernel +
          D2H inside the timed region every step
roofline  HBM: 15 B/word algorithmic (8 in + 7 out) / kernel time vs the
          measured copy bandwidth in MEASURED_PEAKS.json
cpu_baseline  the reference's own CPU path (oracle/_ref, built from
          /root/reference unmodified) on a bounded sample, all host threads
secondary the other BASELINE configs (C1, C3 both paths, C4, C5) measured
          the same way with their own rooflines (N = 1 only)
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

METRIC = "redq_residues_per_s"
UNIT = "residues/s"
N_WORDS = 1 << 26
ND = 7
ALGO_BYTES_PER_WORD = 8 + ND
WORKLOAD = "C2 batched REDQ: 2^26 fp64 words/GPU, p=5, q=2^7, d=6, float_premul + window-4 table -> 7 uint8 residues/word"


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        return float(pk["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_traffic(kernel_key):
    """dram bytes per launch of `kernel_key` from the committed ncu summary."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as f:
            s = json.load(f)
        return s[kernel_key]["dram_bytes_per_launch"]
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed regions."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.samples = []
        self.proc = None
        self.active = False
        self.t = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        self.t = threading.Thread(target=self._read, daemon=True)
        self.t.start()

    def _read(self):
        for line in self.proc.stdout:
            if self.active:
                self.samples.append([x.strip() for x in line.split(",")])

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > i + 2 and s[i + 2].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


# ---------------------------------------------------------------- reference
def run_reference(args, rank):
    """The reference's own CPU implementation (oracle/_ref when built here,
    else the C restatement) on the host cores, same metric/config."""
    import numpy as np

    import oracle as O

    threads = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
    use_ref = O.ref() is not None
    kind = "reference" if use_ref else "port"

    def words_for(n):
        dr = O.draws(0x07100510 + 2, n * ND, 128).reshape(n, ND).astype(np.uint64)
        w = np.zeros(n, np.uint64)
        for j in range(ND):
            w = w * np.uint64(128) + dr[:, j]
        return w.astype(np.float64)

    def run(words):
        if use_ref:
            out, ns, _ = O.ref_redq_f64(5, 128, 6, words, float_mode=True, window=4, threads=threads)
            return ns * 1e-9
        t0 = time.perf_counter()
        O.redq_f64(5, 128, 6, words, float_mode=True, window=4)
        return time.perf_counter() - t0

    # size each step to ~1.5 s of wall time so K+W steps end within minutes
    probe = words_for(1 << 18)
    rate = (1 << 18) / max(run(probe), 1e-6)
    sample = int(min(N_WORDS, max(1 << 16, rate * 1.5)))
    words = words_for(sample)
    for _ in range(args.warmup):
        run(words)
    ts = [run(words) for _ in range(args.steps)]
    t = sum(ts) / len(ts)
    value = ND * sample / t
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded SplitMix64)",
        "config": {"workload": WORKLOAD, "sample_words_per_step": sample},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads if use_ref else 1, "kind": kind,
                         "sample": f"{sample} words of the C2 stream per step (redq_residues_into, float_premul + "
                                   f"window-4 table; -O2 asserts armed as shipped)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


def cpu_baseline_leg():
    """Reference CPU path on the host cores, bounded sample (~5 s)."""
    import numpy as np

    import oracle as O
    threads = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
    if O.ref() is None:
        kind, threads_used = "port", 1
    else:
        kind, threads_used = "reference", threads

    def words_for(n):
        dr = O.draws(0x07100510 + 2, n * ND, 128).reshape(n, ND).astype(np.uint64)
        w = np.zeros(n, np.uint64)
        for j in range(ND):
            w = w * np.uint64(128) + dr[:, j]
        return w.astype(np.float64)

    def run(words):
        if kind == "reference":
            _, ns, _ = O.ref_redq_f64(5, 128, 6, words, float_mode=True, window=4, threads=threads_used)
            return ns * 1e-9
        t0 = time.perf_counter()
        O.redq_f64(5, 128, 6, words, float_mode=True, window=4)
        return time.perf_counter() - t0

    rate = (1 << 18) / max(run(words_for(1 << 18)), 1e-6)
    sample = int(min(N_WORDS, max(1 << 16, rate * 4.0)))
    t = run(words_for(sample))
    return {"value": ND * sample / t, "unit": UNIT, "cores": threads_used, "kind": kind,
            "sample": f"{sample} words of the C2 stream (redq_residues_into, float_premul + window-4 table, "
                      f"reference built -O2 with asserts armed as shipped), {threads_used} threads"}


# ---------------------------------------------------------------------- ours
def run_ours(args, rank, world, local_rank):
    import numpy as np
    import torch

    import paper_0710_0510_b200 as Q

    dist = None
    if world > 1:
        import torch.distributed as dist
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)

    def barrier():
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier(device_ids=[local_rank])

    from paper_0710_0510_b200.sharding import max_over_ranks as _mor
    from paper_0710_0510_b200.sharding import weak_shard

    def max_over_ranks(x):
        return _mor(x, dist, dev)

    clocks = ClockSampler(local_rank)
    clocks.start()

    # inputs: this rank's shard of the seeded C2 stream, generated on device
    first, count = weak_shard(rank, N_WORDS)
    w = torch.empty(count, dtype=torch.float64, device=dev)
    Q.gen_words(Q.C2.seed, count, 128, 6, w, first=first)
    out = torch.empty((N_WORDS, ND), dtype=torch.uint8, device=dev)
    plan = Q.RedqPlan(5, 128, 6, Q.FLOAT_PREMUL).attach_correction(4)

    # ---- value: resident inputs, one REDQ kernel per step
    for _ in range(args.warmup):
        plan.residues(w, out=out)
    plan.sync()
    barrier()
    clocks.active = True
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        plan.residues(w, out=out)
    e1.record()
    barrier()
    clocks.active = False
    plan.sync()
    ms_total = max_over_ranks(e0.elapsed_time(e1))
    ms_step = ms_total / args.steps
    value = world * N_WORDS * ND / (ms_step * 1e-3)
    kernel_ms = e0.elapsed_time(e1) / args.steps  # this rank's kernel (1 launch / step)

    # ---- e2e: host buffers through the C-ABI host entry point
    hw = torch.empty(N_WORDS, dtype=torch.float64, pin_memory=True)
    hw.copy_(w)
    ho = torch.empty((N_WORDS, ND), dtype=torch.uint8, pin_memory=True)
    hw_np, ho_np = hw.numpy(), ho.numpy()
    e2e_steps = max(3, min(args.steps, 10))
    for _ in range(max(1, min(args.warmup, 3))):
        plan.residues(hw_np, out=ho_np)
    barrier()
    clocks.active = True
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        plan.residues(hw_np, out=ho_np)
    t_e2e = time.perf_counter() - t0
    clocks.active = False
    t_e2e = max_over_ranks(t_e2e) / e2e_steps
    e2e_value = world * N_WORDS * ND / t_e2e
    # the e2e output must equal the resident run's
    assert np.array_equal(ho_np[:1 << 20], out[:1 << 20].cpu().numpy()), "e2e output differs from device output"

    peak, peak_src = measured_peaks()
    achieved = ALGO_BYTES_PER_WORD * N_WORDS / (kernel_ms * 1e-3) / 1e9
    traffic = ncu_traffic("redq_c2")

    secondary = None
    if world == 1 and not args.no_secondary:
        clocks.active = True
        secondary = measure_secondary(Q, torch, dev)
        clocks.active = False
    del w, out, hw, ho
    clocks.stop()

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded SplitMix64, generated on device)",
        "config": {"workload": WORKLOAD, "words_per_gpu": N_WORDS, "global_words": world * N_WORDS,
                   "l2": "inputs larger than L2 (512 MiB in + 448 MiB out per GPU per step)",
                   "parallelism": f"dp{world} (independent word shards, no collective)"},
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": world * N_WORDS * 8,
                "d2h_bytes_per_step": world * N_WORDS * ND, "steps": e2e_steps,
                "path": "qpk_redq_residues_f64_host (pinned host buffers; 2M-word chunks: H2D stream -> kernel stream -> D2H stream, 4 buffer slots)"},
        "gpu_launches": args.steps,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic, "peak_source": peak_src,
                     "frac_of_nominal_8TBps": achieved / 8000.0,
                     "kernel": "stream_tma_kernel<RedqOp<7,pow2,w4>>",
                     "algorithmic_bytes_per_launch": ALGO_BYTES_PER_WORD * N_WORDS},
        "clocks": clocks.summary(),
    }
    if secondary is not None:
        line["secondary"] = secondary
    return line


def secondary_cpu_refs(sec):
    """The reference's CPU path timed beside each secondary config (SURVEY
    8(d)): oracle/_ref (the unmodified sources, -O2, asserts armed) on all host
    threads, a bounded sample of the same seeded workload, ~1-3 s each."""
    import numpy as np

    import oracle as O
    if O.ref() is None:
        return
    th = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)

    def entry(value, unit, sample):
        return {"value": value, "unit": unit, "cores": th, "kind": "reference", "sample": sample}

    # C1: fqt_mul per pair (REDQ/FQT path), first 2^20 pairs' worth of draws
    n = 1 << 18
    d = O.draws(0x07100510 + 1, 8 * n, 3).reshape(n, 8)
    _, ns, _ = O.ref_polymul_batch(3, 3, d[:, :4], d[:, 4:], algo=0, threads=th)
    if "c1_polymul" in sec:
        sec["c1_polymul"]["cpu_ref"] = entry(n / (ns * 1e-9), "pairs/s",
                                             f"{n} pairs of the C1 stream, fqt_mul(a,b,3,qadic_for_degree(3,3,53))")
    # C3: fgdp_dot on length-1 vectors (packed) and GfqField::mul (dlog)
    n = 1 << 20
    d = O.draws(0x07100510 + 3, 6 * n, 7).reshape(n, 6)
    rf = O.RefField(7, 3, 256)
    for algo, name, what in ((0, "c3_gfq_mul_packed", "fgdp_dot on length-1 vectors"),
                             (1, "c3_gfq_mul_dlog", "GfqField::mul")):
        _, ns, _ = rf.mul_batch(d[:, :3], d[:, 3:], algo=algo, threads=th)
        if name in sec:
            sec[name]["cpu_ref"] = entry(n / (ns * 1e-9), "products/s", f"{n} products of the C3 stream, {what}")
    # C4 / C5: gfq_matmul (as shipped) on a row slab, GF ops/s = 2 terms/s
    for cid, k, q, nn in ((4, 2, 1 << 16, 4096), (5, 3, 1 << 10, 8192)):
        rows = max(16, th)  # one row slab per host thread at least
        A = O.draws(0x07100510 + cid, rows * nn * k, 3).reshape(rows, nn, k)
        B = O.draws(0x07100510 + cid, nn * nn * k, 3, start=nn * nn * k).reshape(nn, nn, k)
        _, ns, _ = O.RefField(3, k, q).matmul(A, B, 0, rows, algo=0, threads=th)
        name = f"c{cid}_gfq_matmul"
        if name in sec:
            sec[name]["cpu_ref"] = entry(2 * rows * nn * nn / (ns * 1e-9), "GF ops/s",
                                         f"{rows} rows x {nn} x {nn} of C{cid} (gfq_matmul, as shipped), extrapolated rate")
    # K5: fgdp_dot of two long rep vectors
    n = 1 << 24
    v = O.draws(0x5, 2 * n, 27).astype(np.uint32)
    t0 = time.perf_counter()
    O.RefField(3, 3, 1 << 10).dot(v[:n], v[n:])
    dt = time.perf_counter() - t0
    if "k5_fgdp_dot_long" in sec:
        sec["k5_fgdp_dot_long"]["cpu_ref"] = {"value": n / dt, "unit": "GF terms/s", "cores": 1, "kind": "reference",
                                              "sample": f"one fgdp_dot of {n} terms (single call, single thread)"}
    # K6: fqt_mul of two 2^11-coefficient polynomials, C1's params
    n = 1 << 11
    a = O.draws(0x6, 2 * n, 3).astype(np.uint64)
    out = np.zeros(2 * n - 1, np.uint64)
    cost = np.zeros(4, np.uint64)
    t0 = time.perf_counter()
    O.ref().ref_fqt_mul(3, 3, 32, 1, a[:n], n, a[n:], n, out, cost)
    dt = time.perf_counter() - t0
    if "k6_fqt_mul" in sec:
        sec["k6_fqt_mul"]["cpu_ref_q32_d3_nq1"] = {
            "value": n * n / dt, "unit": "coefficient products/s", "cores": 1, "kind": "reference",
            "sample": f"one fqt_mul of two {n}-coefficient polynomials over F_3 (single call, single thread)"}
    # ... and the wide-group parameters of the DMMA kernel (q = 2^13, d = 1, n_q = 409)
    n = 1 << 14
    a = O.draws(0x6, 2 * n, 3).astype(np.uint64)
    out = np.zeros(2 * n - 1, np.uint64)
    t0 = time.perf_counter()
    O.ref().ref_fqt_mul(3, 1, 1 << 13, 409, a[:n], n, a[n:], n, out, cost)
    dt = time.perf_counter() - t0
    if "k6_fqt_mul" in sec:
        sec["k6_fqt_mul"]["cpu_ref_q8192_d1_nq409"] = {
            "value": n * n / dt, "unit": "coefficient products/s", "cores": 1, "kind": "reference",
            "sample": f"one fqt_mul of two {n}-coefficient polynomials over F_3, q=2^13, n_q=409 (single call, single thread)"}
    if "k6_fqt_mul_large" in sec:
        sec["k6_fqt_mul_large"]["cpu_ref"] = {
            "value": n * n / dt, "unit": "coefficient products/s", "cores": 1, "kind": "reference",
            "sample": f"one fqt_mul of two {n}-coefficient polynomials, same params (the rate is size-independent: "
                      "the reference loop is quadratic), single thread"}


def measure_secondary(Q, torch, dev):
    """C1, C3 (both paths), C4, C5 on one GPU; CUDA-event timed."""
    res = {}
    peak_hbm, _ = measured_peaks()
    fp64_peak = Q.probe_fp64(1, 8192)
    dfma_peak = Q.probe_fp64(0, 8192)
    res["fp64_peaks_tflops"] = {"dmma_probe": fp64_peak, "dfma_probe": dfma_peak, "nominal": 37.0}
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    def time_it(fn, reps, warm=3, cold=True):
        for _ in range(warm):
            fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(reps):
            if cold:
                flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        return statistics.median(ts)

    def time_rotating(fns, reps=10):
        """Per-launch time of back-to-back launches cycling through buffer
        sets whose total exceeds L2 (each set was last touched > 126 MB of
        traffic ago); one event pair per batch -- the event clock ticks in
        ~2 us steps, too coarse for a single 10-40 us launch."""
        for fn in fns:
            fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for fn in fns:
                fn()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) / len(fns))
        return statistics.median(ts)

    def time_graph(fns, reps=10):
        """Same as time_rotating with the launches captured in one CUDA graph:
        device time per launch without the Python call overhead."""
        for fn in fns:
            fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for fn in fns:
                fn()
        g.replay()
        torch.cuda.synchronize()
        ts = []
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            g.replay()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) / len(fns))
        return statistics.median(ts)

    # C1: 2^20 polynomial pairs, 15.7 MB per set; 24 sets (377 MB) rotate
    n1 = Q.C1.n
    pm = Q.PolymulPlan(3, 32, 4, 1)
    sets1 = []
    for _ in range(24):
        a1 = torch.empty(n1 * 4, dtype=torch.uint8, device=dev)
        b1 = torch.empty_like(a1)
        Q.gen_pairs(Q.C1.seed, n1, 4, 3, a1, b1)
        sets1.append((a1, b1, torch.empty((n1, 7), dtype=torch.uint8, device=dev)))
    fns = [lambda s=s_: pm(s[0], s[1], out=s[2]) for s_ in sets1]
    eager = time_rotating(fns)
    cold = time_graph(fns)
    hot = time_graph([lambda s=sets1[0]: pm(s[0], s[1], out=s[2])] * 24)
    single = time_it(lambda: pm(sets1[0][0], sets1[0][1], out=sets1[0][2]), 20)
    pm.sync()
    del sets1, fns
    res["c1_polymul"] = {"pairs_per_s_cold": n1 / (cold * 1e-3), "ms_cold": cold, "ms_hot": hot,
                         "timing": "CUDA graph of 24 launches over rotating buffer sets (377 MB > L2)",
                         "ms_eager_python_calls": eager, "ms_single_launch_flushed": single,
                         "GBps_cold": 15 * n1 / (cold * 1e-3) / 1e9, "frac_hbm_cold": 15 * n1 / (cold * 1e-3) / 1e9 / peak_hbm}
    # C3: 2^24 GF(7^3) products, 151 MB per set; 3 sets rotate
    n3 = Q.C3.n
    f3 = Q.GfqField(7, 3, 256)
    sets3 = []
    for _ in range(3):
        a3 = torch.empty(n3 * 3, dtype=torch.uint8, device=dev)
        b3 = torch.empty_like(a3)
        Q.gen_pairs(Q.C3.seed, n3, 3, 7, a3, b3)
        sets3.append((a3, b3, torch.empty((n3, 3), dtype=torch.uint8, device=dev)))
    for path, name in ((0, "packed"), (1, "dlog")):
        ms = time_graph([lambda s=s_, pth=path: f3.mul_batch(s[0], s[1], pth, out=s[2]) for s_ in sets3] * 4)
        single = time_it(lambda pth=path: f3.mul_batch(sets3[0][0], sets3[0][1], pth, out=sets3[0][2]), 20)
        gbs = 9 * n3 / (ms * 1e-3) / 1e9
        res[f"c3_gfq_mul_{name}"] = {"products_per_s": n3 / (ms * 1e-3), "ms": ms, "GBps": gbs,
                                     "frac_hbm": gbs / peak_hbm, "ms_single_launch_flushed": single}
    del sets3
    # K5: GF(3^3) GEMV on reps, 8192 x 8192 (256 MiB of
    # A, streamed once per launch: > L2), and one long fgdp_dot of 2^26 terms
    f5 = Q.GfqField(3, 3, 1 << 10)
    gen = torch.Generator(device=dev).manual_seed(5)
    nn = 8192
    A5 = torch.randint(0, 27, (nn, nn), dtype=torch.int32, device=dev, generator=gen)
    x5 = torch.randint(0, 27, (nn,), dtype=torch.int32, device=dev, generator=gen)
    y5 = torch.empty((nn,), dtype=torch.int32, device=dev)
    ms = time_graph([lambda: f5.gemv(A5, x5, out=y5)] * 4)
    gbs = (nn * nn * 4 + nn * 4 * 2) / (ms * 1e-3) / 1e9
    res["k5_gfq_gemv"] = {"m": nn, "K": nn, "field": "GF(3^3) q=2^10", "ms": ms, "GBps": gbs,
                          "frac_hbm": gbs / peak_hbm, "gf_terms_per_s": nn * nn / (ms * 1e-3)}
    del A5
    nd = 1 << 26
    v1 = torch.randint(0, 27, (1, nd), dtype=torch.int32, device=dev, generator=gen)
    v2 = torch.randint(0, 27, (nd,), dtype=torch.int32, device=dev, generator=gen)
    y1 = torch.empty((1,), dtype=torch.int32, device=dev)
    ms = time_graph([lambda: f5.gemv(v1, v2, out=y1)] * 2)
    gbs = nd * 8 / (ms * 1e-3) / 1e9
    res["k5_fgdp_dot_long"] = {"n": nd, "field": "GF(3^3) q=2^10", "ms": ms, "GBps": gbs, "frac_hbm": gbs / peak_hbm}
    del v1, v2
    # K6: one chunked FQT product of two 2^16-coefficient
    # polynomials over F_3; C1's params (q=2^5, d=3, n_q=1: one REDQ per
    # packed product) and a wide-group packing (q=2^13, d=1, n_q=409)
    n6 = 1 << 16
    a6 = torch.randint(0, 3, (n6,), dtype=torch.uint8, device=dev, generator=gen)
    b6 = torch.randint(0, 3, (n6,), dtype=torch.uint8, device=dev, generator=gen)
    o6 = torch.empty((2 * n6 - 1,), dtype=torch.uint8, device=dev)
    res["k6_fqt_mul"] = {"n": n6, "p": 3}
    for name, (q6, d6, nq6) in (("q32_d3_nq1", (32, 3, 1)), ("q8192_d1_nq409", (1 << 13, 1, 409))):
        pm6 = Q.PolymulPlan(3, q6, d6 + 1, nq6)
        ms = time_graph([lambda: pm6.fqt_mul(a6, b6, out=o6)] * 2)
        chunks = -(-n6 // (d6 + 1))
        wp = chunks * chunks / (ms * 1e-3)
        res["k6_fqt_mul"][name] = {"ms": ms, "coeff_products_per_s": n6 * n6 / (ms * 1e-3),
                                   "word_products_per_s": wp, "redq_per_s": wp / nq6,
                                   "fp64_tflops": 2 * wp / 1e12,
                                   # n_q >= 16 runs on the fp64 tensor pipe (DMMA), n_q = 1 on CUDA cores
                                   "kernel": "fqt_mma_kernel (DMMA)" if nq6 >= 16 else "fqt_conv_step_kernel (SWAR REDQ)",
                                   "frac_fp64_probe": 2 * wp / 1e12 / (fp64_peak if nq6 >= 16 else dfma_peak)}
    # K6 at scale: 2^20-coefficient operands on the DMMA kernel (the 2^16
    # case above is launch/latency dominated)
    nL = 1 << 20
    aL = torch.randint(0, 3, (nL,), dtype=torch.uint8, device=dev, generator=gen)
    bL = torch.randint(0, 3, (nL,), dtype=torch.uint8, device=dev, generator=gen)
    oL = torch.empty((2 * nL - 1,), dtype=torch.uint8, device=dev)
    pmL = Q.PolymulPlan(3, 1 << 13, 2, 409)
    ms = time_it(lambda: pmL.fqt_mul(aL, bL, out=oL), 3, warm=1, cold=False)
    wp = (nL // 2) ** 2 / (ms * 1e-3)
    res["k6_fqt_mul_large"] = {"n": nL, "p": 3, "q": 1 << 13, "d": 1, "n_q": 409, "ms": ms,
                               "coeff_products_per_s": nL * nL / (ms * 1e-3), "fp64_tflops": 2 * wp / 1e12,
                               "kernel": "fqt_mma_kernel (DMMA)", "frac_fp64_probe": 2 * wp / 1e12 / fp64_peak}
    del aL, bL, oL
    # C4, C5: GF(p^k) matrix products (pack + contraction), GF ops/s = 2 n^3 / t
    for cfg in (Q.C4, Q.C5):
        nn, k = cfg.n, cfg.k
        A = torch.empty(nn * nn * k, dtype=torch.uint8, device=dev)
        B = torch.empty_like(A)
        Q.gen_draws(cfg.seed, nn * nn * k, 3, A, start=0)
        Q.gen_draws(cfg.seed, nn * nn * k, 3, B, start=nn * nn * k)
        f = Q.GfqField(3, k, cfg.q)
        Cm = torch.empty((nn, nn, k), dtype=torch.uint8, device=dev)
        ms = time_it(lambda: f.matmul(A, B, nn, nn, nn, cfg.chunk, out=Cm), 5, warm=2, cold=False)
        tf = 2 * nn ** 3 / (ms * 1e-3) / 1e12
        res[f"c{cfg.cid}_gfq_matmul"] = {"gf_ops_per_s": 2 * nn ** 3 / (ms * 1e-3), "ms": ms, "tflops": tf,
                                          "frac_dmma_probe": tf / fp64_peak, "frac_nominal_37": tf / 37.0,
                                          "n": nn, "chunk": cfg.chunk, "repack": "redq"}
        if cfg.cid == 5:
            # the same product with the lane-fold re-pack (same C)
            ms = time_it(lambda: f.matmul(A, B, nn, nn, nn, cfg.chunk, out=Cm, repack="fold"), 5, warm=2, cold=False)
            tf = 2 * nn ** 3 / (ms * 1e-3) / 1e12
            res["c5_gfq_matmul_fold"] = {"gf_ops_per_s": 2 * nn ** 3 / (ms * 1e-3), "ms": ms, "tflops": tf,
                                         "frac_dmma_probe": tf / fp64_peak, "frac_nominal_37": tf / 37.0,
                                         "n": nn, "chunk": cfg.chunk, "repack": "fold"}
        del A, B, Cm
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-secondary", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        if rank == 0:
            run_reference(args, rank)
        return

    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    line = run_ours(args, rank, world, local_rank)
    if rank == 0:
        if world == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline_leg()
            if "secondary" in line:
                secondary_cpu_refs(line["secondary"])
        print(json.dumps(line))
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
