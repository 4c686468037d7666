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
configs   every BASELINE config (C1, C2, C3 on each path, C4, C5) with the
          same legs -- value, roofline, e2e through its C-ABI host entry point,
          cpu_baseline (the reference CPU path, all threads and one thread) --
          N = 1 only; next_rows: the SURVEY 8(f) kernels (K5, K6)
summary   compact per-config values, the LAST key of the line
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
    """dram bytes per launch (read + write) of `kernel_key` from the committed
    ncu summary (profiles/ncu_summary.json: the round-2 captures first)."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as f:
            s = json.load(f)
        entry = s.get("round2", {}).get(kernel_key) or s[kernel_key]
        return entry["dram_bytes_per_launch"]
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
def host_threads():
    return len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


def c2_words(n, first=0):
    """Words [first, first + n) of the seeded C2 stream (the device generator's)."""
    import numpy as np

    import oracle as O
    dr = O.draws(0x07100510 + 2, n * ND, 128, start=first * ND).reshape(n, ND).astype(np.uint64)
    w = np.zeros(n, np.uint64)
    for j in range(ND):
        w = w * np.uint64(128) + dr[:, j]
    return w.astype(np.float64)


def time_cpu(run, steps, warmup):
    """Reference-arm protocol: warm-up calls, then the mean over `steps`
    calls (each returns its own seconds, measured inside the call)."""
    for _ in range(warmup):
        run()
    ts = [run() for _ in range(steps)]
    return sum(ts) / len(ts)


def c2_reference_rate(words, out, threads, steps, warmup):
    """The reference's redq_residues_into (oracle/_ref, unmodified sources,
    float_premul + window-4 table) over `words` on `threads` host threads;
    the C restatement when the reference was not built here."""
    import oracle as O
    use_ref = O.ref() is not None

    def run():
        if use_ref:
            _, ns, _ = O.ref_redq_f64(5, 128, 6, words, float_mode=True, window=4, threads=threads, out=out)
            return ns * 1e-9
        t0 = time.perf_counter()
        O.redq_f64(5, 128, 6, words, float_mode=True, window=4)
        return time.perf_counter() - t0
    t = time_cpu(run, steps, warmup)
    return ND * words.size / t, ("reference" if use_ref else "port"), (threads if use_ref else 1)


def headline_config(world):
    return {"workload": WORKLOAD, "words_per_gpu": N_WORDS, "global_words": world * N_WORDS,
            "l2": "inputs larger than L2 (512 MiB in + 448 MiB out per GPU per step)",
            "parallelism": f"dp{world} (independent word shards, no collective)"}


def run_reference(args, rank):
    """The reference's own CPU implementation on the host cores: the same
    metric, config and 2^26-word workload as our arm (rank 0's shard), every
    step the full workload, all host threads."""
    import numpy as np
    threads = host_threads()
    words = c2_words(N_WORDS)
    out = np.empty((N_WORDS, ND), np.uint8)
    value, kind, cores = c2_reference_rate(words, out, threads, args.steps, args.warmup)
    t = ND * N_WORDS / value
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded SplitMix64)",
        "config": headline_config(args.gpus),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": kind, "cpu_model": cpu_model(),
                         "sample": f"the full {N_WORDS}-word C2 workload per step (redq_residues_into, float_premul + "
                                   "window-4 table; -O2 asserts armed as shipped); output preallocated"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


def cpu_baseline_leg():
    """C2's reference CPU path on the host cores with the reference arm's
    protocol (the full 2^26-word workload, output preallocated, 1 warm-up
    call, mean of 3), all threads and one thread (on a 2^22-word sample)."""
    import numpy as np
    threads = host_threads()
    words = c2_words(N_WORDS)
    out = np.empty((N_WORDS, ND), np.uint8)
    value, kind, cores = c2_reference_rate(words, out, threads, 3, 1)
    one, _, _ = c2_reference_rate(words[:1 << 22], out[:1 << 22], 1, 2, 1)
    return {"value": value, "unit": UNIT, "cores": cores, "kind": kind, "one_thread": one, "cpu_model": cpu_model(),
            "sample": f"the full {N_WORDS}-word C2 workload (redq_residues_into, float_premul + window-4 table, reference "
                      f"built -O2 with asserts armed as shipped), {cores} threads, mean of 3 after 1 warm-up; "
                      "one_thread: 2^22 words on 1 thread"}


def cpu_legs():
    """Every config's reference CPU path (oracle/_ref: the unmodified
    sources) on the host cores, in a process of its own -- CUDA and torch
    initialised in the same process measured the same reference call 1.6x
    slower (scripts/cpu_leg_probe.py) -- with the reference arm's protocol:
    warm-up, mean over calls, outputs preallocated, all threads and one
    thread.  Inputs: the configs' seeded streams regenerated on the host."""
    import numpy as np

    import oracle as O
    th = host_threads()
    out = {"C2": cpu_baseline_leg()}
    if O.ref() is None:
        return out
    model = cpu_model()

    def entry(rate_all, rate_one, unit, sample):
        return {"value": rate_all, "unit": unit, "cores": th, "one_thread": rate_one, "kind": "reference",
                "cpu_model": model, "sample": sample}

    # C1: fqt_mul per pair (the whole 2^20-pair workload per call)
    n1 = 1 << 20
    d = O.draws(0x07100510 + 1, 8 * n1, 3).reshape(n1, 8)
    a, b = np.ascontiguousarray(d[:, :4]), np.ascontiguousarray(d[:, 4:])
    o = np.empty((n1, 7), np.uint8)
    rate = lambda t, n: n / time_cpu(lambda: O.ref_polymul_batch(3, 3, a[:n], b[:n], algo=0, threads=t,
                                                                 out=o[:n])[1] * 1e-9, 3, 1)
    out["C1"] = entry(rate(th, n1), rate(1, 1 << 18), "pairs/s",
                      f"the full {n1}-pair C1 workload per call (fqt_mul per pair, qadic_for_degree(3,3,53)); "
                      "mean of 3 after 1 warm-up; one_thread: 2^18 pairs")
    # C3: 2^22 products of the stream per call, both reference paths
    nc = 1 << 22
    d = O.draws(0x07100510 + 3, 6 * nc, 7).reshape(nc, 6)
    a, b = np.ascontiguousarray(d[:, :3]), np.ascontiguousarray(d[:, 3:])
    o = np.empty((nc, 3), np.uint8)
    rf = O.RefField(7, 3, 256)
    for name, algo, what in (("C3_redq", 0, "fgdp_dot on length-1 vectors"), ("C3_dlog", 1, "GfqField::mul"),
                             ("C3_linear", 0, "fgdp_dot on length-1 vectors")):
        rate = lambda t, n, al=algo: n / time_cpu(lambda: rf.mul_batch(a[:n], b[:n], algo=al, threads=t,
                                                                      out=o[:n])[1] * 1e-9, 3, 1)
        out[name] = entry(rate(th, nc), rate(1, 1 << 20), "products/s",
                          f"2^22 products of the C3 stream per call ({what}); mean of 3 after 1 warm-up; "
                          "one_thread: 2^20 products")
    # C4 / C5: gfq_matmul (as shipped) on a row slab, rate extrapolated
    for cid, k, q, nn in ((4, 2, 1 << 16, 4096), (5, 3, 1 << 10, 8192)):
        rows = max(16, th)
        A = O.draws(0x07100510 + cid, rows * nn * k, 3).reshape(rows, nn, k)
        B = O.draws(0x07100510 + cid, nn * nn * k, 3, start=nn * nn * k).reshape(nn, nn, k)
        rfm = O.RefField(3, k, q)
        cb = np.empty((rows, nn, k), np.uint8)
        rate = lambda t, r: 2 * r * nn * nn / time_cpu(
            lambda: rfm.matmul(A[:r], B, 0, r, algo=0, threads=t, out=cb[:r])[1] * 1e-9, 1, 0)
        out[f"C{cid}"] = entry(rate(th, rows), rate(1, 2), "GF ops/s",
                               f"{rows} rows x {nn} x {nn} of C{cid} per call (gfq_matmul as shipped, row slabs over "
                               "threads), rate extrapolated; one_thread: 2 rows")
    return out


def cpu_legs_subprocess():
    r = subprocess.run([sys.executable, os.path.abspath(__file__), "--cpu-legs"], capture_output=True, text=True,
                       timeout=1800)
    lines = [x for x in r.stdout.splitlines() if x.startswith("{")]
    if r.returncode != 0 or not lines:
        raise RuntimeError("cpu legs failed: " + r.stderr[-2000:])
    return json.loads(lines[-1])


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

    configs = next_rows = None
    if world == 1 and not args.no_secondary:
        clocks.active = True
        configs = measure_configs(Q, torch, dev, peak)
        next_rows = measure_next_rows(Q, torch, dev, peak, configs["fp64_peaks_tflops"]["dmma_probe"])
        clocks.active = False
    del w, out, hw, ho
    clocks.stop()

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded SplitMix64, generated on device)",
        "config": headline_config(world),
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
    if configs is not None:
        configs = {"C2": {"workload": WORKLOAD, "metric": METRIC, "unit": UNIT, "value": value, "ms": ms_step,
                          "roofline": line["roofline"], "e2e": line["e2e"], "cpu_baseline": None}, **configs}
        line["configs"] = configs
        line["next_rows"] = next_rows
    return line


def sig(x, n=3):
    """x rounded to n significant digits (compact summary)."""
    if x is None or x == 0:
        return x
    import math
    return round(x, -int(math.floor(math.log10(abs(x)))) + n - 1)


def measure_configs(Q, torch, dev, peak_hbm):
    """BASELINE configs C1, C3, C4, C5 (C2 is the headline) on one GPU, each
    with the same three legs as the headline: `value` (inputs resident in
    HBM, CUDA-event timed), `e2e` (the same metric through the C-ABI host
    entry point: pinned host buffers, H2D + kernels + D2H inside the timed
    region) and `cpu_baseline` (the reference's own CPU path, oracle/_ref,
    reference-arm protocol), plus the roofline of the dominant kernel."""
    import numpy as np

    import oracle as O
    res = {}
    fp64_peak = Q.probe_fp64(1, 8192)
    dfma_peak = Q.probe_fp64(0, 8192)
    res["fp64_peaks_tflops"] = {"dmma_probe": fp64_peak, "dfma_probe": dfma_peak, "nominal": 37.0,
                                "note": "mma.sync.m8n8k4.f64 / DFMA probe kernels measured in this run "
                                        "(tcgen05 has no f64 kind on sm_100a)"}
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

    def time_graph(fns, reps=10):
        """Per-launch device time of back-to-back launches cycling through
        buffer sets whose total exceeds L2 (each set was last touched > 126 MB
        of traffic ago), captured in one CUDA graph; one event pair per replay
        (the event clock ticks in ~2 us steps, too coarse for one launch)."""
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

    def time_host(fn, steps=5, warm=2):
        """Wall time per call of a synchronous host-buffer C-ABI entry point."""
        for _ in range(warm):
            fn()
        t0 = time.perf_counter()
        for _ in range(steps):
            fn()
        return (time.perf_counter() - t0) / steps

    def pinned(shape, dtype):
        return torch.empty(shape, dtype=dtype, pin_memory=True).numpy()

    def hbm_roof(bytes_per_launch, ms, kernel, ncu_key):
        a = bytes_per_launch / (ms * 1e-3) / 1e9
        return {"bound": "hbm", "achieved": a, "peak": peak_hbm, "unit": "GB/s", "frac": a / peak_hbm,
                "traffic": ncu_traffic(ncu_key), "algorithmic_bytes_per_launch": bytes_per_launch, "kernel": kernel}

    # ---------------------------------------------------------------- C1
    # 2^20 pairs of degree-<4 polynomials over F_3, q = 2^5: 15 B per pair
    # (4 + 4 in, 7 out); 24 sets (377 MB) rotate through the graph
    n1 = Q.C1.n
    pm = Q.PolymulPlan(3, 32, 4, 1)
    sets1 = []
    for _ in range(24):
        a1 = torch.empty(n1 * 4, dtype=torch.uint8, device=dev)
        b1 = torch.empty_like(a1)
        Q.gen_pairs(Q.C1.seed, n1, 4, 3, a1, b1)
        sets1.append((a1, b1, torch.empty((n1, 7), dtype=torch.uint8, device=dev)))
    ms = time_graph([lambda s=s_: pm(s[0], s[1], out=s[2]) for s_ in sets1])
    ms_hot = time_graph([lambda s=sets1[0]: pm(s[0], s[1], out=s[2])] * 24)
    ms_single = time_it(lambda: pm(sets1[0][0], sets1[0][1], out=sets1[0][2]), 20)
    pm.sync()
    ha, hb, ho = pinned((n1, 4), torch.uint8), pinned((n1, 4), torch.uint8), pinned((n1, 7), torch.uint8)
    ha[:] = sets1[0][0].view(n1, 4).cpu().numpy()
    hb[:] = sets1[0][1].view(n1, 4).cpu().numpy()
    t_e2e = time_host(lambda: pm(ha, hb, out=ho), steps=20)
    assert np.array_equal(ho, sets1[0][2].cpu().numpy()), "C1 e2e output differs from the device output"
    del sets1
    cpu = None  # filled from the fresh-process CPU legs (cpu_legs)
    res["C1"] = {"workload": "C1 F_3 polymul: 2^20 pairs of degree-<4 polys, q=2^5 -> 7 residues/pair",
                 "metric": "polymul_pairs_per_s", "unit": "pairs/s", "value": n1 / (ms * 1e-3), "ms": ms,
                 "timing": "CUDA graph of 24 launches over rotating buffer sets (377 MB > L2), per launch",
                 "ms_hot": ms_hot, "ms_single_launch_flushed": ms_single,
                 "roofline": hbm_roof(15 * n1, ms, "stream_direct_kernel<PolymulOp<4,4,CtConst<3,5>>>", "c1_polymul"),
                 "e2e": {"value": n1 / t_e2e, "unit": "pairs/s", "h2d_bytes_per_step": 8 * n1,
                         "d2h_bytes_per_step": 7 * n1, "path": "qpk_polymul_batch_host (pinned host buffers)"},
                 "cpu_baseline": cpu}

    # ---------------------------------------------------------------- C3
    # 2^24 GF(7^3) products, 9 B each (3 + 3 in, 3 out); 3 sets rotate
    n3 = Q.C3.n
    f3 = Q.GfqField(7, 3, 256)
    sets3 = []
    for _ in range(3):
        a3 = torch.empty(n3 * 3, dtype=torch.uint8, device=dev)
        b3 = torch.empty_like(a3)
        Q.gen_pairs(Q.C3.seed, n3, 3, 7, a3, b3)
        sets3.append((a3, b3, torch.empty((n3, 3), dtype=torch.uint8, device=dev)))
    ha, hb, ho = pinned((n3, 3), torch.uint8), pinned((n3, 3), torch.uint8), pinned((n3, 3), torch.uint8)
    ha[:] = sets3[0][0].view(n3, 3).cpu().numpy()
    hb[:] = sets3[0][1].view(n3, 3).cpu().numpy()
    for path, name, what, algo in ((0, "C3_redq", "DQT pack, fp64 product, REDQ, L/H tables (fgdp_dot on length-1 "
                                                  "vectors)", 0),
                                   (1, "C3_dlog", "dlog/Zech (GfqField::mul)", 1),
                                   (2, "C3_linear", "extra: integer word product + lane-wise mod 7 (no REDQ)", 0)):
        ms = time_graph([lambda s=s_, pth=path: f3.mul_batch(s[0], s[1], pth, out=s[2]) for s_ in sets3] * 4)
        single = time_it(lambda pth=path: f3.mul_batch(sets3[0][0], sets3[0][1], pth, out=sets3[0][2]), 20)
        t_e2e = time_host(lambda pth=path: f3.mul_batch(ha, hb, pth, out=ho))
        assert np.array_equal(ho, sets3[0][2].cpu().numpy()), f"{name} e2e output differs from the device output"
        cpu = None
        res[name] = {"workload": f"C3 GF(7^3) elementwise: 2^24 products, q=2^8, path {path}: {what}",
                     "metric": "gf_products_per_s", "unit": "products/s", "value": n3 / (ms * 1e-3), "ms": ms,
                     "timing": "CUDA graph of 12 launches over 3 rotating buffer sets (453 MB > L2), per launch",
                     "ms_single_launch_flushed": single,
                     "roofline": hbm_roof(9 * n3, ms, f"stream_tma_kernel<GfqElemOp<3,CtConst<7,8>,{path}>>",
                                          {0: "c3_redq", 1: "c3_dlog", 2: "c3_linear"}[path]),
                     "e2e": {"value": n3 / t_e2e, "unit": "products/s", "h2d_bytes_per_step": 6 * n3,
                             "d2h_bytes_per_step": 3 * n3,
                             "path": f"qpk_gfq_mul_batch_host path {path} (pinned host buffers)"},
                     "cpu_baseline": cpu}
    del sets3

    # ------------------------------------------------------------ C4, C5
    # GF(p^k) matrix products (K1 pack + K4 DMMA contraction), GF ops/s =
    # 2 n^3 / t (one multiply-add per term = 2 fp64 flops on the tensor pipe)
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
        hA, hB, hC = pinned((nn, nn, k), torch.uint8), pinned((nn, nn, k), torch.uint8), pinned((nn, nn, k), torch.uint8)
        hA[:] = A.view(nn, nn, k).cpu().numpy()
        hB[:] = B.view(nn, nn, k).cpu().numpy()
        t_e2e = time_host(lambda: f.matmul(hA, hB, nn, nn, nn, cfg.chunk, out=hC), steps=3, warm=1)
        assert np.array_equal(hC, Cm.cpu().numpy()), f"C{cfg.cid} e2e output differs from the device output"
        # the reference's own signature: gfq_matmul(GfqMatrix...) on reps
        log = f.tables()["log"]
        wts = np.array([cfg.p ** i for i in range(k)], np.uint32)
        rA = pinned((nn, nn), torch.int32).view(np.uint32)
        rB = pinned((nn, nn), torch.int32).view(np.uint32)
        rA[:] = log[(hA.astype(np.uint32) * wts).sum(axis=2)]   # from_index (gfq.cpp:317-320)
        rB[:] = log[(hB.astype(np.uint32) * wts).sum(axis=2)]
        rC = pinned((nn, nn), torch.int32).view(np.uint32)
        t_rep = time_host(lambda: f.matmul_rep(rA, rB, out=rC), steps=3, warm=1)
        e2e = {"value": 2 * nn ** 3 / t_e2e, "unit": "GF ops/s", "h2d_bytes_per_step": 2 * nn * nn * k,
               "d2h_bytes_per_step": nn * nn * k,
               "path": f"qpk_gfq_matmul_repack_host (coefficient records, chunk {cfg.chunk or 'none'}; pinned host buffers)",
               "rep_api": {"value": 2 * nn ** 3 / t_rep, "h2d_bytes_per_step": 8 * nn * nn,
                           "d2h_bytes_per_step": 4 * nn * nn,
                           "path": "qpk_gfq_matmul_rep_host = gfq_matmul(GfqMatrix, GfqMatrix, GfqField) (reps; "
                                   "the reference's chunk n_q)"}}
        cpu = None
        name = f"C{cfg.cid}"
        res[name] = {"workload": f"C{cfg.cid} GF(3^{k}) matmul {nn}^3, q=2^{cfg.q.bit_length() - 1}"
                                 + (f", delayed REDQ re-pack every {cfg.chunk}" if cfg.chunk else ""),
                     "metric": "gf_ops_per_s", "unit": "GF ops/s", "value": 2 * nn ** 3 / (ms * 1e-3), "ms": ms,
                     "roofline": {"bound": "tensor", "achieved": tf, "peak": fp64_peak, "unit": "TFLOP/s",
                                  "frac": tf / fp64_peak, "peak_source": "fp64 DMMA probe (this run)",
                                  "traffic": ncu_traffic(f"matmul_c{cfg.cid}"),
                                  "frac_of_nominal_37": tf / 37.0, "kernel": "gfq_matmul_kernel (DMMA) + K1 pack"},
                     "e2e": e2e, "cpu_baseline": cpu, "repack": "redq"}
        if cfg.cid == 5:
            ms = time_it(lambda: f.matmul(A, B, nn, nn, nn, cfg.chunk, out=Cm, repack="fold"), 5, warm=2, cold=False)
            tf = 2 * nn ** 3 / (ms * 1e-3) / 1e12
            res["C5_fold"] = {"workload": "C5 with the lane-fold re-pack (same C)", "unit": "GF ops/s",
                              "value": 2 * nn ** 3 / (ms * 1e-3), "ms": ms,
                              "roofline": {"bound": "tensor", "achieved": tf, "peak": fp64_peak, "unit": "TFLOP/s",
                                           "frac": tf / fp64_peak}}
        del A, B, Cm
    return res


def measure_next_rows(Q, torch, dev, peak_hbm, fp64_peak):
    """K5 GF GEMV / long fgdp_dot and K6 chunked FQT."""
    res = {}

    def time_graph(fns, reps=10):
        for fn in fns:
            fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for fn in fns:
                fn()
        ts = []
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            g.replay()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) / len(fns))
        return statistics.median(ts)

    f5 = Q.GfqField(3, 3, 1 << 10)
    gen = torch.Generator(device=dev).manual_seed(5)
    nn = 8192
    A5 = torch.randint(0, 27, (nn, nn), dtype=torch.int32, device=dev, generator=gen)
    x5 = torch.randint(0, 27, (nn,), dtype=torch.int32, device=dev, generator=gen)
    y5 = torch.empty((nn,), dtype=torch.int32, device=dev)
    ms = time_graph([lambda: f5.gemv(A5, x5, out=y5)] * 4)
    gbs = (nn * nn * 4 + nn * 4 * 2) / (ms * 1e-3) / 1e9
    res["K5_gemv"] = {"m": nn, "K": nn, "field": "GF(3^3) q=2^10", "ms": ms, "frac_hbm": gbs / peak_hbm}
    del A5
    nd = 1 << 26
    v1 = torch.randint(0, 27, (1, nd), dtype=torch.int32, device=dev, generator=gen)
    v2 = torch.randint(0, 27, (nd,), dtype=torch.int32, device=dev, generator=gen)
    y1 = torch.empty((1,), dtype=torch.int32, device=dev)
    ms = time_graph([lambda: f5.gemv(v1, v2, out=y1)] * 2)
    res["K5_dot"] = {"n": nd, "ms": ms, "frac_hbm": nd * 8 / (ms * 1e-3) / 1e9 / peak_hbm}
    del v1, v2
    nL = 1 << 20
    aL = torch.randint(0, 3, (nL,), dtype=torch.uint8, device=dev, generator=gen)
    bL = torch.randint(0, 3, (nL,), dtype=torch.uint8, device=dev, generator=gen)
    oL = torch.empty((2 * nL - 1,), dtype=torch.uint8, device=dev)
    pmL = Q.PolymulPlan(3, 1 << 13, 2, 409)
    pmL.fqt_mul(aL, bL, out=oL)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        pmL.fqt_mul(aL, bL, out=oL)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 3
    tf = 2 * (nL // 2) ** 2 / (ms * 1e-3) / 1e12
    res["K6_fqt_2^20"] = {"q": 1 << 13, "d": 1, "n_q": 409, "ms": ms, "frac_fp64": tf / fp64_peak}
    return res


def summary(line):
    """Compact per-config block, printed LAST in the JSON line so that it
    survives a truncated stdout tail: value / roofline fraction / e2e /
    reference CPU (all threads, one thread) per config."""
    out = {}
    for name, c in line.get("configs", {}).items():
        if not isinstance(c, dict) or "value" not in c:
            continue
        e = {"v": sig(c["value"]), "u": c.get("unit"), "frac": sig(c.get("roofline", {}).get("frac"), 2),
             "bound": c.get("roofline", {}).get("bound")}
        if c.get("e2e"):
            e["e2e"] = sig(c["e2e"]["value"])
        if c.get("cpu_baseline"):
            e["cpu"] = sig(c["cpu_baseline"]["value"])
            e["cpu1"] = sig(c["cpu_baseline"].get("one_thread"))
        out[name] = e
    for name, c in line.get("next_rows", {}).items():
        out[name] = {"ms": sig(c["ms"]), "frac": sig(c.get("frac_hbm", c.get("frac_fp64")), 2)}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-secondary", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-legs", action="store_true", help=argparse.SUPPRESS)  # internal: fresh-process CPU legs
    args = ap.parse_args()
    if args.cpu_legs:
        print(json.dumps(cpu_legs()))
        return
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
            legs = cpu_legs_subprocess()
            line["cpu_baseline"] = legs["C2"]
            for name, leg in legs.items():
                if name in line.get("configs", {}):
                    line["configs"][name]["cpu_baseline"] = leg
        if "configs" in line:
            line["summary"] = summary(line)  # last key: survives a truncated stdout tail
        print(json.dumps(line))
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
