#!/usr/bin/env python
"""Generate the committed golden fixtures from the UNMODIFIED reference.

Run in the build container (needs oracle/_ref/libqpack_ref.so, i.e.
/root/reference at build time):

    python tests/golden/make_golden.py            # small fixtures + C1-C4 full checksums
    python tests/golden/make_golden.py --full 5   # add the C5 full checksum (minutes)

Outputs
  tests/golden/c<id>_small.npz  inputs and reference outputs at reduced sizes
  tests/golden/golden.json      per config at FULL BASELINE size: FNV-1a
                                checksum (common.cpp:51-61, bytes promoted to
                                u64) of the reference-generated inputs and of
                                the reference's outputs.

Inputs come from the reference's own SplitMix64 (rng.hpp:13-31), drawn
sequentially with below(n) in the order pinned in configs.py; outputs come
from the reference entry points the survey names per config.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import oracle as O  # noqa: E402
from paper_0710_0510_b200.configs import C1, C2, C3, C4, C5, scaled  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
THREADS = os.cpu_count() or 1


def ref_draws(seed, count, bound):
    out = np.empty(count, np.uint8)
    O.ref().ref_draws_u8(seed, count, bound, out)
    return out


def c2_words(digits: np.ndarray) -> np.ndarray:
    """7 draws per word, first drawn = top digit (acceptance.cpp:52-56)."""
    d = digits.reshape(-1, 7).astype(np.uint64)
    w = np.zeros(d.shape[0], np.uint64)
    for j in range(7):
        w = w * np.uint64(128) + d[:, j]
    return w.astype(np.float64)


def inputs(cfg):
    """Reference-generated inputs for a (possibly scaled) config."""
    if cfg.cid == 1:
        dr = ref_draws(cfg.seed, cfg.n * 8, 3).reshape(cfg.n, 8)
        return dict(a=np.ascontiguousarray(dr[:, :4]), b=np.ascontiguousarray(dr[:, 4:])), dr
    if cfg.cid == 2:
        dr = ref_draws(cfg.seed, cfg.n * 7, 128)
        return dict(words=c2_words(dr)), dr
    if cfg.cid == 3:
        dr = ref_draws(cfg.seed, cfg.n * 6, 7).reshape(cfg.n, 6)
        return dict(a=np.ascontiguousarray(dr[:, :3]), b=np.ascontiguousarray(dr[:, 3:])), dr
    n, k = cfg.n, cfg.k
    dr = ref_draws(cfg.seed, 2 * n * n * k, 3)
    return dict(A=dr[: n * n * k].reshape(n, n, k), B=dr[n * n * k:].reshape(n, n, k)), dr


def outputs(cfg, inp):
    if cfg.cid == 1:
        out, ns, _ = O.ref_polymul_batch(3, 3, inp["a"], inp["b"], algo=0, threads=THREADS)
        return out
    if cfg.cid == 2:
        # float_premul + base-p window-4 table: the variant the GPU mirrors
        out, ns, _ = O.ref_redq_f64(5, 128, 6, inp["words"], float_mode=True, window=4, threads=THREADS)
        return out
    if cfg.cid == 3:
        f = O.RefField(7, 3, 256)
        out, _, _ = f.mul_batch(inp["a"], inp["b"], algo=0, threads=THREADS)
        zech, _, _ = f.mul_batch(inp["a"], inp["b"], algo=1, threads=THREADS)
        assert (out == zech).all(), "reference DQT/L-H path and dlog path disagree"
        return out
    f = O.RefField(3, cfg.k, cfg.q)
    out, _, _ = f.matmul(inp["A"], inp["B"], algo=1, threads=THREADS)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--full", type=int, nargs="*", default=[1, 2, 3, 4],
                    help="configs whose full-size checksums to (re)compute")
    ap.add_argument("--no-small", action="store_true")
    args = ap.parse_args()
    assert O.ref() is not None, "build oracle/_ref first (make -C oracle ref)"

    small = {1: 4096, 2: 4096, 3: 4096, 4: 48, 5: 80}
    if not args.no_small:
        for base in (C1, C2, C3, C4, C5):
            cfg = scaled(base, small[base.cid])
            inp, _ = inputs(cfg)
            out = outputs(cfg, inp)
            np.savez_compressed(os.path.join(HERE, f"c{cfg.cid}_small.npz"), out=out, n=cfg.n, **inp)
            print(f"c{cfg.cid}_small: n={cfg.n} out={out.shape}")

    path = os.path.join(HERE, "golden.json")
    gold = json.load(open(path)) if os.path.exists(path) else {}
    for cid in args.full:
        cfg = {1: C1, 2: C2, 3: C3, 4: C4, 5: C5}[cid]
        t0 = time.time()
        inp, dr = inputs(cfg)
        out = outputs(cfg, inp)
        gold[f"c{cid}"] = dict(
            n=cfg.n, seed=cfg.seed,
            input_draws_checksum=f"{O.checksum_u8(dr):016x}",
            output_checksum=f"{O.checksum_u8(out):016x}",
            output_shape=list(out.shape),
            generator="reference (oracle/_ref) via tests/golden/make_golden.py",
            seconds=round(time.time() - t0, 1),
        )
        print(f"c{cid}: {gold[f'c{cid}']}")
        json.dump(gold, open(path, "w"), indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
