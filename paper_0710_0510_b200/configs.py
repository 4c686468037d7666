"""The five BASELINE.json workloads.

Seeds and draw order are this build's pin (BASELINE.json says only "from
seed"): one SplitMix64 stream per config with seed 0x07100510 + id, values
drawn with below(n) (rng.hpp:25) in the order listed.  Because SplitMix64 is
counter-based, draw j (1-based) is mix(seed + j*gamma) and the device
regenerates the identical inputs in parallel.
"""
from __future__ import annotations

from dataclasses import dataclass

SEED_BASE = 0x07100510


@dataclass(frozen=True)
class Config:
    cid: int
    name: str
    p: int
    q: int
    k: int          # coefficients per input element (or digits per word for C2)
    n: int          # records (C1-C3) or matrix side (C4-C5)
    bound: int      # below(bound) for each draw
    chunk: int = 0  # C5: delayed REDQ re-pack every `chunk` K-steps

    @property
    def seed(self) -> int:
        return SEED_BASE + self.cid


C1 = Config(1, "f3_deg4_polymul", p=3, q=32, k=4, n=1 << 20, bound=3)
C2 = Config(2, "redq_p5_q128_d6", p=5, q=128, k=7, n=1 << 26, bound=128)
C3 = Config(3, "gf7^3_elementwise", p=7, q=256, k=3, n=1 << 24, bound=7)
C4 = Config(4, "gf3^2_matmul_4096", p=3, q=1 << 16, k=2, n=4096, bound=3)
C5 = Config(5, "gf3^3_matmul_8192", p=3, q=1 << 10, k=3, n=8192, bound=3, chunk=64)

CONFIGS = {c.cid: c for c in (C1, C2, C3, C4, C5)}


def scaled(cfg: Config, n: int) -> Config:
    """Same config with a smaller record count / matrix side (parity cases)."""
    return Config(cfg.cid, cfg.name, cfg.p, cfg.q, cfg.k, n, cfg.bound, cfg.chunk)
