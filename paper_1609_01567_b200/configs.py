"""The BASELINE.json configurations, as seeded synthetic codes.

BASELINE.json "configs" (SURVEY.md section 8 shapes):
  C1  n=1024 rate 1/2, var degrees 2/3/8, 1 codeword, 50 iterations (CPU-runnable case)
  C2  n=8192 rate 1/2, batch 4096, 20 iterations
  C3  DVB-S2-shaped n=64800 rate 1/2: 12,960 vars of degree 8, 19,440 of degree 3,
      32,400 of degree 2; check degree 7 (E = 226,800); batch 1024; fixed 10 iterations
  C4  high-degree stress: n=32768, checks of degree 20-1000, vars of degree 17-200, early stop (3 dB)
  C5  C3's code, Eb/N0 0..3 dB sweep, sharded over GPUs with an error-count allreduce
"""

from __future__ import annotations

import functools
import math

from .codes import ParityCheckMatrix, generate_irregular_code

SEED = 1609_01567


def ebno_to_sigma2(ebno_db: float, rate: float) -> float:
    """channel.py:40-44: noise variance at Eb/N0 (dB), code rate R, unit bit energy."""
    if not 0.0 < rate < 1.0:
        raise ValueError("rate must be in (0, 1)")
    return 1.0 / (2.0 * rate * 10.0 ** (ebno_db / 10.0))


@functools.lru_cache(maxsize=None)
def code(name: str) -> ParityCheckMatrix:
    if name == "C1":      # 205*8 + 306*3 + 513*2 = 3584 = 512 * 7
        return generate_irregular_code({8: 205, 3: 306, 2: 513}, 512, seed=SEED + 1)
    if name == "C2":      # 1638*8 + 2458*3 + 4096*2 = 28670 edges over 4096 checks (degree 7 or 6)
        return generate_irregular_code({8: 1638, 3: 2458, 2: 4096}, 4096, seed=SEED + 2)
    if name in ("C3", "C5"):
        return generate_irregular_code({8: 12960, 3: 19440, 2: 32400}, 32400, seed=SEED + 3)
    if name == "C4":
        # high degrees spread over the range: checks of degree 20-1000 (452 checks, 24% of the
        # edges) and variables of degree 17-200 (256 variables, 9% of the edges); the rest are
        # degree-6 / degree-3 variables and checks of degree 5-6.  No degree-2 variables: with a
        # quarter of the edges on weak high-degree checks they would leave uncorrectable bits, and
        # the code must converge (early stop fires at 3 dB: ~70% of frames in 8-20 rounds).
        return generate_irregular_code({200: 16, 120: 16, 60: 32, 30: 64, 17: 128, 6: 4000, 3: 28512}, 16384,
                                       seed=SEED + 4,
                                       check_degrees={1000: 4, 500: 8, 250: 16, 120: 32, 60: 64, 33: 128, 20: 256})
    if name == "C4D":
        # round 1's C4 profile, kept as a second stress code: 16 checks of degree 1000 and 16 variables
        # of degree 200 (21% of the edges) next to degree-2/3/8 variables.  It does not converge (the
        # weak checks leave bits uncorrected), so it is a fixed-work case where the exact mode's
        # O(d^2) ordered products dominate (fast mode vs exact: bench.py other_configs).
        return generate_irregular_code({200: 16, 8: 1024, 3: 15728, 2: 16000}, 16384, seed=SEED + 4,
                                       check_degrees={1000: 16})
    raise KeyError(name)


CONFIGS = {
    "C1": dict(code="C1", batch=1, max_iterations=50, ebno_db=2.0, early_stop=True),
    "C2": dict(code="C2", batch=4096, max_iterations=20, ebno_db=2.0, early_stop=True),
    "C3": dict(code="C3", batch=1024, max_iterations=10, ebno_db=2.0, early_stop=False),
    "C4": dict(code="C4", batch=256, max_iterations=20, ebno_db=3.0, early_stop=True),
    "C5": dict(code="C5", batch=1024, max_iterations=10, ebno_db=(0.0, 1.0, 2.0, 3.0), early_stop=True),
}


def sigma2_for(name: str, ebno_db: float) -> float:
    H = code(CONFIGS[name]["code"])
    return ebno_to_sigma2(ebno_db, (H.n - H.m) / H.n)


def rate(H: ParityCheckMatrix) -> float:
    return (H.n - H.m) / H.n


__all__ = ["CONFIGS", "SEED", "code", "ebno_to_sigma2", "sigma2_for", "rate", "math"]
