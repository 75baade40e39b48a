"""On-chip schedule (onchip.cu): whole decode in one CTA's / cluster's shared memory, bit-exact.

Small codes decode each codeword entirely in shared memory (cluster size 1, 2, 4 or 8 CTAs over
DSMEM).  The results must equal the streaming schedule's and the oracle's (serial.py:150-178)."""

import numpy as np
import pytest

from paper_1609_01567_b200 import CodeTables, ParallelDecoder, configs, generate_irregular_code, priors_awgn_batch

pytestmark = pytest.mark.gpu


def _priors(H, B, ebno_db, seed):
    s2 = configs.ebno_to_sigma2(ebno_db, configs.rate(H))
    rng = np.random.default_rng(seed)
    return priors_awgn_batch(-1.0 + np.sqrt(s2) * rng.standard_normal((B, H.n)), s2)


def _same(a, b):
    return (np.array_equal(a.est_bits, b.est_bits) and np.array_equal(a.syn_bits, b.syn_bits)
            and np.array_equal(a.success, b.success) and np.array_equal(a.iterations, b.iterations))


CODES = {
    "C1": lambda: configs.code("C1"),                                               # 1 CTA
    "C2": lambda: configs.code("C2"),                                               # cluster of 2
    "cs4": lambda: generate_irregular_code({8: 2000, 3: 6000, 2: 12000}, 10000, seed=41),   # cluster of 4
    "cs8": lambda: generate_irregular_code({8: 4000, 3: 12000, 2: 24000}, 20000, seed=43),  # cluster of 8
}


@pytest.mark.parametrize("name,B,ebno,iters,early", [
    ("C1", 70, 2.0, 50, True), ("C1", 1, 1.0, 50, True), ("C1", 33, 1.5, 12, False),
    ("C2", 40, 1.8, 20, True), ("C2", 17, 1.0, 6, False),
    ("cs4", 9, 1.8, 15, True), ("cs8", 5, 1.8, 10, True), ("cs8", 3, 1.0, 4, False),
])
def test_onchip_equals_stream_and_oracle(cuda, name, B, ebno, iters, early):
    from oracle import OracleTables

    H = CODES[name]()
    P = _priors(H, B, ebno, seed=B + iters)
    with ParallelDecoder(CodeTables.from_matrix(H), max_batch=B) as dec:
        on = dec.decode_priors(P, iters, early_stop=early, schedule="onchip")
        st = dec.decode_priors(P, iters, early_stop=early, schedule="stream")
        auto = dec.decode_priors(P, iters, early_stop=early)
    assert _same(on, st) and _same(on, auto)
    k = min(B, 8)
    est, ok, its, z = OracleTables.from_matrix(H).decode_batch(P[:k], iters, fixed_iterations=not early)
    assert np.array_equal(on.estimates()[:k], est) and np.array_equal(on.syndromes()[:k], z)
    assert np.array_equal(on.success[:k].astype(bool), ok) and np.array_equal(on.iterations[:k], its)


def test_onchip_high_degree_forced(cuda):
    # auto mode streams high-degree codes; forcing the on-chip schedule still decodes them exactly
    from oracle import OracleTables

    H = configs.code("C4")
    P = _priors(H, 3, 1.5, seed=5)
    with ParallelDecoder(CodeTables.from_matrix(H), max_batch=3) as dec:
        on = dec.decode_priors(P, 4, early_stop=False, schedule="onchip")
        st = dec.decode_priors(P, 4, early_stop=False)
    assert _same(on, st)
    est, ok, its, z = OracleTables.from_matrix(H).decode_batch(P, 4, fixed_iterations=True)
    assert np.array_equal(on.estimates(), est) and np.array_equal(on.syndromes(), z)


def test_onchip_refuses_codes_that_do_not_fit(cuda):
    H = configs.code("C3")
    with ParallelDecoder(CodeTables.from_matrix(H), max_batch=1) as dec:
        with pytest.raises(ValueError):
            dec.decode_priors(_priors(H, 1, 2.0, seed=1), 2, schedule="onchip")
        with pytest.raises(ValueError):
            dec.decode_priors(_priors(H, 1, 2.0, seed=1), 2, schedule="sideways")


def test_random_codes_all_schedules(cuda):
    # random valid H (every row and column non-empty; degree-1 nodes, dense rows past the
    # register-path degrees), both schedules, both stop modes, against the oracle
    from conftest import random_parity_matrix
    from oracle import OracleTables

    rng = np.random.default_rng(2024)
    for case in range(12):
        H = random_parity_matrix(rng, max_m=48, max_n=96)
        B = int(rng.integers(1, 40))
        it = int(rng.integers(0, 12))
        early = bool(case % 2)
        P = rng.uniform(size=(B, H.n))
        P[rng.uniform(size=P.shape) < 0.05] = 0.0   # saturated priors (serial.py:49 overflow)
        P[rng.uniform(size=P.shape) < 0.05] = 1.0
        est, ok, its, z = OracleTables.from_matrix(H).decode_batch(P, it, fixed_iterations=not early)
        with ParallelDecoder(CodeTables.from_matrix(H), max_batch=B) as dec:
            for sched in ("stream", "onchip"):
                r = dec.decode_priors(P, it, early_stop=early, schedule=sched)
                assert np.array_equal(r.estimates(), est), (case, sched)
                assert np.array_equal(r.syndromes(), z), (case, sched)
                assert np.array_equal(r.success.astype(bool), ok), (case, sched)
                assert np.array_equal(r.iterations, its), (case, sched)
