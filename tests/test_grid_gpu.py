"""Grid schedule (grid.cu): a few codewords in one cooperative launch, bit-identical to the
streaming schedule and the oracle (serial.py:150-178), both stop modes, observations in."""

import numpy as np
import pytest

from paper_1609_01567_b200 import CodeTables, ParallelDecoder, configs, generate_irregular_code, priors_awgn_batch

pytestmark = pytest.mark.gpu


def _frames(H, B, ebno, seed):
    s2 = configs.ebno_to_sigma2(ebno, configs.rate(H))
    rng = np.random.default_rng(seed)
    Y = -1.0 + np.sqrt(s2) * rng.standard_normal((B, H.n))
    return Y, s2, priors_awgn_batch(Y, s2)


def _same(a, b):
    assert np.array_equal(a.est_bits, b.est_bits)
    assert np.array_equal(a.success, b.success)
    assert np.array_equal(a.iterations, b.iterations)
    assert np.array_equal(a.syn_bits, b.syn_bits)


@pytest.mark.parametrize("code,B,ebno,iters", [("C3", 1, 2.0, 50), ("C3", 5, 1.0, 12), ("C2", 8, 1.5, 30),
                                               ("C1", 3, 1.0, 0), ("C1", 7, 0.5, 25), ("C2", 32, 1.25, 20),
                                               ("C3", 13, 2.0, 15), ("C2", 33, 1.5, 20), ("C2", 64, 1.25, 20),
                                               ("C1", 50, 1.0, 30)])
@pytest.mark.parametrize("early", [True, False])
def test_grid_equals_stream_and_oracle(cuda, code, B, ebno, iters, early):
    from oracle import OracleTables

    H = configs.code(code)
    Y, s2, P = _frames(H, B, ebno, seed=B * 31 + iters)
    with ParallelDecoder(CodeTables.from_matrix(H), max_batch=B) as dec:
        g = dec.decode_priors(P, iters, early_stop=early, schedule="grid")
        st = dec.decode_priors(P, iters, early_stop=early, schedule="stream")
        _same(g, st)
        _same(dec.decode_batch(Y, s2, iters, early_stop=early, schedule="grid"), st)  # observations in
    est, ok, its, z = OracleTables.from_matrix(H).decode_batch(P, iters, fixed_iterations=not early)
    assert np.array_equal(g.estimates(), est) and np.array_equal(g.syndromes(), z)
    assert np.array_equal(g.success.astype(bool), ok) and np.array_equal(g.iterations, its)


def test_grid_auto_for_single_frames(cuda):
    # the reference-facing decode(y) of a large code takes the grid schedule (one launch)
    from paper_1609_01567_b200 import _native

    H = configs.code("C2")
    Y, s2, P = _frames(H, 2, 1.5, 7)
    with ParallelDecoder(CodeTables.from_matrix(H), max_batch=1) as dec:
        dec.decode(Y[0], s2, 20)
        k0 = _native.load_library().ldpc_kernel_launches()
        r = dec.decode(Y[1], s2, 20)
        assert _native.load_library().ldpc_kernel_launches() - k0 == 1
        ref = dec.decode_priors(P[1:2], 20, schedule="stream")[0]
        assert np.array_equal(r.estimate, ref.estimate) and r.iterations_used == ref.iterations_used


def test_grid_refusals(cuda):
    H = generate_irregular_code({20: 40, 3: 400, 2: 400}, 400, seed=3)   # a variable degree past 16
    _, _, P = _frames(H, 2, 1.0, 1)
    with ParallelDecoder(CodeTables.from_matrix(H), max_batch=16) as dec:
        with pytest.raises(ValueError):
            dec.decode_priors(P, 5, schedule="grid")
        dec.decode_priors(P, 5)  # auto: streams
    H1 = configs.code("C1")
    _, _, P1 = _frames(H1, 65, 1.0, 2)
    with ParallelDecoder(CodeTables.from_matrix(H1), max_batch=65) as dec:
        with pytest.raises(ValueError):
            dec.decode_priors(P1, 5, schedule="grid")  # more than 64 codewords
