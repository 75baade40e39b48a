"""f4 fp32 fast mode, any node degree: NOT bit-exact.  Tolerance against the
ORACLE (oracle/ldpc_oracle.c, the reference's serial.py:63-178 restated), as stated in DESIGN.md:

  * C-phase (check -> variable, serial.py:92-112): |LLR_fast - LLR_oracle| <= 1e-4
    where the oracle's message is not saturated (1e-6 < r < 1 - 1e-6, |LLR| < 13.8)
  * V-phase (variable -> check, serial.py:63-89): mean |dLLR| <= 2e-4, max <= 0.25 on the same set
    (fp32 loses relative precision in 1 - r once r is within ~1e-7 of 1)
  * decoded frames: >= 98 % identical hard decisions and iteration counts vs the oracle;
    success <=> zero syndrome holds exactly

Nodes of degree <= 16 run the reference's product order in fp32 (kernels_fast.cu); higher degrees
the O(d) kernels (kernels_fastod.cu: prefix x suffix products on the check side, log-ratio sums
on the variable side).  LDPC_FAST_OD=1 sends every degree to the O(d) kernels: the subprocess
test runs the same checks under it."""

import os
import subprocess
import sys

import numpy as np
import pytest

from conftest import ROOT
from paper_1609_01567_b200 import CodeTables, ParallelDecoder, configs, priors_awgn_batch
from paper_1609_01567_b200 import values_to_check, values_to_variable

pytestmark = pytest.mark.gpu

C_PHASE_TOL = 1e-4
V_PHASE_MEAN, V_PHASE_MAX = 2e-4, 0.25
FRAME_AGREEMENT = 0.98


def _llr(x):
    return np.log(x) - np.log1p(-x)


def _unsaturated(x):
    return (x > 1e-6) & (x < 1 - 1e-6)


@pytest.mark.parametrize("code", ["C1", "C3", "C4"])
def test_message_tolerance_vs_oracle(cuda, code):
    from oracle import OracleTables

    H = configs.code(code)
    T, O = CodeTables.from_matrix(H), OracleTables.from_matrix(H)
    rng = np.random.default_rng(7)
    B = 3
    P = rng.uniform(size=(B, H.n))
    R = rng.uniform(size=(B, H.total_edges))
    Q = rng.uniform(size=(B, H.total_edges))
    c_fast = values_to_variable(Q, T, precision="fp32")
    v_fast = values_to_check(P, R, T, precision="fp32")
    for b in range(B):
        c_ref = O.values_to_variable(Q[b])
        ok = _unsaturated(c_ref)
        assert ok.mean() > 0.5
        assert np.abs(_llr(c_fast[b][ok]) - _llr(c_ref[ok])).max() <= C_PHASE_TOL
        v_ref = O.values_to_check(P[b], R[b])
        ok = _unsaturated(v_ref)
        d = np.abs(_llr(v_fast[b][ok]) - _llr(v_ref[ok]))
        assert d.mean() <= V_PHASE_MEAN and d.max() <= V_PHASE_MAX, (d.mean(), d.max())


def test_high_degree_messages_vs_oracle(cuda):
    # one check of degree 1200 and one variable of degree 700 (longer than one 512-row block pass:
    # the two-pass O(d) kernels), plus low-degree filler
    from oracle import OracleTables
    from paper_1609_01567_b200 import ParityCheckMatrix

    n, m = 1400, 720
    ones = {(0, j) for j in range(1200)} | {(i, 1399) for i in range(700)}
    rng = np.random.default_rng(3)
    for j in range(1400):
        for i in rng.choice(np.arange(1, m), size=2, replace=False):
            ones.add((int(i), j))
    for i in range(m):
        ones.add((i, int(rng.integers(n))))
    H = ParityCheckMatrix(n, m, tuple(sorted(ones)))
    T, O = CodeTables.from_matrix(H), OracleTables.from_matrix(H)
    dv, dc = H.degrees()
    assert dc.max() >= 1200 and dv.max() >= 700
    # messages near 1/2 keep the long products away from underflow, so the comparison is meaningful
    P = rng.uniform(0.3, 0.7, size=(2, n))
    R = rng.uniform(0.45, 0.55, size=(2, H.total_edges))
    Q = rng.uniform(0.45, 0.55, size=(2, H.total_edges))
    c_fast = values_to_variable(Q, T, precision="fp32")
    v_fast = values_to_check(P, R, T, precision="fp32")
    for b in range(2):
        c_ref = O.values_to_variable(Q[b])
        ok = _unsaturated(c_ref)
        assert np.abs(_llr(c_fast[b][ok]) - _llr(c_ref[ok])).max() <= C_PHASE_TOL
        v_ref = O.values_to_check(P[b], R[b])
        ok = _unsaturated(v_ref)
        d = np.abs(_llr(v_fast[b][ok]) - _llr(v_ref[ok]))
        assert d.mean() <= V_PHASE_MEAN and d.max() <= V_PHASE_MAX, (d.mean(), d.max())


@pytest.mark.parametrize("code,frames,iters,ebnos", [
    ("C1", 256, 50, (1.0, 1.5, 2.0)),
    ("C2", 64, 20, (1.0, 2.0)),
    ("C4", 32, 20, (3.0, 3.5)),
])
def test_decode_agreement_vs_oracle(cuda, code, frames, iters, ebnos):
    from oracle import OracleTables

    H = configs.code(code)
    T, O = CodeTables.from_matrix(H), OracleTables.from_matrix(H)
    rng = np.random.default_rng(11)
    with ParallelDecoder(T, max_batch=frames) as dec:
        for ebno in ebnos:
            s2 = configs.ebno_to_sigma2(ebno, configs.rate(H))
            P = priors_awgn_batch(-1.0 + np.sqrt(s2) * rng.standard_normal((frames, H.n)), s2)
            fast = dec.decode_priors(P, iters, precision="fp32")
            est, ok, its, z = O.decode_batch(P, iters)
            same = np.all(fast.estimates() == est, axis=1)
            assert same.mean() >= FRAME_AGREEMENT, (ebno, same.mean())
            assert (fast.iterations == its).mean() >= FRAME_AGREEMENT, (ebno, (fast.iterations == its).mean())
            # internal consistency holds exactly in fast mode too: success <=> zero syndrome
            assert np.array_equal(fast.success.astype(bool), ~fast.syndromes().any(axis=1))


def test_fast_mode_high_degree_fixed_iterations(cuda):
    # C4 (checks up to degree 1000) in fast mode, fixed iterations, both schedules' entry points
    import torch

    H = configs.code("C4")
    T = CodeTables.from_matrix(H)
    s2 = configs.ebno_to_sigma2(3.0, configs.rate(H))
    P = priors_awgn_batch(-1.0 + np.sqrt(s2) * np.random.default_rng(2).standard_normal((40, H.n)), s2)
    with ParallelDecoder(T, max_batch=40) as dec:
        host = dec.decode_priors(P, 6, early_stop=False, precision="fp32")
        est, ok, its, syn = dec.decode_device(torch.from_numpy(P).cuda(), 6, early_stop=False, precision="fp32")
        torch.cuda.synchronize()
    assert np.array_equal(est.cpu().numpy().view(np.uint32), host.est_bits)  # deterministic
    assert (host.iterations == 6).all()


def test_all_degrees_through_od_kernels():
    # the same tolerance checks with every degree on the O(d) kernels (LDPC_FAST_OD=1, read once per
    # process, hence a subprocess)
    env = dict(os.environ, LDPC_FAST_OD="1")
    out = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-m", "gpu", "-k",
                          "message_tolerance_vs_oracle or decode_agreement_vs_oracle or high_degree_messages",
                          str(ROOT / "tests" / "test_fast_gpu.py")], capture_output=True, text=True, env=env,
                         cwd=str(ROOT), timeout=900)
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-2000:]


@pytest.mark.parametrize("seed", range(3))
def test_random_high_degree_codes_vs_oracle(cuda, seed):
    # random irregular codes with a few checks / variables past one O(d) block pass (> 512 rows) next
    # to low-degree nodes: message tolerance vs the oracle on random states
    from oracle import OracleTables

    from paper_1609_01567_b200 import generate_irregular_code

    rng = np.random.default_rng(500 + seed)
    m = 1400
    H = generate_irregular_code({600 + 50 * seed: 1, 40: 4, 3: 900, 2: 1000}, m, seed=seed,
                                check_degrees={700 + 100 * seed: 1, 130: 2})
    T, O = CodeTables.from_matrix(H), OracleTables.from_matrix(H)
    P = rng.uniform(0.2, 0.8, size=(2, H.n))
    R = rng.uniform(0.45, 0.55, size=(2, H.total_edges))
    Q = rng.uniform(0.45, 0.55, size=(2, H.total_edges))
    c_fast = values_to_variable(Q, T, precision="fp32")
    v_fast = values_to_check(P, R, T, precision="fp32")
    for b in range(2):
        c_ref = O.values_to_variable(Q[b])
        ok = _unsaturated(c_ref)
        assert np.abs(_llr(c_fast[b][ok]) - _llr(c_ref[ok])).max() <= C_PHASE_TOL
        v_ref = O.values_to_check(P[b], R[b])
        ok = _unsaturated(v_ref)
        d = np.abs(_llr(v_fast[b][ok]) - _llr(v_ref[ok]))
        assert d.mean() <= V_PHASE_MEAN and d.max() <= V_PHASE_MAX, (d.mean(), d.max())
