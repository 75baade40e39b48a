"""Per-phase parity of the CUDA kernels (serial.py:63-147), bit-exact.

Against (a) the reference's outputs (golden fixtures), (b) the CPU oracle on
random batched states of the full-size configs, and (c) the reference's own
phase KATs (test_serial.py:66-181)."""

import numpy as np
import pytest

from conftest import PAIRS_14_7, dense_syndrome, golden_code, random_parity_matrix
from paper_1609_01567_b200 import (
    CodeTables,
    ParityCheckMatrix,
    estimate,
    syndrome,
    values_to_check,
    values_to_variable,
)
from paper_1609_01567_b200 import configs

pytestmark = pytest.mark.gpu


def bits(a):
    return np.ascontiguousarray(a, dtype=np.float64).view(np.uint64)


@pytest.fixture(scope="module")
def tables14(cuda):
    return CodeTables.from_matrix(ParityCheckMatrix(14, 7, PAIRS_14_7))


@pytest.fixture(scope="module")
def chain3(cuda):
    H = ParityCheckMatrix(3, 2, ((0, 0), (0, 1), (1, 1), (1, 2)))
    return H, CodeTables.from_matrix(H)


def test_golden_phases(cuda, golden_tables, golden_phases):
    for name in golden_phases["names"]:
        H = golden_code(golden_tables, name)
        T = CodeTables.from_matrix(H)
        g = lambda k: golden_phases[f"{name}/{k}"]  # noqa: E731
        # batched over the S states at once, and one state at a time
        assert np.array_equal(bits(values_to_check(g("p"), g("r"), T)), bits(g("to_check"))), name
        assert np.array_equal(bits(values_to_variable(g("q"), T)), bits(g("to_variable"))), name
        assert np.array_equal(estimate(g("p"), g("r"), T), g("estimate")), name
        assert np.array_equal(syndrome(g("chat_in"), T), g("syndrome")), name
        assert np.array_equal(bits(values_to_variable(g("q")[1], T)), bits(g("to_variable")[1])), name


@pytest.mark.parametrize("code,B", [("C1", 5), ("C2", 3), ("C3", 2), ("C4", 3)])
def test_random_states_vs_oracle(cuda, code, B):
    from oracle import OracleTables

    H = configs.code(code)
    T = CodeTables.from_matrix(H)
    O = OracleTables.from_matrix(H)
    rng = np.random.default_rng(sum(map(ord, code)))
    P = rng.uniform(size=(B, H.n))
    R = rng.uniform(size=(B, H.total_edges))
    Q = rng.uniform(size=(B, H.total_edges))
    C = rng.integers(0, 2, size=(B, H.n)).astype(np.uint8)
    q = values_to_check(P, R, T)
    r = values_to_variable(Q, T)
    c = estimate(P, R, T)
    z = syndrome(C, T)
    for b in range(B):
        assert np.array_equal(bits(q[b]), bits(O.values_to_check(P[b], R[b]))), (code, b)
        assert np.array_equal(bits(r[b]), bits(O.values_to_variable(Q[b]))), (code, b)
        assert np.array_equal(c[b], O.estimate(P[b], R[b])), (code, b)
        assert np.array_equal(z[b], O.syndrome(C[b])), (code, b)


def test_saturated_golden(cuda, golden_saturated):
    """The reference's outputs on high-SNR states (tests/golden/saturated.npz), all states batched."""
    g = golden_saturated
    for name in g["names"]:
        n, m = (int(x) for x in g[f"{name}/nm"])
        T = CodeTables.from_matrix(ParityCheckMatrix(n, m, g[f"{name}/ones"]))
        k = lambda key: g[f"{name}/{key}"]  # noqa: E731
        assert np.array_equal(bits(values_to_check(k("p"), k("r"), T)), bits(k("to_check"))), name
        assert np.array_equal(bits(values_to_variable(k("q"), T)), bits(k("to_variable"))), name
        assert np.array_equal(estimate(k("p"), k("r"), T), k("estimate")), name


@pytest.mark.parametrize("code,B", [("C1", 4), ("C2", 3), ("C4", 2)])
def test_saturated_states_vs_oracle(cuda, code, B):
    """High-SNR states: messages and priors at exactly 0 / 1 (and -0.0, denormals, tiny values),
    so most variable-side numerators q1 are +-0 over a positive denominator, some denominators are
    0 (the reference's 1/2) and some tiny.  Every slow-path division branch of every variable kernel
    family (ring, register, mid-degree, chains at C4) must give the oracle's bits, signs included."""
    from oracle import OracleTables

    H = configs.code(code)
    T = CodeTables.from_matrix(H)
    O = OracleTables.from_matrix(H)
    rng = np.random.default_rng(7 + sum(map(ord, code)))
    special = np.array([0.0, -0.0, 1.0, 5e-324, 1e-300, 1e-160, 1.0 - 2.0 ** -53, 0.5])

    def draw(shape, frac):
        x = rng.uniform(size=shape)
        pick = rng.uniform(size=shape) < frac
        x[pick] = special[rng.integers(0, special.size, size=int(pick.sum()))]
        return x

    P = draw((B, H.n), 0.5)
    R = draw((B, H.total_edges), 0.6)
    R[:, : H.total_edges // 3] = rng.choice([0.0, 1.0], size=(B, H.total_edges // 3))
    q = values_to_check(P, R, T)
    c = estimate(P, R, T)
    for b in range(B):
        assert np.array_equal(bits(q[b]), bits(O.values_to_check(P[b], R[b]))), (code, b)
        assert np.array_equal(c[b], O.estimate(P[b], R[b])), (code, b)


# ---- test_serial.py KATs, run on the GPU kernels ----------------------------

class TestValuesToCheck:
    def test_degree_one_variable_passes_prior(self, chain3):
        _, T = chain3
        q = values_to_check(np.array([0.3, 0.6, 0.9]), np.array([0.1, 0.2, 0.3, 0.4]), T)
        assert q[int(np.flatnonzero(T.variable.v == 0)[0])] == 0.3
        assert q[int(np.flatnonzero(T.variable.v == 2)[0])] == 0.9

    def test_uniform_messages_return_prior(self, tables14):
        p = np.linspace(0.05, 0.95, 14)
        q = values_to_check(p, np.full(31, 0.5), tables14)
        assert q == pytest.approx(p[tables14.variable.v], abs=1e-15)

    def test_two_term_product(self, chain3):
        _, T = chain3
        q = values_to_check(np.full(3, 0.5), np.full(4, 0.8), T)
        for k in np.flatnonzero(T.variable.v == 1):
            assert q[k] == pytest.approx(0.8, abs=1e-15)

    def test_double_underflow_saturates(self, chain3):
        _, T = chain3
        q = values_to_check(np.array([0.5, 1.0, 0.5]), np.zeros(4), T)
        assert q[int(np.flatnonzero(T.variable.v == 1)[0])] == 0.5

    def test_messages_stay_in_unit_interval(self, tables14):
        rng = np.random.default_rng(3)
        q = values_to_check(rng.uniform(size=(50, 14)), rng.uniform(size=(50, 31)), tables14)
        assert ((0.0 <= q) & (q <= 1.0)).all()


class TestValuesToVariable:
    def test_degree_two_check_reproduces_reference_rounding(self, chain3):
        # serial.py:111 evaluates 1-(0.5+0.5*(1-2q)); for q=0.2 that is 0.19999999999999996,
        # not 0.2 (the reference's own test_serial.py:113-123 expects 0.2 and fails on the
        # reference): the kernel must reproduce the reference arithmetic, not "fix" it.
        _, T = chain3
        q = np.array([0.2, 0.7, 0.6, 0.9])
        r = values_to_variable(q, T)
        chk = T.check
        for pos in range(4):
            target = int(chk.e[pos])
            group = [int(chk.e[i]) for i in range(int(chk.s[pos]), int(chk.s[pos]) + 2)]
            other = next(g for g in group if g != target)
            assert r[target] == 1.0 - (0.5 + 0.5 * (1.0 - 2.0 * q[other]))

    def test_erasure_annihilates(self, tables14):
        assert (values_to_variable(np.full(31, 0.5), tables14) == 0.5).all()

    def test_certain_zero_neighbors(self, tables14):
        assert (values_to_variable(np.zeros(31), tables14) == 0.0).all()

    def test_range_property(self, tables14):
        rng = np.random.default_rng(4)
        r = values_to_variable(rng.uniform(size=(50, 31)), tables14)
        assert ((0.0 <= r) & (r <= 1.0)).all()


class TestEstimate:
    def test_single_edge_decision(self, chain3):
        _, T = chain3
        r = np.full(4, 0.5)
        r[int(np.flatnonzero(T.variable.v == 0)[0])] = 0.8
        assert estimate(np.full(3, 0.5), r, T)[0] == 1

    def test_uniform_messages_decide_by_prior(self, tables14):
        assert (estimate(np.full(14, 0.3), np.full(31, 0.5), tables14) == 0).all()

    def test_exact_tie_decides_one(self, tables14):
        assert (estimate(np.full(14, 0.5), np.full(31, 0.5), tables14) == 1).all()


class TestSyndrome:
    def test_all_zero(self, tables14):
        assert not syndrome(np.zeros(14, dtype=np.uint8), tables14).any()

    def test_unit_vector_lights_adjacent_checks(self, tables14):
        c = np.zeros(14, dtype=np.uint8)
        c[0] = 1
        assert sorted(np.flatnonzero(syndrome(c, tables14)).tolist()) == [0, 2, 3, 5]

    def test_against_dense_oracle(self, cuda):
        rng = np.random.default_rng(12)
        for _ in range(50):
            H = random_parity_matrix(rng)
            c = rng.integers(0, 2, size=(3, H.n)).astype(np.uint8)
            assert np.array_equal(syndrome(c, H), dense_syndrome(H, c))

    def test_length_mismatch(self, tables14):
        with pytest.raises(ValueError):
            syndrome(np.zeros(13, dtype=np.uint8), tables14)


def test_fast_division_is_bitwise_ddiv_rn(cuda):
    """The branch-free division path (common.cuh ddiv_fast) equals __ddiv_rn bit for bit."""
    from paper_1609_01567_b200 import _native

    res = np.zeros(2, dtype=np.int64)
    for seed in (1, 2, 3, 4):
        rc = _native.lib().ldpc_selftest_division(seed, 1 << 28, res.ctypes.data_as(_native.P_i64))
        _native.check(rc, "selftest")
        assert res[0] == 0, f"{res[0]} mismatches"
        assert res[1] > (1 << 26)


def test_unbounded_degree_phases_and_decode(cuda):
    # "no bound on node degree": a check of degree 13000 (past the shared-memory staging of
    # every tile width, so the chains kernel stages in the workspace scratch) and a variable
    # of degree 4000 (same for r / 1-r), bit-exact against the oracle in both phases and a decode
    from oracle import OracleTables
    from paper_1609_01567_b200 import ParallelDecoder, generate_irregular_code, priors_awgn_batch

    H = generate_irregular_code({4000: 1, 2: 15999}, 6000, seed=5, check_degrees={13000: 1})
    dv, dc = H.degrees()
    assert dv.max() == 4000 and dc.max() == 13000
    T = CodeTables.from_matrix(H)
    O = OracleTables.from_matrix(H)
    rng = np.random.default_rng(11)
    B = 2
    P = rng.uniform(size=(B, H.n))
    R = rng.uniform(size=(B, H.total_edges))
    Q = rng.uniform(size=(B, H.total_edges))
    assert np.array_equal(bits(values_to_variable(Q, T)), bits(np.stack([O.values_to_variable(q) for q in Q])))
    assert np.array_equal(bits(values_to_check(P, R, T)), bits(np.stack([O.values_to_check(p, r) for p, r in zip(P, R)])))
    assert np.array_equal(estimate(P, R, T), np.stack([O.estimate(p, r) for p, r in zip(P, R)]))
    s2 = 0.8
    Pd = priors_awgn_batch(-1.0 + np.sqrt(s2) * rng.standard_normal((B, H.n)), s2)
    with ParallelDecoder(T, max_batch=B) as dec:
        res = dec.decode_priors(Pd, 2, early_stop=False)
    est, ok, its, z = O.decode_batch(Pd, 2, fixed_iterations=True)
    assert np.array_equal(res.estimates(), est) and np.array_equal(res.syndromes(), z)
    assert np.array_equal(res.success.astype(bool), ok) and np.array_equal(res.iterations, its)


def test_engine_shared_state_phases(cuda):
    # engine.py:33-76, 157-190: plan_pages / SharedDecodeState / parallel_* write the state in place,
    # equal to the single-phase functions and the oracle, for any page plan
    from oracle import OracleTables
    from paper_1609_01567_b200 import (SharedDecodeState, parallel_estimate, parallel_syndrome, parallel_to_check,
                                       parallel_to_variable, plan_pages)

    H = configs.code("C1")
    T = CodeTables.from_matrix(H)
    O = OracleTables.from_matrix(H)
    rng = np.random.default_rng(8)
    with pytest.raises(ValueError):
        plan_pages(10, 0)
    with pytest.raises(ValueError):
        plan_pages(0, 4)
    for group in (1, 7, 512):
        plan = plan_pages(T.total_edges, group)
        assert plan.page_count == -(-T.total_edges // group) and plan.page_width(plan.page_count - 1) >= 1
        st = SharedDecodeState.allocate(T)
        st.p[:] = rng.uniform(size=H.n)
        st.q[:] = st.p[T.variable.v]                      # serial.py:58
        q_id = st.q
        parallel_to_variable(st, T, plan)
        assert np.array_equal(bits(st.r), bits(O.values_to_variable(st.q)))
        parallel_to_check(st, T, plan)
        assert st.q is q_id and np.array_equal(bits(st.q), bits(O.values_to_check(st.p, st.r)))
        parallel_estimate(st, T, plan)
        assert np.array_equal(st.estimate, O.estimate(st.p, st.r))
        parallel_syndrome(st, T, plan)
        assert np.array_equal(st.syndrome, O.syndrome(st.estimate))


@pytest.mark.parametrize("check_degrees,extra_vars,B", [
    ({17: 40, 24: 40, 30: 40, 32: 40}, {}, 70),            # register path past 16 (V = 1)
    ({33: 30, 40: 30}, {}, 40),                            # just past it: the chains kernel
    ({90: 8, 300: 2}, {17: 30, 33: 10, 120: 3}, 36),       # small chains blocks, both sides
    ({}, {20: 20, 24: 20, 30: 10, 32: 5}, 70),              # variable degrees 17-32: kernels_varmid.cu
    ({}, {40: 10, 48: 6, 64: 4, 65: 2}, 40),                # 33-64 (4-warp blocks), 65: chains
    ({48: 12, 64: 8, 65: 2}, {}, 38),                       # checks 33-64 (kernels_varmid.cu), 65: chains
])
def test_mid_degrees_vs_oracle(cuda, check_degrees, extra_vars, B):
    # DVB-S2's high-rate codes have check degrees 18-30 (rates 4/5 .. 9/10)
    from oracle import OracleTables
    from paper_1609_01567_b200 import ParallelDecoder, generate_irregular_code, priors_awgn_batch

    vdeg = {8: 600, 3: 900, 2: 1800, **extra_vars}
    E = sum(d * c for d, c in vdeg.items())
    m = sum(check_degrees.values()) + (E - sum(d * c for d, c in check_degrees.items())) // 7
    H = generate_irregular_code(vdeg, m, seed=21, check_degrees=check_degrees)
    dc = H.degrees()[1]
    for d in check_degrees:
        assert (dc == d).sum() >= check_degrees[d]
    T = CodeTables.from_matrix(H)
    O = OracleTables.from_matrix(H)
    rng = np.random.default_rng(22)
    Q = rng.uniform(size=(3, H.total_edges))
    assert np.array_equal(bits(values_to_variable(Q, T)), bits(np.stack([O.values_to_variable(q) for q in Q])))
    s2 = 0.5
    P = priors_awgn_batch(-1.0 + np.sqrt(s2) * rng.standard_normal((B, H.n)), s2)
    with ParallelDecoder(T, max_batch=B) as dec:
        for early in (True, False):
            res = dec.decode_priors(P, 12, early_stop=early, schedule="stream")
            est, ok, its, z = O.decode_batch(P, 12, fixed_iterations=not early)
            assert np.array_equal(res.estimates(), est) and np.array_equal(res.syndromes(), z)
            assert np.array_equal(res.success.astype(bool), ok) and np.array_equal(res.iterations, its)
