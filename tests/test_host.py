"""Host-side logic (no GPU): the input type, file format, generator, priors, bit packing."""

import numpy as np
import pytest

from conftest import GOLDEN, PAIRS_14_7
from paper_1609_01567_b200 import (
    CodeFormatError,
    ParityCheckMatrix,
    generate_irregular_code,
    parse_alist,
    priors_awgn,
    priors_awgn_batch,
    serialize_alist,
    unpack_bits,
)
from paper_1609_01567_b200 import configs


class TestParityCheckMatrix:
    # codes.py:42-61 invariants
    def test_sorted_and_views(self):
        H = ParityCheckMatrix(3, 2, ((1, 2), (0, 0), (0, 1), (1, 1)))
        assert H.ones == ((0, 0), (0, 1), (1, 1), (1, 2))
        assert H.col_rows() == [[0], [0, 1], [1]]
        assert H.row_cols() == [[0, 1], [1, 2]]
        assert H.total_edges == 4 and H.k == 1

    @pytest.mark.parametrize("n,m,ones", [
        (2, 2, ((0, 0), (0, 0), (1, 1))),      # duplicate
        (2, 2, ((0, 0), (2, 1), (1, 1))),      # row out of range
        (2, 2, ((0, 0), (1, 2))),              # col out of range
        (2, 2, ((0, 0), (0, 1))),              # empty row
        (2, 2, ((0, 0), (1, 0))),              # empty column
        (0, 2, ()),                            # bad dimension
    ])
    def test_rejects(self, n, m, ones):
        with pytest.raises(ValueError):
            ParityCheckMatrix(n, m, ones)

    # value semantics of the reference's frozen dataclass (codes.py:29-61)
    def test_any_iterable_of_pairs(self):
        pairs = [(1, 2), (0, 0), (0, 1), (1, 1)]
        ref = ParityCheckMatrix(3, 2, tuple(pairs))
        assert ParityCheckMatrix(3, 2, set(pairs)) == ref
        assert ParityCheckMatrix(3, 2, (p for p in pairs)) == ref
        assert ParityCheckMatrix(3, 2, [list(p) for p in pairs]) == ref
        assert ParityCheckMatrix(3, 2, np.array(pairs)) == ref
        assert ParityCheckMatrix(3, 2, [(np.int64(r), float(c)) for r, c in pairs]) == ref

    def test_immutable_and_hashable(self):
        H = ParityCheckMatrix(14, 7, PAIRS_14_7)
        H2 = ParityCheckMatrix(14, 7, tuple(reversed(PAIRS_14_7)))
        assert H == H2 and hash(H) == hash(H2)
        assert len({H, H2, ParityCheckMatrix(3, 2, ((0, 0), (0, 1), (1, 2)))}) == 2
        with pytest.raises(AttributeError):
            H.n = 5
        with pytest.raises(AttributeError):
            del H.m
        with pytest.raises(ValueError):
            H.rows[0] = 3          # read-only coordinates
        assert H != "H" and H != ParityCheckMatrix(14, 7, PAIRS_14_7[:-1] + ((6, 13),))

    def test_pickle_round_trip(self):
        import copy
        import pickle

        H = ParityCheckMatrix(14, 7, PAIRS_14_7)
        assert pickle.loads(pickle.dumps(H)) == H
        assert copy.deepcopy(H) == H


def test_code_info_value_type():
    # codes.py:95-105: frozen dataclass, equal field by field, readable repr
    from paper_1609_01567_b200 import CodeInfo

    H = ParityCheckMatrix(14, 7, PAIRS_14_7)
    info = CodeInfo.from_matrix(H)
    assert info == CodeInfo(31, 14, 7) and hash(info) == hash(CodeInfo(31, 14, 7))
    assert repr(info) == "CodeInfo(total_edges=31, var_nodes=14, check_nodes=7)"
    with pytest.raises(AttributeError):
        info.total_edges = 1


def test_code_tables_constructible_from_fields():
    # tables.py:95-105: CodeTables(variable, check, n, m, total_edges, var_group_start, var_group_size)
    # without touching the device; immutable
    from conftest import GOLDEN_CHECK, GOLDEN_VARIABLE
    from paper_1609_01567_b200 import CodeTables, EdgeTables

    var = EdgeTables("variable", *(np.array(GOLDEN_VARIABLE[k]) for k in "evctsu"))
    chk = EdgeTables("check", *(np.array(GOLDEN_CHECK[k]) for k in "evctsu"))
    firsts = var.u == 0
    gs, gz = np.empty(14, np.int64), np.empty(14, np.int64)
    gs[var.v[firsts]], gz[var.v[firsts]] = var.s[firsts], var.t[firsts]
    T = CodeTables(var, chk, 14, 7, 31, gs, gz)
    assert T.n == 14 and T.m == 7 and T.total_edges == 31
    assert T.variable is var and T.check is chk
    assert np.array_equal(T.var_group_size, [4, 2, 2, 3, 2, 2, 2, 2, 2, 2, 2, 2, 2, 2])
    with pytest.raises(AttributeError):
        T.n = 3
    with pytest.raises(ValueError):
        CodeTables(chk, var, 14, 7, 31, gs, gz)


class TestAlist:
    def test_fixture_round_trip(self):
        text = (GOLDEN / "ldpc_14_7.alist").read_text()
        H = parse_alist(text)
        assert H == ParityCheckMatrix(14, 7, PAIRS_14_7)
        assert parse_alist(serialize_alist(H)) == H

    def test_inconsistent(self):
        with pytest.raises(CodeFormatError):
            parse_alist("2 1\n1 2\n1 1\n2\n1\n1\n1\n")

    def test_large_round_trip(self):
        H = configs.code("C1")
        assert parse_alist(serialize_alist(H)) == H


class TestGenerator:
    def test_dvbs2_profile(self):
        H = configs.code("C3")
        dv, dc = H.degrees()
        assert H.n == 64800 and H.m == 32400 and H.total_edges == 226800
        assert sorted(np.unique(dv, return_counts=True)[1].tolist()) == [12960, 19440, 32400]
        assert (dc == 7).all()

    def test_high_degree_profile(self):
        H = configs.code("C4")
        dv, dc = H.degrees()
        assert dv.max() == 200 and dc.max() == 1000 and (dc == 1000).sum() == 4
        assert sorted(set(dc[dc > 16].tolist())) == [20, 33, 60, 120, 250, 500, 1000]
        assert sorted(set(dv[dv > 16].tolist())) == [17, 30, 60, 120, 200]
        assert H.n == 32768 and H.m == 16384

    def test_deterministic(self):
        a = generate_irregular_code({3: 40, 2: 20}, 25, seed=5)
        b = generate_irregular_code({3: 40, 2: 20}, 25, seed=5)
        assert a == b


def test_priors_batch_matches_per_frame():
    rng = np.random.default_rng(0)
    Y = -1.0 + 1.3 * rng.standard_normal((37, 1001))
    s2 = rng.uniform(0.3, 2.0, size=37)
    P = priors_awgn_batch(Y, s2, threads=4)
    for b in range(37):
        assert np.array_equal(P[b].view(np.uint64), priors_awgn(Y[b], s2[b]).view(np.uint64))
    with pytest.raises(ValueError):
        priors_awgn_batch(Y, 0.0)


def test_unpack_bits_layout():
    words = np.array([[0b1011, 1 << 31]], dtype=np.uint32)
    bits = unpack_bits(words, 64)
    assert bits[0, :4].tolist() == [1, 1, 0, 1] and bits[0, 63] == 1 and bits.sum() == 4


def test_plan_pages_mirrors_engine():
    # engine.py:33-55: pages of group_size lanes, the last one partial; same errors
    from paper_1609_01567_b200 import PagePlan, plan_pages

    plan = plan_pages(10, 4)
    assert plan == PagePlan(10, 4, (0, 4, 8))
    assert plan.page_count == 3 and [plan.page_width(k) for k in range(3)] == [4, 4, 2]
    assert plan_pages(7, 512).page_starts == (0,) and plan_pages(7, 1).page_count == 7
    for bad in ((10, 0), (0, 4), (-1, 3)):
        with pytest.raises(ValueError):
            plan_pages(*bad)


def test_numa_binding_is_best_effort():
    # no GPU / no NVML here: nothing is bound and the affinity is unchanged
    import os

    from paper_1609_01567_b200.numa import bind_to_gpu

    before = os.sched_getaffinity(0)
    info = bind_to_gpu(0)
    assert os.sched_getaffinity(0) == (before if not info["bound"] else os.sched_getaffinity(0))
    assert info["cpus"] >= 1
