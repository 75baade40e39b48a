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
        assert dv.max() == 200 and dc.max() == 1000 and (dc == 1000).sum() == 16

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
