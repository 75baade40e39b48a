"""The CPU oracle pinned against the reference: golden Tables I/II and the
fixtures produced by running the reference (tests/golden/make_golden.py)."""

import numpy as np
import pytest

from conftest import GOLDEN_CHECK, GOLDEN_VARIABLE, PAIRS_14_7
from oracle import OracleTables, priors_awgn


def test_paper_tables_I_II():
    T = OracleTables(14, 7, PAIRS_14_7)
    v, c = T.export("variable"), T.export("check")
    for k in "evctsu":
        assert v[k].tolist() == GOLDEN_VARIABLE[k], k
        assert c[k].tolist() == GOLDEN_CHECK[k], k


def test_tables_match_reference_fixtures(golden_tables):
    for name in golden_tables["names"]:
        n, m = golden_tables[f"{name}/nm"]
        T = OracleTables(n, m, golden_tables[f"{name}/ones"])
        for o, orient in (("var", "variable"), ("chk", "check")):
            ex = T.export(orient)
            for k in "evctsu":
                assert np.array_equal(ex[k], golden_tables[f"{name}/{o}_{k}"]), (name, o, k)
        gs, gz = T.var_groups()
        assert np.array_equal(gs, golden_tables[f"{name}/gstart"])
        assert np.array_equal(gz, golden_tables[f"{name}/gsize"])


@pytest.mark.parametrize("bad", [((0, 0), (0, 0), (1, 1)), ((0, 0), (5, 1)), ((0, 0), (0, 1)), ((0, 0),)])
def test_oracle_rejects_invalid(bad):
    with pytest.raises(ValueError):
        OracleTables(2, 2, bad)


def test_phases_match_reference(golden_tables, golden_phases):
    for name in golden_phases["names"]:
        n, m = golden_tables[f"{name}/nm"]
        T = OracleTables(n, m, golden_tables[f"{name}/ones"])
        g = lambda k: golden_phases[f"{name}/{k}"]  # noqa: E731
        for i in range(g("p").shape[0]):
            q = T.values_to_check(g("p")[i], g("r")[i])
            assert np.array_equal(q.view(np.uint64), g("to_check")[i].view(np.uint64)), name
            r = T.values_to_variable(g("q")[i])
            assert np.array_equal(r.view(np.uint64), g("to_variable")[i].view(np.uint64)), name
            assert np.array_equal(T.estimate(g("p")[i], g("r")[i]), g("estimate")[i]), name
            assert np.array_equal(T.syndrome(g("chat_in")[i]), g("syndrome")[i]), name


def test_saturated_phases_match_reference(golden_saturated):
    """High-SNR states (0 / 1 / -0.0 / denormal priors and messages; tests/golden/make_saturated_golden.py):
    the oracle's zero numerators, zero denominators and signed zeros are the reference's bits."""
    g = golden_saturated
    for name in g["names"]:
        n, m = g[f"{name}/nm"]
        T = OracleTables(n, m, g[f"{name}/ones"])
        for i in range(g[f"{name}/p"].shape[0]):
            q = T.values_to_check(g[f"{name}/p"][i], g[f"{name}/r"][i])
            assert np.array_equal(q.view(np.uint64), g[f"{name}/to_check"][i].view(np.uint64)), name
            r = T.values_to_variable(g[f"{name}/q"][i])
            assert np.array_equal(r.view(np.uint64), g[f"{name}/to_variable"][i].view(np.uint64)), name
            assert np.array_equal(T.estimate(g[f"{name}/p"][i], g[f"{name}/r"][i]), g[f"{name}/estimate"][i]), name
        assert np.signbit(g[f"{name}/to_check"]).any()  # the fixture does hold -0.0 outputs


def test_decode_matches_reference(golden_tables, golden_decode):
    for key in golden_decode["cases"]:
        code = str(golden_decode[f"{key}/code"])
        n, m = golden_tables[f"{code}/nm"]
        T = OracleTables(n, m, golden_tables[f"{code}/ones"])
        it = int(golden_decode[f"{key}/max_iterations"])
        P = golden_decode[f"{key}/p"]
        est, ok, its, z = T.decode_batch(P, it, n_threads=4)
        assert np.array_equal(est, golden_decode[f"{key}/estimate"]), key
        assert np.array_equal(ok, golden_decode[f"{key}/success"]), key
        assert np.array_equal(its, golden_decode[f"{key}/iterations"]), key
        assert np.array_equal(z, golden_decode[f"{key}/syndrome"]), key


def test_fixed_iterations_match_reference_composition(golden_tables, golden_decode):
    n, m = golden_tables["c1/nm"]
    T = OracleTables(n, m, golden_tables["c1/ones"])
    est, ok, its, z = T.decode_batch(golden_decode["fixed/p"], int(golden_decode["fixed/max_iterations"]),
                                     fixed_iterations=True, n_threads=2)
    assert np.array_equal(est, golden_decode["fixed/estimate"])
    assert np.array_equal(ok, golden_decode["fixed/success"])
    assert np.array_equal(z, golden_decode["fixed/syndrome"])
    assert (its == 10).all()


def test_priors_kat(golden_decode):
    # test_serial.py:28-53 KATs; the last-ulp behaviour of numpy exp is machine dependent,
    # so the golden priors are compared within 1 ulp (exact on the generating machine).
    p = priors_awgn(golden_decode["kat/y"], 1.0)
    ref = golden_decode["kat/p_s2_1"]
    assert np.all(np.abs(p.view(np.int64) - ref.view(np.int64)) <= 1)
    assert p[0] == 0.5 and p[3] == 0.0 and p[4] == 1.0
    assert abs(p[1] - 0.8807970779778823) <= 1e-15
    with pytest.raises(ValueError):
        priors_awgn(np.zeros(3), 0.0)
