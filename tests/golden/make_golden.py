"""Generate the golden fixtures by running the REFERENCE package (edgeldpc).

Run in the build container, where the read-only reference is mounted:

    PYTHONPATH=/root/reference/pkg/src:/root/repo python tests/golden/make_golden.py

It writes small compressed .npz files next to this script.  They are the only
thing that travels to the GPU box: no test reads /root/reference at run time.
Contents:
  tables.npz   ones + all 12 table arrays + var groups for the paper's (14,7)
               code (Tables I/II), the 1x1 code, chain3, the reference's own
               Gallager (96,48) fixture code, 20 random matrices
               (conftest.random_parity_matrix) and config C1's irregular code.
  phases.npz   seeded random states and the reference's values_to_check,
               values_to_variable, estimate and syndrome outputs.
  decode.npz   priors (reference priors_awgn, i.e. numpy exp on this machine),
               decode_awgn results, and a fixed-iteration run composed from the
               reference's exported phase functions (no early exit).
  channel.npz  xorshift128+ / derive_state KATs, exact received frames and the
               reference ber_sweep points + CSV for the (96,48) and (14,7) codes.
"""

from __future__ import annotations

import pathlib
import sys

import numpy as np

HERE = pathlib.Path(__file__).resolve().parent
REF_TESTS = pathlib.Path("/root/reference/pkg/tests")

import edgeldpc as ref  # noqa: E402  (reference, PYTHONPATH)

sys.path.insert(0, str(REF_TESTS))
from conftest import PAIRS_14_7, random_parity_matrix  # noqa: E402

sys.path.insert(0, str(HERE.parent.parent))
from paper_1609_01567_b200 import configs  # noqa: E402


def codes() -> dict:
    out = {
        "h14": ref.ParityCheckMatrix(14, 7, PAIRS_14_7),
        "one": ref.ParityCheckMatrix(1, 1, ((0, 0),)),
        "chain3": ref.ParityCheckMatrix(3, 2, ((0, 0), (0, 1), (1, 1), (1, 2))),
        "h96": ref.generate_gallager_code(96, 3, 6, seed=1),
    }
    rng = np.random.default_rng(11)
    for i in range(20):
        out[f"rand{i:02d}"] = random_parity_matrix(rng, max_m=24, max_n=40)
    c1 = configs.code("C1")
    out["c1"] = ref.ParityCheckMatrix(c1.n, c1.m, c1.ones)
    return out


def save_tables(cs: dict) -> None:
    d = {"names": np.array(list(cs))}
    for name, H in cs.items():
        T = ref.CodeTables.from_matrix(H)
        ones = np.array(H.ones, dtype=np.int32).reshape(-1, 2)
        d[f"{name}/nm"] = np.array([H.n, H.m], dtype=np.int64)
        d[f"{name}/ones"] = ones
        for o, tb in (("var", T.variable), ("chk", T.check)):
            for k in "evctsu":
                d[f"{name}/{o}_{k}"] = getattr(tb, k).astype(np.int32)
        d[f"{name}/gstart"] = T.var_group_start.astype(np.int32)
        d[f"{name}/gsize"] = T.var_group_size.astype(np.int32)
    np.savez_compressed(HERE / "tables.npz", **d)
    # the (14,7) code as alist text, written by the reference serializer (codes.py:186-198)
    (HERE / "ldpc_14_7.alist").write_text(ref.serialize_alist(cs["h14"]))


def save_phases(cs: dict) -> None:
    rng = np.random.default_rng(20240917)
    d = {}
    names = ["h14", "chain3", "h96", "c1", "rand03", "rand07"]
    d["names"] = np.array(names)
    for name in names:
        H = cs[name]
        T = ref.CodeTables.from_matrix(H)
        S = 3
        P = rng.uniform(size=(S, H.n))
        R = rng.uniform(size=(S, H.total_edges))
        Q = rng.uniform(size=(S, H.total_edges))
        # include saturated values (0, 1, 0.5) the KATs exercise
        P[0, : min(3, H.n)] = [0.0, 1.0, 0.5][: min(3, H.n)]
        R[0, : min(3, H.total_edges)] = [0.0, 1.0, 0.5][: min(3, H.total_edges)]
        Q[0, : min(3, H.total_edges)] = [0.0, 1.0, 0.5][: min(3, H.total_edges)]
        C = rng.integers(0, 2, size=(S, H.n)).astype(np.uint8)
        d[f"{name}/p"] = P
        d[f"{name}/r"] = R
        d[f"{name}/q"] = Q
        d[f"{name}/chat_in"] = C
        d[f"{name}/to_check"] = np.stack([ref.values_to_check(P[i], R[i], T) for i in range(S)])
        d[f"{name}/to_variable"] = np.stack([ref.values_to_variable(Q[i], T) for i in range(S)])
        d[f"{name}/estimate"] = np.stack([ref.estimate(P[i], R[i], T) for i in range(S)])
        d[f"{name}/syndrome"] = np.stack([ref.syndrome(C[i], H) for i in range(S)])
    np.savez_compressed(HERE / "phases.npz", **d)


def fixed_iterations(y, s2, iters, T, H):
    """Reference phase functions composed without the early exit (serial.py:165-178 minus 169/176)."""
    st = ref.initialize(y, s2, T)
    r = ref.values_to_variable(st.q, T)
    c = ref.estimate(st.p, r, T)
    for _ in range(iters):
        q = ref.values_to_check(st.p, r, T)
        r = ref.values_to_variable(q, T)
        c = ref.estimate(st.p, r, T)
    z = ref.syndrome(c, H)
    return c, (not z.any()), iters, z


def save_decode(cs: dict) -> None:
    rng = np.random.default_rng(1609)
    d = {}
    cases = []
    # (14,7): the reference's single-flip test inputs (test_serial.py:198-207) and noisy frames
    H = cs["h14"]
    ys = []
    for flip in range(14):
        y = np.full(14, -1.0)
        y[flip] = 1.0
        ys.append(y)
    for _ in range(26):
        ys.append(-1.0 + 1.1 * rng.standard_normal(14))
    cases.append(("h14_s05", "h14", np.array(ys[:14]), 0.5, 10))
    cases.append(("h14_s10", "h14", np.array(ys[14:]), 1.0, 5))
    # (96,48) Gallager code, 60 noisy frames at sigma2 = 0.63 (SPEC.md parallel-engine example)
    cases.append(("h96", "h96", -1.0 + np.sqrt(0.63) * rng.standard_normal((60, 96)), 0.63, 50))
    # C1 irregular n=1024: 2 dB and 1 dB, 50 iterations (BASELINE config 1)
    H1 = cs["c1"]
    for db, cnt in ((2.0, 24), (1.0, 24), (0.0, 8)):
        s2 = configs.ebno_to_sigma2(db, (H1.n - H1.m) / H1.n)
        cases.append((f"c1_{db:.0f}dB", "c1", -1.0 + np.sqrt(s2) * rng.standard_normal((cnt, H1.n)), s2, 50))
    d["cases"] = np.array([c[0] for c in cases])
    for key, code, Y, s2, iters in cases:
        H = cs[code]
        T = ref.CodeTables.from_matrix(H)
        P = np.stack([ref.priors_awgn(y, s2) for y in Y])
        res = [ref.decode_awgn(y, s2, iters, T, H) for y in Y]
        d[f"{key}/code"] = np.array(code)
        if code in ("h14", "h96"):
            d[f"{key}/y"] = Y
        d[f"{key}/sigma2"] = np.array(s2)
        d[f"{key}/max_iterations"] = np.array(iters)
        d[f"{key}/p"] = P
        d[f"{key}/estimate"] = np.stack([r.estimate for r in res])
        d[f"{key}/success"] = np.array([r.success for r in res])
        d[f"{key}/iterations"] = np.array([r.iterations_used for r in res], dtype=np.int32)
        d[f"{key}/syndrome"] = np.stack([r.syndrome for r in res])
    # fixed-iteration composition on C1 (the benchmark's fixed-work mode), 10 rounds
    H1 = cs["c1"]
    T1 = ref.CodeTables.from_matrix(H1)
    s2 = configs.ebno_to_sigma2(1.5, 0.5)
    Y = -1.0 + np.sqrt(s2) * rng.standard_normal((8, H1.n))
    fx = [fixed_iterations(y, s2, 10, T1, H1) for y in Y]
    d["fixed/code"] = np.array("c1")
    d["fixed/p"] = np.stack([ref.priors_awgn(y, s2) for y in Y])
    d["fixed/max_iterations"] = np.array(10)
    d["fixed/estimate"] = np.stack([f[0] for f in fx])
    d["fixed/success"] = np.array([f[1] for f in fx])
    d["fixed/syndrome"] = np.stack([f[3] for f in fx])
    # prior KATs (test_serial.py:28-53)
    yk = np.array([0.0, 1.0, -1.0, -1e6, 1e6, 0.3, -2.5])
    d["kat/y"] = yk
    d["kat/p_s2_1"] = ref.priors_awgn(yk, 1.0)
    np.savez_compressed(HERE / "decode.npz", **d)


def save_channel(cs: dict) -> None:
    """rng.py / channel.py outputs: RNG KATs, exact received frames, reference ber_sweep points."""
    d = {}
    st = ref.RngState(1, 2)
    outs = []
    for _ in range(64):
        st, x = ref.rng_next(st)
        outs.append(x)
    d["rng/outputs_1_2"] = np.array(outs, dtype=np.uint64)
    keys = [(0, 0, 0), (5, 1, 7), (2**40 + 3, 2, 11)]
    d["rng/derive_keys"] = np.array(keys, dtype=np.uint64)
    d["rng/derive_states"] = np.array([[ref.derive_state(*k).s0, ref.derive_state(*k).s1] for k in keys], dtype=np.uint64)
    Y = np.stack([ref.transmit_all_zero(96, 0.63, ref.derive_state(5, 0, f))[1] for f in range(6)])
    d["channel/y_h96_seed5"] = Y
    for name, code, pts, frames, it, seed in (("h96", "h96", (1.0, 2.0, 3.0), 24, 20, 5),
                                             ("h14", "h14", (0.0, 2.0), 16, 10, 9)):
        P = ref.ber_sweep(cs[code], pts, frames, max_iterations=it, seed=seed, decoders_in_flight=1)
        d[f"ber/{name}/args"] = np.array([frames, it, seed])
        d[f"ber/{name}/ebno"] = np.array(pts)
        d[f"ber/{name}/points"] = np.array([[p.ebno_db, p.sigma2, p.frames, p.bit_errors, p.ber, p.mean_iterations,
                                              p.failures] for p in P])
        d[f"ber/{name}/csv"] = np.array(ref.ber_csv(P))
    np.savez_compressed(HERE / "channel.npz", **d)


if __name__ == "__main__":
    cs = codes()
    save_tables(cs)
    save_phases(cs)
    save_decode(cs)
    save_channel(cs)
    for f in sorted(HERE.glob("*.npz")):
        print(f.name, f.stat().st_size, "bytes")
