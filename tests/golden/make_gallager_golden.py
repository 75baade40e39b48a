"""Golden vectors for the regular code generator, made by RUNNING the reference.

  PYTHONPATH=/root/reference/pkg/src python tests/golden/make_gallager_golden.py

Writes tests/golden/gallager.npz: for each (n, wc, wr, seed) the reference's
generate_gallager_code (codes.py:241-294) edge list, plus derive_state / shuffle /
randrange outputs of rng.py (the generator's stream).
"""
import pathlib

import numpy as np

from edgeldpc import codes, rng

CASES = [(12, 2, 4, 3), (96, 3, 6, 0), (96, 3, 6, 1), (30, 2, 3, 7), (200, 4, 8, 5), (64, 3, 4, 11),
         (20, 4, 5, 2), (9, 3, 3, 4), (1000, 3, 6, 2)]
out = {}
for k, (n, wc, wr, seed) in enumerate(CASES):
    H = codes.generate_gallager_code(n, wc, wr, seed)
    out[f"g{k}/params"] = np.array([n, wc, wr, seed], dtype=np.int64)
    out[f"g{k}/ones"] = np.array(H.ones, dtype=np.int64).reshape(-1, 2)
st = rng.derive_state(5, 6, 7)
items = list(range(50))
st2 = rng.shuffle(items, st)
st3, draws = st2, []
for b in (1, 2, 7, 1000, 2**40 + 3):
    st3, v = rng.randrange(st3, b)
    draws.append(v)
out["rng/state"] = np.array([st.s0, st.s1, st2.s0, st2.s1, st3.s0, st3.s1], dtype=np.uint64)
out["rng/shuffled"] = np.array(items, dtype=np.int64)
out["rng/draws"] = np.array(draws, dtype=np.uint64)
out["cases"] = np.array(len(CASES))
np.savez_compressed(pathlib.Path(__file__).with_name("gallager.npz"), **out)
print("wrote", len(CASES), "codes")
