"""Golden fixture for saturated (high-SNR) message states, made by running the REFERENCE package.

    PYTHONPATH=/root/reference/pkg/src:/root/repo python tests/golden/make_saturated_golden.py

Writes saturated.npz next to this script: for config C1's code and the paper's (14,7) code, seeded
states whose priors and messages sit at exactly 0 / 1, -0.0, denormals and tiny values (so most
variable-side numerators are +-0 over a positive denominator, some denominators are 0 and some
tiny), and the reference's values_to_check (serial.py:63-89), values_to_variable (serial.py:92-112)
and estimate (serial.py:115-133) outputs on them.  Nothing at run time reads /root/reference.
"""

from __future__ import annotations

import pathlib
import sys

import numpy as np

HERE = pathlib.Path(__file__).resolve().parent

import edgeldpc as ref  # noqa: E402  (reference, PYTHONPATH)

sys.path.insert(0, "/root/reference/pkg/tests")
from conftest import PAIRS_14_7  # noqa: E402  (the reference's own (14,7) fixture)

sys.path.insert(0, str(HERE.parent.parent))
from paper_1609_01567_b200 import configs  # noqa: E402

SPECIAL = np.array([0.0, -0.0, 1.0, 5e-324, 1e-300, 1e-160, 1.0 - 2.0 ** -53, 0.5])
STATES = 3


def saturated_states(rng, n, E):
    def draw(size, frac):
        x = rng.uniform(size=size)
        pick = rng.uniform(size=size) < frac
        x[pick] = SPECIAL[rng.integers(0, SPECIAL.size, size=int(pick.sum()))]
        return x

    P = draw((STATES, n), 0.5)
    R = draw((STATES, E), 0.6)
    R[:, : E // 3] = rng.choice([0.0, 1.0], size=(STATES, E // 3))
    Q = draw((STATES, E), 0.6)
    return P, R, Q


def main() -> None:
    H1 = configs.code("C1")
    codes = {
        "C1": ref.ParityCheckMatrix(H1.n, H1.m, tuple(zip(H1.rows.tolist(), H1.cols.tolist()))),
        "h14": ref.ParityCheckMatrix(14, 7, PAIRS_14_7),
    }
    rng = np.random.default_rng(20261017)
    out = {"names": np.array(list(codes))}
    for name, H in codes.items():
        T = ref.CodeTables.from_matrix(H)
        P, R, Q = saturated_states(rng, H.n, H.total_edges)
        out[f"{name}/nm"] = np.array([H.n, H.m])
        out[f"{name}/ones"] = np.array(H.ones, dtype=np.int64)
        out[f"{name}/p"], out[f"{name}/r"], out[f"{name}/q"] = P, R, Q
        out[f"{name}/to_check"] = np.stack([ref.values_to_check(P[s], R[s], T) for s in range(STATES)])
        out[f"{name}/to_variable"] = np.stack([ref.values_to_variable(Q[s], T) for s in range(STATES)])
        out[f"{name}/estimate"] = np.stack([ref.estimate(P[s], R[s], T) for s in range(STATES)]).astype(np.uint8)
    np.savez_compressed(HERE / "saturated.npz", **out)
    print("wrote", HERE / "saturated.npz", {k: v.shape for k, v in out.items()})


if __name__ == "__main__":
    main()
