"""Randomized bit-exact parity campaign against the CPU oracle (test infrastructure on the checker side).

python tools/parity_campaign.py [minutes] [seed0]
Each case draws a random irregular code (variable degrees 1-300, some checks up to degree 700), a
batch size, an iteration budget, a stop mode, a schedule and an Eb/N0, decodes through the public API
(host buffers, pageable or pinned) and compares estimate bits, success, iterations and syndromes with
the oracle.  Prints one line per case and a summary; exit status 1 on any mismatch."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
sys.path.insert(0, "oracle")
from oracle import OracleTables  # noqa: E402

from paper_1609_01567_b200 import (CodeTables, ParallelDecoder, configs, generate_irregular_code,  # noqa: E402
                                   priors_awgn_batch)

minutes = float(sys.argv[1]) if len(sys.argv) > 1 else 10.0
seed0 = int(sys.argv[2]) if len(sys.argv) > 2 else 0
t_end = time.time() + 60 * minutes
cases = bad = frames = 0
while time.time() < t_end:
    seed = seed0 + cases
    rng = np.random.default_rng(seed)
    m = int(rng.integers(40, 3000))
    prof = {2: int(rng.integers(m // 4, m)), 3: int(rng.integers(0, m)), int(rng.integers(4, 12)): int(rng.integers(1, m // 3 + 2))}
    if rng.random() < 0.4:
        prof[int(rng.integers(17, min(300, m)))] = int(rng.integers(1, 6))
    checks = None
    E = sum(d * c for d, c in prof.items())
    if rng.random() < 0.4 and E > 4 * m:
        dmax = int(rng.integers(17, min(700, E // 4)))
        checks = {dmax: 1, int(rng.integers(17, dmax + 1)): int(rng.integers(1, 4))}
    try:
        H = generate_irregular_code(prof, m, seed=seed, check_degrees=checks)
    except (ValueError, RuntimeError):
        cases += 1
        continue
    B = int(rng.choice([1, 2, 31, 32, 33, 63, 64, 65, 100, 128, 200, 257, 400, 700]))
    iters = int(rng.integers(0, 31))
    early = bool(rng.random() < 0.7)
    schedule = str(rng.choice(["auto", "stream"]))
    ebno = float(rng.uniform(0.0, 4.0))
    rate = max(configs.rate(H), 0.05) if H.n > H.m else 0.5
    s2 = configs.ebno_to_sigma2(ebno, rate)
    P = priors_awgn_batch(-1.0 + np.sqrt(s2) * rng.standard_normal((B, H.n)), s2)
    if rng.random() < 0.3:
        P = torch.from_numpy(P).pin_memory().numpy()
    with ParallelDecoder(CodeTables.from_matrix(H), max_batch=B) as dec:
        res = dec.decode_priors(P, iters, early_stop=early, schedule=schedule)
    est, ok, its, z = OracleTables.from_matrix(H).decode_batch(np.ascontiguousarray(P), iters,
                                                                 fixed_iterations=not early)
    same = (np.array_equal(res.estimates(), est) and np.array_equal(res.success.astype(bool), ok)
            and np.array_equal(res.iterations, its) and np.array_equal(res.syndromes(), z))
    dv, dc = H.degrees()
    print(f"case {cases} seed {seed}: n={H.n} m={H.m} E={H.total_edges} dv<={dv.max()} dc<={dc.max()} B={B} "
          f"iters={iters} early={early} schedule={schedule} ebno={ebno:.2f} mean_its={its.mean():.2f} "
          f"{'OK' if same else 'MISMATCH'}", flush=True)
    cases += 1
    frames += B
    bad += 0 if same else 1
print(f"summary: {cases} cases, {frames} frames, {bad} mismatching cases")
sys.exit(1 if bad else 0)
