"""fp32 fast mode vs the oracle on random codes: hard-decision and iteration agreement per case.

python tools/fast_campaign.py [minutes] [seed0]
Random irregular codes (variable degrees up to 300, checks up to 700), batches, budgets and Eb/N0;
each case decodes in fast mode (precision="fp32", early stop) and with the CPU oracle (exact), and
reports the fraction of frames whose hard decisions and iteration counts agree.  Summary at the end:
frame-weighted agreement and its worst case."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "oracle")
from oracle import OracleTables  # noqa: E402

from paper_1609_01567_b200 import (CodeTables, ParallelDecoder, configs, generate_irregular_code,  # noqa: E402
                                   priors_awgn_batch)

minutes = float(sys.argv[1]) if len(sys.argv) > 1 else 10.0
seed0 = int(sys.argv[2]) if len(sys.argv) > 2 else 0
only = [int(x) for x in sys.argv[3].split(",")] if len(sys.argv) > 3 else None  # replay these seeds
t_end = time.time() + 60 * minutes
cases = frames = same_est = same_its = conv_frames = conv_same_est = 0
worst = 1.0
while time.time() < t_end and (only is None or cases < len(only)):
    seed = only[cases] if only else seed0 + cases
    rng = np.random.default_rng(seed)
    m = int(rng.integers(100, 3000))
    prof = {2: int(rng.integers(m // 4, m)), 3: int(rng.integers(m // 4, m)),
            int(rng.integers(4, 12)): int(rng.integers(1, m // 3 + 2))}
    if rng.random() < 0.4:
        prof[int(rng.integers(17, min(300, m)))] = int(rng.integers(1, 6))
    E = sum(d * c for d, c in prof.items())
    checks = None
    if rng.random() < 0.4 and E > 4 * m:
        dmax = int(rng.integers(17, min(700, E // 4)))
        checks = {dmax: 1}
    cases += 1
    try:
        H = generate_irregular_code(prof, m, seed=seed, check_degrees=checks)
    except (ValueError, RuntimeError):
        continue
    if H.n <= H.m:
        continue
    B = int(rng.choice([32, 64, 100, 256]))
    iters = int(rng.integers(5, 31))
    ebno = float(rng.uniform(0.5, 4.0))
    s2 = configs.ebno_to_sigma2(ebno, configs.rate(H))
    P = priors_awgn_batch(-1.0 + np.sqrt(s2) * rng.standard_normal((B, H.n)), s2)
    with ParallelDecoder(CodeTables.from_matrix(H), max_batch=B) as dec:
        r = dec.decode_priors(P, iters, precision="fp32")
    est, ok, its, _ = OracleTables.from_matrix(H).decode_batch(P, iters)
    same = np.all(r.estimates() == est, axis=1)
    se = int(same.sum())
    si = int((r.iterations == its).sum())
    conv = ok.astype(bool)  # frames the exact decoder converged on
    conv_same = int(same[conv].sum())
    conv_n = int(conv.sum())
    frames += B
    conv_frames += conv_n
    conv_same_est += conv_same
    same_est += se
    same_its += si
    worst = min(worst, se / B)
    dv, dc = H.degrees()
    print(f"case {cases} seed {seed}: n={H.n} dv<={dv.max()} dc<={dc.max()} B={B} iters={iters} ebno={ebno:.2f} "
          f"frames identical {se / B:.3f} iterations identical {si / B:.3f} "
          f"converged frames {conv_n} identical {conv_same / max(conv_n, 1):.3f}", flush=True)
print(f"summary: {cases} cases, {frames} frames; identical hard decisions {same_est / max(frames, 1):.4f}, "
      f"identical iteration counts {same_its / max(frames, 1):.4f}, worst case {worst:.3f}; frames the exact "
      f"decoder converged on: {conv_frames}, identical {conv_same_est / max(conv_frames, 1):.5f}")
