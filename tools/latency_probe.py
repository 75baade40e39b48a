"""Single-frame latency of the reference-facing call ParallelDecoder.decode(y, sigma2, max_iterations)
(engine.py:363) at C1 and C3, wall clock per call (host in, host out), early stop at 2 dB."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from paper_1609_01567_b200 import CodeTables, ParallelDecoder, configs  # noqa: E402

for name, iters in (("C1", 50), ("C3", 50)):
    H = configs.code(name)
    s2 = configs.sigma2_for(name, 2.0)
    rng = np.random.default_rng(9)
    Y = -1.0 + np.sqrt(s2) * rng.standard_normal((40, H.n))
    with ParallelDecoder(CodeTables.from_matrix(H), max_batch=1) as dec:
        for y in Y[:5]:
            dec.decode(y, s2, iters)
        ts, its = [], []
        for y in Y[5:]:
            t0 = time.perf_counter()
            r = dec.decode(y, s2, iters)
            ts.append(time.perf_counter() - t0)
            its.append(r.iterations_used)
    ts = np.array(ts) * 1e3
    print(f"{name}: n={H.n} median {np.median(ts):.3f} ms (p90 {np.percentile(ts, 90):.3f}) per frame, "
          f"mean iterations {np.mean(its):.1f}")
