"""Time the synchronous host API (decode_priors, C3, B=1024, 10 fixed iterations) under the
sub-batch plan in LDPC_E2E_PLAN / LDPC_E2E_GROWTH / LDPC_E2E_LANES (read once per process).

  for p in "" 64,64,128,192,256,320; do LDPC_E2E_PLAN=$p python tools/e2e_plan_probe.py; done
"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from paper_1609_01567_b200 import CodeTables, ParallelDecoder, configs  # noqa: E402
from paper_1609_01567_b200.decoder import BatchResult, priors_awgn_batch  # noqa: E402

B, I = 1024, 10
H = configs.code("C3")
s2 = configs.sigma2_for("C3", 2.0)
rng = np.random.default_rng(5)
P = torch.from_numpy(priors_awgn_batch(-1.0 + np.sqrt(s2) * rng.standard_normal((B, H.n)), s2)).pin_memory().numpy()
n, m = H.n, H.m
pin = lambda shape, dt: torch.empty(shape, dtype=dt).pin_memory().numpy()  # noqa: E731
res = BatchResult(pin((B, (n + 31) // 32), torch.int32).view(np.uint32), pin((B,), torch.uint8),
                  pin((B,), torch.int32), pin((B, (m + 31) // 32), torch.int32).view(np.uint32), n, m)
with ParallelDecoder(CodeTables.from_matrix(H), max_batch=B) as dec:
    for _ in range(4):
        dec.decode_priors(P, I, early_stop=False, out=res)
    ts = []
    for _ in range(12):
        t0 = time.perf_counter()
        dec.decode_priors(P, I, early_stop=False, out=res)
        ts.append(time.perf_counter() - t0)
ts = np.array(ts) * 1e3
print(f"plan={os.environ.get('LDPC_E2E_PLAN', '')!r} growth={os.environ.get('LDPC_E2E_GROWTH', '')!r} "
      f"lanes={os.environ.get('LDPC_E2E_LANES', '')!r}: median {np.median(ts):.2f} ms  min {ts.min():.2f}  "
      f"-> {B * n / np.median(ts) / 1e6:.3f} Gbit/s")
