"""Device decode rate of a DVB-S2 rate-9/10-shaped code (check degree 29/30: the register path
past degree 16) against the HBM roofline, B=1024, 10 fixed iterations.

  python tools/highrate_probe.py            # LDPC_* kernel switches apply as usual
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from paper_1609_01567_b200 import CodeTables, ParallelDecoder, generate_irregular_code  # noqa: E402
from paper_1609_01567_b200.decoder import priors_awgn_batch  # noqa: E402

B, I = 1024, 10
# default: DVB-S2 rate-9/10 shape (check degrees 29/30); --deg40: rate ~0.93 (check degrees 39/40)
H = (generate_irregular_code({3: 60000, 2: 4800}, 4800, seed=940) if "--deg40" in sys.argv
     else generate_irregular_code({4: 5832, 3: 52488, 2: 6480}, 6480, seed=910))
n, m, E = H.n, H.m, H.total_edges
dc = H.degrees()[1]
s2 = 1.0 / (2 * 0.9 * 10 ** (4.0 / 10))
rng = np.random.default_rng(1)
P = torch.from_numpy(priors_awgn_batch(-1.0 + np.sqrt(s2) * rng.standard_normal((B, n)), s2)).cuda()
with ParallelDecoder(CodeTables.from_matrix(H), max_batch=B) as dec:
    ws = dec.workspace(B)
    outs = dec.alloc_outputs(B, P.device)
    for _ in range(3):
        dec.decode_device(P, I, early_stop=False, workspace=ws, outputs=outs)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    K = 10
    for _ in range(K):
        dec.decode_device(P, I, early_stop=False, workspace=ws, outputs=outs)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / K
# bytes/cw = 8E(4I+2) + 8n(I+2) + (n/8)(2I+2)
bpc = 8 * E * (4 * I + 2) + 8 * n * (I + 2) + (n / 8) * (2 * I + 2)
peak = json.loads(open(os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json")).read()).get("hbm_gbs", 6554.6)
gbs = bpc * B / (ms / 1e3) / 1e9
print(json.dumps({"code": f"rate-9/10-shaped n={n} m={m} E={E} check degrees {sorted(set(dc.tolist()))}",
                  "ms_per_decode": round(ms, 3), "coded_Gbit_s": round(B * n / ms / 1e6, 3),
                  "algorithmic_GBps": round(gbs, 1), "frac_of_copy_peak": round(gbs / peak, 3)}))
