"""Device decode rate of a code whose variable degrees include 24 and 30 (5G-NR-BG1-like heavy
columns, past the register path's 16): the small-block chains kernels carry those nodes.
B=1024, 10 fixed iterations; prints per-kernel-class times and the roofline fraction."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from paper_1609_01567_b200 import CodeTables, ParallelDecoder, _native, generate_irregular_code  # noqa: E402
from paper_1609_01567_b200.decoder import priors_awgn_batch  # noqa: E402

B, I = 1024, 10
vdeg = {30: 1000, 24: 1000, 8: 2000, 3: 12000, 2: 16000}
E = sum(d * c for d, c in vdeg.items())
H = generate_irregular_code(vdeg, E // 7, seed=77)
n, m = H.n, H.m
s2 = 0.6
rng = np.random.default_rng(1)
P = torch.from_numpy(priors_awgn_batch(-1.0 + np.sqrt(s2) * rng.standard_normal((B, n)), s2)).cuda()
with ParallelDecoder(CodeTables.from_matrix(H), max_batch=B) as dec:
    ws, outs = dec.workspace(B), dec.alloc_outputs(B, P.device)
    for _ in range(3):
        dec.decode_device(P, I, early_stop=False, workspace=ws, outputs=outs)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(5):
        dec.decode_device(P, I, early_stop=False, workspace=ws, outputs=outs)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    prof = _native.Profile()
    dec.decode_device(P, I, early_stop=False, workspace=ws, outputs=outs, profile=prof)
    torch.cuda.synchronize()
bpc = 8 * E * (4 * I + 2) + 8 * n * (I + 2) + (n / 8) * (2 * I + 2)
peak = json.loads(open(os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json")).read()).get("hbm_gbs", 6554.6)
gbs = bpc * B / (ms / 1e3) / 1e9
print(json.dumps({"code": f"n={n} m={m} E={E} var degrees {sorted(vdeg)}", "ms_per_decode": round(ms, 3),
                  "frac_of_copy_peak": round(gbs / peak, 3),
                  "kernel_ms": {k: round(v["ms"], 3) for k, v in prof.as_dict().items()}}))
