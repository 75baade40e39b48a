"""fp32 fast mode (f4) at C3: device time per decode and per kernel class, against the fp32 roofline
(w = 4 bytes per message)."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from paper_1609_01567_b200 import CodeTables, ParallelDecoder, _native, configs  # noqa: E402
from paper_1609_01567_b200.decoder import priors_awgn_batch  # noqa: E402

B, I = 1024, 10
H = configs.code("C3")
s2 = configs.sigma2_for("C3", 2.0)
rng = np.random.default_rng(1)
P = torch.from_numpy(priors_awgn_batch(-1.0 + np.sqrt(s2) * rng.standard_normal((B, H.n)), s2)).cuda()
with ParallelDecoder(CodeTables.from_matrix(H), max_batch=B) as dec:
    ws, outs = dec.workspace(B), dec.alloc_outputs(B, P.device)
    run = lambda prof=None: dec.decode_device(P, I, early_stop=False, workspace=ws, outputs=outs,  # noqa: E731
                                              precision="fp32", profile=prof)
    for _ in range(3):
        run()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(10):
        run()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    prof = _native.Profile()
    run(prof)
    torch.cuda.synchronize()
n, E = H.n, H.total_edges
bpc = 4 * E * (4 * I + 2) + 4 * n * (I + 2) + (n / 8) * (2 * I + 2)
peak = json.loads(open(os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json")).read()).get("hbm_gbs", 6554.6)
print(json.dumps({"ms_per_decode": round(ms, 3), "coded_Gbit_s": round(B * n / ms / 1e6, 3),
                  "frac_of_copy_peak": round(bpc * B / (ms / 1e3) / 1e9 / peak, 3),
                  "kernel_ms": {k: round(v["ms"], 3) for k, v in prof.as_dict().items()}}))
