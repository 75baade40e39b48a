"""Layout kernel with and without the fused AWGN prior (k_transpose_priors<0|1>), C3, B=1024:
event-timed decodes with max_iterations=0 from priors and from observations (the difference is the
prior arithmetic), and a target for `ncu -k regex:k_transpose_priors`."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from paper_1609_01567_b200 import CodeTables, ParallelDecoder, configs  # noqa: E402
from paper_1609_01567_b200.decoder import priors_awgn_batch  # noqa: E402

B = 1024
H = configs.code("C3")
s2 = configs.sigma2_for("C3", 2.0)
rng = np.random.default_rng(3)
Y = -1.0 + np.sqrt(s2) * rng.standard_normal((B, H.n))
Yd = torch.from_numpy(Y).cuda()
Pd = torch.from_numpy(priors_awgn_batch(Y, s2)).cuda()
S = torch.full((B,), s2, dtype=torch.float64, device="cuda")
with ParallelDecoder(CodeTables.from_matrix(H), max_batch=B) as dec:
    ws, outs = dec.workspace(B), dec.alloc_outputs(B, Yd.device)
    for name, run in (("priors", lambda: dec.decode_device(Pd, 0, workspace=ws, outputs=outs)),
                      ("observations", lambda: dec.decode_device_awgn(Yd, S, 0, workspace=ws, outputs=outs))):
        run()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(20):
            run()
        e1.record()
        torch.cuda.synchronize()
        print(f"{name:13s} 0-iteration decode (layout + pre-pass + estimate + syndrome): {e0.elapsed_time(e1) / 20:.3f} ms")
