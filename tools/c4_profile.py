"""C4 (high-degree stress) decode for profiling: python tools/c4_profile.py [fp64|fp32] [reps]
Run under ncu (see tools/c4_ncu.sh); prints the device time per decode when run plainly."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1609_01567_b200 import CodeTables, ParallelDecoder, configs, priors_awgn_batch  # noqa: E402

prec = sys.argv[1] if len(sys.argv) > 1 else "fp64"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
C = configs.CONFIGS["C4"]
H = configs.code("C4")
B, it = C["batch"], C["max_iterations"]
s2 = configs.ebno_to_sigma2(C["ebno_db"], configs.rate(H))
P = priors_awgn_batch(-1.0 + np.sqrt(s2) * np.random.default_rng(5).standard_normal((B, H.n)), s2)
Pd = torch.from_numpy(P).cuda()
with ParallelDecoder(CodeTables.from_matrix(H), max_batch=B) as d:
    ws, o = d.workspace(B), d.alloc_outputs(B, Pd.device)
    d.decode_device(Pd, it, workspace=ws, outputs=o, precision=prec)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        d.decode_device(Pd, it, workspace=ws, outputs=o, precision=prec)
    e1.record()
    torch.cuda.synchronize()
    print(prec, "ms per decode", e0.elapsed_time(e1) / reps, "mean iterations", o[2].float().mean().item())
