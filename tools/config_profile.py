"""One config's decode for profiling / timing: python tools/config_profile.py CODE B ITERS EBNO EARLY(0|1) PREC [reps]
Decodes once (warm-up, eager) and then `reps` times (graph replay); prints ms per decode.  Under ncu,
the second half of the launches belongs to the timed decodes (reps = 1)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1609_01567_b200 import CodeTables, ParallelDecoder, configs, priors_awgn_batch  # noqa: E402

code, B, it, eb, early, prec = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), float(sys.argv[4]), \
    sys.argv[5] == "1", sys.argv[6]
reps = int(sys.argv[7]) if len(sys.argv) > 7 else 1
H = configs.code(code)
s2 = configs.ebno_to_sigma2(eb, configs.rate(H))
P = priors_awgn_batch(-1.0 + np.sqrt(s2) * np.random.default_rng(5).standard_normal((B, H.n)), s2)
Pd = torch.from_numpy(P).cuda()
with ParallelDecoder(CodeTables.from_matrix(H), max_batch=B) as d:
    ws, o = d.workspace(B), d.alloc_outputs(B, Pd.device)
    d.decode_device(Pd, it, early_stop=early, workspace=ws, outputs=o, precision=prec)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        d.decode_device(Pd, it, early_stop=early, workspace=ws, outputs=o, precision=prec)
    e1.record()
    torch.cuda.synchronize()
    print(code, B, it, eb, early, prec, "ms per decode", round(e0.elapsed_time(e1) / reps, 3),
          "mean iterations", o[2].float().mean().item())
