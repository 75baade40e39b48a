import sys
import numpy as np, torch
sys.path.insert(0, ".")
from paper_1609_01567_b200 import CodeTables, ParallelDecoder, configs, priors_awgn_batch
H = configs.code("C1")
s2 = configs.ebno_to_sigma2(2.0, configs.rate(H))
for B in (1, 8, 32, 64, 296):
    P = torch.from_numpy(priors_awgn_batch(-1.0 + np.sqrt(s2) * np.random.default_rng(3).standard_normal((B, H.n)), s2)).cuda()
    with ParallelDecoder(CodeTables.from_matrix(H), max_batch=B) as d:
        ws, o = d.workspace(B), d.alloc_outputs(B, P.device)
        row = []
        for sched in ("auto", "onchip", "grid", "stream"):
            if sched == "grid" and B > 32: row.append((sched, None)); continue
            for _ in range(3): d.decode_device(P, 50, workspace=ws, outputs=o, schedule=sched)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(20): d.decode_device(P, 50, workspace=ws, outputs=o, schedule=sched)
            e1.record(); torch.cuda.synchronize()
            row.append((sched, round(e0.elapsed_time(e1) / 20, 3)))
        print("C1 B=", B, row, flush=True)
