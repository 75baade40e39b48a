"""Grid schedule vs streaming for small batches (device time per decode, early stop, 2 dB)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1609_01567_b200 import CodeTables, ParallelDecoder, configs  # noqa: E402
from paper_1609_01567_b200.decoder import priors_awgn_batch  # noqa: E402

for name, it in (("C3", 50), ("C2", 50)):
    H = configs.code(name)
    s2 = configs.sigma2_for(name, 2.0)
    rng = np.random.default_rng(3)
    P = torch.from_numpy(priors_awgn_batch(-1.0 + np.sqrt(s2) * rng.standard_normal((64, H.n)), s2)).cuda()
    with ParallelDecoder(CodeTables.from_matrix(H), max_batch=64) as dec:
        for B in (1, 4, 8, 16, 32, 48, 64):
            Pb = P[:B].contiguous()
            ws, outs = dec.workspace(B), dec.alloc_outputs(B, P.device)
            row = []
            for sched in ("grid", "stream"):
                for _ in range(2):
                    dec.decode_device(Pb, it, workspace=ws, outputs=outs, schedule=sched)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda.synchronize()
                e0.record()
                for _ in range(10):
                    dec.decode_device(Pb, it, workspace=ws, outputs=outs, schedule=sched)
                e1.record()
                torch.cuda.synchronize()
                row.append(e0.elapsed_time(e1) / 10)
            print(f"{name} B={B:3d}: grid {row[0]:.3f} ms, stream {row[1]:.3f} ms")
