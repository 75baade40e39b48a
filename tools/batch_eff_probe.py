"""Device decode time per codeword vs batch size (C3, 10 fixed iterations): the efficiency of the
sub-batches the synchronous host decoder pipelines (64, 128, 192, 256, 384) against B = 1024."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from paper_1609_01567_b200 import CodeTables, ParallelDecoder, configs  # noqa: E402
from paper_1609_01567_b200.decoder import priors_awgn_batch  # noqa: E402

H = configs.code("C3")
s2 = configs.sigma2_for("C3", 2.0)
rng = np.random.default_rng(4)
P = torch.from_numpy(priors_awgn_batch(-1.0 + np.sqrt(s2) * rng.standard_normal((1024, H.n)), s2)).cuda()
base = None
with ParallelDecoder(CodeTables.from_matrix(H), max_batch=1024) as dec:
    for B in (1024, 64, 128, 192, 256, 384, 512):
        Pb = P[:B].contiguous()
        ws, outs = dec.workspace(B), dec.alloc_outputs(B, P.device)
        for _ in range(3):
            dec.decode_device(Pb, 10, early_stop=False, workspace=ws, outputs=outs)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(10):
            dec.decode_device(Pb, 10, early_stop=False, workspace=ws, outputs=outs)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 10
        per = ms / B * 1e3
        base = base or per
        print(f"B={B:5d}: {ms:7.3f} ms, {per:6.2f} us/codeword, efficiency vs B=1024 {base / per:.3f}")
