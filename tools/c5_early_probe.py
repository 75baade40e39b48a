"""C5 early stop: device-timed decode per call at several Eb/N0, decode_device (host priors) and
decode_channel (device channel), compaction on/off via LDPC_COMPACT in the environment."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1609_01567_b200 import CodeTables, ParallelDecoder, configs, priors_awgn_batch  # noqa: E402

H = configs.code("C5")
prec = sys.argv[1] if len(sys.argv) > 1 else "fp64"
B = 1024
with ParallelDecoder(CodeTables.from_matrix(H), max_batch=B) as d:
    ws, o = d.workspace(B), d.alloc_outputs(B, torch.device("cuda"))
    for eb in (2.0, 3.0, 3.5):
        s2 = configs.ebno_to_sigma2(eb, configs.rate(H))
        P = torch.from_numpy(priors_awgn_batch(-1.0 + np.sqrt(s2) * np.random.default_rng(5).standard_normal((B, H.n)),
                                               s2)).cuda()
        res = {}
        for label, fn in (("device", lambda: d.decode_device(P, 10, workspace=ws, outputs=o, precision=prec)),
                          ("channel", lambda: d.decode_channel(7, 0, 0, B, s2, 10, workspace=ws, outputs=o, precision=prec)),
                          ("fixed", lambda: d.decode_device(P, 10, early_stop=False, workspace=ws, outputs=o, precision=prec))):
            for _ in range(3):
                fn()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(5):
                fn()
            e1.record()
            torch.cuda.synchronize()
            res[label] = (round(e0.elapsed_time(e1) / 5, 2), round(o[2].float().mean().item(), 2))
        print(eb, res, flush=True)
