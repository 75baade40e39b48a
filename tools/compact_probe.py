"""Early-stop compaction probe: device-timed decode per call, compaction threshold sweep.

python tools/compact_probe.py  (runs LDPC_COMPACT = 0 / 50 / 75 / 90 / 100 in subprocesses)
Prints ms per decode for C2 (B=4096, 20 its, 2 dB, early stop), fixed 20 its, C5 at 3 dB, C4 at 3 dB."""
import json
import os
import subprocess
import sys

SRC = r"""
import sys, json, numpy as np, torch
sys.path.insert(0, '.')
from paper_1609_01567_b200 import CodeTables, ParallelDecoder, configs, priors_awgn_batch
res = {}
for label, code, B, it, early, eb in (("C2", "C2", 4096, 20, True, 2.0), ("C2_fixed", "C2", 4096, 20, False, 2.0),
                                      ("C5_3dB", "C5", 1024, 10, True, 3.0), ("C5_2dB", "C5", 1024, 10, True, 2.0),
                                      ("C4", "C4", 256, 20, True, 3.0)):
    H = configs.code(code)
    s2 = configs.ebno_to_sigma2(eb, configs.rate(H))
    P = priors_awgn_batch(-1.0 + np.sqrt(s2) * np.random.default_rng(5).standard_normal((B, H.n)), s2)
    Pd = torch.from_numpy(P).cuda()
    with ParallelDecoder(CodeTables.from_matrix(H), max_batch=B) as d:
        ws, o = d.workspace(B), d.alloc_outputs(B, Pd.device)
        for _ in range(3):
            d.decode_device(Pd, it, early_stop=early, workspace=ws, outputs=o)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            d.decode_device(Pd, it, early_stop=early, workspace=ws, outputs=o)
        e1.record()
        torch.cuda.synchronize()
        res[label] = (round(e0.elapsed_time(e1) / 10, 3), round(o[2].float().mean().item(), 2))
print(json.dumps(res))
"""
for v in sys.argv[1:] or ["0", "50", "75", "90", "100"]:
    out = subprocess.run([sys.executable, "-c", SRC], capture_output=True, text=True,
                         env=dict(os.environ, LDPC_COMPACT=v))
    print("LDPC_COMPACT=%s" % v, out.stdout.strip() or out.stderr[-2000:], flush=True)
