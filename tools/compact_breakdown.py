"""Per-class device time of one early-stop decode (eager, event-timed) with compaction on/off,
plus the stopping-round histogram.  python tools/compact_breakdown.py [code B iters ebno]"""
import json
import os
import subprocess
import sys

SRC = r"""
import sys, json, numpy as np, torch
sys.path.insert(0, '.')
from paper_1609_01567_b200 import CodeTables, ParallelDecoder, configs, priors_awgn_batch, _native
code, B, it, eb = %r, %d, %d, %f
H = configs.code(code)
s2 = configs.ebno_to_sigma2(eb, configs.rate(H))
P = priors_awgn_batch(-1.0 + np.sqrt(s2) * np.random.default_rng(5).standard_normal((B, H.n)), s2)
Pd = torch.from_numpy(P).cuda()
with ParallelDecoder(CodeTables.from_matrix(H), max_batch=B) as d:
    ws, o = d.workspace(B), d.alloc_outputs(B, Pd.device)
    d.decode_device(Pd, it, workspace=ws, outputs=o)
    prof = _native.Profile()
    for _ in range(5):
        d.decode_device(Pd, it, workspace=ws, outputs=o, profile=prof)
    torch.cuda.synchronize()
    pd = prof.as_dict()
    print(json.dumps({k: round(v["ms"] / 5, 3) for k, v in pd.items()}), "launches", {k: v["launches"] // 5 for k, v in pd.items()})
    its = o[2].cpu().numpy()
    h = np.bincount(its, minlength=it + 1)
    print("stop-round histogram", h.tolist(), "mean", its.mean())
"""
args = sys.argv[1:] or ["C2", "4096", "20", "2.0"]
for v in ("0", "75"):
    out = subprocess.run([sys.executable, "-c", SRC % (args[0], int(args[1]), int(args[2]), float(args[3]))],
                         capture_output=True, text=True, env=dict(os.environ, LDPC_COMPACT=v))
    print("LDPC_COMPACT=%s" % v, out.stdout.strip() or out.stderr[-2000:], flush=True)
