"""CUPTI timeline (torch.profiler) of one decode of a config: span, GPU-busy time (union of kernel
intervals over all streams), idle gaps, and per-kernel totals.
python tools/config_timeline.py CODE B ITERS EBNO EARLY(0|1) PREC"""
import collections
import sys

import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, ".")
from paper_1609_01567_b200 import CodeTables, ParallelDecoder, configs, priors_awgn_batch  # noqa: E402

code, B, it, eb, early, prec = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), float(sys.argv[4]), \
    sys.argv[5] == "1", sys.argv[6]
H = configs.code(code)
s2 = configs.ebno_to_sigma2(eb, configs.rate(H))
P = priors_awgn_batch(-1.0 + np.sqrt(s2) * np.random.default_rng(5).standard_normal((B, H.n)), s2)
Pd = torch.from_numpy(P).cuda()
with ParallelDecoder(CodeTables.from_matrix(H), max_batch=B) as d:
    ws, o = d.workspace(B), d.alloc_outputs(B, Pd.device)
    for _ in range(3):
        d.decode_device(Pd, it, early_stop=early, workspace=ws, outputs=o, precision=prec)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        d.decode_device(Pd, it, early_stop=early, workspace=ws, outputs=o, precision=prec)
        torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type.name == "CUDA" and e.name.startswith(("void", "ldpc", "_Z"))
      or (e.device_type.name == "CUDA" and "k_" in e.name)]
iv = sorted((e.time_range.start, e.time_range.end, e.name) for e in ev)
t0, t1 = iv[0][0], max(x[1] for x in iv)
busy, cur_s, cur_e, gaps = 0, iv[0][0], iv[0][1], []
for s, e, _ in iv[1:]:
    if s > cur_e:
        busy += cur_e - cur_s
        gaps.append(s - cur_e)
        cur_s, cur_e = s, e
    else:
        cur_e = max(cur_e, e)
busy += cur_e - cur_s
tot = collections.defaultdict(float)
cnt = collections.Counter()
for s, e, n in iv:
    k = n.split("(")[0].replace("void ", "").replace("ldpc::", "").replace("(anonymous namespace)::", "")
    tot[k] += e - s
    cnt[k] += 1
print(f"{code} B={B} {prec} early={early}: span {(t1 - t0) / 1e3:.3f} ms, GPU busy {busy / 1e3:.3f} ms, "
      f"{len(gaps)} gaps totalling {sum(gaps) / 1e3:.3f} ms, {len(iv)} kernels, kernel-time sum {sum(tot.values()) / 1e3:.3f} ms")
for k, v in sorted(tot.items(), key=lambda x: -x[1])[:14]:
    print(f"  {k[:60]:60s} n={cnt[k]:4d} {v / 1e3:8.3f} ms")
