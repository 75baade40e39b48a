"""Per-stream busy intervals of one decode_priors call (CUPTI via torch.profiler), with GPU idle gaps."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from bench import synthetic_priors  # noqa: E402
from paper_1609_01567_b200 import CodeTables, ParallelDecoder, configs  # noqa: E402
from paper_1609_01567_b200.decoder import BatchResult  # noqa: E402

H = configs.code("C3")
B = 1024
T = CodeTables.from_matrix(H)
dec = ParallelDecoder(T, max_batch=B, sub_batch=int(sys.argv[1]) if len(sys.argv) > 1 else 0)
P, _ = synthetic_priors(H, B, 2.0, 1)
Pp = torch.from_numpy(P).pin_memory().numpy()
pin = lambda shape, dt: torch.empty(shape, dtype=dt).pin_memory().numpy()  # noqa: E731
n, m = H.n, H.m
res = BatchResult(pin((B, (n + 31) // 32), torch.int32).view(np.uint32), pin((B,), torch.uint8),
                  pin((B,), torch.int32), pin((B, (m + 31) // 32), torch.int32).view(np.uint32), n, m)
for _ in range(3):
    dec.decode_priors(Pp, 10, early_stop=False, out=res)
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    for _ in range(2):
        dec.decode_priors(Pp, 10, early_stop=False, out=res)
prof.export_chrome_trace("gpurun_out/e2e_trace2.json")
ev = [e for e in json.load(open("gpurun_out/e2e_trace2.json"))["traceEvents"] if e.get("ph") == "X"]
gpu = [e for e in ev if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")]
t0 = min(e["ts"] for e in gpu)
ker = sorted((e["ts"] - t0, e["ts"] - t0 + e["dur"], e["args"].get("stream")) for e in gpu if e["cat"] == "kernel")
cpy = sorted((e["ts"] - t0, e["ts"] - t0 + e["dur"], e["name"][:20]) for e in gpu if e["cat"] == "gpu_memcpy" and e["dur"] > 50)
print("H2D/D2H > 50us:", [(round(a / 1e3, 2), round(b / 1e3, 2), nm) for a, b, nm in cpy])
# union of kernel intervals -> idle gaps
gaps, cur_end = [], None
for a, b, st in ker:
    if cur_end is not None and a > cur_end + 5:
        gaps.append((round(cur_end / 1e3, 3), round((a - cur_end) / 1e3, 3)))
    cur_end = b if cur_end is None else max(cur_end, b)
print("kernel span ms", round(ker[0][0] / 1e3, 3), "->", round(cur_end / 1e3, 3))
print("idle gaps > 5us (start ms, len ms):", gaps[:40], "total idle ms", round(sum(g[1] for g in gaps), 3))
