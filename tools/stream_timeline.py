"""CUPTI timeline of the streaming API (decode_priors_async, two in flight): GPU idle gaps, copies."""
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
dec = ParallelDecoder(CodeTables.from_matrix(H), max_batch=B)
P, _ = synthetic_priors(H, B, 2.0, 1)
Pp = torch.from_numpy(P).pin_memory().numpy()
pin = lambda shape, dt: torch.empty(shape, dtype=dt).pin_memory().numpy()  # noqa: E731
n, m = H.n, H.m
outs = [BatchResult(pin((B, (n + 31) // 32), torch.int32).view(np.uint32), pin((B,), torch.uint8),
                    pin((B,), torch.int32), pin((B, (m + 31) // 32), torch.int32).view(np.uint32), n, m)
        for _ in range(2)]


def steps(k):
    pend = []
    for i in range(k):
        pend.append(dec.decode_priors_async(Pp, 10, early_stop=False, out=outs[i % 2]))
        if len(pend) == 2:
            pend.pop(0).wait()
    for q in pend:
        q.wait()


steps(4)
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA, torch.profiler.ProfilerActivity.CPU]) as prof:
    steps(4)
prof.export_chrome_trace("gpurun_out/stream_trace.json")
ev = [e for e in json.load(open("gpurun_out/stream_trace.json"))["traceEvents"] if e.get("ph") == "X"]
gpu = [e for e in ev if e.get("cat") in ("kernel", "gpu_memcpy")]
t0 = min(e["ts"] for e in gpu)
ker = sorted((e["ts"] - t0, e["ts"] - t0 + e["dur"]) for e in gpu if e["cat"] == "kernel")
cpy = sorted((round((e["ts"] - t0) / 1e3, 2), round(e["dur"] / 1e3, 2), e["name"][:12]) for e in gpu
             if e["cat"] == "gpu_memcpy" and e["dur"] > 100)
print("copies >100us (start ms, dur ms):", cpy)
gaps, cur = [], None
for a, b in ker:
    if cur is not None and a > cur + 5:
        gaps.append((round(cur / 1e3, 2), round((a - cur) / 1e3, 3)))
    cur = b if cur is None else max(cur, b)
print("kernels", round(ker[0][0] / 1e3, 2), "->", round(cur / 1e3, 2), "gaps:", gaps)
rt = sorted((round((e["ts"] - t0) / 1e3, 2), round(e["dur"] / 1e3, 3), e["name"][:28]) for e in ev
            if e.get("cat") == "cuda_runtime" and e["dur"] > 200)
print("slow runtime calls:", rt)
