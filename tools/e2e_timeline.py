"""Timeline of one ParallelDecoder.decode_priors call (CUPTI via torch.profiler): memcpy vs kernels per stream."""
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
    dec.decode_priors(Pp, 10, early_stop=False, out=res)
prof.export_chrome_trace("gpurun_out/e2e_trace.json")
ev = [e for e in json.load(open("gpurun_out/e2e_trace.json"))["traceEvents"] if e.get("ph") == "X"]
t0 = min(e["ts"] for e in ev)
rows = sorted(((e["ts"] - t0, e["dur"], e.get("args", {}).get("stream"), e["name"][:40]) for e in ev))
segs = {}
for ts, dur, st, name in rows:
    kind = "memcpy" if "emcpy" in name else "kernel"
    segs.setdefault((st, kind), []).append((ts, ts + dur))
for (st, kind), s in sorted(segs.items(), key=lambda x: str(x[0])):
    busy = sum(b - a for a, b in s)
    print(f"stream {st} {kind:6s}: n={len(s):4d} first={s[0][0]/1e3:7.2f}ms last_end={max(b for a,b in s)/1e3:7.2f}ms busy={busy/1e3:7.2f}ms")
end = max(ts + dur for ts, dur, _, _ in rows)
print("total span ms", end / 1e3)
# memcpy segments
for ts, dur, st, name in rows:
    if "emcpy" in name and dur > 100:
        print(f"  {name:40s} stream={st} start={ts/1e3:7.2f} dur={dur/1e3:6.2f}ms")
