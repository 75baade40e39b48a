"""Where the C5 sweep's time goes: ber_sweep(channel="device") wall clock vs its decodes alone."""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_1609_01567_b200 import CodeTables, ParallelDecoder, channel as ch, configs  # noqa: E402

H = configs.code("C5")
ch.ber_sweep(H, [0.0], 1024, max_iterations=10, batch=1024, channel="device")   # warm-up
torch.cuda.synchronize()
t0 = time.perf_counter()
ch.ber_sweep(H, [0.0, 1.0, 2.0, 3.0], 4096, max_iterations=10, seed=1, batch=1024, channel="device")
torch.cuda.synchronize()
t1 = time.perf_counter()
print(f"ber_sweep 4 points x 4096 frames: {1e3 * (t1 - t0):.1f} ms")
with ParallelDecoder(CodeTables.from_matrix(H), max_batch=1024) as dec:
    dev = torch.device("cuda", 0)
    ws, outs = dec.workspace(1024), dec.alloc_outputs(1024, dev)
    counts = torch.zeros(4, dtype=torch.int64, device=dev)
    s2 = configs.sigma2_for("C5", 3.0)
    for rep in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for b in range(16):
            dec.decode_channel(1, 3, b * 1024, 1024, s2, 10, workspace=ws, outputs=outs)
            dec.count_errors(outs, counts)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        print(f"16 decode_channel calls: {1e3 * (t1 - t0):.1f} ms ({1e3 * (t1 - t0) / 16:.2f} ms each)")
