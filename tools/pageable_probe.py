"""e2e with pageable numpy buffers vs pinned (C3, 1024 codewords, 10 fixed iterations).
python tools/pageable_probe.py  -> ms per decode_priors call, pinned and pageable"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1609_01567_b200 import CodeTables, ParallelDecoder, configs, priors_awgn_batch  # noqa: E402
from paper_1609_01567_b200.decoder import BatchResult  # noqa: E402

H = configs.code("C3")
B = 1024
s2 = configs.ebno_to_sigma2(2.0, 0.5)
P = priors_awgn_batch(-1.0 + np.sqrt(s2) * np.random.default_rng(1).standard_normal((B, H.n)), s2)
P_pin = torch.from_numpy(P).pin_memory().numpy()
n, m = H.n, H.m
pin = lambda shape, dt: torch.empty(shape, dtype=dt).pin_memory().numpy()  # noqa: E731
res = BatchResult(pin((B, (n + 31) // 32), torch.int32).view(np.uint32), pin((B,), torch.uint8),
                  pin((B,), torch.int32), pin((B, (m + 31) // 32), torch.int32).view(np.uint32), n, m)
with ParallelDecoder(CodeTables.from_matrix(H), max_batch=B) as dec:
    for label, fn in (("pinned", lambda: dec.decode_priors(P_pin, 10, early_stop=False, out=res)),
                      ("pageable", lambda: dec.decode_priors(P, 10, early_stop=False))):
        for _ in range(3):
            fn()
        t0 = time.perf_counter()
        for _ in range(10):
            fn()
        print(label, "ms", round((time.perf_counter() - t0) / 10 * 1e3, 2), flush=True)
    # host memcpy bandwidth of numpy into pinned memory, for scale
    t0 = time.perf_counter()
    for _ in range(5):
        np.copyto(P_pin, P)
    print("numpy copy into pinned GB/s", round(5 * P.nbytes / (time.perf_counter() - t0) / 1e9, 1))
