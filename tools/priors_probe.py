import sys, time, os
sys.path.insert(0, ".")
import numpy as np, torch
from paper_1609_01567_b200 import decoder as D
n, B = 64800, 1024
rng = np.random.default_rng(1)
Y = -1.0 + 0.8 * rng.standard_normal((B, n))
Yp = torch.from_numpy(Y).pin_memory().numpy()
for rep in range(2):
    t = time.perf_counter(); P = D.priors_awgn_batch(Yp, 0.63); print("batch fresh out", time.perf_counter() - t)
out = torch.empty((B, n), dtype=torch.float64).pin_memory().numpy()
def work(b):
    with np.errstate(over="ignore"):
        np.divide(1.0, 1.0 + np.exp(-2.0 * Yp[b] / 0.63), out=out[b])
from concurrent.futures import ThreadPoolExecutor
for nt in (1, 4, 8, 16, 32):
    pool = ThreadPoolExecutor(nt)
    list(pool.map(work, range(B)))
    t = time.perf_counter(); list(pool.map(work, range(B))); print("threads", nt, "pinned out", round(time.perf_counter() - t, 4))
# in-place ufunc chain without temporaries
tmp = [np.empty(n) for _ in range(32)]
def work2(b):
    tt = tmp[b % 32]
    with np.errstate(over="ignore"):
        np.multiply(Yp[b], -2.0, out=tt); np.divide(tt, 0.63, out=tt); np.exp(tt, out=tt); np.add(tt, 1.0, out=tt)
        np.divide(1.0, tt, out=out[b])
pool = ThreadPoolExecutor(16)
list(pool.map(work2, range(B)))
t = time.perf_counter(); list(pool.map(work2, range(B))); print("16 threads, no temporaries", round(time.perf_counter() - t, 4))
print(os.cpu_count())
