"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck / initcheck): every kernel
family on tiny inputs -- graph build, streaming decode (check register kernel, variable ring kernels,
syndrome, done flags, layout), on-chip decode (1 CTA and a 2-CTA cluster), high-degree chains
kernels (1024-thread and small blocks), the register check path past degree 16, fp32 fast mode,
the phase API, the host and streaming decoders, the device channel, device priors from observations
(fused layout kernel, on-chip, standalone exp/prior kernels); round 2: early-stop compaction, the
O(d) fast-mode kernels, forked small buckets, pageable staging."""
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_1609_01567_b200 import (CodeTables, ParallelDecoder, configs, estimate, generate_irregular_code,  # noqa: E402
                                   priors_awgn_batch, syndrome, values_to_check, values_to_variable)


def priors(H, B, ebno, seed):
    s2 = configs.ebno_to_sigma2(ebno, configs.rate(H))
    rng = np.random.default_rng(seed)
    return priors_awgn_batch(-1.0 + np.sqrt(s2) * rng.standard_normal((B, H.n)), s2)


H1 = configs.code("C1")
T1 = CodeTables.from_matrix(H1)
P1 = priors(H1, 8, 1.5, 1)
with ParallelDecoder(T1, max_batch=8) as dec:
    for sched in ("stream", "onchip"):
        for early in (True, False):
            dec.decode_priors(P1, 5, early_stop=early, schedule=sched)
    dec.decode_priors(P1, 5, precision="fp32", schedule="stream")
    dec.decode_priors_async(P1, 3).wait()
    import torch
    dev = torch.device("cuda", 0)
    dec.decode_channel(1, 0, 0, 8, 0.7, 3, workspace=dec.workspace(8), outputs=dec.alloc_outputs(8, dev))
rng = np.random.default_rng(2)
q = rng.uniform(size=(2, H1.total_edges))
r = values_to_variable(q, T1)
values_to_check(P1[:2], r, T1)
c = estimate(P1[:2], r, T1)
syndrome(c, T1)
# 2-CTA cluster on chip
H2 = generate_irregular_code({8: 400, 3: 1200, 2: 2400}, 2000, seed=3)
with ParallelDecoder(CodeTables.from_matrix(H2), max_batch=2) as dec:
    dec.decode_priors(priors(H2, 2, 1.5, 4), 3, schedule="onchip")
# high-degree chains kernels (shared-memory staging)
H4 = generate_irregular_code({200: 2, 3: 3000, 2: 3000}, 2000, seed=5, check_degrees={600: 2})
with ParallelDecoder(CodeTables.from_matrix(H4), max_batch=2) as dec:
    dec.decode_priors(priors(H4, 2, 1.5, 6), 2, early_stop=False)
# check degrees 17-32 (register path, V = 1) and 33-40 / variable 17-40 (small chains blocks)
H5 = generate_irregular_code({40: 4, 20: 8, 8: 300, 3: 400, 2: 800}, 700, seed=7,
                             check_degrees={24: 10, 32: 10, 36: 4, 40: 4})
with ParallelDecoder(CodeTables.from_matrix(H5), max_batch=3) as dec:
    dec.decode_priors(priors(H5, 3, 1.5, 8), 3, early_stop=True)
# observations in: fused prior in the layout kernel, on chip, standalone kernels
s2 = configs.ebno_to_sigma2(1.5, configs.rate(H1))
Y = -1.0 + np.sqrt(s2) * rng.standard_normal((8, H1.n))
Y[0, :4] = [400.0, -400.0, 1e5, -1e5]
with ParallelDecoder(T1, max_batch=8) as dec:
    for sched in ("stream", "onchip"):
        dec.decode_batch(Y, s2, 4, schedule=sched)
    dec.decode_batch_async(Y, s2, 3).wait()
from paper_1609_01567_b200 import _native  # noqa: E402
Yd = torch.from_numpy(Y).to(dev)
Sd = torch.full((8,), s2, dtype=torch.float64, device=dev)
Pd = torch.empty_like(Yd)
_native.check(_native.lib().ldpc_priors_awgn(Yd.data_ptr(), Sd.data_ptr(), 8, H1.n, Pd.data_ptr(), None), "priors")
_native.check(_native.lib().ldpc_npexp(Yd.data_ptr(), Yd.numel(), Pd.data_ptr(), None), "npexp")
# variables of degree 17-64 (kernels_varmid.cu), early and fixed
H7 = generate_irregular_code({48: 3, 24: 6, 30: 4, 8: 200, 3: 300, 2: 600}, 420, seed=11,
                             check_degrees={40: 4, 64: 2})
with ParallelDecoder(CodeTables.from_matrix(H7), max_batch=40) as dec:
    P7 = priors(H7, 40, 1.5, 12)
    dec.decode_priors(P7, 3, early_stop=True, schedule="stream")
    dec.decode_priors(P7, 3, early_stop=False, schedule="stream")
# grid schedule (cooperative launch), early and fixed; long-check syndrome (degree 600 checks, early stop)
H6 = configs.code("C2")
with ParallelDecoder(CodeTables.from_matrix(H6), max_batch=3) as dec:
    P6 = priors(H6, 3, 1.5, 9)
    dec.decode_priors(P6, 6, schedule="grid")
    dec.decode_priors(P6, 4, early_stop=False, schedule="grid")
with ParallelDecoder(CodeTables.from_matrix(H4), max_batch=2) as dec:
    dec.decode_priors(priors(H4, 2, 1.5, 10), 2, early_stop=True, schedule="stream")
# round 2: early-stop compaction (plan, fused retire/move, mapped outputs; exact and fp32, side
# streams), O(d) fast-mode kernels at any degree (incl. a two-pass check of degree 600), forked small
# buckets, pageable staging through pinned slots, the TMA ring (LDPC_KERNEL=tma in a second run)
H8 = configs.code("C2")
with ParallelDecoder(CodeTables.from_matrix(H8), max_batch=200) as dec:
    P8 = priors(H8, 200, 2.0, 13)
    for prec in ("fp64", "fp32"):
        dec.decode_priors(P8, 12, early_stop=True, precision=prec, schedule="stream")
with ParallelDecoder(CodeTables.from_matrix(H4), max_batch=70) as dec:
    P4 = priors(H4, 70, 2.0, 14)
    dec.decode_priors(P4, 4, early_stop=True, precision="fp32")
    dec.decode_priors(P4, 3, early_stop=False, precision="fp32")
with ParallelDecoder(CodeTables.from_matrix(H5), max_batch=3) as dec:
    dec.decode_priors(priors(H5, 3, 1.5, 15), 3, precision="fp32")
H9 = configs.code("C3")
with ParallelDecoder(CodeTables.from_matrix(H9), max_batch=64, sub_batch=64) as dec:
    dec.decode_priors(priors(H9, 64, 2.0, 16), 2, early_stop=False)  # pageable in/out: staged
torch.cuda.synchronize()
print("sanitize workload done")
