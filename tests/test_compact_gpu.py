"""Per-codeword early stop (serial.py:169-177, engine.py:341-347): live codewords are compacted
into dense chunks on the device (compact.cu) so the work follows each codeword's stopping round.
Results must be bit-identical to the oracle and to the uncompacted decode, whatever the
compaction points are (LDPC_COMPACT=<pct> threshold, 0 = off; LDPC_COMPACT_MODE=fill|stable; read once per
process)."""

from __future__ import annotations

import os
import subprocess
import sys

import numpy as np
import pytest

from conftest import ROOT
from paper_1609_01567_b200 import CodeTables, ParallelDecoder, configs, priors_awgn_batch

pytestmark = pytest.mark.gpu


def _frames(code, B, ebno, seed):
    H = configs.code(code)
    s2 = configs.ebno_to_sigma2(ebno, configs.rate(H))
    rng = np.random.default_rng(seed)
    return H, priors_awgn_batch(-1.0 + np.sqrt(s2) * rng.standard_normal((B, H.n)), s2)


@pytest.mark.parametrize("code,B,ebno,iters", [
    ("C2", 512, 2.0, 20),
    ("C2", 200, 1.5, 20),
    ("C1", 700, 1.5, 50),
    ("C4", 130, 3.0, 20),
])
def test_compacted_decode_vs_oracle(cuda, code, B, ebno, iters):
    from oracle import OracleTables

    H, P = _frames(code, B, ebno, seed=B + iters)
    with ParallelDecoder(CodeTables.from_matrix(H), max_batch=B) as dec:
        res = dec.decode_priors(P, iters, schedule="stream")
    est, ok, its, z = OracleTables.from_matrix(H).decode_batch(P, iters)
    assert len(set(its.tolist())) > 3  # codewords stop at many different rounds
    assert np.array_equal(res.iterations, its)
    assert np.array_equal(res.success.astype(bool), ok)
    assert np.array_equal(res.estimates(), est)
    assert np.array_equal(res.syndromes(), z)


_RUN = r"""
import sys, numpy as np, torch
sys.path.insert(0, {root!r})
from paper_1609_01567_b200 import CodeTables, ParallelDecoder, configs, priors_awgn_batch
H = configs.code({code!r})
s2 = configs.ebno_to_sigma2({ebno}, configs.rate(H))
P = priors_awgn_batch(-1.0 + np.sqrt(s2) * np.random.default_rng(4).standard_normal(({B}, H.n)), s2)
out = {{}}
with ParallelDecoder(CodeTables.from_matrix(H), max_batch={B}) as dec:
    for prec in ("fp64", "fp32"):
        r = dec.decode_priors(P, {iters}, precision=prec, schedule="stream")
        out[prec + "_est"], out[prec + "_syn"] = r.est_bits, r.syn_bits
        out[prec + "_ok"], out[prec + "_it"] = r.success, r.iterations
        e, o, i, z = dec.decode_device(torch.from_numpy(P).cuda(), {iters}, precision=prec)
        torch.cuda.synchronize()
        out[prec + "_dev_est"], out[prec + "_dev_it"] = e.cpu().numpy(), i.cpu().numpy()
    # device channel (f1) through the same decode sequence
    d = dec.alloc_outputs({B}, torch.device("cuda"))
    dec.decode_channel(7, 0, 0, {B}, s2, {iters}, outputs=d)
    torch.cuda.synchronize()
    out["chan_est"], out["chan_it"] = d[0].cpu().numpy(), d[2].cpu().numpy()
np.savez({path!r}, **out)
"""


def _run(tmp_path, env_value, code, B, ebno, iters):
    pct, _, mode = env_value.partition(":")
    path = str(tmp_path / f"out_{pct}_{mode}.npz")
    env = dict(os.environ, LDPC_COMPACT=pct, LDPC_COMPACT_MODE=mode or "fill")
    src = _RUN.format(root=str(ROOT), code=code, B=B, ebno=ebno, iters=iters, path=path)
    r = subprocess.run([sys.executable, "-c", src], capture_output=True, text=True, env=env, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    return np.load(path)


@pytest.mark.parametrize("code,B,ebno,iters", [("C2", 448, 2.0, 20), ("C4", 192, 3.0, 20)])
def test_compaction_points_do_not_change_results(cuda, tmp_path, code, B, ebno, iters):
    # off, the default threshold, and compaction at every round that frees a chunk; live codewords
    # moved into the stopped positions (fill, default) or shifted down in order (stable)
    modes = ("75", "80", "100", "80:stable", "100:stable")
    runs = {v: _run(tmp_path, v, code, B, ebno, iters) for v in ("0",) + modes}
    base = runs["0"]
    assert len(set(base["fp64_it"].tolist())) > 3
    for v in modes:
        for k in base.files:
            assert np.array_equal(runs[v][k], base[k]), (v, k)


@pytest.mark.parametrize("seed", range(4))
def test_compaction_random_codes_vs_oracle(cuda, seed):
    # random irregular codes (some high degrees), batches that do not fill their last chunk, early
    # stop at an SNR where frames stop at many different rounds: bit-exact vs the oracle
    from oracle import OracleTables

    from paper_1609_01567_b200 import generate_irregular_code

    rng = np.random.default_rng(100 + seed)
    m = int(rng.integers(300, 900))
    prof = {int(rng.integers(4, 9)): int(rng.integers(20, 80)), 3: int(rng.integers(200, 600)), 2: m}
    extra = {int(rng.integers(17, 70)): 2} if seed % 2 else None
    H = generate_irregular_code(prof, m, seed=seed, check_degrees=extra)
    B = int(rng.integers(65, 330))
    s2 = configs.ebno_to_sigma2(1.0 + 0.5 * seed, configs.rate(H))
    P = priors_awgn_batch(-1.0 + np.sqrt(s2) * rng.standard_normal((B, H.n)), s2)
    with ParallelDecoder(CodeTables.from_matrix(H), max_batch=B) as dec:
        res = dec.decode_priors(P, 25, schedule="stream")
    est, ok, its, z = OracleTables.from_matrix(H).decode_batch(P, 25)
    assert np.array_equal(res.iterations, its) and np.array_equal(res.success.astype(bool), ok)
    assert np.array_equal(res.estimates(), est) and np.array_equal(res.syndromes(), z)


def test_concurrent_decoders_and_shared_decoder(cuda):
    # host threads: two decoders at once (each its own streams, fork sets and compaction side
    # streams) and two threads sharing one decoder (serialised by its lock); early stop with
    # compaction and forked high-degree buckets (C4) -- every result equals the oracle
    import threading

    from oracle import OracleTables

    H = configs.code("C4")
    T = CodeTables.from_matrix(H)
    frames = [_frames("C4", 96, 3.0, seed=s)[1] for s in range(4)]
    O = OracleTables.from_matrix(H)
    want = [O.decode_batch(P, 12) for P in frames]
    got, errors = [None] * 4, []

    def run(dec, i):
        try:
            got[i] = dec.decode_priors(frames[i], 12, schedule="stream")
        except Exception as e:  # pragma: no cover - reported below
            errors.append(e)

    with ParallelDecoder(T, max_batch=96) as d0, ParallelDecoder(T, max_batch=96) as d1:
        ts = [threading.Thread(target=run, args=(d0, 0)), threading.Thread(target=run, args=(d1, 1)),
              threading.Thread(target=run, args=(d0, 2)), threading.Thread(target=run, args=(d1, 3))]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
    assert not errors, errors
    for res, (est, ok, its, z) in zip(got, want):
        assert np.array_equal(res.iterations, its) and np.array_equal(res.estimates(), est)
        assert np.array_equal(res.success.astype(bool), ok) and np.array_equal(res.syndromes(), z)
