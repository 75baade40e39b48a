"""Channel, frame seeding and the sharded BER sweep (rng.py, channel.py), on CPU.

The decoder here is the CPU oracle injected through ber_sweep's decode_fn
seam, so these tests exercise the host logic -- seeding, shard ranges, the
int64[4] fold and its allreduce -- without a GPU.  The multi-rank case runs
two gloo processes and must reproduce the single-process points exactly."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import GOLDEN, golden_code
from paper_1609_01567_b200 import channel as ch


@pytest.fixture(scope="module")
def gch():
    return np.load(GOLDEN / "channel.npz")


def test_rng_matches_reference(gch):
    st = ch.RngState(1, 2)
    outs = []
    for _ in range(64):
        st, x = ch.rng_next(st)
        outs.append(x)
    assert np.array_equal(np.array(outs, dtype=np.uint64), gch["rng/outputs_1_2"])
    for k, s in zip(gch["rng/derive_keys"], gch["rng/derive_states"]):
        d = ch.derive_state(*(int(x) for x in k))
        assert (d.s0, d.s1) == (int(s[0]), int(s[1]))


def test_exact_channel_matches_reference(gch):
    states = [ch.derive_state(5, 0, f) for f in range(6)]
    Y = ch.transmit_all_zero_batch(96, 0.63, states, exact=True)
    assert np.array_equal(Y.view(np.uint64), gch["channel/y_h96_seed5"].view(np.uint64))


def test_native_channel_matches_reference(gch):
    # csrc/host_channel.cpp: the reference's scalar channel (libm log/cos/sin) in C, on threads
    Y = ch.transmit_all_zero_frames(96, 0.63, seed=5, point=0, frame0=0, count=6, threads=3)
    assert np.array_equal(Y.view(np.uint64), gch["channel/y_h96_seed5"].view(np.uint64))


@pytest.mark.parametrize("n,point,frame0,threads", [(101, 2, 7, 1), (64800 // 8 + 1, 3, 1000, 4), (1, 0, 0, 0)])
def test_native_channel_matches_scalar_path(n, point, frame0, threads):
    Y = ch.transmit_all_zero_frames(n, 0.7943, seed=11, point=point, frame0=frame0, count=5, threads=threads)
    for i in range(5):
        want = ch.transmit_all_zero(n, 0.7943, ch.derive_state(11, point, frame0 + i))[1]
        assert np.array_equal(Y[i].view(np.uint64), want.view(np.uint64))


def test_native_channel_rejects_bad_sigma2():
    with pytest.raises(ValueError):
        ch.transmit_all_zero_frames(8, 0.0, 1, 0, 0, 2)


def test_vectorised_uniforms_are_exact():
    states = [ch.derive_state(3, 1, f) for f in range(5)]
    U = ch.uniforms_batch(states, 40)
    for i, s in enumerate(states):
        for k in range(40):
            s, u = ch.rng_uniform01(s)
            assert U[i, k] == u


def test_vectorised_channel_close_to_exact():
    states = [ch.derive_state(3, 1, f) for f in range(4)]
    a = ch.transmit_all_zero_batch(101, 0.8, states, exact=True)
    b = ch.transmit_all_zero_batch(101, 0.8, states, exact=False)
    assert np.allclose(a, b, rtol=0, atol=1e-13)


def test_shard_ranges_cover_frames():
    for frames in (1, 7, 64, 1000):
        for world in (1, 2, 3, 8):
            got = [f for r in range(world) for f in range(*ch.shard_range(frames, r, world))]
            assert got == list(range(frames))


def oracle_decode_fn(H):
    """Test-only decode_fn: the CPU oracle stands in for the GPU decoder."""
    from oracle import OracleTables, priors_awgn

    O = OracleTables.from_matrix(H)

    def run(Y, sigma2, max_iterations, counts):
        P = np.stack([priors_awgn(y, sigma2) for y in Y])
        est, ok, its, _ = O.decode_batch(P, max_iterations, n_threads=2)
        counts += torch.tensor([int(est.sum()), int((~ok).sum()), int(its.sum()), len(Y)], dtype=torch.int64)

    return run


def _points_array(points):
    return np.array([[p.ebno_db, p.sigma2, p.frames, p.bit_errors, p.ber, p.mean_iterations, p.failures]
                     for p in points])


@pytest.mark.parametrize("name", ["h96", "h14"])
def test_ber_sweep_matches_reference(gch, golden_tables, name):
    H = golden_code(golden_tables, name)
    frames, it, seed = (int(x) for x in gch[f"ber/{name}/args"])
    pts = ch.ber_sweep(H, gch[f"ber/{name}/ebno"], frames, max_iterations=it, seed=seed, batch=7,
                       decode_fn=oracle_decode_fn(H), exact_channel=True)
    assert np.array_equal(_points_array(pts), gch[f"ber/{name}/points"])
    assert ch.ber_csv(pts) == str(gch[f"ber/{name}/csv"])


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank_main(rank, world, port, name, out_q):
    import sys

    from conftest import ROOT

    sys.path.insert(0, str(ROOT / "oracle"))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import numpy as _np

        from conftest import GOLDEN as G, golden_code as gc

        gt = _np.load(G / "tables.npz")
        g = _np.load(G / "channel.npz")
        H = gc(gt, name)
        frames, it, seed = (int(x) for x in g[f"ber/{name}/args"])
        pts = ch.ber_sweep(H, g[f"ber/{name}/ebno"], frames, max_iterations=it, seed=seed, batch=5,
                           decode_fn=oracle_decode_fn(H), exact_channel=True)
        out_q.put((rank, _points_array(pts)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name", ["h96"])
def test_ber_sweep_two_ranks_gloo(gch, name):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, 2, port, name, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(2):
        assert np.array_equal(res[r], gch[f"ber/{name}/points"])
