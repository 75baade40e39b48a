"""Multi-rank execution of the GPU decoder: codeword shards per rank, one int64[4]
allreduce of {bit errors, failures, iterations, frames} per Eb/N0 point (reference fold:
channel.py:218-231 / SPEC ber_sweep, channel.py:83-137).

A gpurun box has one GPU, and NCCL refuses two ranks on one device, so the ranks share cuda:0 and
fold over gloo -- the decode itself is the real CUDA path on every rank.  The bench's multi-rank flow
is run the same way (LDPC_BENCH_ONE_GPU=1) and its folded counters are checked against two
single-rank runs over the same frames."""

from __future__ import annotations

import json
import multiprocessing as mp
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

from conftest import GOLDEN, ROOT, golden_code

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _points_array(points):
    return np.array([[p.ebno_db, p.sigma2, p.frames, p.bit_errors, p.ber, p.mean_iterations, p.failures]
                     for p in points])


def _sweep(kind):
    """One rank's sweep; rank/world come from torch.distributed when initialised."""
    from paper_1609_01567_b200 import channel as ch, configs

    if kind == "host":  # the reference's channel bit for bit, golden (14,7)/(96,48) fixtures
        gt = np.load(GOLDEN / "tables.npz")
        g = np.load(GOLDEN / "channel.npz")
        H = golden_code(gt, "h96")
        frames, it, seed = (int(x) for x in g["ber/h96/args"])
        pts = ch.ber_sweep(H, g["ber/h96/ebno"], frames, max_iterations=it, seed=seed, batch=5, exact_channel=True)
    else:  # f1 device channel on C1, early stop
        H = configs.code("C1")
        pts = ch.ber_sweep(H, [1.0, 2.0], 300, max_iterations=30, seed=9, batch=64, channel="device")
    return _points_array(pts), ch.ber_csv(pts)


def _rank_main(rank, world, port, kind, out_q):
    import torch
    import torch.distributed as dist

    sys.path.insert(0, str(ROOT))
    sys.path.insert(0, str(ROOT / "tests"))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        out_q.put((rank, _sweep(kind)))
    finally:
        dist.destroy_process_group()


def _two_ranks(kind):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, 2, port, kind, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return res


def test_ber_sweep_two_ranks_gpu_decoder_host_channel(cuda):
    g = np.load(GOLDEN / "channel.npz")
    res = _two_ranks("host")
    for r in range(2):
        pts, csv = res[r]
        assert np.array_equal(pts, g["ber/h96/points"])  # the reference's own BerPoints
        assert csv == str(g["ber/h96/csv"])
    one_pts, one_csv = _sweep("host")  # this process: world size 1
    assert np.array_equal(one_pts, res[0][0]) and one_csv == res[0][1]


def test_ber_sweep_two_ranks_gpu_decoder_device_channel(cuda):
    res = _two_ranks("device")
    one_pts, one_csv = _sweep("device")
    for r in range(2):
        assert np.array_equal(res[r][0], one_pts)  # per-frame seeds: independent of the shard count
        assert res[r][1] == one_csv
    assert one_pts[:, 2].tolist() == [300, 300]


def _bench(extra, nproc=1):
    args = ["--config", "C2", "--batch", "128", "--iters", "5", "--steps", "3", "--warmup", "3", "--no-e2e",
            "--no-cpu", "--no-fast", "--no-configs"] + extra
    env = dict(os.environ, LDPC_BENCH_ONE_GPU="1")
    if nproc == 1:
        cmd = [sys.executable, str(ROOT / "bench.py")] + args
    else:
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
               "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), str(ROOT / "bench.py"),
               "--gpus", str(nproc)] + args
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env, cwd=str(ROOT))
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-3000:]  # rank 0 alone prints
    return json.loads(lines[0])


def test_bench_two_ranks_folds_counts(cuda):
    two = _bench(["--seed", "1000"], nproc=2)  # rank r draws with seed 1000 + r
    a, b = _bench(["--seed", "1000"]), _bench(["--seed", "1001"])
    assert two["n_gpus"] == 2 and a["n_gpus"] == 1
    steps = 3 + 3 + 3  # warmup + timed + per-class profiled steps
    assert two["counts"]["frames"] == 2 * 128 * steps
    for k in ("bit_errors", "failures", "iterations", "frames"):
        assert two["counts"][k] == a["counts"][k] + b["counts"][k], k
    assert two["value"] > 0 and two["gpu_launches"] > 0
