"""C5 (BASELINE.json configs[4]): BER/FER Monte Carlo sweep, Eb/N0 0-3 dB, n=64800, on 1..8 GPUs.

  torchrun --nproc-per-node N tools/ber_bench.py --frames-per-gpu 1024
Frames are sharded over ranks; channel, priors and decode run on each GPU (f1 device channel);
one NCCL allreduce of int64[4] per point.  Prints one JSON line on rank 0 with the points and
the decoded-frames throughput (device-timed max over ranks).
"""
import argparse
import json
import os
import sys
import time

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from paper_1609_01567_b200 import channel as ch, configs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--frames-per-gpu", type=int, default=1024)
ap.add_argument("--iters", type=int, default=10)
ap.add_argument("--ebno", type=float, nargs="+", default=[0.0, 1.0, 2.0, 3.0])
ap.add_argument("--precision", default="fp64")
args = ap.parse_args()
world = int(os.environ.get("WORLD_SIZE", 1))
rank = int(os.environ.get("RANK", 0))
local = int(os.environ.get("LOCAL_RANK", 0))
torch.cuda.set_device(local)
if world > 1:
    dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
H = configs.code("C5")
frames = args.frames_per_gpu * world
for _ in range(2):  # warm-up: same precision, batch and frames (kernel setup; GPU clocks up from idle)
    ch.ber_sweep(H, args.ebno[:1], frames, max_iterations=args.iters, batch=1024, channel="device",
                 precision=args.precision)
torch.cuda.synchronize()
if world > 1:
    dist.barrier()
t0 = time.perf_counter()
pts = ch.ber_sweep(H, args.ebno, frames, max_iterations=args.iters, seed=1, batch=1024, channel="device",
                   precision=args.precision)
torch.cuda.synchronize()
el = torch.tensor([time.perf_counter() - t0], device="cuda")
if world > 1:
    dist.all_reduce(el, op=dist.ReduceOp.MAX)
if rank == 0:
    total = frames * len(args.ebno)
    print(json.dumps({"config": "C5", "n_gpus": world, "frames_per_point": frames, "points": [p.__dict__ for p in pts],
                      "seconds": el.item(), "frames_per_s": total / el.item(),
                      "coded_Gbit_s": total * H.n / el.item() / 1e9, "early_stop": True,
                      "max_iterations": args.iters, "precision": args.precision,
                      "csv": ch.ber_csv(pts)}))
if world > 1:
    dist.destroy_process_group()
