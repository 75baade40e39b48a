#!/usr/bin/env python
"""Benchmark: decoded coded Gbit/s of the B200 LDPC decoder (BASELINE.json metric).

Workload (BASELINE.json configs[2]): DVB-S2-shaped
irregular rate-1/2 code, n = 64800, E = 226,800, batch 1024 codewords per
GPU, fixed 10 iterations (early stop off, fixed work), all-zero codeword over
BPSK/AWGN at Eb/N0 = 2 dB (synthetic, seeded).  One step = one decode of the
batch + the error-count reduction (NCCL allreduce across ranks when N > 1).

  python bench.py [--gpus N --steps K --warmup W]           # our arm
  python bench.py --impl reference [...]                     # reference CPU arm
  torchrun --nproc-per-node N bench.py --gpus N ...          # N > 1 (weak scaling)

Prints ONE JSON line on rank 0.  ``value`` is device-timed (CUDA events, max
over ranks) with the priors already resident in HBM; ``e2e`` is the same
metric through the public host API (ParallelDecoder.decode_priors: pinned host
priors -> device -> packed results back to host every step).  The per-step
working set (2.4 GB per GPU) is far larger than the 126 MB L2, so no L2
flush is needed between steps.
"""

from __future__ import annotations

import argparse
import json
import os
import pathlib
import subprocess
import sys
import time

import numpy as np

ROOT = pathlib.Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "decoded coded Gbit/s at 10 iters (n=64800), 1/2/4/8 B200; % of HBM roofline"
UNIT = "Gbit/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--config", default="C3")
    ap.add_argument("--batch", type=int, default=None)
    ap.add_argument("--iters", type=int, default=None)
    ap.add_argument("--ebno", type=float, default=2.0)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-fast", action="store_true", help="skip the fp32 fast-mode leg")
    ap.add_argument("--no-configs", action="store_true", help="skip the other-BASELINE-configs leg")
    ap.add_argument("--cpu-seconds", type=float, default=15.0, help="target CPU time of the cpu_baseline sample")
    ap.add_argument("--sub-batch", type=int, default=0, help="e2e pipeline sub-batch (0 = decoder default)")
    ap.add_argument("--seed", type=int, default=1000, help="rank r draws its synthetic frames with seed + r")
    return ap.parse_args()


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)),
            int(os.environ.get("WORLD_SIZE", 1)))


def synthetic_observations(H, B, ebno_db, seed):
    """All-zero codeword, BPSK 0 -> -1, AWGN (channel.py:1-8): channel outputs y [B, n] and sigma^2."""
    from paper_1609_01567_b200 import configs

    s2 = configs.ebno_to_sigma2(ebno_db, configs.rate(H))
    rng = np.random.default_rng(seed)
    return -1.0 + np.sqrt(s2) * rng.standard_normal((B, H.n)), s2


def synthetic_priors(H, B, ebno_db, seed):
    """All-zero codeword, BPSK 0 -> -1, AWGN (channel.py:1-8); priors by the reference's numpy expression."""
    from paper_1609_01567_b200 import configs, priors_awgn_batch

    s2 = configs.ebno_to_sigma2(ebno_db, configs.rate(H))
    rng = np.random.default_rng(seed)
    Y = -1.0 + np.sqrt(s2) * rng.standard_normal((B, H.n))
    return priors_awgn_batch(Y, s2), s2


def workload_desc(cfg, H, B, iters, ebno):
    return {"workload": f"{cfg}: DVB-S2-shaped irregular LDPC n={H.n} m={H.m} E={H.total_edges} rate 1/2 "
                        f"(var deg 8/3/2, check deg 7), batch {B} codewords per GPU, fixed {iters} iterations",
            "code": cfg, "n": H.n, "edges": H.total_edges, "batch_per_gpu": B, "iterations": iters,
            "early_stop": False, "ebno_db": ebno,
            "l2": "no flush needed: per-step working set ~2.4 GB/GPU >> 126 MB L2"}


# ---- CPU reference (oracle port of the reference decoder, test-infrastructure) ----

def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown CPU"


def cpu_reference_rate(H, P, iters, seconds):
    """Time the oracle (C restatement of serial.py) on host threads over the workload's frames.

    Decodes every frame of P when that fits ~2x the time budget (it does at C3 on the GPU box's
    16 threads: 1024 frames in ~2 s), else a bounded prefix of it.  Returns (Gbit/s, cores, frames,
    secs, outputs) with outputs = (estimate [F, n] u8, success [F] bool, iterations [F] i32,
    syndrome [F, m] u8) of frames P[:F], the checker for the timed GPU run (parity)."""
    sys.path.insert(0, str(ROOT / "oracle"))
    from oracle import OracleTables  # noqa: E402  (checker / CPU baseline only)

    O = OracleTables.from_matrix(H)
    cores = os.cpu_count() or 1
    t = time.perf_counter()
    O.decode_batch(P[:1], iters, fixed_iterations=True, n_threads=1)
    per_frame = time.perf_counter() - t
    budget = int(2 * seconds * cores / max(per_frame, 1e-3))
    frames = len(P) if budget >= len(P) else max(cores, (budget // cores) * cores)
    Ps = np.ascontiguousarray(P[:frames])
    t = time.perf_counter()
    outs = O.decode_batch(Ps, iters, fixed_iterations=True, n_threads=cores)
    secs = time.perf_counter() - t
    return frames * H.n / secs / 1e9, cores, frames, secs, outs


def parity_vs_oracle(outs_dev, ref, n, m):
    """Compare the timed GPU run's outputs (device tensors) with the oracle's on the same frames."""
    from paper_1609_01567_b200 import unpack_bits

    est_o, ok_o, its_o, z_o = ref
    F = len(ok_o)
    est, ok, its, syn = (t[:F].cpu().numpy() for t in outs_dev)
    bad_est = ~(unpack_bits(est.view(np.uint32), n) == est_o).all(axis=1)
    bad_ok = ok.astype(bool) != ok_o.astype(bool)
    bad_its = its != its_o
    bad_syn = ~(unpack_bits(syn.view(np.uint32), m) == z_o).all(axis=1)
    bad = bad_est | bad_ok | bad_its | bad_syn
    return {"frames": int(F), "mismatches": int(bad.sum()),
            "fields": {"estimate": int(bad_est.sum()), "success": int(bad_ok.sum()),
                       "iterations": int(bad_its.sum()), "syndrome": int(bad_syn.sum())},
            "checked": "outputs of the last timed decode_device step vs the C oracle (oracle/) on the same "
                       "priors: estimate bits, success, iterations, syndrome bits; bit-exact"}


def survey_bytes_per_codeword(E, n, iters, w=8):
    """w*E*(4I+2) + w*n*(I+2) + (n/8)*(2I+2) algorithmic HBM bytes per codeword."""
    return w * E * (4 * iters + 2) + w * n * (iters + 2) + (n / 8) * (2 * iters + 2)


PARALLELISM = "dp%d: independent codeword shards, NCCL allreduce of error counts"


def run_reference(args):
    rank, _, world = dist_env()
    if rank != 0:
        return
    from paper_1609_01567_b200 import configs

    cfg = args.config
    C = configs.CONFIGS[cfg]
    H = configs.code(C["code"])
    B = args.batch or C["batch"]
    iters = args.iters if args.iters is not None else C["max_iterations"]
    sys.path.insert(0, str(ROOT / "oracle"))
    from oracle import OracleTables

    O = OracleTables.from_matrix(H)
    cores = os.cpu_count() or 1
    # 64 frames per thread per step: long enough that thread start-up and the tail of the last
    # frames do not understate the CPU (2 frames per thread read ~15% low in round 1)
    P, _ = synthetic_priors(H, 64 * cores, args.ebno, seed=7)
    times = []
    for step in range(args.warmup + args.steps):
        t = time.perf_counter()
        O.decode_batch(P, iters, fixed_iterations=True, n_threads=cores)
        dt = time.perf_counter() - t
        if step >= args.warmup:
            times.append(dt)
    secs = float(np.sum(times))
    value = len(P) * H.n * args.steps / secs / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * secs / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic: all-zero codeword, BPSK/AWGN at %.1f dB, seeded numpy normals" % args.ebno,
        "config": dict(workload_desc(cfg, H, B, iters, args.ebno), parallelism=PARALLELISM % world),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": f"each step {len(P)} frames ({len(P) // cores} per thread) of the workload's "
                                   f"code (fixed {iters} iterations) decoded by the C restatement of the reference "
                                   f"decoder (oracle/) on {cores} host threads ({cpu_model()})",
                         "note": "a C port of the reference's serial.py, ~20x faster per core than the reference's "
                                 "own numpy ParallelDecoder (see python_engine)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "python_engine": reference_python_engine(H, iters, args.ebno),
    }
    print(json.dumps(line), flush=True)


def _py_engine_worker(args):
    """One process: the reference's own ParallelDecoder (baseline/_ref, unmodified) on frames of H."""
    path, n, m, rows, cols, Y, s2, iters = args
    sys.path.insert(0, path)
    import edgeldpc
    from edgeldpc.engine import ParallelDecoder as RefDecoder

    Href = edgeldpc.ParityCheckMatrix(n, m, tuple(zip(rows.tolist(), cols.tolist())))
    T = edgeldpc.CodeTables.from_matrix(Href)
    dec = RefDecoder(T, 512, n_threads=1)
    t = time.perf_counter()
    its = [dec.decode(y, s2, iters).iterations_used for y in Y]
    return time.perf_counter() - t, its


def reference_python_engine(H, iters, ebno, frames_per_core=1):
    """Context only: the reference's own numpy engine, unmodified, from
    baseline/_ref (pip --target install of /root/reference), one frame per host core in a process pool.
    None when the install is absent."""
    ref = ROOT / "baseline" / "_ref"
    if not (ref / "edgeldpc").is_dir():
        return None
    from concurrent.futures import ProcessPoolExecutor

    cores = os.cpu_count() or 1
    Y, s2 = synthetic_observations(H, cores * frames_per_core, ebno, seed=11)
    chunks = [Y[i::cores] for i in range(cores)]
    t = time.perf_counter()
    try:
        with ProcessPoolExecutor(cores) as ex:
            per = list(ex.map(_py_engine_worker,
                              [(str(ref), H.n, H.m, H.rows, H.cols, c, s2, iters) for c in chunks]))
    except Exception as e:  # context figure only; never fails the arm
        return {"error": repr(e)[:200]}
    wall = time.perf_counter() - t
    busy = max(p[0] for p in per)
    its = [i for p in per for i in p[1]]
    return {"value": len(Y) * H.n / busy / 1e9, "unit": UNIT, "cores": cores, "frames": len(Y),
            "mean_iterations": float(np.mean(its)),
            "seconds_decode_max_worker": busy, "seconds_wall_incl_table_build": wall,
            "path": "baseline/_ref edgeldpc.engine.ParallelDecoder(tables, 512, n_threads=1).decode, one process "
                    "per core (context for the port's speed; not the reference arm's value)"}


# ---- clocks sampler ---------------------------------------------------------------

class ClockSampler:
    """nvidia-smi -lms sampling of SM clocks and throttle reasons during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index, period_ms=50):
        self.cmd = ["nvidia-smi", "-i", str(device_index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                    "-lms", str(period_ms)]
        self.proc = None
        self.samples = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(self.cmd, stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            time.sleep(0.3)  # first sample lands before the timed region starts
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc is None:
            return
        time.sleep(0.1)
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            out = ""
        for line in (out or "").splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 9:
                self.samples.append(parts)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}

        def num(x):
            try:
                return float(x)
            except ValueError:
                return None

        sm = [v for v in (num(s[1]) for s in self.samples) if v is not None]
        mx = [v for v in (num(s[2]) for s in self.samples) if v is not None]
        pw = [v for v in (num(s[3]) for s in self.samples) if v is not None]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[5 + i] == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "power_w_max": max(pw) if pw else None, "reasons": reasons, "samples": len(self.samples)}


def load_traffic(kernel_class):
    """dram bytes per launch from the committed `ncu --set full` summary (profiles/), or None."""
    f = ROOT / "profiles" / "ncu_traffic.json"
    if not f.exists():
        return None
    try:
        d = json.loads(f.read_text())
        return d.get(kernel_class, {}).get("dram_bytes_per_launch")
    except Exception:
        return None


# ---- our arm ----------------------------------------------------------------------

def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_1609_01567_b200 import CodeTables, ParallelDecoder, _native, configs

    rank, local_rank, world = dist_env()
    # LDPC_BENCH_ONE_GPU=1 (testing the multi-rank flow on a one-GPU box): every rank on cuda:0,
    # gloo instead of NCCL (NCCL refuses two ranks on one device).  Never used for reported numbers.
    one_gpu = os.environ.get("LDPC_BENCH_ONE_GPU") == "1"
    if one_gpu:
        local_rank = 0
    if world > 1:
        torch.cuda.set_device(local_rank)
        if one_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local_rank}"))
    dev = torch.device(f"cuda:{local_rank}")
    torch.cuda.set_device(dev)
    from paper_1609_01567_b200.numa import bind_to_gpu

    all_cpus = os.sched_getaffinity(0)
    numa = bind_to_gpu(local_rank)  # host copies from the CPUs (and memory) nearest this rank's GPU
    cfg = args.config
    C = configs.CONFIGS[cfg]
    H = configs.code(C["code"])
    B = args.batch or C["batch"]
    iters = args.iters if args.iters is not None else C["max_iterations"]
    T = CodeTables.from_matrix(H)
    dec = ParallelDecoder(T, max_batch=B, sub_batch=args.sub_batch)
    P_host, _ = synthetic_priors(H, B, args.ebno, seed=args.seed + rank)
    P_pin = torch.from_numpy(P_host).pin_memory()
    P_dev = P_pin.to(dev, non_blocking=True)
    ws = dec.workspace(B)
    outs = dec.alloc_outputs(B, dev)
    counts = torch.zeros(4, dtype=torch.int64, device=dev)       # whole run, all ranks
    step_counts = torch.zeros(4, dtype=torch.int64, device=dev)  # one step, folded over ranks
    stream = torch.cuda.current_stream()

    def step(profile=None):
        dec.decode_device(P_dev, iters, early_stop=False, workspace=ws, outputs=outs, profile=profile)
        step_counts.zero_()
        dec.count_errors(outs, step_counts)
        if world > 1:
            dist.all_reduce(step_counts)  # the only collective: int64[4] error counters
        counts.add_(step_counts)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    # timed region: K steps, barrier + synchronize on both sides, CUDA events, max over ranks
    L = _native.load_library()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = L.ldpc_kernel_launches()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(torch.cuda.current_device()) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            step()
        ev1.record(stream)
        torch.cuda.synchronize()
    launches = L.ldpc_kernel_launches() - launches0
    timed_outs = tuple(t.clone() for t in outs)  # the last timed step's results (checked below)
    if world > 1:
        dist.barrier()
    ms = ev0.elapsed_time(ev1)
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    ms_step = ms_max / args.steps
    value = world * B * H.n / (ms_step / 1e3) / 1e9

    # per-kernel-class event timing over K profiled steps (same stream, same work)
    prof = _native.Profile()
    for _ in range(args.steps):
        step(profile=prof)
    torch.cuda.synchronize()
    pd = prof.as_dict()
    dom = max(("check", "variable"), key=lambda k: pd[k]["ms"])
    per_launch_bytes = pd[dom]["bytes"] / max(pd[dom]["launches"], 1)
    per_launch_ms = pd[dom]["ms"] / max(pd[dom]["launches"], 1)
    peaks = {}
    try:
        peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
    except Exception:
        pass
    peak = float(peaks.get("hbm_gbs", 6650.0))
    achieved = per_launch_bytes / (per_launch_ms / 1e3) / 1e9
    step_ms_prof = sum(v["ms"] for v in pd.values()) / args.steps
    # step level with SURVEY.md 8(d)'s formula (layout passes and the transpose not counted)
    survey_bpc = survey_bytes_per_codeword(H.total_edges, H.n, iters)
    step_survey_GBps = B * survey_bpc / (ms_step / 1e3) / 1e9
    class_frac = {k: (v["bytes"] / (v["ms"] / 1e3) / 1e9) / peak for k, v in pd.items()
                  if k in ("check", "variable", "estimate") and v["ms"] > 0}

    # e2e through the public host API: pinned priors in, packed results out, every step
    e2e = e2e_stream = e2e_from_y = e2e_pageable = None
    if not args.no_e2e:
        from paper_1609_01567_b200.decoder import BatchResult

        n, m = H.n, H.m
        pin = lambda shape, dt: torch.empty(shape, dtype=dt).pin_memory().numpy()  # noqa: E731
        res = BatchResult(pin((B, (n + 31) // 32), torch.int32).view(np.uint32), pin((B,), torch.uint8),
                          pin((B,), torch.int32), pin((B, (m + 31) // 32), torch.int32).view(np.uint32), n, m)
        Pn = P_pin.numpy()
        for _ in range(max(1, args.warmup)):
            dec.decode_priors(Pn, iters, early_stop=False, out=res)
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            dec.decode_priors(Pn, iters, early_stop=False, out=res)
        el = time.perf_counter() - t0
        tt = torch.tensor([el], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        el = float(tt.item())
        e2e = {"value": world * B * n * args.steps / el / 1e9, "unit": UNIT,
               "h2d_bytes_per_step": int(Pn.nbytes),
               "d2h_bytes_per_step": int(res.est_bits.nbytes + res.success.nbytes + res.iterations.nbytes
                                         + res.syn_bits.nbytes),
               "ms_per_step": 1e3 * el / args.steps,
               "path": "ParallelDecoder.decode_priors (ldpc_decoder_decode_host: pinned H2D, decode, D2H; "
                       "geometric sub-batches over a copy stream and two compute streams)"}
        # the same call as a plain caller makes it (engine.py:363-372 takes any array): pageable numpy
        # priors in, fresh (pageable) result arrays out; staged through the decoder's pinned slots
        Pn_pageable = np.array(Pn, copy=True)
        for _ in range(max(1, args.warmup)):
            dec.decode_priors(Pn_pageable, iters, early_stop=False)
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            dec.decode_priors(Pn_pageable, iters, early_stop=False)
        el_pg = time.perf_counter() - t0
        tp = torch.tensor([el_pg], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(tp, op=dist.ReduceOp.MAX)
        el_pg = float(tp.item())
        e2e_pageable = {"value": world * B * n * args.steps / el_pg / 1e9, "unit": UNIT,
                        "h2d_bytes_per_step": int(Pn_pageable.nbytes), "d2h_bytes_per_step": e2e["d2h_bytes_per_step"],
                        "ms_per_step": 1e3 * el_pg / args.steps,
                        "vs_pinned": e2e["ms_per_step"] / (1e3 * el_pg / args.steps),
                        "path": "ParallelDecoder.decode_priors on a plain numpy array, fresh numpy results "
                                "(pageable input staged through pinned slots by host copy threads, overlapped "
                                "with the H2D DMA; results through pinned buffers)"}
        # streaming API (two batches in flight: the H2D of step k+1 overlaps the decode of step k)
        outs2 = [res, BatchResult(pin((B, (n + 31) // 32), torch.int32).view(np.uint32), pin((B,), torch.uint8),
                                  pin((B,), torch.int32), pin((B, (m + 31) // 32), torch.int32).view(np.uint32),
                                  n, m)]

        def stream_steps(k):
            pend = []
            for i in range(k):
                pend.append(dec.decode_priors_async(Pn, iters, early_stop=False, out=outs2[i % 2]))
                if len(pend) == 2:
                    pend.pop(0).wait()
            for q in pend:
                q.wait()

        # from channel observations: decode_batch(Y, sigma2), the reference's decode(y, sigma2) per frame
        # batched -- priors formed on the device, bit-identical to the host's numpy (priors.cuh), when the
        # probe says so; else by the reference's numpy expression on the host threads, then decode_priors
        from paper_1609_01567_b200.decoder import device_priors_exact

        dev_priors = device_priors_exact(dev.index or 0)
        Y_host, s2_y = synthetic_observations(H, B, args.ebno, seed=2000 + rank)
        Y_pin = torch.from_numpy(Y_host).pin_memory().numpy()
        for _ in range(max(1, args.warmup)):
            dec.decode_batch(Y_pin, s2_y, iters, early_stop=False, out=res)
        t0 = time.perf_counter()
        for _ in range(args.steps):
            dec.decode_batch(Y_pin, s2_y, iters, early_stop=False, out=res)
        el_y = time.perf_counter() - t0
        ty = torch.tensor([el_y], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(ty, op=dist.ReduceOp.MAX)
        el_y = float(ty.item())
        e2e_from_y = {"value": world * B * n * args.steps / el_y / 1e9, "unit": UNIT,
                      "h2d_bytes_per_step": int(Y_host.nbytes), "d2h_bytes_per_step": e2e["d2h_bytes_per_step"],
                      "ms_per_step": 1e3 * el_y / args.steps,
                      "device_priors": dev_priors,
                      "path": ("ParallelDecoder.decode_batch(Y, sigma2) (ldpc_decoder_decode_awgn_host): pinned H2D of "
                               "the observations, priors formed in the layout kernel with numpy's exp algorithm "
                               "(bit-identical; probe passed), decode, D2H" if dev_priors else
                               "ParallelDecoder.decode_batch(Y, sigma2): priors by the reference's numpy expression "
                               f"on {min(32, os.cpu_count() or 1)} host threads inside the timed region (this host's "
                               "np.exp differs from the device prior), then decode_priors")}
        stream_steps(max(2, args.warmup))
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        stream_steps(args.steps)
        el = time.perf_counter() - t0
        tt = torch.tensor([el], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        el = float(tt.item())
        e2e_stream = {"value": world * B * n * args.steps / el / 1e9, "unit": UNIT,
                      "h2d_bytes_per_step": e2e["h2d_bytes_per_step"], "d2h_bytes_per_step": e2e["d2h_bytes_per_step"],
                      "ms_per_step": 1e3 * el / args.steps,
                      "path": "ParallelDecoder.decode_priors_async / wait (ldpc_decoder_submit: whole-batch decode, "
                              "two batches in flight)"}

    # f4 fast mode (fp32, not bit-exact): same workload, device-timed, agreement with the exact run
    fast = None
    if not args.no_fast:
        outs32 = dec.alloc_outputs(B, dev)
        for _ in range(args.warmup):
            dec.decode_device(P_dev, iters, early_stop=False, workspace=ws, outputs=outs32, precision="fp32")
        torch.cuda.synchronize()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        for _ in range(args.steps):
            dec.decode_device(P_dev, iters, early_stop=False, workspace=ws, outputs=outs32, precision="fp32")
        f1.record(stream)
        torch.cuda.synchronize()
        fms = f0.elapsed_time(f1) / args.steps
        same = (outs32[0] == outs[0]).all(dim=1).float().mean().item()
        fast = {"value": world * B * H.n / (fms / 1e3) / 1e9, "unit": UNIT, "dtype": "f32", "ms_per_step": fms,
                "identical_frames_vs_f64": same,
                "note": "f4 fast mode, fp32: the reference's product order for degrees <= 16 (approximate division), "
                        "O(d) prefix/suffix checks and log-ratio-sum variables above; not bit-exact, tolerance vs the "
                        "oracle in DESIGN.md / tests/test_fast_gpu.py",
                "roofline_frac": (B * survey_bytes_per_codeword(H.total_edges, H.n, iters, w=4) / (fms / 1e3) / 1e9)
                                 / peak}

    # the other BASELINE.json configs (parity-test cases, reported for reference, not the headline):
    # device-timed decode per call through decode_device with the automatic schedule
    others = None
    if world == 1 and not args.no_configs and cfg == "C3":
        others = {}
        # (label, code, batch, iterations, early stop, Eb/N0, precision); C2/C4 at the config's Eb/N0
        runs = (("C1", "C1", 1, 50, True, 2.0, "fp64"),
                ("C2", "C2", 4096, 20, True, 2.0, "fp64"),
                ("C2_fixed", "C2", 4096, 20, False, 2.0, "fp64"),
                ("C4", "C4", 256, 20, True, 3.0, "fp64"),
                ("C4_fast_fp32", "C4", 256, 20, True, 3.0, "fp32"),
                ("C4D_fixed", "C4D", 256, 20, False, 2.0, "fp64"),
                ("C4D_fixed_fast_fp32", "C4D", 256, 20, False, 2.0, "fp32"),
                ("C5_3dB", "C5", 1024, 10, True, 3.0, "fp64"))
        for label, name, B_o, it_o, early_o, eb_o, prec_o in runs:
            H_o = configs.code(name)
            T_o = CodeTables.from_matrix(H_o)
            P_o = torch.from_numpy(synthetic_priors(H_o, B_o, eb_o, seed=5)[0]).to(dev)
            with ParallelDecoder(T_o, max_batch=B_o) as d_o:
                ws_o, outs_o = d_o.workspace(B_o), d_o.alloc_outputs(B_o, dev)
                for _ in range(3):
                    d_o.decode_device(P_o, it_o, early_stop=early_o, workspace=ws_o, outputs=outs_o,
                                      precision=prec_o)
                reps = 20 if B_o < 64 else 5
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda.synchronize()
                e0.record(stream)
                for _ in range(reps):
                    d_o.decode_device(P_o, it_o, early_stop=early_o, workspace=ws_o, outputs=outs_o,
                                      precision=prec_o)
                e1.record(stream)
                torch.cuda.synchronize()
                ms_o = e0.elapsed_time(e1) / reps
                its_o = outs_o[2].float()
            others[label] = {"batch": B_o, "max_iterations": it_o, "early_stop": early_o, "ebno_db": eb_o,
                             "precision": prec_o, "ms_per_decode": ms_o,
                             "coded_Gbit_s": B_o * H_o.n / (ms_o / 1e3) / 1e9,
                             "mean_iterations": its_o.mean().item(), "max_iterations_used": its_o.max().item(),
                             "n": H_o.n, "edges": H_o.total_edges}
            del P_o, ws_o, outs_o
        # fp64-pipe activity of the high-degree (O(d^2)) kernels at C4, from the committed ncu metric
        # list of one C4 decode (a profiler number, so not measured here: profiles/ncu_c4_fp64.json)
        try:
            c4k = json.loads((ROOT / "profiles" / "ncu_c4_fp64.json").read_text())["kernels"]
            chains = {k: {"fp64_pipe_pct": v["fp64_pipe_pct"], "sm_active_balance": v["sm_active_balance"],
                          "share_of_decode": v["share"]}
                      for k, v in c4k.items() if "chains" in k and v["launches"] > 2}
            others["C4"]["fp64_pipe"] = {"kernels": chains, "source": "profiles/ncu_c4_fp64.json (tools/c4_ncu.sh: "
                                         "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active, "
                                         "sm__cycles_active avg/max, one C4 decode under ncu)"}
        except Exception:
            pass
        if "C4" in others and "C4_fast_fp32" in others:
            others["C4_fast_fp32"]["speedup_vs_exact"] = others["C4"]["ms_per_decode"] / others["C4_fast_fp32"]["ms_per_decode"]
        if "C4D_fixed" in others and "C4D_fixed_fast_fp32" in others:
            others["C4D_fixed_fast_fp32"]["speedup_vs_exact"] = (others["C4D_fixed"]["ms_per_decode"]
                                                                  / others["C4D_fixed_fast_fp32"]["ms_per_decode"])
        if "C2" in others and "C2_fixed" in others:
            others["C2"]["vs_fixed_iterations"] = others["C2"]["ms_per_decode"] / others["C2_fixed"]["ms_per_decode"]
        # the reference-facing single-frame call at C3 (engine.py:363 decode(y, sigma2)): host in,
        # host out, wall clock; one cooperative grid launch per frame (grid.cu)
        Y1, s2_1 = synthetic_observations(H, 12, args.ebno, seed=77)
        with ParallelDecoder(T, max_batch=1) as d1:
            for y in Y1[:3]:
                d1.decode(y, s2_1, 50)
            lat, its1 = [], []
            for y in Y1[3:]:
                t0 = time.perf_counter()
                r1 = d1.decode(y, s2_1, 50)
                lat.append(time.perf_counter() - t0)
                its1.append(r1.iterations_used)
        others["C3_single_frame"] = {"batch": 1, "max_iterations": 50, "early_stop": True,
                                     "ms_per_decode_wall": 1e3 * float(np.median(lat)),
                                     "mean_iterations": float(np.mean(its1)),
                                     "path": "ParallelDecoder.decode(y, sigma2): H2D of y, device prior, "
                                             "grid schedule (one cooperative launch), D2H"}

    cpu = parity = None
    if rank == 0 and world == 1 and not args.no_cpu:
        os.sched_setaffinity(0, all_cpus)  # the CPU baseline gets every host thread
        v, cores, frames, secs, ref_outs = cpu_reference_rate(H, P_host, iters, args.cpu_seconds)
        cpu = {"value": v, "unit": UNIT, "cores": cores, "kind": "port",
               "sample": f"{frames} frames of the workload (fixed {iters} iterations) in {secs:.1f} s by the C "
                         f"restatement of the reference decoder (oracle/) on {cores} host threads ({cpu_model()})"}
        parity = parity_vs_oracle(timed_outs, ref_outs, H.n, H.m)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic: all-zero codeword, BPSK/AWGN at %.1f dB, seeded numpy normals; priors by the "
                    "reference's numpy expression" % args.ebno,
            "config": dict(workload_desc(cfg, H, B, iters, args.ebno), parallelism=PARALLELISM % world),
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": load_traffic(dom), "kernel": dom,
                         "algorithmic_bytes_per_launch": per_launch_bytes, "launch_ms": per_launch_ms,
                         "peak_source": "MEASURED_PEAKS.json hbm_gbs (measured copy)" if peaks else "fallback 6.65 TB/s",
                         "step": {"bytes_per_codeword": survey_bpc, "GBps": step_survey_GBps,
                                  "frac": step_survey_GBps / peak,
                                  "formula": "SURVEY.md 8(d): 8*E*(4I+2) + 8*n*(I+2) + (n/8)*(2I+2) per codeword "
                                             "/ device-timed ms_per_step"},
                         "class_frac": class_frac,
                         "kernel_ms_per_step": {k: v["ms"] / args.steps for k, v in pd.items()}},
            "parity": parity,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "e2e_stream": e2e_stream,
            "e2e_from_y": e2e_from_y,
            "e2e_pageable": e2e_pageable,
            "fast_fp32": fast,
            "other_configs": others,
            "gpu_launches": int(launches),
            "numa": numa,
            "clocks": clk.summary(),
            "counts": {"bit_errors": int(counts[0]), "failures": int(counts[1]), "iterations": int(counts[2]),
                       "frames": int(counts[3])},
        }
        print(json.dumps(line), flush=True)
    dec.close()
    if world > 1:
        dist.destroy_process_group()
    if parity is not None and parity["mismatches"]:
        sys.stderr.write(f"PARITY FAILURE: {parity['mismatches']} of {parity['frames']} frames differ from the oracle\n")
        sys.exit(3)


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
