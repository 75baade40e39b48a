"""AWGN channel, frame seeding and the BER sweep, sharded over GPUs.

Mirrors the reference's channel/RNG layer (edgeldpc/rng.py:34-80,
channel.py:31-148): xorshift128+ with per-frame states derived from
(seed, point, frame), BPSK 0 -> -1 over AWGN via Box-Muller, and ber_sweep's
fold of (bit errors, iterations, failures) in frame order.

Multi-GPU: frames of every Eb/N0 point are split into
contiguous per-rank ranges; each rank decodes its own frames on its own GPU
and the only collective is one allreduce of int64[4] = {bit errors, failures,
iterations, frames} per point.  Integer sums are exact, so the BerPoints are
identical for any number of ranks (and to the single-process reference).

Channel arithmetic: the integer RNG is exact.  ``exact_channel=True`` runs
Box-Muller with the same libm calls as Python's math module, in C on host
threads (csrc/host_channel.cpp, ``transmit_all_zero_frames``), exactly like
channel.py:31-37, so y -- and with the bit-exact decoder the whole BerPoint --
equals the reference's.  The default vectorised path uses numpy's log/cos/sin,
which may differ from libm in the last ulp (statistically identical noise, not
bit-identical; the reference's channel arithmetic is itself untested).  ber_sweep
uses the exact native channel by default.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

MASK64 = (1 << 64) - 1
_GOLDEN = 0x9E3779B97F4A7C15
DEFAULT_BATCH = 1024


# ---- rng.py:34-80 -------------------------------------------------------------

@dataclass(frozen=True)
class RngState:
    s0: int
    s1: int

    def __post_init__(self):
        if not (0 <= self.s0 <= MASK64 and 0 <= self.s1 <= MASK64):
            raise ValueError("state words must be unsigned 64-bit integers")
        if self.s0 == 0 and self.s1 == 0:
            raise ValueError("all-zero state is a fixed point of xorshift128+")


def rng_next(state: RngState) -> tuple[RngState, int]:
    """xorshift128+ (23/18/5), rng.py:34-41."""
    x, y = state.s0, state.s1
    x ^= (x << 23) & MASK64
    x ^= x >> 18
    x ^= y ^ (y >> 5)
    return RngState(y, x), (x + y) & MASK64


def u01_from_bits(x: int) -> float:
    """Top 53 bits + 1, scaled by 2^-53: a double in (0, 1] (rng.py:44-50)."""
    return ((x >> 11) + 1) * 2.0**-53


def rng_uniform01(state: RngState) -> tuple[RngState, float]:
    state, x = rng_next(state)
    return state, u01_from_bits(x)


def _mix64(z: int) -> int:
    z &= MASK64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
    return z ^ (z >> 31)


def derive_state(*keys: int) -> RngState:
    """splitmix64-style per-frame state (rng.py:67-80)."""
    acc = 0
    for k in keys:
        acc = _mix64((acc + _GOLDEN + (k & MASK64)) & MASK64)
    s0 = _mix64((acc + _GOLDEN) & MASK64)
    s1 = _mix64((acc + 2 * _GOLDEN) & MASK64)
    if s0 == 0 and s1 == 0:
        s1 = _GOLDEN
    return RngState(s0, s1)


# ---- channel.py:31-67 -------------------------------------------------------

def shuffle(items: list, state: RngState) -> RngState:
    """rng.py:84-90: Fisher-Yates from the last position down; the partner of position i is the
    high 64 bits of x * (i + 1) for the next output x.  In place; returns the advanced state."""
    for i in range(len(items) - 1, 0, -1):
        state, x = rng_next(state)
        j = (x * (i + 1)) >> 64
        items[i], items[j] = items[j], items[i]
    return state


def randrange(state: RngState, bound: int) -> tuple[RngState, int]:
    """rng.py:93-96: an integer in [0, bound), the high 64 bits of x * bound."""
    state, x = rng_next(state)
    return state, (x * bound) >> 64


def box_muller(u1: float, u2: float) -> tuple[float, float]:
    """Standard normal pair from two uniforms, u1 in (0, 1] (channel.py:31-37)."""
    if u1 <= 0.0:
        raise ValueError("u1 must be positive")
    radius = math.sqrt(-2.0 * math.log(u1))
    angle = 2.0 * math.pi * u2
    return radius * math.cos(angle), radius * math.sin(angle)


def ebno_to_sigma2(ebno_db: float, rate: float) -> float:
    """channel.py:40-44."""
    if not 0.0 < rate < 1.0:
        raise ValueError("rate must be in (0, 1)")
    return 1.0 / (2.0 * rate * 10.0 ** (ebno_db / 10.0))


def transmit_all_zero(n: int, sigma2: float, state: RngState) -> tuple[RngState, np.ndarray]:
    """y_j = -1 + sigma z_j, pairs of uniforms per normal pair (channel.py:47-67)."""
    if sigma2 <= 0.0:
        raise ValueError("sigma2 must be positive")
    sigma = math.sqrt(sigma2)
    y = np.empty(n)
    i = 0
    while i < n:
        state, u1 = rng_uniform01(state)
        state, u2 = rng_uniform01(state)
        z0, z1 = box_muller(u1, u2)
        y[i] = -1.0 + sigma * z0
        i += 1
        if i < n:
            y[i] = -1.0 + sigma * z1
            i += 1
    return state, y


def uniforms_batch(states: list[RngState], count: int) -> np.ndarray:
    """[F, count] uniforms of F independent xorshift128+ streams, integer-exact, vectorised over frames."""
    s0 = np.array([s.s0 for s in states], dtype=np.uint64)
    s1 = np.array([s.s1 for s in states], dtype=np.uint64)
    out = np.empty((len(states), count), dtype=np.float64)
    scale = np.float64(2.0**-53)
    with np.errstate(over="ignore"):
        for k in range(count):
            x, y = s0, s1
            x = x ^ (x << np.uint64(23))
            x = x ^ (x >> np.uint64(18))
            x = x ^ (y ^ (y >> np.uint64(5)))
            s0, s1 = y, x
            out[:, k] = (((x + y) >> np.uint64(11)) + np.uint64(1)).astype(np.float64) * scale
    return out


def transmit_all_zero_batch(n: int, sigma2: float, states: list[RngState], exact: bool = False) -> np.ndarray:
    """Received frames [F, n] for the all-zero codeword, one seeded stream per frame."""
    if sigma2 <= 0.0:
        raise ValueError("sigma2 must be positive")
    if exact:
        return np.stack([transmit_all_zero(n, sigma2, s)[1] for s in states]) if states else np.empty((0, n))
    pairs = (n + 1) // 2
    u = uniforms_batch(states, 2 * pairs)
    u1, u2 = u[:, 0::2], u[:, 1::2]
    radius = np.sqrt(-2.0 * np.log(u1))
    angle = 2.0 * math.pi * u2
    z = np.empty((len(states), 2 * pairs))
    z[:, 0::2] = radius * np.cos(angle)
    z[:, 1::2] = radius * np.sin(angle)
    return -1.0 + math.sqrt(sigma2) * z[:, :n]


def transmit_all_zero_frames(n: int, sigma2: float, seed: int, point: int, frame0: int, count: int,
                             threads: int = 0, out: np.ndarray | None = None) -> np.ndarray:
    """Frames frame0..frame0+count-1 of Eb/N0 point ``point`` ([count, n]), each from
    derive_state(seed, point, frame) (channel.py:112), bit-identical to transmit_all_zero
    (the same libm log/cos/sin calls; csrc/host_channel.cpp), on ``threads`` host threads."""
    import ctypes

    from . import _native

    if sigma2 <= 0.0:
        raise ValueError("sigma2 must be positive")
    if out is None:
        out = np.empty((count, n), dtype=np.float64)
    elif out.shape != (count, n) or out.dtype != np.float64 or not out.flags.c_contiguous:
        raise ValueError("out must be a C-contiguous float64 [count, n] array")
    rc = _native.load_library().ldpc_channel_awgn_host(int(seed) & MASK64, int(point) & MASK64,
                                                        int(frame0) & MASK64, int(count), int(n), float(sigma2),
                                                        ctypes.c_void_p(out.ctypes.data), int(threads))
    _native.check(rc, "ldpc_channel_awgn_host")
    return out


# ---- channel.py:70-148 ------------------------------------------------------

@dataclass(frozen=True)
class BerPoint:
    ebno_db: float
    sigma2: float
    frames: int
    bit_errors: int
    ber: float
    mean_iterations: float
    failures: int


def shard_range(frames: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous frame range of one rank (frames [lo, hi))."""
    return frames * rank // world, frames * (rank + 1) // world


def _dist_info():
    try:
        import torch.distributed as dist

        if dist.is_available() and dist.is_initialized():
            return dist, dist.get_rank(), dist.get_world_size()
    except Exception:
        pass
    return None, 0, 1


def gpu_decode_counts(decoder, early_stop: bool = True, precision: str = "fp64"):
    """decode_fn for ber_sweep: GPU decode of a batch, error counts accumulated on the device."""
    import torch

    from .decoder import priors_awgn_batch

    from .decoder import device_priors_exact

    def run(Y, sigma2, max_iterations, counts):
        if device_priors_exact(counts.device.index or 0):   # priors formed on the device, bit-identical
            Yd = torch.from_numpy(np.ascontiguousarray(Y)).to(counts.device)
            S = torch.full((Yd.shape[0],), float(sigma2), dtype=torch.float64, device=counts.device)
            outs = decoder.decode_device_awgn(Yd, S, max_iterations, early_stop=early_stop, syndrome_out=False,
                                              precision=precision)
        else:
            P = torch.from_numpy(priors_awgn_batch(Y, sigma2)).to(counts.device)
            outs = decoder.decode_device(P, max_iterations, early_stop=early_stop, syndrome_out=False,
                                         precision=precision)
        decoder.count_errors(outs, counts)

    return run


def ber_sweep(H, ebno_points, frames: int, max_iterations: int = 50, seed: int = 0, group_size: int = 512,
              decoders_in_flight: int = 1, rate: float | None = None, *, batch: int = DEFAULT_BATCH, decode_fn=None,
              exact_channel: bool = True, device=None, channel: str = "host",
              precision: str = "fp64", early_stop: bool = True) -> list[BerPoint]:
    """channel.py:83-137 on the GPU, frames sharded over torch.distributed ranks.

    The first eight parameters are the reference's, in its order; ``group_size`` and
    ``decoders_in_flight`` are validated and otherwise unused (the GPU decodes ``batch``
    frames per call instead of pages and decoders in flight).
    decode_fn(Y [b, n], sigma2, max_iterations, counts) must add
    [bit errors, failures, iterations, frames] of the batch into the int64[4]
    tensor ``counts``; the default decodes on this rank's GPU.
    exact_channel=True (default) draws the noise with the reference's scalar math in C on
    host threads (bit-identical BerPoints); False uses numpy's vectorised log/cos/sin
    (statistically identical noise).
    channel="device" (f1) generates the noise and priors on the GPU as well
    (integer-exact RNG streams, device transcendentals: statistical parity).
    precision="fp32" selects the fast mode; early_stop=False runs every frame for max_iterations
    (the reference always stops early).
    """
    if group_size < 1:
        raise ValueError("group_size must be at least 1")
    if decoders_in_flight < 1:
        raise ValueError("decoders_in_flight must be at least 1")
    if channel not in ("host", "device"):
        raise ValueError("channel must be 'host' or 'device'")
    if channel == "device":
        return _ber_sweep_device(H, ebno_points, frames, max_iterations, seed, batch, rate, precision, early_stop)
    import torch

    if frames < 1:
        raise ValueError("frames must be at least 1")
    if batch < 1:
        raise ValueError("batch must be at least 1")
    dist, rank, world = _dist_info()
    R = rate if rate is not None else (H.n - H.m) / H.n
    decoder = None
    if decode_fn is None:
        from .decoder import ParallelDecoder
        from .numa import bind_to_gpu
        from .tables import CodeTables

        bind_to_gpu(torch.cuda.current_device())  # host channel threads and copies near this rank's GPU

        decoder = ParallelDecoder(CodeTables.from_matrix(H), max_batch=batch)
        decode_fn = gpu_decode_counts(decoder, early_stop, precision)
        device = device or torch.device("cuda", torch.cuda.current_device())
    device = device or torch.device("cpu")
    lo, hi = shard_range(frames, rank, world)
    points = []
    try:
        for index, ebno_db in enumerate(ebno_points):
            sigma2 = ebno_to_sigma2(float(ebno_db), R)
            counts = torch.zeros(4, dtype=torch.int64, device=device)
            for b0 in range(lo, hi, batch):
                fr = range(b0, min(hi, b0 + batch))
                if exact_channel:   # the reference's channel bit for bit, native threads
                    Y = transmit_all_zero_frames(H.n, sigma2, seed, index, b0, len(fr))
                else:
                    states = [derive_state(seed, index, f) for f in fr]   # channel.py:112
                    Y = transmit_all_zero_batch(H.n, sigma2, states)
                decode_fn(Y, sigma2, max_iterations, counts)
            if dist is not None:
                dist.all_reduce(counts)                                # the only collective
            c = [int(x) for x in counts.cpu().tolist()]
            assert c[3] == frames, "frame count mismatch after the allreduce"
            points.append(BerPoint(ebno_db=float(ebno_db), sigma2=sigma2, frames=frames, bit_errors=c[0],
                                   ber=c[0] / (frames * H.n), mean_iterations=c[2] / frames, failures=c[1]))
    finally:
        if decoder is not None:
            decoder.close()
    return points


def _ber_sweep_device(H, ebno_points, frames, max_iterations, seed, batch, rate, precision, early_stop=True):
    """f1 path: channel, priors, decode and the error fold all on this rank's GPU."""
    import torch

    from .decoder import ParallelDecoder
    from .tables import CodeTables

    if frames < 1:
        raise ValueError("frames must be at least 1")
    dist, rank, world = _dist_info()
    R = rate if rate is not None else (H.n - H.m) / H.n
    dev = torch.device("cuda", torch.cuda.current_device())
    from .numa import bind_to_gpu

    bind_to_gpu(dev.index)
    lo, hi = shard_range(frames, rank, world)
    points = []
    with ParallelDecoder(CodeTables.from_matrix(H), max_batch=batch) as dec:
        ws = dec.workspace(batch)
        outs = dec.alloc_outputs(batch, dev)
        for index, ebno_db in enumerate(ebno_points):
            sigma2 = ebno_to_sigma2(float(ebno_db), R)
            counts = torch.zeros(4, dtype=torch.int64, device=dev)
            for b0 in range(lo, hi, batch):
                b = min(hi, b0 + batch) - b0
                o = tuple(x[:b] for x in outs)
                dec.decode_channel(seed, index, b0, b, sigma2, max_iterations, early_stop=early_stop, workspace=ws,
                                   outputs=o,
                                   precision=precision)
                dec.count_errors(o, counts)
            if dist is not None:
                dist.all_reduce(counts)
            c = [int(x) for x in counts.cpu().tolist()]
            points.append(BerPoint(ebno_db=float(ebno_db), sigma2=sigma2, frames=frames, bit_errors=c[0],
                                   ber=c[0] / (frames * H.n), mean_iterations=c[2] / frames, failures=c[1]))
    return points


def ber_csv(points: list[BerPoint]) -> str:
    """channel.py:140-148: full-precision (round-trip) floats."""
    lines = ["ebno_db,sigma2,frames,bit_errors,ber,mean_iterations,failures"]
    for pt in points:
        lines.append(f"{pt.ebno_db!r},{pt.sigma2!r},{pt.frames},{pt.bit_errors},"
                     f"{pt.ber!r},{pt.mean_iterations!r},{pt.failures}")
    return "\n".join(lines) + "\n"
