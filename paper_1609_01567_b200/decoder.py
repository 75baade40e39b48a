"""The decoder API of the reference, backed by the B200 kernels.

Reference interface mirrored here (edgeldpc):
  priors_awgn, initialize, MessageState, DecodeResult    serial.py:22-60
  values_to_check / values_to_variable / estimate / syndrome  serial.py:63-147
  decode_awgn                                            serial.py:150-178
  ParallelDecoder(tables, group_size, n_threads).decode  engine.py:220-420
  parallel_decode_awgn                                   engine.py:423-440

Same names, argument meaning and errors (ValueError for sigma2 <= 0, length
mismatches, negative max_iterations, group_size/n_threads < 1; RuntimeError
after close).  Results are bit-identical to the reference on the same inputs.
Added for throughput: ``ParallelDecoder.decode_batch`` (B frames per call,
host buffers, pipelined copies) and ``decode_device`` (device tensors, for
benchmarks and multi-GPU sharding).  ``group_size`` and ``n_threads`` are
accepted for compatibility; the CUDA grid replaces the reference's pages and
worker pool.

Priors are computed on the host with the reference's own numpy expression
(serial.py:49-50): numpy's exp is machine dependent in the last ulp, and bit
parity requires the same priors, so they cross to the device as fp64.
"""

from __future__ import annotations

import ctypes
import os
import threading
import weakref
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass

import numpy as np

from . import _native
from .codes import ParityCheckMatrix
from .tables import CodeTables

DEFAULT_MAX_ITERATIONS = 50   # serial.py:19
DEFAULT_GROUP_SIZE = 512      # engine.py:30


@dataclass
class MessageState:
    """Priors p (per variable) and edge messages q, r (serial.py:22-28)."""

    p: np.ndarray
    q: np.ndarray
    r: np.ndarray


@dataclass
class DecodeResult:
    """serial.py:31-36."""

    estimate: np.ndarray
    success: bool
    iterations_used: int
    syndrome: np.ndarray


def priors_awgn(y, sigma2: float) -> np.ndarray:
    """P(bit = 1) for BPSK over AWGN, serial.py:39-50 (same numpy expression)."""
    if sigma2 <= 0:
        raise ValueError("sigma2 must be positive")
    y = np.asarray(y, dtype=np.float64)
    with np.errstate(over="ignore"):  # exp overflow saturates p to exactly 0.0
        return 1.0 / (1.0 + np.exp(-2.0 * y / sigma2))


_prior_pool = None


def priors_awgn_batch(Y, sigma2, threads: int | None = None, out: np.ndarray | None = None) -> np.ndarray:
    """priors_awgn over a [B, n] batch, rows fanned out over host threads.

    Element-wise identical to calling priors_awgn per frame (numpy's exp does
    not depend on array position; tests/test_host.py pins this).  sigma2 may
    be a scalar or a per-frame [B] array.
    """
    global _prior_pool
    Y = np.ascontiguousarray(Y, dtype=np.float64)
    if Y.ndim != 2:
        raise ValueError("Y must be [B, n]")
    s2 = np.broadcast_to(np.asarray(sigma2, dtype=np.float64), (Y.shape[0],))
    if (s2 <= 0).any():
        raise ValueError("sigma2 must be positive")
    if out is None:
        out = np.empty_like(Y)
    elif out.shape != Y.shape or out.dtype != np.float64 or not out.flags.c_contiguous:
        raise ValueError("out must be a C-contiguous float64 array shaped like Y")
    nt = threads or min(32, os.cpu_count() or 1)
    if nt <= 1 or Y.shape[0] == 1:
        for b in range(Y.shape[0]):
            out[b] = priors_awgn(Y[b], float(s2[b]))
        return out
    if _prior_pool is None:
        _prior_pool = ThreadPoolExecutor(max_workers=nt)

    def work(b):
        with np.errstate(over="ignore"):
            np.divide(1.0, 1.0 + np.exp(-2.0 * Y[b] / float(s2[b])), out=out[b])

    list(_prior_pool.map(work, range(Y.shape[0])))
    return out


def initialize(y, sigma2: float, tables: CodeTables) -> MessageState:
    """serial.py:53-60 (host): q copies each edge's prior, r starts at 1/2."""
    p = priors_awgn(y, sigma2)
    if len(p) != tables.n:
        raise ValueError(f"expected {tables.n} observations, got {len(p)}")
    return MessageState(p, p[tables.variable.v], np.full(tables.total_edges, 0.5))


# ---- device priors (observation input) -------------------------------------------

_exact = {}
_exact_mu = threading.Lock()


def _exp_probe_inputs() -> np.ndarray:
    """Fixed inputs on which candidate float64 exp implementations disagree: ~5% of
    random arguments separate numpy's SVML exp from glibc's, so 2^17 of them (plus
    both special-case regions and the rare path's bounds) leave no doubt."""
    rng = np.random.default_rng(160901567)
    edges = np.array([0.0, -0.0, np.inf, -np.inf, np.nan, 1e-300, -1e-300, 2.0 ** -54, -(2.0 ** -54),
                      709.78, 709.79, 707.70327135170, 707.70327135171, -707.70327135171, -708.39641853226,
                      -708.39641853227, -745.13321910194, -745.13321910195, -740.0, -720.0])
    return np.concatenate([rng.uniform(-40.0, 40.0, 1 << 17), rng.uniform(-746.0, 710.0, 1 << 14),
                           rng.uniform(-746.0, -700.0, 1 << 12), rng.uniform(700.0, 710.0, 1 << 12),
                           rng.normal(0.0, 1e-9, 1 << 10), edges])


def device_priors_exact(device: int = 0) -> bool:
    """Whether the device prior (csrc/priors.cuh) reproduces this host's np.exp bit for bit.

    The reference forms priors with numpy (serial.py:49-50), whose float64 exp is
    machine dependent; the device runs the algorithm numpy uses on AVX512_SKX hosts.
    Checked once per process and device on _exp_probe_inputs(); when it fails the
    decoder forms priors on the host with numpy instead, so results stay identical
    to the reference either way.  LDPC_DEVICE_PRIORS=0 forces host priors.
    """
    if os.environ.get("LDPC_DEVICE_PRIORS", "") == "0":
        return False
    with _exact_mu:
        if device in _exact:
            return _exact[device]
        torch = _torch()
        x = _exp_probe_inputs()
        with np.errstate(all="ignore"):
            want = np.exp(x)
        xd = torch.from_numpy(x).to(f"cuda:{device}")
        out = torch.empty_like(xd)
        with torch.cuda.device(device):
            _native.check(_native.lib().ldpc_npexp(_ptr(xd), x.size, _ptr(out), _native.current_stream_handle(device)),
                          "ldpc_npexp")
        got = out.cpu().numpy()
        same = (got.view(np.uint64) == want.view(np.uint64)) | (np.isnan(got) & np.isnan(want))
        _exact[device] = bool(same.all())
        return _exact[device]


# ---- device plumbing ----------------------------------------------------------

def _torch():
    import torch

    return torch


def _workspace(graph, B: int):
    torch = _torch()
    nbytes = int(_native.lib().ldpc_workspace_bytes(graph.handle, int(B)))
    return torch.empty(nbytes, dtype=torch.uint8, device=f"cuda:{graph.device}"), nbytes


def _ptr(t) -> ctypes.c_void_p:
    return ctypes.c_void_p(t.data_ptr())


def _tables_of(obj) -> CodeTables:
    if isinstance(obj, CodeTables):
        return obj
    if isinstance(obj, ParityCheckMatrix):
        # device tables of a matrix passed where the reference takes H (syndrome, decode_awgn),
        # kept while the matrix lives
        tables = _H_TABLES.get(obj)
        if tables is None:
            tables = CodeTables.from_matrix(obj)
            _H_TABLES[obj] = tables
        return tables
    raise TypeError("expected CodeTables or ParityCheckMatrix")


class _IdentityKeyed(dict):
    """id(matrix) -> tables, dropped when the matrix is collected."""

    def get(self, obj, default=None):
        return super().get(id(obj), default)

    def __setitem__(self, obj, tables):
        key = id(obj)
        super().__setitem__(key, tables)
        weakref.finalize(obj, self.pop, key, None)


_H_TABLES = _IdentityKeyed()


def _as_batch(a, width: int, what: str) -> tuple[np.ndarray, bool]:
    a = np.asarray(a, dtype=np.float64)
    single = a.ndim == 1
    a2 = a.reshape(1, -1) if single else a
    if a2.ndim != 2 or a2.shape[1] != width:
        raise ValueError(f"expected {width} {what}, got {a.shape[-1] if a.ndim else 0}")
    return np.ascontiguousarray(a2), single


def _dev(a: np.ndarray, device: int):
    return _torch().from_numpy(a).to(f"cuda:{device}")


# ---- single phases (serial.py:63-147 signatures, any batch) -------------------

SCHEDULES = ("auto", "stream", "onchip", "grid")


def _flags(early_stop: bool, precision: str, schedule: str = "auto") -> int:
    """schedule: "auto" decodes small codes entirely on chip (one CTA or thread-block cluster per
    codeword, onchip.cu), a few codewords of larger codes in one cooperative launch (grid.cu), and
    streams the rest; "stream" / "onchip" / "grid" force one (identical results)."""
    if precision not in ("fp64", "fp32"):
        raise ValueError("precision must be 'fp64' (exact) or 'fp32' (fast mode)")
    if schedule not in SCHEDULES:
        raise ValueError(f"schedule must be one of {SCHEDULES}")
    return ((_native.FLAG_EARLY_STOP if early_stop else _native.FLAG_FIXED_ITERS)
            | (_native.FLAG_FP32 if precision == "fp32" else 0)
            | (_native.FLAG_STREAMING if schedule == "stream" else 0)
            | (_native.FLAG_ONCHIP if schedule == "onchip" else 0)
            | (_native.FLAG_GRID if schedule == "grid" else 0))


def values_to_check(p, r, tables: CodeTables, precision: str = "fp64") -> np.ndarray:
    """V-phase (serial.py:63-89) on the GPU; p [n] or [B,n], r [E] or [B,E] canonical order.

    precision="fp32" runs the fast-mode kernel (not bit-exact; DESIGN.md states the tolerance)."""
    T = _tables_of(tables)
    P, single = _as_batch(p, T.n, "priors")
    R, _ = _as_batch(r, T.total_edges, "messages")
    if P.shape[0] != R.shape[0]:
        raise ValueError("batch mismatch between p and r")
    _flags(True, precision)
    B = P.shape[0]
    g = T.graph
    torch = _torch()
    ws, nb = _workspace(g, B)
    dp, dr = _dev(P, g.device), _dev(R, g.device)
    dq = torch.empty_like(dr)
    if precision == "fp32":
        rc = _native.lib().ldpc_phase_f32(g.handle, 0, _ptr(dp), _ptr(dr), _ptr(dq), B, _ptr(ws), nb,
                                          _native.current_stream_handle(g.device))
    else:
        rc = _native.lib().ldpc_phase_to_check(g.handle, _ptr(dp), _ptr(dr), _ptr(dq), B, _ptr(ws), nb,
                                               _native.current_stream_handle(g.device))
    _native.check(rc, "values_to_check")
    q = dq.cpu().numpy()
    return q[0] if single else q


def values_to_variable(q, tables: CodeTables, precision: str = "fp64") -> np.ndarray:
    """C-phase (serial.py:92-112) on the GPU; q [E] or [B,E] canonical order (precision as values_to_check)."""
    T = _tables_of(tables)
    Q, single = _as_batch(q, T.total_edges, "messages")
    _flags(True, precision)
    B = Q.shape[0]
    g = T.graph
    torch = _torch()
    ws, nb = _workspace(g, B)
    dq = _dev(Q, g.device)
    dr = torch.empty_like(dq)
    if precision == "fp32":
        rc = _native.lib().ldpc_phase_f32(g.handle, 1, None, _ptr(dq), _ptr(dr), B, _ptr(ws), nb,
                                          _native.current_stream_handle(g.device))
    else:
        rc = _native.lib().ldpc_phase_to_variable(g.handle, _ptr(dq), _ptr(dr), B, _ptr(ws), nb,
                                                  _native.current_stream_handle(g.device))
    _native.check(rc, "values_to_variable")
    r = dr.cpu().numpy()
    return r[0] if single else r


def estimate(p, r, tables: CodeTables) -> np.ndarray:
    """Hard decision (serial.py:115-133) on the GPU."""
    T = _tables_of(tables)
    P, single = _as_batch(p, T.n, "priors")
    R, _ = _as_batch(r, T.total_edges, "messages")
    B = P.shape[0]
    g = T.graph
    torch = _torch()
    ws, nb = _workspace(g, B)
    dp, dr = _dev(P, g.device), _dev(R, g.device)
    dc = torch.empty((B, T.n), dtype=torch.uint8, device=dp.device)
    _native.check(_native.lib().ldpc_phase_estimate(g.handle, _ptr(dp), _ptr(dr), _ptr(dc), B, _ptr(ws), nb,
                                                    _native.current_stream_handle(g.device)), "estimate")
    c = dc.cpu().numpy()
    return c[0] if single else c


def syndrome(c_hat, H) -> np.ndarray:
    """z = H c_hat mod 2 (serial.py:136-147) on the GPU; H may be a ParityCheckMatrix or CodeTables."""
    T = _tables_of(H)
    c = np.asarray(c_hat)
    single = c.ndim == 1
    c2 = (c.reshape(1, -1) if single else c)
    if c2.shape[-1] != T.n:
        raise ValueError(f"estimate length {c2.shape[-1]} does not match n={T.n}")
    c2 = np.ascontiguousarray(c2.astype(np.int64) & 1, dtype=np.uint8)
    B = c2.shape[0]
    g = T.graph
    torch = _torch()
    ws, nb = _workspace(g, B)
    dc = _dev(c2, g.device)
    dz = torch.empty((B, T.m), dtype=torch.uint8, device=dc.device)
    _native.check(_native.lib().ldpc_phase_syndrome(g.handle, _ptr(dc), _ptr(dz), B, _ptr(ws), nb,
                                                    _native.current_stream_handle(g.device)), "syndrome")
    z = dz.cpu().numpy()
    return z[0] if single else z


# ---- batch results -------------------------------------------------------------

def unpack_bits(words: np.ndarray, width: int) -> np.ndarray:
    """[B, ceil(width/32)] uint32 little-bit-order rows -> [B, width] uint8."""
    w = np.ascontiguousarray(words, dtype=np.uint32)
    return np.unpackbits(w.view(np.uint8), axis=-1, bitorder="little")[..., :width]


class BatchResult:
    """Results of B frames: packed estimate/syndrome bits, flags and counts."""

    def __init__(self, est_bits, success, iterations, syn_bits, n: int, m: int):
        self.est_bits = est_bits
        self.success = success
        self.iterations = iterations
        self.syn_bits = syn_bits
        self.n, self.m = n, m

    def __len__(self) -> int:
        return len(self.success)

    def estimates(self) -> np.ndarray:
        return unpack_bits(self.est_bits, self.n)

    def syndromes(self) -> np.ndarray:
        return unpack_bits(self.syn_bits, self.m)

    def __getitem__(self, i: int) -> DecodeResult:
        return DecodeResult(unpack_bits(self.est_bits[i:i + 1], self.n)[0], bool(self.success[i]),
                            int(self.iterations[i]), unpack_bits(self.syn_bits[i:i + 1], self.m)[0])


# ---- the decoder ----------------------------------------------------------------

# ---- engine.py's page plan and shared-state phase API (engine.py:33-76, 157-190) ------------
# The reference sweeps pages of `group_size` lanes with worker threads; here the CUDA grid
# replaces the pages, so the plan is kept for API compatibility (results do not depend on it,
# in the reference either) and the parallel_* entry points run the GPU phase kernels on the
# state's arrays, writing their outputs in place like the reference.

@dataclass(frozen=True)
class PagePlan:
    """engine.py:33-47: split of total_edges lanes into pages of at most group_size."""

    total_edges: int
    group_size: int
    page_starts: tuple

    @property
    def page_count(self) -> int:
        return len(self.page_starts)

    def page_width(self, page: int) -> int:
        """Active lanes in a page; trailing lanes of the last page idle."""
        return min(self.group_size, self.total_edges - self.page_starts[page])


def plan_pages(total_edges: int, group_size: int) -> PagePlan:
    """engine.py:50-55, same errors."""
    if group_size < 1:
        raise ValueError("group_size must be at least 1")
    if total_edges < 1:
        raise ValueError("total_edges must be at least 1")
    return PagePlan(total_edges, group_size, tuple(range(0, total_edges, group_size)))


@dataclass
class SharedDecodeState:
    """engine.py:58-76: the arrays one decode works on (host numpy, updated in place)."""

    p: np.ndarray          # n priors
    q: np.ndarray          # E variable-to-check messages
    r: np.ndarray          # E check-to-variable messages
    estimate: np.ndarray   # n hard bits
    syndrome: np.ndarray   # m parity bits

    @classmethod
    def allocate(cls, tables) -> "SharedDecodeState":
        T = _tables_of(tables)
        return cls(p=np.zeros(T.n), q=np.zeros(T.total_edges), r=np.full(T.total_edges, 0.5),
                   estimate=np.zeros(T.n, dtype=np.uint8), syndrome=np.zeros(T.m, dtype=np.uint8))


def parallel_to_check(state: SharedDecodeState, tables, plan: PagePlan | None = None) -> None:
    """engine.py:157-163: variable-to-check update on the GPU; writes state.q."""
    state.q[...] = values_to_check(state.p, state.r, tables)


def parallel_to_variable(state: SharedDecodeState, tables, plan: PagePlan | None = None) -> None:
    """engine.py:166-172: check-to-variable update on the GPU; writes state.r."""
    state.r[...] = values_to_variable(state.q, tables)


def parallel_estimate(state: SharedDecodeState, tables, plan: PagePlan | None = None) -> None:
    """engine.py:175-181: hard decision on the GPU; writes state.estimate."""
    state.estimate[...] = estimate(state.p, state.r, tables)


def parallel_syndrome(state: SharedDecodeState, tables, plan: PagePlan | None = None) -> None:
    """engine.py:184-190: syndrome on the GPU; writes state.syndrome."""
    state.syndrome[...] = syndrome(state.estimate, tables)


class PendingDecode:
    """One in-flight ParallelDecoder.decode_priors_async batch; keeps its host buffers alive."""

    def __init__(self, decoder, ticket: int, P, result: BatchResult):
        self._decoder, self._ticket, self._P, self._result = decoder, ticket, P, result
        self._done = False

    def wait(self) -> BatchResult:
        if not self._done:
            self._decoder._wait(self._ticket)
            self._done = True
            self._P = None
        return self._result


class ParallelDecoder:
    """GPU drop-in for edgeldpc.engine.ParallelDecoder (engine.py:220-420).

    One instance owns a device decode context for up to ``max_batch`` frames
    (pipelined host<->device copies over two streams).  Reentrant use from
    several threads is serialised by the native context (engine.py:223-226
    allows concurrent decode calls on one n_threads == 1 instance).
    """

    def __init__(self, tables, group_size: int = DEFAULT_GROUP_SIZE, n_threads: int = 1, *,
                 max_batch: int = 1024, sub_batch: int = 0):
        if group_size < 1:
            raise ValueError("group_size must be at least 1")      # engine.py:51-52
        if n_threads < 1:
            raise ValueError("n_threads must be at least 1")       # engine.py:234-235
        if max_batch < 1:
            raise ValueError("max_batch must be at least 1")
        self.tables = _tables_of(tables)
        self.group_size = group_size
        self.n_threads = n_threads
        self.max_batch = int(max_batch)
        L = _native.lib()
        h = ctypes.c_void_p()
        _native.check(L.ldpc_decoder_create(self.tables.graph.handle, self.max_batch, int(sub_batch),
                                            ctypes.byref(h)), "ldpc_decoder_create")
        self._h = h
        self._closed = False
        self._pinned = None
        self._lock = threading.RLock()

    # engine.py:363-398
    def decode(self, y, sigma2: float, max_iterations: int = DEFAULT_MAX_ITERATIONS) -> DecodeResult:
        if self._closed:
            raise RuntimeError("decoder is closed")
        if max_iterations < 0:
            raise ValueError("max_iterations must be non-negative")
        if device_priors_exact(self.tables.graph.device):
            if sigma2 <= 0:
                raise ValueError("sigma2 must be positive")
            y = np.ascontiguousarray(y, dtype=np.float64)
            if y.ndim != 1 or len(y) != self.tables.n:
                raise ValueError(f"expected {self.tables.n} observations, got {len(y)}")
            return self._run(y.reshape(1, -1), np.full(1, float(sigma2)), max_iterations, True, None, "fp64",
                             "auto")[0]
        p = priors_awgn(y, sigma2)
        if p.ndim != 1 or len(p) != self.tables.n:
            raise ValueError(f"expected {self.tables.n} observations, got {len(p)}")
        return self.decode_priors(p.reshape(1, -1), max_iterations)[0]

    def decode_batch(self, Y, sigma2, max_iterations: int = DEFAULT_MAX_ITERATIONS,
                     early_stop: bool = True, precision: str = "fp64", schedule: str = "auto",
                     out: BatchResult | None = None) -> BatchResult:
        """B received frames [B, n] (sigma2 scalar or [B]) -> BatchResult (into ``out`` if given)."""
        if self._closed:
            raise RuntimeError("decoder is closed")
        Y = np.asarray(Y, dtype=np.float64)
        if Y.ndim != 2 or Y.shape[1] != self.tables.n:
            raise ValueError(f"expected frames of {self.tables.n} observations")
        B, n, m = Y.shape[0], self.tables.n, self.tables.m
        s2 = np.broadcast_to(np.asarray(sigma2, dtype=np.float64), (B,))
        if device_priors_exact(self.tables.graph.device):
            # observations go to the device as they are; the priors are formed there (priors.cuh),
            # bit-identical to numpy's.  Pinned Y (torch pin_memory) copies at full speed.
            if (s2 <= 0).any():
                raise ValueError("sigma2 must be positive")
            return self._run(np.ascontiguousarray(Y), np.ascontiguousarray(s2), max_iterations, early_stop, out,
                             precision, schedule)
        res = out if out is not None else BatchResult(np.empty((B, (n + 31) // 32), np.uint32), np.empty(B, np.uint8), np.empty(B, np.int32),
                          np.empty((B, (m + 31) // 32), np.uint32), n, m)
        # priors go into a reused pinned buffer (no page faults, full-speed copies), max_batch frames at a
        # time; the buffer is shared by the instance, so concurrent calls hold the (reentrant) lock across
        # forming the priors and decoding them
        with self._lock:
            buf = self._pinned_priors()
            for c0 in range(0, B, self.max_batch):
                c1 = min(B, c0 + self.max_batch)
                P = priors_awgn_batch(Y[c0:c1], s2[c0:c1], out=buf[:c1 - c0])
                self.decode_priors(P, max_iterations, early_stop, precision=precision, schedule=schedule,
                                   out=BatchResult(res.est_bits[c0:c1], res.success[c0:c1], res.iterations[c0:c1],
                                                   res.syn_bits[c0:c1], n, m))
        return res

    def _pinned_priors(self) -> np.ndarray:
        """The instance's pinned [max_batch, n] priors buffer (caller holds self._lock)."""
        if self._pinned is None:
            torch = _torch()
            self._pinned = torch.empty((self.max_batch, self.tables.n), dtype=torch.float64).pin_memory().numpy()
        return self._pinned

    def decode_priors(self, P, max_iterations: int = DEFAULT_MAX_ITERATIONS, early_stop: bool = True,
                      out: BatchResult | None = None, precision: str = "fp64", schedule: str = "auto") -> BatchResult:
        """Host priors [B, n] -> host BatchResult.  Pinned buffers (torch ``pin_memory()``) are copied
        directly; plain numpy arrays are staged through the decoder's pinned slots by host copy threads
        (about 0.9 of the pinned rate at C3).

        precision="fp32": fast mode, same algorithm in fp32 (not bit-exact; DESIGN.md tolerance)."""
        if self._closed:
            raise RuntimeError("decoder is closed")
        if max_iterations < 0:
            raise ValueError("max_iterations must be non-negative")
        P = np.ascontiguousarray(P, dtype=np.float64)
        if P.ndim != 2 or P.shape[1] != self.tables.n:
            raise ValueError(f"expected priors of shape [B, {self.tables.n}]")
        return self._run(P, None, max_iterations, early_stop, out, precision, schedule)

    def _run(self, P, s2, max_iterations, early_stop, out, precision, schedule) -> BatchResult:
        """Host [B, n] priors (s2 None) or observations with per-frame sigma2 [B] -> BatchResult."""
        B = P.shape[0]
        n, m = self.tables.n, self.tables.m
        res = out if out is not None else BatchResult(np.empty((B, (n + 31) // 32), np.uint32),
                                                      np.empty(B, np.uint8), np.empty(B, np.int32),
                                                      np.empty((B, (m + 31) // 32), np.uint32), n, m)
        L = _native.lib()
        flags = _flags(early_stop, precision, schedule)
        if B > self.max_batch:
            # several chunks: two in flight through the streaming slots, so the copy of chunk k+1
            # overlaps the decode of chunk k (results identical to the per-chunk synchronous call)
            pending = []
            for c0 in range(0, B, self.max_batch):
                c1 = min(B, c0 + self.max_batch)
                view = BatchResult(res.est_bits[c0:c1], res.success[c0:c1], res.iterations[c0:c1],
                                   res.syn_bits[c0:c1], n, m)
                pending.append(self._submit(P[c0:c1], None if s2 is None else s2[c0:c1], max_iterations,
                                            early_stop, view, precision, schedule))
                if len(pending) == 2:
                    pending.pop(0).wait()
            for job in pending:
                job.wait()
            return res
        with self._lock:
            outs = (res.est_bits.ctypes.data, res.success.ctypes.data, res.iterations.ctypes.data,
                    res.syn_bits.ctypes.data)
            if s2 is None:
                rc = L.ldpc_decoder_decode_host(self._h, P.ctypes.data, B, int(max_iterations), flags, *outs)
            else:
                rc = L.ldpc_decoder_decode_awgn_host(self._h, P.ctypes.data, s2.ctypes.data, B, int(max_iterations),
                                                     flags, *outs)
            if rc == _native.LDPC_ECUDA or rc == _native.LDPC_ECLOSED:
                self._closed = True   # engine.py:389-392: poisoned after a device fault
            _native.check(rc, "decode")
        return res

    def decode_priors_async(self, P, max_iterations: int = DEFAULT_MAX_ITERATIONS, early_stop: bool = True,
                            out: BatchResult | None = None, precision: str = "fp64",
                            schedule: str = "auto") -> "PendingDecode":
        """Streaming variant of decode_priors (no reference counterpart): enqueue the H2D copy,
        the decode and the D2H copy of one batch (B <= max_batch) and return at once; call
        ``.wait()`` on the result for the BatchResult.  Two batches can be in flight, so the
        copy of batch k+1 overlaps the decode of batch k.  Results equal decode_priors'.
        ``P`` and ``out`` should be pinned (torch ``pin_memory()``) for asynchronous copies."""
        if self._closed:
            raise RuntimeError("decoder is closed")
        if max_iterations < 0:
            raise ValueError("max_iterations must be non-negative")
        P = np.ascontiguousarray(P, dtype=np.float64)
        if P.ndim != 2 or P.shape[1] != self.tables.n:
            raise ValueError(f"expected priors of shape [B, {self.tables.n}]")
        return self._submit(P, None, max_iterations, early_stop, out, precision, schedule)

    def decode_batch_async(self, Y, sigma2, max_iterations: int = DEFAULT_MAX_ITERATIONS, early_stop: bool = True,
                           out: BatchResult | None = None, precision: str = "fp64",
                           schedule: str = "auto") -> "PendingDecode":
        """Streaming variant of decode_batch: observations [B, n] (B <= max_batch, pinned for
        asynchronous copies) in, priors formed on the device.  Needs device_priors_exact()."""
        if self._closed:
            raise RuntimeError("decoder is closed")
        if not device_priors_exact(self.tables.graph.device):
            raise RuntimeError("this host's np.exp differs from the device prior; use decode_priors_async")
        if max_iterations < 0:
            raise ValueError("max_iterations must be non-negative")
        Y = np.ascontiguousarray(Y, dtype=np.float64)
        if Y.ndim != 2 or Y.shape[1] != self.tables.n:
            raise ValueError(f"expected frames of {self.tables.n} observations")
        s2 = np.ascontiguousarray(np.broadcast_to(np.asarray(sigma2, dtype=np.float64), (Y.shape[0],)))
        if (s2 <= 0).any():
            raise ValueError("sigma2 must be positive")
        return self._submit(Y, s2, max_iterations, early_stop, out, precision, schedule)

    def _submit(self, P, s2, max_iterations, early_stop, out, precision, schedule) -> "PendingDecode":
        B = P.shape[0]
        if not 1 <= B <= self.max_batch:
            raise ValueError(f"batch {B} outside 1..{self.max_batch}")
        n, m = self.tables.n, self.tables.m
        res = out if out is not None else BatchResult(np.empty((B, (n + 31) // 32), np.uint32),
                                                      np.empty(B, np.uint8), np.empty(B, np.int32),
                                                      np.empty((B, (m + 31) // 32), np.uint32), n, m)
        ticket = ctypes.c_int64(-1)
        L = _native.lib()
        flags = _flags(early_stop, precision, schedule)
        outs = (res.est_bits.ctypes.data, res.success.ctypes.data, res.iterations.ctypes.data,
                res.syn_bits.ctypes.data, ctypes.byref(ticket))
        with self._lock:
            if s2 is None:
                rc = L.ldpc_decoder_submit(self._h, P.ctypes.data, B, int(max_iterations), flags, *outs)
            else:
                rc = L.ldpc_decoder_submit_awgn(self._h, P.ctypes.data, s2.ctypes.data, B, int(max_iterations),
                                                flags, *outs)
            if rc == _native.LDPC_ECUDA or rc == _native.LDPC_ECLOSED:
                self._closed = True
            _native.check(rc, "decode")
        return PendingDecode(self, ticket.value, (P, s2), res)

    def decode_stream(self, batches, max_iterations: int = DEFAULT_MAX_ITERATIONS, early_stop: bool = True,
                      precision: str = "fp64"):
        """Yield a BatchResult per host priors batch of ``batches``, keeping two batches in flight."""
        pending = []
        for P in batches:
            pending.append(self.decode_priors_async(P, max_iterations, early_stop, precision=precision))
            if len(pending) == 2:
                yield pending.pop(0).wait()
        while pending:
            yield pending.pop(0).wait()

    def _wait(self, ticket: int) -> None:
        with self._lock:
            if self._h is None:
                raise RuntimeError("decoder is closed")
            rc = _native.lib().ldpc_decoder_wait(self._h, int(ticket))
            if rc == _native.LDPC_ECUDA or rc == _native.LDPC_ECLOSED:
                self._closed = True
            _native.check(rc, "decode")

    def decode_device(self, P_dev, max_iterations: int, early_stop: bool = True, workspace=None,
                      outputs=None, profile: "_native.Profile | None" = None, syndrome_out: bool = True,
                      precision: str = "fp64", schedule: str = "auto"):
        """Device priors tensor [B, n] fp64 -> device tensors (est_bits, success, iters, syn_bits).

        Stream-ordered on torch's current stream; no host synchronisation
        unless ``profile`` is given (event timings are resolved at the end).
        """
        if self._closed:
            raise RuntimeError("decoder is closed")
        torch = _torch()
        g = self.tables.graph
        B = int(P_dev.shape[0])
        if P_dev.dtype != torch.float64 or P_dev.dim() != 2 or P_dev.shape[1] != g.n or not P_dev.is_contiguous():
            raise ValueError("P_dev must be a contiguous float64 [B, n] CUDA tensor")
        if workspace is None:
            workspace, nb = _workspace(g, B)
        else:
            nb = workspace.numel()
        if outputs is None:
            outputs = self.alloc_outputs(B, P_dev.device)
        est, ok, its, syn = outputs
        flags = _flags(early_stop, precision, schedule)
        rc = _native.lib().ldpc_decode(g.handle, _ptr(P_dev), B, int(max_iterations), flags, _ptr(est), _ptr(ok),
                                       _ptr(its), _ptr(syn) if syndrome_out else None, _ptr(workspace), nb,
                                       _native.current_stream_handle(g.device),
                                       ctypes.byref(profile) if profile is not None else None)
        _native.check(rc, "ldpc_decode")
        return outputs

    def decode_device_awgn(self, Y_dev, sigma2_dev, max_iterations: int, early_stop: bool = True, workspace=None,
                           outputs=None, syndrome_out: bool = True, precision: str = "fp64",
                           schedule: str = "auto"):
        """Device observations [B, n] fp64 + sigma2 [B] fp64 -> device outputs; the priors are
        formed on the device (priors.cuh; bit-identical to numpy's on AVX512_SKX hosts)."""
        if self._closed:
            raise RuntimeError("decoder is closed")
        torch = _torch()
        g = self.tables.graph
        B = int(Y_dev.shape[0])
        if Y_dev.dtype != torch.float64 or Y_dev.dim() != 2 or Y_dev.shape[1] != g.n or not Y_dev.is_contiguous():
            raise ValueError("Y_dev must be a contiguous float64 [B, n] CUDA tensor")
        if sigma2_dev.dtype != torch.float64 or sigma2_dev.numel() != B or not sigma2_dev.is_contiguous():
            raise ValueError("sigma2_dev must be a contiguous float64 [B] CUDA tensor")
        if workspace is None:
            workspace, nb = _workspace(g, B)
        else:
            nb = workspace.numel()
        if outputs is None:
            outputs = self.alloc_outputs(B, Y_dev.device)
        est, ok, its, syn = outputs
        rc = _native.lib().ldpc_decode_awgn(g.handle, _ptr(Y_dev), _ptr(sigma2_dev), B, int(max_iterations),
                                            _flags(early_stop, precision, schedule), _ptr(est), _ptr(ok), _ptr(its),
                                            _ptr(syn) if syndrome_out else None, _ptr(workspace), nb,
                                            _native.current_stream_handle(g.device), None)
        _native.check(rc, "ldpc_decode_awgn")
        return outputs

    def decode_channel(self, seed: int, point: int, frame0: int, B: int, sigma2: float, max_iterations: int,
                       early_stop: bool = True, workspace=None, outputs=None, precision: str = "fp64"):
        """f1: frames frame0..frame0+B-1 of Eb/N0 point `point` generated on the device (all-zero
        codeword over AWGN, the reference's per-frame xorshift128+ streams) and decoded; device outputs."""
        if self._closed:
            raise RuntimeError("decoder is closed")
        if sigma2 <= 0:
            raise ValueError("sigma2 must be positive")
        g = self.tables.graph
        torch = _torch()
        if workspace is None:
            workspace, nb = _workspace(g, B)
        else:
            nb = workspace.numel()
        if outputs is None:
            outputs = self.alloc_outputs(B, torch.device("cuda", g.device))
        est, ok, its, syn = outputs
        rc = _native.lib().ldpc_decode_channel(g.handle, int(seed) & (2**64 - 1), int(point), int(frame0), int(B),
                                               float(sigma2), int(max_iterations), _flags(early_stop, precision),
                                               _ptr(est), _ptr(ok), _ptr(its), None, _ptr(workspace), nb,
                                               _native.current_stream_handle(g.device))
        _native.check(rc, "ldpc_decode_channel")
        return outputs

    def alloc_outputs(self, B: int, device):
        torch = _torch()
        n, m = self.tables.n, self.tables.m
        return (torch.empty((B, (n + 31) // 32), dtype=torch.int32, device=device),
                torch.empty(B, dtype=torch.uint8, device=device),
                torch.empty(B, dtype=torch.int32, device=device),
                torch.empty((B, (m + 31) // 32), dtype=torch.int32, device=device))

    def workspace(self, B: int):
        return _workspace(self.tables.graph, B)[0]

    def count_errors(self, outputs, counts_dev):
        """Accumulate [bit errors, failures, iterations, frames] (all-zero codeword) into int64[4]."""
        est, ok, its, _ = outputs
        rc = _native.lib().ldpc_count_errors(self.tables.graph.handle, _ptr(est), _ptr(ok), _ptr(its),
                                             int(ok.shape[0]), _ptr(counts_dev),
                                             _native.current_stream_handle(self.tables.graph.device))
        _native.check(rc, "ldpc_count_errors")

    # engine.py:400-420
    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            _native.load_library().ldpc_decoder_destroy(self._h)
            self._h = None
        self._closed = True

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


GpuDecoder = ParallelDecoder


def decode_awgn(y, sigma2: float, max_iterations: int, tables, H: ParityCheckMatrix | None = None) -> DecodeResult:
    """serial.py:150-178 signature, decoded on the GPU."""
    if max_iterations < 0:
        raise ValueError("max_iterations must be non-negative")
    T = _tables_of(tables)
    if H is not None and (H.n != T.n or H.m != T.m):
        raise ValueError("H does not match the tables")
    with ParallelDecoder(T, max_batch=1) as dec:
        return dec.decode(y, sigma2, max_iterations)


def parallel_decode_awgn(y, sigma2: float, max_iterations: int, tables, H: ParityCheckMatrix | None = None,
                         group_size: int = DEFAULT_GROUP_SIZE, n_threads: int = 1) -> DecodeResult:
    """engine.py:423-440: one-shot decode through a throwaway decoder."""
    T = _tables_of(tables)
    if H is not None and (H.n != T.n or H.m != T.m):
        raise ValueError("H does not match the tables")
    with ParallelDecoder(T, group_size=group_size, n_threads=n_threads, max_batch=1) as dec:
        return dec.decode(y, sigma2, max_iterations)
