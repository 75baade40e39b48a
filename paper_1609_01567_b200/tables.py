"""Edge tables, built on the device (north_star kernel 1).

Mirrors the reference's table layer (edgeldpc/tables.py:33-121): the six
address-iterator arrays e, v, c, t, s, u in variable and check orientation,
``CodeTables.from_matrix`` and the per-variable CSR (var_group_start/size).
Construction runs the G1 builder in libldpc_b200.so (device sort of unique
edge keys, CSR scan, slot mapping, degree buckets); the host arrays of the
reference interface are exported lazily from the device graph.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _native
from .codes import ParityCheckMatrix

VARIABLE = "variable"
CHECK = "check"


@dataclass(frozen=True)
class EdgeTables:
    """One orientation of the six per-edge iterator arrays (tables.py:33-47)."""

    orientation: str
    e: np.ndarray
    v: np.ndarray
    c: np.ndarray
    t: np.ndarray
    s: np.ndarray
    u: np.ndarray

    @property
    def total_edges(self) -> int:
        return len(self.e)


class DeviceGraph:
    """Owner of one ldpc_graph handle (immutable, shareable across threads)."""

    def __init__(self, H: ParityCheckMatrix):
        L = _native.lib()
        rows = np.ascontiguousarray(H.rows, dtype=np.int32)
        cols = np.ascontiguousarray(H.cols, dtype=np.int32)
        h = ctypes.c_void_p()
        rc = L.ldpc_graph_create(H.n, H.m, len(rows), rows.ctypes.data_as(_native.P_i32),
                                 cols.ctypes.data_as(_native.P_i32), _native.current_stream_handle(),
                                 ctypes.byref(h))
        _native.check(rc, "ldpc_graph_create")
        self.handle = h
        info = np.zeros(8, dtype=np.int64)
        _native.check(L.ldpc_graph_info(h, info.ctypes.data_as(_native.P_i64)))
        self.n, self.m, self.E, self.max_dv, self.max_dc = (int(x) for x in info[:5])
        self.device = int(info[7])

    def buckets(self, side: str) -> list[tuple[int, int]]:
        L = _native.lib()
        sd = _native.VARIABLE if side == VARIABLE else _native.CHECK
        cnt = L.ldpc_graph_get_buckets(self.handle, sd, None, None, 0)
        deg = np.zeros(max(cnt, 1), dtype=np.int32)
        num = np.zeros(max(cnt, 1), dtype=np.int32)
        L.ldpc_graph_get_buckets(self.handle, sd, deg.ctypes.data_as(_native.P_i32),
                                 num.ctypes.data_as(_native.P_i32), cnt)
        return list(zip(deg[:cnt].tolist(), num[:cnt].tolist()))

    def export(self, orientation: str) -> EdgeTables:
        L = _native.lib()
        arrs = [np.empty(self.E, dtype=np.int64) for _ in range(6)]
        rc = L.ldpc_graph_get_tables(self.handle, _native.VARIABLE if orientation == VARIABLE else _native.CHECK,
                                     *[a.ctypes.data_as(_native.P_i64) for a in arrs])
        _native.check(rc, "ldpc_graph_get_tables")
        return EdgeTables(orientation, *arrs)

    def var_groups(self) -> tuple[np.ndarray, np.ndarray]:
        L = _native.lib()
        st = np.empty(self.n, dtype=np.int64)
        sz = np.empty(self.n, dtype=np.int64)
        _native.check(L.ldpc_graph_get_var_groups(self.handle, st.ctypes.data_as(_native.P_i64),
                                                  sz.ctypes.data_as(_native.P_i64)))
        return st, sz

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            try:
                _native.load_library().ldpc_graph_destroy(h)
            except Exception:
                pass
            self.handle = None


class CodeTables:
    """Both orientations plus node/edge counts (tables.py:95-116), device-resident.

    Constructible like the reference's frozen dataclass from its seven fields
    ``CodeTables(variable, check, n, m, total_edges, var_group_start,
    var_group_size)``; the device graph is then built on first use from the
    variable-oriented (c, v) pairs.  ``from_matrix`` builds the device graph
    first (G1 builder) and exports the reference's host arrays lazily.
    Immutable: attribute assignment raises, like the reference's.
    """

    def __init__(self, variable: EdgeTables, check: EdgeTables, n: int, m: int, total_edges: int,
                 var_group_start: np.ndarray, var_group_size: np.ndarray):
        if variable.orientation != VARIABLE or check.orientation != CHECK:
            raise ValueError("expected variable- and check-oriented edge tables")
        self._set(_graph=None, _var=variable, _chk=check, _groups=(var_group_start, var_group_size),
                  n=int(n), m=int(m), total_edges=int(total_edges))

    def _set(self, **kw):
        for k, v in kw.items():
            object.__setattr__(self, k, v)

    def __setattr__(self, name, value):
        raise AttributeError(f"cannot assign to field {name!r}: CodeTables is immutable")

    @classmethod
    def _of_graph(cls, graph: DeviceGraph) -> "CodeTables":
        self = cls.__new__(cls)
        self._set(_graph=graph, _var=None, _chk=None, _groups=None, n=graph.n, m=graph.m, total_edges=graph.E)
        return self

    @classmethod
    def from_matrix(cls, H: ParityCheckMatrix) -> "CodeTables":
        # no back-reference to H: a matrix-keyed cache of tables must not keep its key alive
        return cls._of_graph(DeviceGraph(H))

    @property
    def graph(self) -> DeviceGraph:
        """The device graph (G1), built from the variable tables' (c, v) pairs when the tables
        were constructed field by field."""
        if self._graph is None:
            v = self._var
            H = ParityCheckMatrix(self.n, self.m, np.stack([np.asarray(v.c), np.asarray(v.v)], axis=1))
            if H.total_edges != self.total_edges:
                raise ValueError("total_edges does not match the edge tables")
            self._set(_graph=DeviceGraph(H))
        return self._graph

    @property
    def variable(self) -> EdgeTables:
        if self._var is None:
            self._set(_var=self._graph.export(VARIABLE))
        return self._var

    @property
    def check(self) -> EdgeTables:
        if self._chk is None:
            self._set(_chk=self._graph.export(CHECK))
        return self._chk

    @property
    def var_group_start(self) -> np.ndarray:
        if self._groups is None:
            self._set(_groups=self._graph.var_groups())
        return self._groups[0]

    @property
    def var_group_size(self) -> np.ndarray:
        if self._groups is None:
            self._set(_groups=self._graph.var_groups())
        return self._groups[1]

    def buckets(self, side: str = VARIABLE) -> list[tuple[int, int]]:
        """Degree buckets [(degree, node count)] of one side, ascending degree."""
        return self.graph.buckets(side)

    def __repr__(self) -> str:
        return f"CodeTables(n={self.n}, m={self.m}, total_edges={self.total_edges})"


def build_variable_tables(H: ParityCheckMatrix) -> EdgeTables:
    """tables.py:66-77, through the device builder."""
    return CodeTables.from_matrix(H).variable


def build_check_tables(variable_tables: EdgeTables) -> EdgeTables:
    """tables.py:80-92: regroup variable-oriented tables by check node."""
    if variable_tables.orientation != VARIABLE:
        raise ValueError("input must be variable-oriented tables")
    n = int(variable_tables.v.max()) + 1
    m = int(variable_tables.c.max()) + 1
    H = ParityCheckMatrix(n, m, np.stack([variable_tables.c, variable_tables.v], axis=1))
    return CodeTables.from_matrix(H).check


def edge_set(tables: EdgeTables) -> set[tuple[int, int]]:
    """(row, col) pairs encoded by the tables (tables.py:119-121)."""
    return set(zip(tables.c.tolist(), tables.v.tolist()))
