"""CPU oracle for the b-tree exact close-neighbor search (arXiv 1910.02639).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  The product package ``paper_1910_02639_b200`` never imports it and
shares no code with it.

The arithmetic lives in ``btree_oracle.c`` (plain C, fp64, no FMA); this module
only compiles it and marshals numpy arrays through ctypes.

Parity status: Eq. 1-5, the predicate, the brute force and the tree walk are
pinned by tests/test_oracle_pins.py.  Tree *shapes* at scale are "parity
unpinned" beyond the structural invariants (the paper prints none).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "btree_oracle.c")
# ORACLE_LIB: an alternative build of the same source (the sanitizer test)
_LIB = os.environ.get("ORACLE_LIB") or os.path.join(_HERE, "liboracle.so")

CFLAGS = ["-O2", "-std=c11", "-fPIC", "-shared", "-ffp-contract=off",
          "-fno-fast-math", "-fopenmp", "-Wall", "-Wno-unknown-pragmas"]


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (no FMA contraction, no fast-math)."""
    if os.environ.get("ORACLE_LIB"):
        return _LIB
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, _SRC, "-o", tmp, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


class Stats(C.Structure):
    _fields_ = [("n", C.c_int64), ("nodes", C.c_int64), ("leaves", C.c_int64),
                ("halvings", C.c_int64), ("overfull", C.c_int64),
                ("max_leaf", C.c_int64), ("depth", C.c_int32), ("root_b", C.c_int32)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


_lib = None
_P = C.c_void_p


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_LIB)
        L.orc_branching_factor.argtypes = [C.c_int64, C.c_int64]
        L.orc_branching_factor_k.argtypes = [C.c_int64, C.c_int64, C.c_int]
        L.orc_branching_factor_k.restype = C.c_int
        L.orc_branching_factor.restype = C.c_int
        L.orc_cell_coord.argtypes = [C.c_double, C.c_double, C.c_double, C.c_int]
        L.orc_cell_coord.restype = C.c_int
        L.orc_cell_id.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int]
        L.orc_cell_id.restype = C.c_int64
        L.orc_ratio.argtypes = [_P, C.c_int64, C.c_double, C.c_int64]
        L.orc_ratio.restype = C.c_double
        L.orc_range.argtypes = [C.c_double, C.c_double, C.c_double, C.c_double, C.c_int,
                                C.POINTER(C.c_int), C.POINTER(C.c_int)]
        L.orc_range.restype = None
        L.orc_root_box.argtypes = [_P, C.c_int64, _P, _P]
        L.orc_root_box.restype = None
        L.orc_build.argtypes = [_P, C.c_int64, C.c_int32, C.c_double, C.c_double, C.c_int32]
        L.orc_build.restype = _P
        L.orc_build_policy.argtypes = [_P, C.c_int64, C.c_int32, C.c_double, C.c_double, C.c_int32, C.c_int]
        L.orc_build_policy.restype = _P
        L.orc_free.argtypes = [_P]
        L.orc_free.restype = None
        L.orc_get_stats.argtypes = [_P, C.POINTER(Stats)]
        L.orc_get_stats.restype = C.c_int
        L.orc_get_box.argtypes = [_P, _P, _P]
        L.orc_get_box.restype = None
        L.orc_get_order.argtypes = [_P, _P, _P, _P, _P]
        L.orc_get_order.restype = C.c_int64
        L.orc_count.argtypes = [_P, _P, _P, _P, C.c_int64, _P, C.c_int]
        L.orc_count.restype = None
        L.orc_rows.argtypes = [_P, _P, _P, _P, C.c_int64, _P, _P, C.c_int]
        L.orc_rows.restype = C.c_int
        L.orc_brute_count.argtypes = [_P, _P, C.c_int64, _P, C.c_int64, _P, C.c_int]
        L.orc_brute_count.restype = None
        L.orc_brute_rows.argtypes = [_P, _P, C.c_int64, _P, C.c_int64, _P, _P, C.c_int]
        L.orc_brute_rows.restype = C.c_int
        L.orc_brute_count_sym.argtypes = [_P, _P, C.c_int64, _P, C.c_int64, _P, C.c_int]
        L.orc_brute_count_sym.restype = None
        L.orc_brute_rows_sym.argtypes = [_P, _P, C.c_int64, _P, C.c_int64, _P, _P, C.c_int]
        L.orc_brute_rows_sym.restype = C.c_int
        L.orc_w_m4.argtypes = [C.c_double]
        L.orc_w_m4.restype = C.c_double
        L.orc_density.argtypes = [_P, _P, _P, _P, _P, C.c_int64, _P, C.c_int]
        L.orc_density.restype = None
        L.orc_brute_density.argtypes = [_P, _P, _P, C.c_int64, _P, C.c_int64, _P, C.c_int]
        L.orc_brute_density.restype = None
        L.orc_max_threads.argtypes = []
        L.orc_max_threads.restype = C.c_int
        _lib = L
    return _lib


def _ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _f64(a, shape=None):
    a = np.ascontiguousarray(a, dtype=np.float64)
    if shape is not None:
        a = a.reshape(shape)
    return a


def default_threads() -> int:
    return max(1, os.cpu_count() or 1)


# ---- Eq. 1 - 5 helpers (exposed for the pins) -------------------------------
POLICIES = {"btree": 0, "octree": 1, "btree2d": 2, "quadtree": 3}


def branching_factor_k(n: int, s: int, k: int) -> int:
    return lib().orc_branching_factor_k(n, s, k)


def branching_factor(n: int, s: int) -> int:
    return lib().orc_branching_factor(n, s)


def cell_coord(x: float, lo: float, hi: float, b: int) -> int:
    return lib().orc_cell_coord(x, lo, hi, b)


def cell_id(c1: int, c2: int, c3: int, b: int) -> int:
    return lib().orc_cell_id(c1, c2, c3, b)


def ratio(counts, alpha: float, s: int) -> float:
    c = np.ascontiguousarray(counts, dtype=np.int64)
    return lib().orc_ratio(_ptr(c), c.size, alpha, s)


def search_range(x: float, R: float, lo: float, hi: float, b: int):
    a, z = C.c_int(), C.c_int()
    lib().orc_range(x, R, lo, hi, b, C.byref(a), C.byref(z))
    return a.value, z.value


def root_box(pos):
    pos = _f64(pos, (-1, 3))
    lo = np.zeros(3)
    hi = np.zeros(3)
    lib().orc_root_box(_ptr(pos), pos.shape[0], _ptr(lo), _ptr(hi))
    return lo, hi


# ---- tree ------------------------------------------------------------------
class Tree:
    """b-tree built by the oracle's BuildTree (Alg. 1)."""

    def __init__(self, pos, bucket_size: int = 64, max_empty: float = 0.5,
                 alpha: float = 0.5, depth_cap: int = 64, policy: str = "btree"):
        self.pos = _f64(pos, (-1, 3))
        self.n = self.pos.shape[0]
        self._h = lib().orc_build_policy(_ptr(self.pos), self.n, bucket_size, max_empty, alpha, depth_cap,
                                         POLICIES[policy])
        if not self._h:
            raise ValueError("oracle: invalid build arguments")

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and _lib is not None:
            try:
                _lib.orc_free(h)
            except Exception:
                pass
            self._h = None

    def stats(self) -> dict:
        s = Stats()
        lib().orc_get_stats(self._h, C.byref(s))
        return s.as_dict()

    def box(self):
        lo = np.zeros(3)
        hi = np.zeros(3)
        lib().orc_get_box(self._h, _ptr(lo), _ptr(hi))
        return lo, hi

    def order(self):
        """(perm, leaf_begin, leaf_count, leaf_depth) in depth-first leaf order."""
        nl = lib().orc_get_order(self._h, None, None, None, None)
        perm = np.empty(self.n, dtype=np.int32)
        lb = np.empty(nl, dtype=np.int64)
        lc = np.empty(nl, dtype=np.int32)
        ld = np.empty(nl, dtype=np.int32)
        lib().orc_get_order(self._h, _ptr(perm), _ptr(lb), _ptr(lc), _ptr(ld))
        return perm, lb, lc, ld

    def count(self, h, queries=None, threads: int | None = None):
        h = _f64(h)
        q = None if queries is None else np.ascontiguousarray(queries, dtype=np.int64)
        nq = self.n if q is None else q.size
        counts = np.empty(nq, dtype=np.int32)
        lib().orc_count(self._h, _ptr(self.pos), _ptr(h), _ptr(q), nq, _ptr(counts),
                        threads or default_threads())
        return counts

    def neighbors(self, h, queries=None, threads: int | None = None):
        """(counts int32, offsets int64 [nq+1], idx int32) with rows ascending."""
        h = _f64(h)
        q = None if queries is None else np.ascontiguousarray(queries, dtype=np.int64)
        counts = self.count(h, q, threads)
        offsets = np.zeros(counts.size + 1, dtype=np.int64)
        np.cumsum(counts, out=offsets[1:])
        idx = np.empty(int(offsets[-1]), dtype=np.int32)
        rc = lib().orc_rows(self._h, _ptr(self.pos), _ptr(h), _ptr(q), counts.size,
                            _ptr(offsets), _ptr(idx), threads or default_threads())
        if rc != 0:
            raise RuntimeError("oracle: row length changed between passes")
        return counts, offsets, idx

    def density(self, h, mass, queries=None, threads: int | None = None):
        """SPH density (reading R21: M4 cubic spline, support 2h, gather h):
        rho_i = m_i W(0, h_i) + sum over the tree walk's N(i) of m_j W(r_ij, h_i)."""
        h = _f64(h)
        mass = _f64(mass)
        q = None if queries is None else np.ascontiguousarray(queries, dtype=np.int64)
        nq = self.n if q is None else q.size
        rho = np.empty(nq, dtype=np.float64)
        lib().orc_density(self._h, _ptr(self.pos), _ptr(h), _ptr(mass), _ptr(q), nq, _ptr(rho),
                          threads or default_threads())
        return rho


def w_m4(q: float) -> float:
    """The M4 cubic spline shape w(q) of the density consumer (R21)."""
    return lib().orc_w_m4(float(q))


def brute_density(pos, h, mass, queries=None, threads: int | None = None):
    """SPH density by the plain definition (every j != i passing the predicate)."""
    pos = _f64(pos, (-1, 3))
    h = _f64(h)
    mass = _f64(mass)
    n = pos.shape[0]
    q = None if queries is None else np.ascontiguousarray(queries, dtype=np.int64)
    nq = n if q is None else q.size
    rho = np.empty(nq, dtype=np.float64)
    lib().orc_brute_density(_ptr(pos), _ptr(h), _ptr(mass), n, _ptr(q), nq, _ptr(rho),
                            threads or default_threads())
    return rho


def brute_force(pos, h, queries=None, threads: int | None = None, symmetric: bool = False):
    """O(n^2) plain definition: (counts, offsets, idx), rows ascending.
    symmetric: the max(h_i, h_j) criterion (reading R22)."""
    pos = _f64(pos, (-1, 3))
    h = _f64(h)
    n = pos.shape[0]
    q = None if queries is None else np.ascontiguousarray(queries, dtype=np.int64)
    nq = n if q is None else q.size
    counts = np.empty(nq, dtype=np.int32)
    count_fn = lib().orc_brute_count_sym if symmetric else lib().orc_brute_count
    rows_fn = lib().orc_brute_rows_sym if symmetric else lib().orc_brute_rows
    count_fn(_ptr(pos), _ptr(h), n, _ptr(q), nq, _ptr(counts), threads or default_threads())
    offsets = np.zeros(nq + 1, dtype=np.int64)
    np.cumsum(counts, out=offsets[1:])
    idx = np.empty(int(offsets[-1]), dtype=np.int32)
    rc = rows_fn(_ptr(pos), _ptr(h), n, _ptr(q), nq, _ptr(offsets), _ptr(idx), threads or default_threads())
    if rc != 0:
        raise RuntimeError("oracle brute force: row length changed between passes")
    return counts, offsets, idx
