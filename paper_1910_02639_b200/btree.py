"""Thin ctypes binding of libbtree.so (include/btree.h).

Argument marshalling only: every step of the path runs in the CUDA library.
PyTorch supplies device memory (tensors) and the current stream; it computes
nothing here.  There is no CPU fallback: if libbtree.so is missing or a call
fails, this module raises.
"""
from __future__ import annotations

import ctypes as C
import os

import torch

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("BT_LIB") or os.path.join(_PKG, "libbtree.so")  # BT_LIB: A/B experiments

BT_OK, BT_ERR_ARG, BT_ERR_INPUT, BT_ERR_CAPACITY, BT_ERR_CUDA, BT_ERR_OOM = range(6)
_NAMES = {0: "BT_OK", 1: "BT_ERR_ARG", 2: "BT_ERR_INPUT", 3: "BT_ERR_CAPACITY", 4: "BT_ERR_CUDA",
          5: "BT_ERR_OOM"}

# every symbol include/btree.h declares
EXPORTS = ["bt_build", "bt_build_ex", "bt_build_policy", "bt_find_neighbors", "bt_fill_neighbors",
           "bt_find_neighbors_sym", "bt_fill_neighbors_sym", "bt_density", "bt_set_partition", "bt_set_tree_order",
           "bt_reorder", "bt_free",
           "bt_search_host", "bt_set_stream", "bt_set_exact_only", "bt_release_cache", "bt_last_error", "bt_last_status", "bt_tree_stats",
           "bt_tree_order", "bt_profile_enable", "bt_profile_reset", "bt_profile_get"]


# bt_build_policy's policies (include/btree.h)
POLICIES = {"btree": 0, "octree": 1, "btree2d": 2, "quadtree": 3}


class BtreeError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{_NAMES.get(code, code)}: {msg}")
        self.code = code


class Stats(C.Structure):
    _fields_ = [("n", C.c_int64), ("nodes", C.c_int64), ("leaves", C.c_int64),
                ("halvings", C.c_int64), ("overfull", C.c_int64), ("max_leaf", C.c_int64),
                ("depth", C.c_int32), ("root_b", C.c_int32), ("units", C.c_int64),
                ("box_lo", C.c_double * 3), ("box_hi", C.c_double * 3),
                ("total_pairs", C.c_int64), ("max_count", C.c_int64), ("staged", C.c_int64),
                ("tests", C.c_int64), ("exact_tests", C.c_int64), ("loaded", C.c_int64),
                ("mask_words", C.c_int64), ("cand_slots", C.c_int64), ("list_entries", C.c_int64),
                ("big_units", C.c_int64), ("rows_over_ngmax", C.c_int64),
                ("mask_words_nonzero", C.c_int64)]

    def as_dict(self):
        d = {}
        for k, _ in self._fields_:
            v = getattr(self, k)
            d[k] = list(v) if k.startswith("box") else v
        return d


_lib = None
_P = C.c_void_p


def lib():
    """Load libbtree.so (raises if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not found: run __graft_entry__.build() "
                              "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        L.bt_build.argtypes = [_P, C.c_int64, C.c_int32, C.c_double]
        L.bt_build.restype = _P
        L.bt_build_ex.argtypes = [_P, C.c_int64, C.c_int32, C.c_double, C.c_double, C.c_int32]
        L.bt_build_ex.restype = _P
        L.bt_build_policy.argtypes = [_P, C.c_int64, C.c_int32, C.c_double, C.c_double, C.c_int32, C.c_int32]
        L.bt_build_policy.restype = _P
        L.bt_find_neighbors.argtypes = [_P, _P, C.c_int32, _P, _P, _P]
        L.bt_find_neighbors.restype = C.c_int
        L.bt_fill_neighbors.argtypes = [_P, _P, _P, _P, C.c_int64]
        L.bt_fill_neighbors.restype = C.c_int
        L.bt_find_neighbors_sym.argtypes = [_P, _P, C.c_int32, _P, _P, _P]
        L.bt_find_neighbors_sym.restype = C.c_int
        L.bt_fill_neighbors_sym.argtypes = [_P, _P, _P, _P, C.c_int64]
        L.bt_fill_neighbors_sym.restype = C.c_int
        L.bt_set_partition.argtypes = [_P, C.c_int32, C.c_int32]
        L.bt_set_partition.restype = C.c_int
        L.bt_set_tree_order.argtypes = [_P, C.c_int]
        L.bt_set_tree_order.restype = C.c_int
        L.bt_reorder.argtypes = [_P, _P, C.c_int32, _P]
        L.bt_reorder.restype = C.c_int
        L.bt_density.argtypes = [_P, _P, _P, _P]
        L.bt_density.restype = C.c_int
        L.bt_free.argtypes = [_P]
        L.bt_free.restype = None
        L.bt_search_host.argtypes = [_P, _P, C.c_int64, C.c_int32, C.c_double, _P, _P, _P, C.c_int64]
        L.bt_search_host.restype = C.c_int
        L.bt_set_stream.argtypes = [_P]
        L.bt_set_stream.restype = C.c_int
        L.bt_release_cache.argtypes = []
        L.bt_release_cache.restype = C.c_int
        L.bt_set_exact_only.argtypes = [C.c_int]
        L.bt_set_exact_only.restype = C.c_int
        L.bt_last_error.argtypes = []
        L.bt_last_error.restype = C.c_char_p
        L.bt_last_status.argtypes = []
        L.bt_last_status.restype = C.c_int
        L.bt_tree_stats.argtypes = [_P, C.POINTER(Stats)]
        L.bt_tree_stats.restype = C.c_int
        L.bt_tree_order.argtypes = [_P, _P, _P, _P, _P]
        L.bt_tree_order.restype = C.c_int
        L.bt_profile_enable.argtypes = [C.c_int]
        L.bt_profile_enable.restype = C.c_int
        L.bt_profile_reset.argtypes = []
        L.bt_profile_reset.restype = C.c_int
        L.bt_profile_get.argtypes = [C.c_int, C.POINTER(C.c_char_p), C.POINTER(C.c_double),
                                     C.POINTER(C.c_int64)]
        L.bt_profile_get.restype = C.c_int
        _lib = L
    return _lib


def _check(rc: int):
    if rc != BT_OK:
        raise BtreeError(rc, lib().bt_last_error().decode())


def _ptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def _use_current_stream(device=None):
    """Hand torch's current stream of `device` (the tensors' GPU) to the library."""
    lib().bt_set_stream(C.c_void_p(torch.cuda.current_stream(device).cuda_stream))


def _dev_f64(t, shape_last=None, n=None, device=None, name="tensor"):
    """A contiguous CUDA float64 tensor of shape [n, shape_last] (or [n])."""
    if not isinstance(t, torch.Tensor) or not t.is_cuda or t.dtype != torch.float64:
        raise TypeError(f"{name}: expected a CUDA float64 tensor")
    if shape_last is not None and (t.dim() != 2 or t.shape[1] != shape_last):
        raise TypeError(f"{name}: expected shape [n, {shape_last}]")
    if shape_last is None and t.dim() != 1:
        raise TypeError(f"{name}: expected a 1-D tensor")
    if n is not None and t.shape[0] != n:
        raise ValueError(f"{name}: expected {n} rows, got {t.shape[0]}")
    if device is not None and t.device != device:
        raise ValueError(f"{name}: on {t.device}, the tree is on {device}")
    return t.contiguous()


def _dev_out(t, dtype, numel, device, name):
    """A caller-supplied CUDA output buffer: dtype, device, contiguity, size >= numel."""
    if not isinstance(t, torch.Tensor) or not t.is_cuda or t.dtype != dtype or not t.is_contiguous():
        raise TypeError(f"{name}: expected a contiguous CUDA {dtype} tensor")
    if t.device != device:
        raise ValueError(f"{name}: on {t.device}, the tree is on {device}")
    if t.numel() < numel:
        raise ValueError(f"{name}: needs >= {numel} elements, has {t.numel()}")
    return t


class Tree:
    """b-tree over n particles (bt_build).  pos: CUDA float64 [n, 3]."""

    def __init__(self, pos: torch.Tensor, bucket_size: int = 64, max_empty: float = 0.5,
                 alpha: float | None = None, depth_cap: int | None = None, policy: str = "btree"):
        pos = _dev_f64(pos, 3, name="pos")
        self.n = pos.shape[0]
        self.device = pos.device
        if policy not in POLICIES:
            raise ValueError(f"policy must be one of {sorted(POLICIES)}")
        with torch.cuda.device(self.device):
            self._h = self._build(pos, bucket_size, max_empty, alpha, depth_cap, policy)

    def _build(self, pos, bucket_size, max_empty, alpha, depth_cap, policy):
        _use_current_stream(self.device)
        if policy != "btree":
            h = lib().bt_build_policy(_ptr(pos), self.n, int(bucket_size), float(max_empty),
                                      0.5 if alpha is None else float(alpha),
                                      64 if depth_cap is None else int(depth_cap), POLICIES[policy])
        elif alpha is None and depth_cap is None:
            h = lib().bt_build(_ptr(pos), self.n, int(bucket_size), float(max_empty))
        else:
            h = lib().bt_build_ex(_ptr(pos), self.n, int(bucket_size), float(max_empty),
                                  0.5 if alpha is None else float(alpha),
                                  64 if depth_cap is None else int(depth_cap))
        if not h:
            raise BtreeError(lib().bt_last_status(), lib().bt_last_error().decode())
        return h

    def free(self):
        h = getattr(self, "_h", None)
        if h:
            with torch.cuda.device(self.device):
                _use_current_stream(self.device)
                lib().bt_free(h)
            self._h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass

    def _handle(self):
        if not self._h:
            raise BtreeError(BT_ERR_ARG, "tree already freed")
        return self._h

    def count(self, h: torch.Tensor, symmetric: bool = False, ngmax: int = 512):
        """Count-only call: (counts int32 [n], offsets int64 [n+1]).  symmetric:
        the max(h_i, h_j) criterion (bt_find_neighbors_sym); ngmax only sets
        the threshold of stats()["rows_over_ngmax"]."""
        h = _dev_f64(h, n=self.n, device=self.device, name="h")
        counts = torch.empty(self.n, dtype=torch.int32, device=self.device)
        offsets = torch.empty(self.n + 1, dtype=torch.int64, device=self.device)
        with torch.cuda.device(self.device):
            _use_current_stream(self.device)
            fn = lib().bt_find_neighbors_sym if symmetric else lib().bt_find_neighbors
            _check(fn(self._handle(), _ptr(h), int(ngmax), _ptr(counts), _ptr(offsets), None))
        return counts, offsets

    def fill(self, h: torch.Tensor, offsets: torch.Tensor, out: torch.Tensor | None = None,
             symmetric: bool = False):
        h = _dev_f64(h, n=self.n, device=self.device, name="h")
        _dev_out(offsets, torch.int64, self.n + 1, self.device, "offsets")
        if offsets.numel() != self.n + 1:
            raise ValueError(f"offsets: expected {self.n + 1} entries, got {offsets.numel()}")
        total = int(offsets[-1].item())
        if out is None:
            out = torch.empty(max(total, 1), dtype=torch.int32, device=self.device)
        _dev_out(out, torch.int32, 0, self.device, "out")
        with torch.cuda.device(self.device):
            _use_current_stream(self.device)
            fn = lib().bt_fill_neighbors_sym if symmetric else lib().bt_fill_neighbors
            _check(fn(self._handle(), _ptr(h), _ptr(offsets), _ptr(out), out.numel()))
        return out[:total]

    def density(self, h: torch.Tensor, mass: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        """SPH density rho [n] fp64 (bt_density: M4 spline, neighbor search fused in)."""
        h = _dev_f64(h, n=self.n, device=self.device, name="h")
        mass = _dev_f64(mass, n=self.n, device=self.device, name="mass")
        if out is None:
            out = torch.empty(self.n, dtype=torch.float64, device=self.device)
        _dev_out(out, torch.float64, self.n, self.device, "out")
        with torch.cuda.device(self.device):
            _use_current_stream(self.device)
            _check(lib().bt_density(self._handle(), _ptr(h), _ptr(mass), _ptr(out)))
        return out

    def find_neighbors(self, h: torch.Tensor, ngmax: int | None = None,
                       counts=None, offsets=None, nbr_idx=None, symmetric: bool = False):
        """(counts, offsets, nbr_idx) for every particle.

        ngmax given: one bt_find_neighbors call into a buffer of n*ngmax slots
        (or the caller's nbr_idx).  ngmax None: count-only call, exact
        allocation, then bt_fill_neighbors.  symmetric: the max(h_i, h_j)
        criterion (bt_find_neighbors_sym / bt_fill_neighbors_sym).
        """
        h = _dev_f64(h, n=self.n, device=self.device, name="h")
        if ngmax is None:
            counts, offsets = self.count(h, symmetric)
            return counts, offsets, self.fill(h, offsets, symmetric=symmetric)
        if counts is None:
            counts = torch.empty(self.n, dtype=torch.int32, device=self.device)
        if offsets is None:
            offsets = torch.empty(self.n + 1, dtype=torch.int64, device=self.device)
        if nbr_idx is None:
            nbr_idx = torch.empty(max(self.n * int(ngmax), 1), dtype=torch.int32, device=self.device)
        _dev_out(counts, torch.int32, self.n, self.device, "counts")
        _dev_out(offsets, torch.int64, self.n + 1, self.device, "offsets")
        # the library's capacity is n * ngmax slots (BJ): the buffer must hold them
        _dev_out(nbr_idx, torch.int32, self.n * int(ngmax), self.device, "nbr_idx")
        with torch.cuda.device(self.device):
            _use_current_stream(self.device)
            fn = lib().bt_find_neighbors_sym if symmetric else lib().bt_find_neighbors
            _check(fn(self._handle(), _ptr(h), int(ngmax), _ptr(counts), _ptr(offsets), _ptr(nbr_idx)))
        return counts, offsets, nbr_idx

    def set_partition(self, part: int, nparts: int):
        """Restrict later searches to part `part` of `nparts` (bt_set_partition):
        rows of other parts' particles come back empty."""
        _check(lib().bt_set_partition(self._handle(), int(part), int(nparts)))
        return self

    def set_tree_order(self, on: bool = True):
        """Index space of later searches (bt_set_tree_order): with on, h, mass,
        counts, offsets rows, rho and neighbor indices are tree positions
        (particles reordered along the walk's curve)."""
        _check(lib().bt_set_tree_order(self._handle(), 1 if on else 0))
        return self

    def reorder(self, x: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        """x (caller order, fp64 [n] or [n, c]) gathered into tree order by
        bt_reorder: out[k] = x[perm[k]]."""
        if not isinstance(x, torch.Tensor) or x.dtype != torch.float64 or x.device != self.device:
            raise ValueError(f"x: expected a float64 tensor on {self.device}")
        if x.shape[0] != self.n or x.dim() > 2 or not x.is_contiguous():
            raise ValueError(f"x: expected a contiguous [{self.n}] or [{self.n}, c] tensor")
        ncomp = 1 if x.dim() == 1 else x.shape[1]
        if out is None:
            out = torch.empty_like(x)
        _dev_out(out, torch.float64, x.numel(), self.device, "out")
        if out.data_ptr() == x.data_ptr():
            raise ValueError("out: must not alias x")
        with torch.cuda.device(self.device):
            _use_current_stream(self.device)
            _check(lib().bt_reorder(self._handle(), _ptr(x), int(ncomp), _ptr(out)))
        return out

    def stats(self) -> dict:
        s = Stats()
        _check(lib().bt_tree_stats(self._handle(), C.byref(s)))
        return s.as_dict()

    def order(self):
        """(perm int32 [n], leaf_begin int64, leaf_count int32, leaf_depth int32) on the device."""
        L = self.stats()["leaves"]
        perm = torch.empty(max(self.n, 1), dtype=torch.int32, device=self.device)
        lb = torch.empty(max(L, 1), dtype=torch.int64, device=self.device)
        lc = torch.empty(max(L, 1), dtype=torch.int32, device=self.device)
        ld = torch.empty(max(L, 1), dtype=torch.int32, device=self.device)
        with torch.cuda.device(self.device):
            _use_current_stream(self.device)
            _check(lib().bt_tree_order(self._handle(), _ptr(perm), _ptr(lb), _ptr(lc), _ptr(ld)))
        return perm[:self.n], lb[:L], lc[:L], ld[:L]


def build(pos, bucket_size: int = 64, max_empty: float = 0.5, **kw) -> Tree:
    return Tree(pos, bucket_size, max_empty, **kw)


def search_host(pos, h, bucket_size: int = 64, max_empty: float = 0.5, capacity: int | None = None,
                counts=None, offsets=None, nbr=None):
    """End-to-end on host (preferably pinned) tensors via bt_search_host."""
    def host(t, dtype, shape, name):
        if not isinstance(t, torch.Tensor) or t.is_cuda or t.dtype != dtype or not t.is_contiguous():
            raise TypeError(f"{name}: expected a contiguous CPU {dtype} tensor")
        if shape is not None and tuple(t.shape) != shape:
            raise ValueError(f"{name}: expected shape {shape}, got {tuple(t.shape)}")
        return t
    if not isinstance(pos, torch.Tensor) or pos.dim() != 2:
        raise TypeError("pos: expected a CPU float64 tensor [n, 3]")
    n = pos.shape[0]
    host(pos, torch.float64, (n, 3), "pos")
    host(h, torch.float64, (n,), "h")
    if counts is None:
        counts = torch.empty(n, dtype=torch.int32).pin_memory()
    if offsets is None:
        offsets = torch.empty(n + 1, dtype=torch.int64).pin_memory()
    if nbr is None:
        nbr = torch.empty(max(capacity or 1, 1), dtype=torch.int32).pin_memory()
    host(counts, torch.int32, (n,), "counts")
    host(offsets, torch.int64, (n + 1,), "offsets")
    host(nbr, torch.int32, None, "nbr")
    cap = nbr.numel() if capacity is None else int(capacity)
    if cap > nbr.numel() or cap < 0:
        raise ValueError(f"capacity {cap} exceeds nbr's {nbr.numel()} elements")
    _use_current_stream()
    _check(lib().bt_search_host(_ptr(pos), _ptr(h), n, int(bucket_size), float(max_empty), _ptr(counts),
                                _ptr(offsets), _ptr(nbr), cap))
    return counts, offsets, nbr[:int(offsets[n])]


def release_cache():
    """Return this thread's cached device blocks to the driver."""
    _check(lib().bt_release_cache())


def set_exact_only(on: bool = True):
    """Validation knob: every pair decided by the fp64 predicate itself."""
    lib().bt_set_exact_only(1 if on else 0)


def profile_enable(on: bool = True):
    lib().bt_profile_enable(1 if on else 0)


def profile_reset():
    lib().bt_profile_reset()


def profile() -> dict:
    """{name: (ms accumulated, launches)} from the library's CUDA-event phases."""
    k = lib().bt_profile_get(0, None, None, None)
    names = (C.c_char_p * max(k, 1))()
    ms = (C.c_double * max(k, 1))()
    la = (C.c_int64 * max(k, 1))()
    k = lib().bt_profile_get(k, names, ms, la)
    return {names[i].decode(): (ms[i], la[i]) for i in range(k)}
