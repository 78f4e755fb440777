"""TEST INFRASTRUCTURE ONLY — ctypes bindings for the CPU oracles.

* ``Oracle``    : oracle/liboracle.so, the plain-C restatement (oracle.c).
* ``Reference`` : oracle/_ref/libqref.so, the unmodified reference library
                  (/root/reference/proj/src/*.cpp) behind ref_shim.cpp.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may import this module, and only as the checker or
the timed CPU baseline.  The product package never imports it.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libqref.so")

_u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")

KIND = {"quesadilla": 0, "topk": 1, "radix": 2, "comparison": 3}


class OracleError(Exception):
    def __init__(self, code: int, msg: str = ""):
        super().__init__(f"status {code}: {msg}")
        self.code = code


def _u32(a):
    return np.ascontiguousarray(a, dtype=np.uint32)


class Oracle:
    """The C restatement (oracle/oracle.c)."""

    def __init__(self, path: str = ORACLE_SO):
        self.lib = C.CDLL(path)
        L = self.lib
        L.qo_plan.argtypes = [_u32p, C.c_uint32, C.c_uint32, _u32p, C.c_uint32,
                              C.POINTER(C.c_uint32)]
        L.qo_partial_sort.argtypes = [C.c_uint32, _u32p, C.c_uint64, _u32p, _f64p,
                                      _u32p, C.c_uint32, C.c_uint32]
        L.qo_transpose.argtypes = [C.c_uint32, _u32p, C.c_uint64, _u32p, _f64p,
                                   _u32p, C.c_int, C.c_uint32, C.c_int, _u32p,
                                   C.c_uint32, C.POINTER(C.c_uint32)]
        L.qo_bucket_starts.argtypes = [C.c_uint32, C.c_uint64, _u32p, _u32p,
                                       C.c_uint32, _u64p]
        L.qo_bucket_starts.restype = C.c_uint64
        L.qo_is_sorted.argtypes = [C.c_uint32, C.c_uint64, _u32p, _u32p]
        L.qo_sort_rows_by.argtypes = [C.c_uint32, C.c_uint64, _u32p, _f64p, C.c_uint64,
                                      C.c_uint64, _u32p, C.c_uint32]
        L.qo_relabel_target.argtypes = [_u32p, _u32p, C.c_uint32, _u32p]

    def sort_rows_by(self, rank, coords, values, row_begin, row_end, keys):
        c = _u32(coords).copy()
        v = np.ascontiguousarray(values, np.float64).copy()
        k = _u32(keys) if len(keys) else np.zeros(1, np.uint32)
        s = self.lib.qo_sort_rows_by(rank, len(v), c, v, row_begin, row_end, k, len(keys))
        if s:
            raise OracleError(s)
        return c, v

    def relabel_target(self, source, target):
        out = np.zeros(len(target), np.uint32)
        s = self.lib.qo_relabel_target(_u32(source), _u32(target), len(target), out)
        if s:
            raise OracleError(s)
        return [int(x) for x in out]

    def plan(self, target, want: int = 0):
        t = _u32(target)
        steps = np.zeros(256, np.uint32)
        n = C.c_uint32(0)
        s = self.lib.qo_plan(t, len(t), want, steps, 128, C.byref(n))
        if s:
            raise OracleError(s)
        return [(int(steps[2 * i]), int(steps[2 * i + 1])) for i in range(n.value)]

    def partial_sort(self, dims, coords, values, prefix, mode):
        dims = _u32(dims)
        c = _u32(coords).copy()
        v = np.ascontiguousarray(values, np.float64).copy()
        p = _u32(prefix) if len(prefix) else np.zeros(1, np.uint32)
        s = self.lib.qo_partial_sort(len(dims), dims, len(v), c, v, p, len(prefix), mode)
        if s:
            raise OracleError(s)
        return c, v

    def transpose(self, dims, coords, values, target, strategy="quesadilla", k=0,
                  verify_input=False):
        dims = _u32(dims)
        c = _u32(coords).copy()
        v = np.ascontiguousarray(values, np.float64).copy()
        steps = np.zeros(256, np.uint32)
        n = C.c_uint32(0)
        s = self.lib.qo_transpose(len(dims), dims, len(v), c, v, _u32(target),
                                  KIND[strategy], k, int(verify_input), steps, 128,
                                  C.byref(n))
        if s:
            raise OracleError(s)
        return c, v, [(int(steps[2 * i]), int(steps[2 * i + 1])) for i in range(n.value)]

    def bucket_starts(self, rank, coords, modes):
        c = _u32(coords)
        nnz = len(c) // rank if rank else 0
        out = np.zeros(max(nnz, 1), np.uint64)
        m = _u32(modes) if len(modes) else np.zeros(1, np.uint32)
        n = self.lib.qo_bucket_starts(rank, nnz, c, m, len(modes), out)
        return out[:n].copy()

    def is_sorted(self, rank, coords, order):
        c = _u32(coords)
        return bool(self.lib.qo_is_sorted(rank, len(c) // rank, c, _u32(order)))


class Reference:
    """The reference library itself (oracle/_ref/libqref.so)."""

    def __init__(self, path: str = REF_SO):
        self.lib = C.CDLL(path)
        L = self.lib
        L.qref_last_error.restype = C.c_char_p
        L.qref_transpose.argtypes = [C.c_uint32, _u32p, C.c_uint64, _u32p, _f64p,
                                     _u32p, C.c_int, C.c_uint32, C.c_uint32, C.c_int,
                                     _u32p, C.c_uint32, C.POINTER(C.c_uint32)]
        L.qref_partial_sort.argtypes = [C.c_uint32, _u32p, C.c_uint64, _u32p, _f64p,
                                        _u32p, C.c_uint32, C.c_uint32, C.c_uint32]
        L.qref_plan.argtypes = [_u32p, C.c_uint32, C.c_uint32, _u32p, C.c_uint32,
                                C.POINTER(C.c_uint32)]
        L.qref_min_plan_bruteforce.argtypes = [_u32p, C.c_uint32, C.POINTER(C.c_int),
                                               C.POINTER(C.c_int)]
        L.qref_required_sort_count.argtypes = [_u32p, _u32p, C.c_uint32,
                                               C.POINTER(C.c_int)]
        L.qref_pass_histogram.argtypes = [C.c_uint32, np.ctypeslib.ndpointer(
            np.int64, flags="C_CONTIGUOUS"), C.c_uint32]
        L.qref_generate.argtypes = [C.c_uint32, _u32p, C.c_uint64, C.c_uint64, C.c_int,
                                    _u32p, _f64p]
        L.qref_bucket_starts.argtypes = [C.c_uint32, _u32p, C.c_uint64, _u32p, _f64p,
                                         _u32p, C.c_uint32, _u64p,
                                         C.POINTER(C.c_uint64)]
        L.qref_is_sorted.argtypes = [C.c_uint32, _u32p, C.c_uint64, _u32p, _f64p,
                                     _u32p, C.POINTER(C.c_int)]
        L.qref_ctx_create.restype = C.c_void_p
        L.qref_ctx_create.argtypes = [C.c_uint32, _u32p, C.c_uint64, _u32p, _f64p]
        L.qref_ctx_destroy.argtypes = [C.c_void_p]
        L.qref_ctx_reset.argtypes = [C.c_void_p, _u32p, _f64p]
        L.qref_ctx_transpose.argtypes = [C.c_void_p, _u32p, C.c_uint32]
        L.qref_ctx_read.argtypes = [C.c_void_p, _u32p, _f64p]
        L.qref_default_workers.restype = C.c_uint
        L.qref_read_tns.restype = C.c_void_p
        L.qref_read_tns.argtypes = [C.c_char_p, C.c_void_p, C.c_uint32, C.c_int, C.c_int,
                                    C.POINTER(C.c_int)]
        L.qref_parse_error_line.restype = C.c_uint64
        L.qref_tensor_info.argtypes = [C.c_void_p, C.POINTER(C.c_uint32),
                                       C.POINTER(C.c_uint64)]
        L.qref_tensor_copy.argtypes = [C.c_void_p, _u32p, _u32p, _f64p]
        L.qref_tensor_free.argtypes = [C.c_void_p]
        L.qref_write_tns.argtypes = [C.c_uint32, _u32p, C.c_uint64, _u32p, _f64p, C.c_char_p]

    def _check(self, s):
        if s:
            raise OracleError(s, self.lib.qref_last_error().decode())

    def read_tns(self, path, declared_dims=None, canonicalize=True):
        """io.hpp:40-41.  Raises OracleError(4, what) with .line for ParseError."""
        decl = None if declared_dims is None else _u32(declared_dims)
        st = C.c_int(0)
        h = self.lib.qref_read_tns(str(path).encode(),
                                   None if decl is None or len(decl) == 0 else decl.ctypes.data,
                                   0 if decl is None else len(decl), int(decl is not None),
                                   int(bool(canonicalize)), C.byref(st))
        if st.value:
            e = OracleError(st.value, self.lib.qref_last_error().decode())
            e.line = int(self.lib.qref_parse_error_line())
            raise e
        r, n = C.c_uint32(0), C.c_uint64(0)
        self.lib.qref_tensor_info(h, C.byref(r), C.byref(n))
        dims = np.zeros(max(r.value, 1), np.uint32)
        coords = np.zeros(max(n.value * r.value, 1), np.uint32)
        values = np.zeros(max(n.value, 1), np.float64)
        self.lib.qref_tensor_copy(h, dims, coords, values)
        self.lib.qref_tensor_free(h)
        return dims[: r.value], coords[: n.value * r.value], values[: n.value]

    def write_tns(self, dims, coords, values, path):
        """io.hpp:47 (shortest round-trip values, 1-based indices)."""
        d = _u32(dims)
        self._check(self.lib.qref_write_tns(len(d), d, len(values), _u32(coords),
                                            np.ascontiguousarray(values, np.float64),
                                            str(path).encode()))

    def sort_rows_by(self, dims, coords, values, row_begin, row_end, keys):
        dims = _u32(dims)
        c = _u32(coords).copy()
        v = np.ascontiguousarray(values, np.float64).copy()
        k = _u32(keys) if len(keys) else np.zeros(1, np.uint32)
        self.lib.qref_sort_rows_by.argtypes = [C.c_uint32, _u32p, C.c_uint64, _u32p, _f64p,
                                               C.c_uint64, C.c_uint64, _u32p, C.c_uint32]
        self._check(self.lib.qref_sort_rows_by(len(dims), dims, len(v), c, v, row_begin, row_end,
                                               k, len(keys)))
        return c, v

    def relabel_target(self, source, target):
        out = np.zeros(len(target), np.uint32)
        self.lib.qref_relabel_target.argtypes = [_u32p, _u32p, C.c_uint32, _u32p]
        self._check(self.lib.qref_relabel_target(_u32(source), _u32(target), len(target), out))
        return [int(x) for x in out]

    def transpose(self, dims, coords, values, target, strategy="quesadilla", k=0,
                  workers=1, verify_input=False):
        dims = _u32(dims)
        c = _u32(coords).copy()
        v = np.ascontiguousarray(values, np.float64).copy()
        steps = np.zeros(256, np.uint32)
        n = C.c_uint32(0)
        self._check(self.lib.qref_transpose(len(dims), dims, len(v), c, v, _u32(target),
                                            KIND[strategy], k, workers, int(verify_input),
                                            steps, 128, C.byref(n)))
        return c, v, [(int(steps[2 * i]), int(steps[2 * i + 1])) for i in range(n.value)]

    def partial_sort(self, dims, coords, values, prefix, mode, workers=1):
        dims = _u32(dims)
        c = _u32(coords).copy()
        v = np.ascontiguousarray(values, np.float64).copy()
        p = _u32(prefix) if len(prefix) else np.zeros(1, np.uint32)
        self._check(self.lib.qref_partial_sort(len(dims), dims, len(v), c, v, p,
                                               len(prefix), mode, workers))
        return c, v

    def plan(self, target, want: int = 0):
        t = _u32(target)
        steps = np.zeros(256, np.uint32)
        n = C.c_uint32(0)
        self._check(self.lib.qref_plan(t, len(t), want, steps, 128, C.byref(n)))
        return [(int(steps[2 * i]), int(steps[2 * i + 1])) for i in range(n.value)]

    def min_plan_bruteforce(self, target):
        a, b = C.c_int(0), C.c_int(0)
        t = _u32(target)
        self._check(self.lib.qref_min_plan_bruteforce(t, len(t), C.byref(a), C.byref(b)))
        return a.value, b.value

    def pass_histogram(self, rank):
        h = np.zeros(16, np.int64)
        self._check(self.lib.qref_pass_histogram(rank, h, 16))
        return {i: int(x) for i, x in enumerate(h) if x}

    def generate(self, dims, nnz, seed, distinct=False):
        dims = _u32(dims)
        c = np.zeros(nnz * len(dims), np.uint32)
        v = np.zeros(nnz, np.float64)
        self._check(self.lib.qref_generate(len(dims), dims, nnz, seed, int(distinct), c, v))
        return c, v

    def bucket_starts(self, dims, coords, values, modes):
        dims = _u32(dims)
        c = _u32(coords)
        v = np.ascontiguousarray(values, np.float64)
        out = np.zeros(max(len(v), 1), np.uint64)
        n = C.c_uint64(0)
        m = _u32(modes) if len(modes) else np.zeros(1, np.uint32)
        self._check(self.lib.qref_bucket_starts(len(dims), dims, len(v), c, v, m,
                                                len(modes), out, C.byref(n)))
        return out[: n.value].copy()

    def default_workers(self):
        return int(self.lib.qref_default_workers())


def reference_available() -> bool:
    return os.path.exists(REF_SO)
