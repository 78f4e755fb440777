"""quesadilla_b200 — B200-native Quesadilla sparse-tensor transposition.

Python mirror of the reference's C++ transpose API (arxiv 2005.10427 artifact,
/root/reference/proj/include/quesadilla/*.hpp) over the C ABI in
``include/quesadilla_b200.h`` (``lib/libquesadilla_b200.so``, sm_100a).

Same names, argument meaning and error behaviour as the reference:

=========================  ================================================
reference (C++)            here
=========================  ================================================
CooTensor                  CooTensor (dims, AoS uint32 coords, f64 values)
Ordering / ModeSet         Ordering
PlanStep / SortPlan        PlanStep / SortPlan
quesadilla_plan            quesadilla_plan      (host planner, Alg. 3)
prefix_plan                prefix_plan
required_sort_count        required_sort_count
apply_transition           apply_transition / simulate_plan
SortStrategy               SortStrategy (+ parse_strategy, strategy_pass_cost)
TransposeOptions           TransposeOptions
Workspace                  Workspace (device workspace on one GPU)
transpose_inplace          transpose_inplace    (GPU, bit-exact)
transpose                  transpose
partial_sort               partial_sort
full_radix_transpose etc.  full_radix_transpose / topk_transpose /
                           comparison_transpose
is_sorted_under            is_sorted_under (host check, for convenience)
std::invalid_argument      InvalidArgument (ValueError)
std::out_of_range          OutOfRange (IndexError)
=========================  ================================================

There is no CPU fallback: importing works anywhere, but every transpose runs
as CUDA kernels and raises ``DeviceError`` when no GPU is visible.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("QD_LIB_PATH") or os.path.join(_HERE, "lib", "libquesadilla_b200.so")

QD_OK, QD_INVALID_ARGUMENT, QD_OUT_OF_RANGE, QD_CUDA_ERROR, QD_NCCL_ERROR, QD_NO_DEVICE = range(6)
KINDS = {"quesadilla": 0, "topk": 1, "radix": 2, "comparison": 3}


QD_PARSE_ERROR = 6


class InvalidArgument(ValueError):
    """std::invalid_argument"""


class OutOfRange(IndexError):
    """std::out_of_range (a coordinate exceeds its dimension)"""

    def __init__(self, msg, row=None, mode=None):
        super().__init__(msg)
        self.row, self.mode = row, mode


class DeviceError(RuntimeError):
    """CUDA failure or no device (the library has no CPU path)."""


class ParseError(RuntimeError):
    """quesadilla::ParseError (io.hpp:15-22): str() is "line N: ...", .line() is N."""

    def __init__(self, msg, line=0, kind=0, field=0):
        super().__init__(msg)
        self._line, self.kind, self.field = line, kind, field

    def line(self) -> int:
        return self._line


class TnsTensorC(C.Structure):
    _fields_ = [("rank", C.c_uint32), ("nnz", C.c_uint64), ("dims", C.POINTER(C.c_uint32)),
                ("coords", C.POINTER(C.c_uint32)), ("values", C.POINTER(C.c_double))]


class TnsErrorC(C.Structure):
    _fields_ = [("line", C.c_uint64), ("kind", C.c_uint32), ("field", C.c_uint32),
                ("got", C.c_uint32), ("expected", C.c_uint32), ("token_offset", C.c_uint64),
                ("token_len", C.c_uint64)]


class PlanStepC(C.Structure):
    _fields_ = [("prefix_len", C.c_uint32), ("mode", C.c_uint32)]


class OptionsC(C.Structure):
    _fields_ = [
        ("verify_input", C.c_int),
        ("workers", C.c_uint32),
        ("pass_log", C.POINTER(PlanStepC)),
        ("pass_log_capacity", C.c_uint32),
        ("pass_log_len", C.POINTER(C.c_uint32)),
        ("boundaries", C.POINTER(C.c_uint64)),
        ("n_boundaries", C.POINTER(C.c_uint64)),
    ]


_u32p = C.POINTER(C.c_uint32)
_f64p = C.POINTER(C.c_double)
_lib = None


def lib():
    """The loaded CUDA library; raises if it was not built (no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
            )
        L = C.CDLL(LIB_PATH)
        L.qd_last_error.restype = C.c_char_p
        L.qd_workspace_create.argtypes = [C.c_int, C.POINTER(C.c_void_p)]
        L.qd_workspace_destroy.argtypes = [C.c_void_p]
        L.qd_workspace_bytes.argtypes = [C.c_void_p]
        L.qd_workspace_bytes.restype = C.c_uint64
        L.qd_workspace_launches.argtypes = [C.c_void_p]
        L.qd_workspace_launches.restype = C.c_uint64
        L.qd_workspace_slices.argtypes = [C.c_void_p]
        L.qd_workspace_slices.restype = C.c_uint64
        L.qd_profile_enable.argtypes = [C.c_void_p, C.c_int]
        L.qd_profile_reset.argtypes = [C.c_void_p]
        L.qd_profile_get.argtypes = [C.c_void_p, C.c_int, C.POINTER(C.c_uint64),
                                     C.POINTER(C.c_double), C.POINTER(C.c_double)]
        L.qd_last_error_detail.argtypes = [C.POINTER(C.c_uint64), C.POINTER(C.c_uint32)]
        L.qd_quesadilla_plan.argtypes = [_u32p, C.c_uint32, C.POINTER(PlanStepC), C.c_uint32, _u32p]
        L.qd_prefix_plan.argtypes = [_u32p, C.c_uint32, C.c_uint32, C.POINTER(PlanStepC),
                                     C.c_uint32, _u32p]
        L.qd_required_sort_count.argtypes = [_u32p, _u32p, C.c_uint32, C.POINTER(C.c_int)]
        L.qd_apply_transition.argtypes = [_u32p, C.c_uint32, PlanStepC, _u32p]
        L.qd_strategy_pass_cost.argtypes = [C.c_int, C.c_uint32, _u32p, C.c_uint32,
                                            C.POINTER(C.c_int), C.POINTER(C.c_int)]
        L.qd_transpose_inplace.argtypes = [C.c_uint32, _u32p, C.c_uint64, _u32p, _f64p, _u32p,
                                           C.c_int, C.c_uint32, C.POINTER(OptionsC), C.c_void_p]
        L.qd_transpose_inplace_async.argtypes = L.qd_transpose_inplace.argtypes
        L.qd_workspace_synchronize.argtypes = [C.c_void_p]
        L.qd_transpose_device.argtypes = [C.c_uint32, _u32p, C.c_uint64, C.c_void_p, C.c_void_p,
                                          C.c_void_p, C.c_void_p, _u32p, C.c_int, C.c_uint32,
                                          C.POINTER(OptionsC), C.c_void_p, C.c_void_p]
        L.qd_partial_sort.argtypes = [C.c_uint32, _u32p, C.c_uint64, _u32p, _f64p, _u32p,
                                      C.c_uint32, C.c_uint32, C.c_void_p]
        L.qd_sort_rows_by.argtypes = [C.c_uint32, _u32p, C.c_uint64, _u32p, _f64p, C.c_uint64,
                                      C.c_uint64, _u32p, C.c_uint32, C.c_void_p]
        L.qd_sort_rows_by_device.argtypes = [C.c_uint32, _u32p, C.c_uint64, C.c_void_p,
                                             C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint64,
                                             C.c_uint64, _u32p, C.c_uint32, C.c_void_p,
                                             C.c_void_p]
        L.qd_relabel_target.argtypes = [_u32p, _u32p, C.c_uint32, _u32p]
        L.qd_csf_device.argtypes = [C.c_uint32, C.c_uint64, C.c_void_p, _u32p,
                                    C.POINTER(C.c_void_p), C.POINTER(C.c_void_p),
                                    C.POINTER(C.c_uint64), C.c_void_p, C.c_void_p]
        L.qd_partial_sort_device.argtypes = [C.c_uint32, _u32p, C.c_uint64, C.c_void_p, C.c_void_p,
                                             C.c_void_p, C.c_void_p, _u32p, C.c_uint32, C.c_uint32,
                                             C.c_void_p, C.c_void_p]
        L.qd_is_sorted_device.argtypes = [C.c_uint32, C.c_uint64, C.c_void_p, _u32p,
                                          C.POINTER(C.c_int), C.c_void_p, C.c_void_p]
        L.qd_bucket_starts_device.argtypes = [C.c_uint32, C.c_uint64, C.c_void_p, _u32p, C.c_uint32,
                                              C.c_void_p, C.POINTER(C.c_uint64), C.c_void_p,
                                              C.c_void_p]
        L.qd_mode_histogram_device.argtypes = [C.c_uint32, C.c_uint64, C.c_void_p, C.c_uint32,
                                               C.c_uint32, C.c_void_p, C.c_void_p, C.c_void_p]
        L.qd_partition_rows_device.argtypes = [C.c_uint32, C.c_uint64, C.c_void_p, C.c_void_p,
                                               C.c_uint32, C.c_uint32, C.c_void_p, C.c_uint32,
                                               C.c_void_p, C.c_void_p, C.POINTER(C.c_uint64),
                                               C.c_void_p, C.c_void_p]
        _u64p = C.POINTER(C.c_uint64)
        L.qd_partition_rows_to_peers_device.argtypes = [
            C.c_uint32, C.c_uint64, C.c_void_p, C.c_void_p, C.c_uint32, C.c_uint32, C.c_void_p,
            C.c_uint32, _u64p, _u64p, _u64p, _u64p, C.c_void_p, C.c_void_p]
        L.qd_read_tns.argtypes = [C.c_char_p, C.c_uint64, C.c_void_p, C.c_uint32, C.c_int,
                                  C.c_int, C.POINTER(TnsTensorC), C.POINTER(TnsErrorC),
                                  C.c_void_p]
        L.qd_tns_free.argtypes = [C.POINTER(TnsTensorC)]
        L.qd_write_tns.argtypes = [C.c_uint32, C.c_uint64, _u32p, _f64p,
                                   C.POINTER(C.c_void_p), C.POINTER(C.c_uint64), C.c_void_p]
        L.qd_text_free.argtypes = [C.c_void_p]
        L.qd_comm_unique_id.argtypes = [C.c_void_p]
        L.qd_comm_create.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_void_p)]
        L.qd_hub_create.argtypes = [C.c_int, C.POINTER(C.c_void_p)]
        L.qd_hub_destroy.argtypes = [C.c_void_p]
        L.qd_comm_create_emulated.argtypes = [C.c_void_p, C.c_int, C.c_void_p,
                                              C.POINTER(C.c_void_p)]
        L.qd_comm_destroy.argtypes = [C.c_void_p]
        L.qd_sharded_transpose_device.argtypes = [
            C.c_void_p, C.c_uint32, _u32p, C.c_uint64, C.c_void_p, C.c_void_p, C.c_void_p,
            C.c_void_p, C.c_uint64, C.POINTER(C.c_uint64), _u32p, C.c_int, C.c_uint32,
            C.c_void_p, C.c_void_p, C.POINTER(ShardStatsC)]
        _lib = L
    return _lib


class ShardStatsC(C.Structure):
    _fields_ = [("exchanged", C.c_int), ("rows_out", C.c_uint64), ("bytes_sent", C.c_uint64),
                ("bytes_received", C.c_uint64), ("exchange_ms", C.c_float)]


def _check(status: int):
    if status == QD_OK:
        return
    L = lib()
    msg = L.qd_last_error().decode()
    if status == QD_INVALID_ARGUMENT:
        raise InvalidArgument(msg)
    if status == QD_OUT_OF_RANGE:
        row, mode = C.c_uint64(0), C.c_uint32(0)
        L.qd_last_error_detail(C.byref(row), C.byref(mode))
        raise OutOfRange(msg, row.value, mode.value)
    raise DeviceError(msg)


def _arr_u32(x) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(x, dtype=np.uint32))


def _ptr_u32(a: np.ndarray):
    return a.ctypes.data_as(_u32p)


# ---------------------------------------------------------------------------
# core types (ordering.hpp, plan.hpp, coo.hpp)
# ---------------------------------------------------------------------------
MAX_RANK = 64


class Ordering:
    """A permutation of 0..r-1, highest comparison priority first."""

    def __init__(self, modes: Sequence[int]):
        modes = [int(m) for m in modes]
        r = len(modes)
        if r == 0 or r > MAX_RANK:
            raise InvalidArgument(f"ordering rank must be in 1..{MAX_RANK}")
        seen = set()
        for m in modes:  # the reference's checks and messages (ordering.cpp:13-31)
            if m < 0 or m >= r:
                raise InvalidArgument(f"ordering contains mode {m} outside 0..{r - 1}")
            if m in seen:
                raise InvalidArgument(f"ordering repeats mode {m}")
            seen.add(m)
        self._m = tuple(modes)

    @staticmethod
    def simple(rank: int) -> "Ordering":
        return Ordering(range(rank))

    def rank(self) -> int:
        return len(self._m)

    def modes(self):
        return list(self._m)

    def at(self, i: int) -> int:
        return self._m[i]

    def position_of(self, m: int) -> int:
        if m not in self._m:
            raise InvalidArgument(f"mode {m} does not appear in the ordering")
        return self._m.index(m)

    def is_simple(self) -> bool:
        return self._m == tuple(range(len(self._m)))

    def __iter__(self):
        return iter(self._m)

    def __len__(self):
        return len(self._m)

    def __eq__(self, o):
        return isinstance(o, Ordering) and o._m == self._m

    def __hash__(self):
        return hash(self._m)

    def __repr__(self):
        return f"Ordering({list(self._m)})"


def _from_chars_u32(tok: str):
    """std::from_chars into an unsigned (32-bit): ASCII digits only, no sign or
    spaces, None on a parse failure or overflow."""
    if not tok or any(c < "0" or c > "9" for c in tok):
        return None
    v = int(tok)
    return v if v < 2**32 else None


def parse_ordering(text: str) -> Ordering:
    """'2134' (1-based digits) or '10,2,1' (ordering.cpp:68-99)."""
    if not text:
        raise InvalidArgument("empty ordering")
    if "," in text:
        vals = []
        for tok in text.split(","):
            if not _from_chars_u32(tok):
                raise InvalidArgument(f"bad ordering element '{tok}'")
            vals.append(int(tok) - 1)
        return Ordering(vals)
    if any(c < "1" or c > "9" for c in text):
        raise InvalidArgument("ordering digits must be 1-9; use the comma form for larger ranks")
    return Ordering([ord(c) - ord("1") for c in text])


def format_ordering(o: Ordering) -> str:
    if o.rank() <= 9:
        return "".join(chr(ord("1") + m) for m in o)
    return ",".join(str(m + 1) for m in o)


@dataclass(frozen=True)
class PlanStep:
    prefix_len: int = 0
    mode: int = 0

    def bucketed(self) -> bool:
        return self.prefix_len > 0


@dataclass
class SortPlan:
    target: Ordering
    steps: List[PlanStep]


@dataclass(frozen=True)
class PlanCost:
    total_passes: int = 0
    bucketed_passes: int = 0


def _ord(target) -> Ordering:
    return target if isinstance(target, Ordering) else Ordering(target)


def _plan_call(fn, target: Ordering, *extra) -> List[PlanStep]:
    t = _arr_u32(target.modes())
    steps = (PlanStepC * 128)()
    n = C.c_uint32(0)
    _check(fn(_ptr_u32(t), len(t), *extra, steps, 128, C.byref(n)))
    return [PlanStep(steps[i].prefix_len, steps[i].mode) for i in range(n.value)]


def quesadilla_plan(target) -> SortPlan:
    target = _ord(target)
    return SortPlan(target, _plan_call(lib().qd_quesadilla_plan, target))


def prefix_plan(target, prefix_len: int) -> SortPlan:
    target = _ord(target)
    return SortPlan(target, _plan_call(lib().qd_prefix_plan, target, prefix_len))


def required_sort_count(source, target) -> int:
    s, t = _ord(source), _ord(target)
    if s.rank() != t.rank():
        raise InvalidArgument("source and target ranks differ")
    out = C.c_int(0)
    a, b = _arr_u32(s.modes()), _arr_u32(t.modes())
    _check(lib().qd_required_sort_count(_ptr_u32(a), _ptr_u32(b), len(a), C.byref(out)))
    return out.value


def apply_transition(current, step: PlanStep) -> Ordering:
    cur = _arr_u32(_ord(current).modes())
    nxt = np.zeros_like(cur)
    _check(lib().qd_apply_transition(_ptr_u32(cur), len(cur),
                                     PlanStepC(step.prefix_len, step.mode), _ptr_u32(nxt)))
    return Ordering(nxt.tolist())


def simulate_plan(plan: SortPlan) -> Ordering:
    o = Ordering.simple(plan.target.rank())
    for s in plan.steps:
        o = apply_transition(o, s)
    return o


def plan_cost(plan: SortPlan) -> PlanCost:
    return PlanCost(len(plan.steps), sum(1 for s in plan.steps if s.bucketed()))


@dataclass(frozen=True)
class SortStrategy:
    kind: str = "quesadilla"  # quesadilla | topk | radix | comparison
    k: int = 0

    @staticmethod
    def quesadilla():
        return SortStrategy("quesadilla", 0)

    @staticmethod
    def top_k(k: int):
        return SortStrategy("topk", int(k))

    @staticmethod
    def splatt_style():
        return SortStrategy("topk", 1)

    @staticmethod
    def full_radix():
        return SortStrategy("radix", 0)

    @staticmethod
    def comparison_sort():
        return SortStrategy("comparison", 0)

    def name(self) -> str:
        return {"quesadilla": "quesadilla", "radix": "radix", "comparison": "comparison"}.get(
            self.kind, f"top{self.k}")


def parse_strategy(name: str) -> SortStrategy:
    """transpose.cpp:22-41"""
    if name == "quesadilla":
        return SortStrategy.quesadilla()
    if name == "radix":
        return SortStrategy.full_radix()
    if name in ("comparison", "qsort"):
        return SortStrategy.comparison_sort()
    if name == "splatt":
        return SortStrategy.splatt_style()
    if len(name) > 3 and name.startswith("top") and (_from_chars_u32(name[3:]) or 0) >= 1:
        return SortStrategy.top_k(int(name[3:]))
    raise InvalidArgument(f"unknown strategy '{name}' (expected quesadilla, top<K>, radix, "
                          "comparison, splatt or qsort)")


def strategy_pass_cost(s: SortStrategy, target) -> PlanCost:
    t = _arr_u32(_ord(target).modes())
    a, b = C.c_int(0), C.c_int(0)
    _check(lib().qd_strategy_pass_cost(KINDS[s.kind], s.k, _ptr_u32(t), len(t), C.byref(a),
                                       C.byref(b)))
    return PlanCost(a.value, b.value)


@dataclass
class CooTensor:
    """N rows of `rank` uint32 coordinates (row-major AoS) + one f64 value each."""

    dims: np.ndarray
    coords: np.ndarray
    values: np.ndarray

    def __post_init__(self):
        self.dims = _arr_u32(self.dims)
        self.coords = _arr_u32(self.coords).reshape(-1)
        self.values = np.ascontiguousarray(np.asarray(self.values, dtype=np.float64)).reshape(-1)

    def rank(self) -> int:
        return len(self.dims)

    def nnz(self) -> int:
        return len(self.values)

    def coord(self, row: int, mode: int) -> int:
        return int(self.coords[row * self.rank() + mode])

    def row(self, i: int):
        r = self.rank()
        return self.coords[i * r:(i + 1) * r]

    def copy(self) -> "CooTensor":
        return CooTensor(self.dims.copy(), self.coords.copy(), self.values.copy())

    def check_valid(self):
        """coo.cpp:8-30"""
        r = self.rank()
        if r == 0:
            raise InvalidArgument("tensor rank must be positive")
        if (self.dims == 0).any():
            raise InvalidArgument("dimensions must be positive")
        if len(self.coords) != r * self.nnz():
            raise InvalidArgument("coordinate storage does not match value count")
        if self.nnz() and (self.coords.reshape(-1, r) >= self.dims).any():
            raise InvalidArgument("coordinate out of range")

    def __eq__(self, o):
        """Bit equality (stricter than the reference's defaulted operator==)."""
        return (isinstance(o, CooTensor) and np.array_equal(self.dims, o.dims)
                and np.array_equal(self.coords, o.coords)
                and np.array_equal(self.values.view(np.uint64), o.values.view(np.uint64)))


def is_sorted_under(t: CooTensor, ord_) -> bool:
    """Host convenience check (coo.cpp:32-49); the device one is is_sorted_device."""
    o = _ord(ord_)
    if o.rank() != t.rank():
        raise InvalidArgument("ordering rank does not match tensor rank")
    if t.nnz() < 2:
        return True
    c = t.coords.reshape(-1, t.rank())[:, o.modes()].astype(np.int64)
    d = c[1:] - c[:-1]
    nz = d != 0
    first = np.where(nz.any(1), nz.argmax(1), 0)
    return bool((d[np.arange(len(d)), first] >= 0).all())


@dataclass
class ParallelConfig:
    workers: int = 1


@dataclass
class TransposeOptions:
    verify_input: bool = False
    parallel: ParallelConfig = field(default_factory=ParallelConfig)
    pass_log: Optional[list] = None
    # when a list: receives the output's leading-mode run starts + nnz
    boundaries: Optional[list] = None


class Workspace:
    """Device workspace (sort.hpp:14-21): cached HBM buffers on one GPU.
    Reusable across calls, never concurrently."""

    def __init__(self, device: int = 0):
        h = C.c_void_p()
        _check(lib().qd_workspace_create(device, C.byref(h)))
        self._h = h

    @property
    def handle(self):
        return self._h

    def bytes(self) -> int:
        return int(lib().qd_workspace_bytes(self._h))

    def launches(self) -> int:
        return int(lib().qd_workspace_launches(self._h))

    def slices(self) -> int:
        """Slices the last synchronous host-buffer call was pipelined in (1: whole)."""
        return int(lib().qd_workspace_slices(self._h))

    PROFILE_CLASSES = ("scatter", "hist", "local", "runs", "other")

    def profile(self, enable: bool = True):
        """Live per-kernel-class CUDA-event timing inside the library."""
        lib().qd_profile_enable(self._h, int(enable))

    def profile_reset(self):
        lib().qd_profile_reset(self._h)

    def profile_stats(self) -> dict:
        out = {}
        for i, name in enumerate(self.PROFILE_CLASSES):
            n, ms, b = C.c_uint64(0), C.c_double(0), C.c_double(0)
            _check(lib().qd_profile_get(self._h, i, C.byref(n), C.byref(ms), C.byref(b)))
            out[name] = {"launches": n.value, "ms": ms.value, "bytes": b.value}
        return out

    def synchronize(self):
        """Wait for this workspace's asynchronous calls (transpose_inplace_async)."""
        _check(lib().qd_workspace_synchronize(self._h))
        self._pending = []

    def close(self):
        if self._h:
            lib().qd_workspace_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_default_ws = {}


def _ws(ws):
    if ws is not None:
        return ws
    import threading
    key = threading.get_ident()
    if key not in _default_ws:
        _default_ws[key] = Workspace(0)
    return _default_ws[key]


def _options(opts: Optional[TransposeOptions], nnz: int):
    o = OptionsC()
    keep = {}
    if opts is None:
        o.workers = 1
        return o, keep
    o.verify_input = int(bool(opts.verify_input))
    o.workers = int(opts.parallel.workers)
    if opts.pass_log is not None:
        keep["log"] = (PlanStepC * 4096)()
        keep["n"] = C.c_uint32(0)
        o.pass_log = keep["log"]
        o.pass_log_capacity = 4096
        o.pass_log_len = C.pointer(keep["n"])
    if opts.boundaries is not None:
        keep["b"] = np.zeros(nnz + 1, np.uint64)
        keep["nb"] = C.c_uint64(0)
        o.boundaries = keep["b"].ctypes.data_as(C.POINTER(C.c_uint64))
        o.n_boundaries = C.pointer(keep["nb"])
    return o, keep


def _finish_options(opts, keep):
    if opts is None:
        return
    if opts.pass_log is not None:
        opts.pass_log.extend(PlanStep(keep["log"][i].prefix_len, keep["log"][i].mode)
                             for i in range(keep["n"].value))
    if opts.boundaries is not None:
        opts.boundaries.extend(int(x) for x in keep["b"][: keep["nb"].value])


def transpose_inplace(tensor: CooTensor, target, strategy: SortStrategy = SortStrategy(),
                      ws: Optional[Workspace] = None,
                      opts: Optional[TransposeOptions] = None) -> None:
    """transpose.hpp:59-61 — reorder `tensor` (simply sorted) into `target` order, in place.
    The tensor is left untouched when an exception is raised."""
    target = _ord(target)
    if target.rank() != tensor.rank():
        raise InvalidArgument("target ordering rank does not match tensor")
    w = _ws(ws)
    o, keep = _options(opts, tensor.nnz())
    t = _arr_u32(target.modes())
    _check(lib().qd_transpose_inplace(
        tensor.rank(), _ptr_u32(tensor.dims), tensor.nnz(), _ptr_u32(tensor.coords),
        tensor.values.ctypes.data_as(_f64p), _ptr_u32(t), KINDS[strategy.kind], strategy.k,
        C.byref(o), w.handle))
    _finish_options(opts, keep)


def transpose_inplace_async(tensor: CooTensor, target, strategy: SortStrategy = SortStrategy(),
                            ws: Optional[Workspace] = None,
                            opts: Optional[TransposeOptions] = None) -> None:
    """transpose_inplace that returns after enqueueing the input copy; the
    device work and output copy complete by ws.synchronize(), which raises the
    first device-side error (that call's tensor untouched).  Argument errors
    raise at once.  The tensor's arrays must stay alive (and should be
    pinned) until then."""
    target = _ord(target)
    if target.rank() != tensor.rank():
        raise InvalidArgument("target ordering rank does not match tensor")
    w = _ws(ws)
    o, keep = _options(opts, tensor.nnz())
    t = _arr_u32(target.modes())
    _check(lib().qd_transpose_inplace_async(
        tensor.rank(), _ptr_u32(tensor.dims), tensor.nnz(), _ptr_u32(tensor.coords),
        tensor.values.ctypes.data_as(_f64p), _ptr_u32(t), KINDS[strategy.kind], strategy.k,
        C.byref(o), w.handle))
    _finish_options(opts, keep)
    if not hasattr(w, "_pending"):
        w._pending = []
    w._pending.append(tensor)  # keep the host arrays alive until synchronize()


def transpose(tensor: CooTensor, target, strategy: SortStrategy = SortStrategy(),
              opts: Optional[TransposeOptions] = None, ws: Optional[Workspace] = None) -> CooTensor:
    """transpose.hpp:64-66 — copying wrapper."""
    out = tensor.copy()
    transpose_inplace(out, target, strategy, ws, opts)
    return out


def full_radix_transpose(tensor, target, opts=None, ws=None):
    return transpose(tensor, target, SortStrategy.full_radix(), opts, ws)


def comparison_transpose(tensor, target, ws=None):
    return transpose(tensor, target, SortStrategy.comparison_sort(), None, ws)


def topk_transpose(tensor, target, k, opts=None, ws=None):
    return transpose(tensor, target, SortStrategy.top_k(k), opts, ws)


def partial_sort(tensor: CooTensor, prefix: Sequence[int], mode: int,
                 ws: Optional[Workspace] = None) -> None:
    """sort.hpp:32-33 — one stable histogram pass on `mode`, bucketed on `prefix`."""
    w = _ws(ws)
    p = _arr_u32(list(prefix) or [0])
    _check(lib().qd_partial_sort(tensor.rank(), _ptr_u32(tensor.dims), tensor.nnz(),
                                 _ptr_u32(tensor.coords), tensor.values.ctypes.data_as(_f64p),
                                 _ptr_u32(p), len(prefix), int(mode), w.handle))


def sort_rows_by(tensor: CooTensor, row_begin: int, row_end: int, key_modes: Sequence[int],
                 ws: Optional[Workspace] = None) -> None:
    """sort.hpp:38-39 — stable sort of rows [row_begin, row_end) by key_modes
    (priority order), in place; no range check, like the reference."""
    w = _ws(ws)
    k = _arr_u32(list(key_modes) or [0])
    _check(lib().qd_sort_rows_by(tensor.rank(), _ptr_u32(tensor.dims), tensor.nnz(),
                                 _ptr_u32(tensor.coords), tensor.values.ctypes.data_as(_f64p),
                                 int(row_begin), int(row_end), _ptr_u32(k), len(key_modes),
                                 w.handle))


def canonicalize(tensor: CooTensor, ws: Optional[Workspace] = None) -> None:
    """read_tns's canonicalisation (io.cpp:36-38): stable sort into the simple
    ordering from any row order."""
    sort_rows_by(tensor, 0, tensor.nnz(), list(range(tensor.rank())), ws)


def relabel_target(source, target) -> Ordering:
    """planner.hpp:51-55."""
    s, t = _ord(source), _ord(target)
    if s.rank() != t.rank():
        raise InvalidArgument("source and target ranks differ")
    out = np.zeros(t.rank(), np.uint32)
    _check(lib().qd_relabel_target(_ptr_u32(_arr_u32(s.modes())), _ptr_u32(_arr_u32(t.modes())),
                                   t.rank(), _ptr_u32(out)))
    return Ordering([int(x) for x in out])


def parallel_partial_sort(tensor, prefix, mode, ws=None, cfg: ParallelConfig = ParallelConfig()):
    """parallel.hpp:35-37 — identical output; the GPU is the parallelism."""
    if cfg.workers == 0:
        raise InvalidArgument("worker count must be at least 1")
    partial_sort(tensor, prefix, mode, ws)


# ---------------------------------------------------------------------------
# device-resident entry points (raw device pointers, e.g. torch data_ptr())
# ---------------------------------------------------------------------------

def transpose_device(rank: int, dims, nnz: int, coords_in: int, values_in: int, coords_out: int,
                     values_out: int, target, strategy: SortStrategy = SortStrategy(),
                     ws: Optional[Workspace] = None, stream: int = 0,
                     opts: Optional[TransposeOptions] = None) -> None:
    """Out-of-place transpose of device buffers (pointers as ints)."""
    w = _ws(ws)
    d = _arr_u32(dims)
    t = _arr_u32(_ord(target).modes())
    o, keep = _options(opts, 0)
    if opts is not None and opts.boundaries is not None:
        raise InvalidArgument("use transpose_device_boundaries for device boundaries")
    _check(lib().qd_transpose_device(rank, _ptr_u32(d), nnz, C.c_void_p(coords_in),
                                     C.c_void_p(values_in), C.c_void_p(coords_out),
                                     C.c_void_p(values_out), _ptr_u32(t), KINDS[strategy.kind],
                                     strategy.k, C.byref(o), w.handle, C.c_void_p(stream)))
    _finish_options(opts, keep)


def transpose_device_boundaries(rank, dims, nnz, coords_in, values_in, coords_out, values_out,
                                target, boundaries_out: int, strategy=SortStrategy(), ws=None,
                                stream: int = 0) -> int:
    """As transpose_device, also writing the leading-mode run starts + nnz to the device
    buffer `boundaries_out` (capacity nnz + 1 uint64); returns the entry count."""
    w = _ws(ws)
    d = _arr_u32(dims)
    t = _arr_u32(_ord(target).modes())
    o = OptionsC()
    o.workers = 1
    nb = C.c_uint64(0)
    o.boundaries = C.cast(C.c_void_p(boundaries_out), C.POINTER(C.c_uint64))
    o.n_boundaries = C.pointer(nb)
    _check(lib().qd_transpose_device(rank, _ptr_u32(d), nnz, C.c_void_p(coords_in),
                                     C.c_void_p(values_in), C.c_void_p(coords_out),
                                     C.c_void_p(values_out), _ptr_u32(t), KINDS[strategy.kind],
                                     strategy.k, C.byref(o), w.handle, C.c_void_p(stream)))
    return nb.value


def partial_sort_device(rank, dims, nnz, coords_in, values_in, coords_out, values_out, prefix,
                        mode, ws=None, stream=0):
    w = _ws(ws)
    d = _arr_u32(dims)
    p = _arr_u32(list(prefix) or [0])
    _check(lib().qd_partial_sort_device(rank, _ptr_u32(d), nnz, C.c_void_p(coords_in),
                                        C.c_void_p(values_in), C.c_void_p(coords_out),
                                        C.c_void_p(values_out), _ptr_u32(p), len(prefix), mode,
                                        w.handle, C.c_void_p(stream)))


def sort_rows_by_device(rank, dims, nnz, coords_in, values_in, coords_out, values_out,
                        row_begin, row_end, key_modes, ws=None, stream=0):
    w = _ws(ws)
    d = _arr_u32(dims)
    k = _arr_u32(list(key_modes) or [0])
    _check(lib().qd_sort_rows_by_device(rank, _ptr_u32(d), nnz, C.c_void_p(coords_in),
                                        C.c_void_p(values_in), C.c_void_p(coords_out),
                                        C.c_void_p(values_out), int(row_begin), int(row_end),
                                        _ptr_u32(k), len(key_modes), w.handle, C.c_void_p(stream)))


def is_sorted_device(rank, nnz, coords, order, ws=None, stream=0) -> bool:
    w = _ws(ws)
    o = _arr_u32(_ord(order).modes())
    out = C.c_int(0)
    _check(lib().qd_is_sorted_device(rank, nnz, C.c_void_p(coords), _ptr_u32(o), C.byref(out),
                                     w.handle, C.c_void_p(stream)))
    return bool(out.value)


def bucket_starts_device(rank, nnz, coords, modes, starts_out: int, ws=None, stream=0) -> int:
    w = _ws(ws)
    m = _arr_u32(list(modes) or [0])
    n = C.c_uint64(0)
    _check(lib().qd_bucket_starts_device(rank, nnz, C.c_void_p(coords), _ptr_u32(m), len(modes),
                                         C.c_void_p(starts_out), C.byref(n), w.handle,
                                         C.c_void_p(stream)))
    return n.value


def csf_device(coords, rank: int, order, ws=None, stream=0):
    """CSF level arrays of a device tensor sorted under `order` (torch int32
    coords, nnz*rank): returns (pos, crd) lists of torch tensors, level k =
    runs of equal order[0..k] (qd_csf_device)."""
    import torch
    w = _ws(ws)
    o = _arr_u32(_ord(order).modes())
    nnz = coords.numel() // rank
    pos = [torch.empty(max(nnz + 1, 2), dtype=torch.int64, device=coords.device)
           for _ in range(rank)]
    crd = [torch.empty(max(nnz, 1), dtype=torch.int32, device=coords.device) for _ in range(rank)]
    pp = (C.c_void_p * rank)(*[p.data_ptr() for p in pos])
    cp = (C.c_void_p * rank)(*[c.data_ptr() for c in crd])
    nf = (C.c_uint64 * rank)()
    _check(lib().qd_csf_device(rank, nnz, C.c_void_p(coords.data_ptr()), _ptr_u32(o), pp, cp, nf,
                               w.handle, C.c_void_p(stream)))
    n = [int(x) for x in nf]
    pos = [pos[0][:2]] + [pos[k][: n[k - 1] + 1] for k in range(1, rank)]
    crd = [crd[k][: n[k]] for k in range(rank)]
    return pos, crd


def mode_histogram_device(rank, nnz, coords, mode, dim, hist_out: int, ws=None, stream=0):
    w = _ws(ws)
    _check(lib().qd_mode_histogram_device(rank, nnz, C.c_void_p(coords), mode, dim,
                                          C.c_void_p(hist_out), w.handle, C.c_void_p(stream)))


def partition_rows_device(rank, nnz, coords_in, values_in, mode, dim, lookup, n_parts,
                          coords_out, values_out, ws=None, stream=0) -> List[int]:
    w = _ws(ws)
    counts = (C.c_uint64 * n_parts)()
    _check(lib().qd_partition_rows_device(rank, nnz, C.c_void_p(coords_in), C.c_void_p(values_in),
                                          mode, dim, C.c_void_p(lookup), n_parts,
                                          C.c_void_p(coords_out), C.c_void_p(values_out), counts,
                                          w.handle, C.c_void_p(stream)))
    return [int(x) for x in counts]


def partition_rows_to_peers_device(rank, nnz, coords_in, values_in, mode, dim, lookup, n_parts,
                                   peer_coords, peer_values, peer_row_offsets, ws=None,
                                   stream=0) -> List[int]:
    """qd_partition_rows_to_peers_device: part p's rows written to device
    addresses peer_coords[p] / peer_values[p] from row peer_row_offsets[p]."""
    w = _ws(ws)
    counts = (C.c_uint64 * n_parts)()
    arr = lambda xs: (C.c_uint64 * n_parts)(*[int(x) for x in xs])  # noqa: E731
    _check(lib().qd_partition_rows_to_peers_device(
        rank, nnz, C.c_void_p(coords_in), C.c_void_p(values_in), mode, dim, C.c_void_p(lookup),
        n_parts, arr(peer_coords), arr(peer_values), arr(peer_row_offsets), counts, w.handle,
        C.c_void_p(stream)))
    return [int(x) for x in counts]




# ---- .tns text format (io.hpp:24-47) ------------------------------------------

def read_tns_text(text: bytes, declared_dims=None, canonicalize: bool = True,
                  ws: Optional[Workspace] = None) -> CooTensor:
    """read_tns (io.cpp:42-126) over a file's bytes, parsed on the GPU
    (qd_read_tns).  Raises ParseError exactly where and with the text the
    reference would; InvalidArgument for check_valid failures (coo.cpp:8-16)."""
    L = lib()
    w = _ws(ws)
    decl = None if declared_dims is None else _arr_u32(declared_dims)
    out, err = TnsTensorC(), TnsErrorC()
    st = L.qd_read_tns(bytes(text), len(text),
                       None if decl is None or len(decl) == 0 else decl.ctypes.data,
                       0 if decl is None else len(decl), int(decl is not None),
                       int(bool(canonicalize)), C.byref(out), C.byref(err), w.handle)
    if st == QD_PARSE_ERROR:
        raise ParseError(L.qd_last_error().decode(), err.line, err.kind, err.field)
    _check(st)
    # the rows stay in the library's buffers (no copy); freed with the arrays
    owner = _TnsOwner(out)
    r, n = out.rank, out.nnz
    dims = np.ctypeslib.as_array(out.dims, (r,)).copy() if r else np.zeros(0, np.uint32)
    coords = owner.view(out.coords, C.c_uint32, n * r, np.uint32)
    values = owner.view(out.values, C.c_double, n, np.float64)
    return CooTensor(dims, coords, values)


class _TnsOwner:
    """Owns a qd_tns_tensor; numpy views keep it alive, qd_tns_free on collection."""

    def __init__(self, t):
        self.t = t

    def view(self, ptr, ctype, count, dtype):
        if count == 0:
            return np.zeros(0, dtype)
        buf = (ctype * count).from_address(C.addressof(ptr.contents))
        buf._owner = self
        return np.frombuffer(buf, dtype=dtype)

    def __del__(self):
        try:
            lib().qd_tns_free(C.byref(self.t))
        except Exception:
            pass


def read_tns(path, declared_dims=None, canonicalize: bool = True,
             ws: Optional[Workspace] = None) -> CooTensor:
    """read_tns(path, ReadOptions) (io.hpp:40-41); the file is read on the host,
    everything after that runs on the GPU."""
    try:
        with open(path, "rb") as f:
            text = f.read()
    except OSError:
        raise RuntimeError(f"cannot open '{path}' for reading")
    return read_tns_text(text, declared_dims, canonicalize, ws)


def write_tns_text(tensor: CooTensor, ws: Optional[Workspace] = None) -> memoryview:
    """write_tns's file contents (io.cpp:128-152), formatted on the GPU
    (qd_write_tns): 1-based indices, shortest round-trip values.  Returns a
    read-only view of the library's buffer (no copy; bytes(...) copies)."""
    L = lib()
    w = _ws(ws)
    t = tensor
    p, n = C.c_void_p(), C.c_uint64(0)
    c = np.ascontiguousarray(t.coords, np.uint32)
    v = np.ascontiguousarray(t.values, np.float64)
    _check(L.qd_write_tns(t.rank(), t.nnz(), c.ctypes.data_as(_u32p), v.ctypes.data_as(_f64p),
                          C.byref(p), C.byref(n), w.handle))
    if not n.value:
        L.qd_text_free(p)
        return memoryview(b"")
    buf = (C.c_char * n.value).from_address(p.value)
    buf._owner = _TextOwner(p.value)
    return memoryview(buf).cast("B").toreadonly()


class _TextOwner:
    def __init__(self, addr):
        self.addr = addr

    def __del__(self):
        try:
            lib().qd_text_free(C.c_void_p(self.addr))
        except Exception:
            pass


def write_tns(tensor: CooTensor, path, ws: Optional[Workspace] = None) -> None:
    """write_tns(tensor, path) (io.hpp:47): text formatted on the GPU, written
    to the file straight from the library's buffer."""
    try:
        f = open(path, "wb")
    except OSError:
        raise RuntimeError(f"cannot open '{path}' for writing")
    with f:
        f.write(write_tns_text(tensor, ws))


__all__ = [n for n in dir() if not n.startswith("_")]


# --- sharded transpose over NCCL (qd_sharded_transpose_device) ----

def comm_unique_id() -> bytes:
    """ncclGetUniqueId (128 bytes) for rank 0 to broadcast to every rank."""
    buf = (C.c_uint8 * 128)()
    _check(lib().qd_comm_unique_id(buf))
    return bytes(buf)


class Hub:
    """Emulated ranks (tests): threads of one process on one device."""

    def __init__(self, nranks: int):
        h = C.c_void_p()
        _check(lib().qd_hub_create(nranks, C.byref(h)))
        self._h = h

    def close(self):
        if getattr(self, "_h", None):
            lib().qd_hub_destroy(self._h)
            self._h = None


class Comm:
    """One rank of a sharded-transpose communicator: NCCL (ncclCommInitRank on
    `device`, from the 128-byte unique id of rank 0) or, with `hub`, the
    emulated transport (ws = this rank's workspace)."""

    def __init__(self, nranks: int = 1, rank: int = 0, device: int = 0, unique_id: bytes = None,
                 hub: "Hub" = None, ws: "Workspace" = None):
        h = C.c_void_p()
        if hub is not None:
            _check(lib().qd_comm_create_emulated(hub._h, rank, ws.handle, C.byref(h)))
        else:
            uid = (C.c_uint8 * 128).from_buffer_copy(unique_id or comm_unique_id())
            _check(lib().qd_comm_create(uid, nranks, rank, device, C.byref(h)))
        self._h = h
        self.nranks, self.rank = nranks if hub is None else None, rank

    def close(self):
        if getattr(self, "_h", None):
            lib().qd_comm_destroy(self._h)
            self._h = None


def sharded_transpose_device(comm: Comm, rank: int, dims, nnz: int, coords_in: int,
                             values_in: int, coords_out: int, values_out: int, out_capacity: int,
                             target, strategy: SortStrategy = SortStrategy(),
                             ws: Optional[Workspace] = None, stream: int = 0):
    """This rank's slice of the global input -> its slice of the global output
    (device pointers as ints; collective over `comm`).  Returns (rows_out,
    stats dict)."""
    w = _ws(ws)
    d = _arr_u32(dims)
    t = _arr_u32(_ord(target).modes())
    n_out = C.c_uint64(0)
    st = ShardStatsC()
    _check(lib().qd_sharded_transpose_device(
        comm._h, rank, _ptr_u32(d), nnz, C.c_void_p(coords_in), C.c_void_p(values_in),
        C.c_void_p(coords_out), C.c_void_p(values_out), out_capacity, C.byref(n_out),
        _ptr_u32(t), KINDS[strategy.kind], strategy.k, w.handle, C.c_void_p(stream),
        C.byref(st)))
    return n_out.value, {"exchanged": bool(st.exchanged), "rows_out": st.rows_out,
                         "bytes_sent": st.bytes_sent, "bytes_received": st.bytes_received,
                         "exchange_ms": st.exchange_ms}
