"""Python mirror of the reference ``tridpart`` API for the partition-solve path.

Same names, argument meaning and error behaviour as the reference C++20
headers (/root/reference/proj/include/tridpart), so code and tests written
against the reference read the same here:

    sys = generate_system(10_000, 1)            # host arrays
    x = solve_partition(sys, RecursionPolicy([4]))
    residual_inf(sys, x)

Every solve runs on the B200 through the C-ABI (``include/tridpart_b200.h``);
the predictors run as host C++ in the same library (bit-exact with the
reference, see ``tp_knn.cpp``). Inputs may be numpy arrays (host path:
H2D, device solve, D2H) or contiguous float64 CUDA torch tensors (device
path, on torch's current stream).
"""
from __future__ import annotations

import ctypes as C
import json
import os
import threading
from dataclasses import dataclass, field
from typing import Callable, Dict, List, Optional, Sequence

import numpy as np

from . import _lib
from ._lib import TpError, lib

_D = C.POINTER(C.c_double)
_I64 = C.POINTER(C.c_int64)
_I32 = C.POINTER(C.c_int32)

kPivotFloor = 1e-30          # tridiagonal.hpp:15-16
kMaxRecursionDepth = 4       # policy.hpp:11
kModelFormatVersion = 1      # io.hpp:24
kObservationsHeader = "N,precision,device,streams,m,time_ms,is_opt,corrected_m,opt_R"  # io.hpp:21-22


# ----------------------------------------------------------------- errors.hpp
class Error(RuntimeError):
    """Base of all library errors (errors.hpp:10-13)."""


class ZeroPivotError(Error):
    """errors.hpp:16-24. ``row`` is the row within the partition level's
    system (``level`` 0 = the input system)."""

    def __init__(self, row: int, level: int = 0, msg: Optional[str] = None):
        super().__init__(msg or f"zero pivot at row {row}")
        self._row = int(row)
        self.level = int(level)

    def row(self) -> int:
        return self._row


class InvalidSizeError(Error):
    pass


class DepthOutOfRangeError(Error):
    pass


class EmptyTrainingSetError(Error):
    def __init__(self, msg: str = "training set is empty"):
        super().__init__(msg)


class KTooLargeError(Error):
    pass


class MalformedHeaderError(Error):
    pass


class BadNumberError(Error):
    pass


class VersionMismatchError(Error):
    pass


class SchemaError(Error):
    pass


class DeviceError(Error):
    """CUDA failure inside the solver (no reference analogue)."""


def _raise(status: int, err: TpError):
    if status == _lib.OK:
        return
    msg = err.msg.decode(errors="replace")
    if status == _lib.ZERO_PIVOT:
        raise ZeroPivotError(err.row, err.level, msg)
    cls = {
        _lib.INVALID_SIZE: InvalidSizeError,
        _lib.DEPTH_OUT_OF_RANGE: DepthOutOfRangeError,
        _lib.EMPTY_TRAINING_SET: EmptyTrainingSetError,
        _lib.K_TOO_LARGE: KTooLargeError,
        _lib.MALFORMED_HEADER: MalformedHeaderError,
        _lib.BAD_NUMBER: BadNumberError,
        _lib.IO: Error,
        _lib.CUDA: DeviceError,
        _lib.INVALID_ARGUMENT: ValueError,
    }.get(status, Error)
    raise cls(msg)


def _call(fn, *args):
    err = TpError()
    st = fn(*args, C.byref(err))
    _raise(st, err)


# ----------------------------------------------------------------- contexts
class Context:
    """One tp_ctx: device, stream, workspace and CUDA-graph cache."""

    def __init__(self, device: int = 0):
        self.device = int(device)
        h = C.c_void_p()
        _call(lib.tp_ctx_create, self.device, C.byref(h))
        self.handle = h

    def close(self):
        if self.handle:
            lib.tp_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_stream(self, stream_ptr: int):
        _call(lib.tp_ctx_set_stream, self.handle, C.c_void_p(stream_ptr))

    def set_graphs(self, enabled: bool):
        _call(lib.tp_ctx_set_graphs, self.handle, 1 if enabled else 0)

    def set_grid(self, enabled: bool = True, min_rows: int = 80_000):
        """The one-kernel grid solve of one-level policies (k_grid_solve): on/off
        and the smallest n it takes (below ~8e4 rows the level path is faster)."""
        _call(lib.tp_ctx_set_grid, self.handle, 1 if enabled else 0, int(min_rows))

    def last_launch_count(self) -> int:
        return int(lib.tp_ctx_last_launch_count(self.handle))

    def last_kernels(self) -> list:
        """The last solve's kernels, "name:Llevel" in launch order (k_reset not listed)."""
        n = int(lib.tp_ctx_last_kernels(self.handle, None, 0))
        buf = C.create_string_buffer(n + 1)
        lib.tp_ctx_last_kernels(self.handle, buf, n + 1)
        return [k for k in buf.value.decode().split(",") if k]


_tls = threading.local()


def context(device: Optional[int] = None) -> Context:
    """Per-thread default context (the reference is reentrant; a tp_ctx is not)."""
    if device is None:
        device = 0
        try:
            import torch
            if torch.cuda.is_available():
                device = torch.cuda.current_device()
        except ImportError:
            pass
    cache = getattr(_tls, "ctx", None)
    if cache is None:
        cache = _tls.ctx = {}
    if device not in cache:
        cache[device] = Context(device)
    return cache[device]


def torch_stream() -> int:
    """cudaStream_t of torch's current stream. torch's default stream is the
    legacy NULL stream: pass cudaStreamLegacy (0x1) for it, because a NULL
    stream argument means "the context's own stream" in the C-ABI."""
    import torch

    return torch.cuda.current_stream().cuda_stream or 0x1


# ----------------------------------------------------------- tridiagonal.hpp
def _is_torch(a) -> bool:
    return type(a).__module__.startswith("torch")


class TridiagonalSystem:
    """SoA system (tridiagonal.hpp:22-46): row i reads
    sub[i]*x[i-1] + diag[i]*x[i] + super[i]*x[i+1] = rhs[i].

    Element type as TridiagonalSystem<Real>: float64 by default, float32 when
    ``dtype`` is float32 or the arrays already are float32."""

    def __init__(self, sub, diag, super, rhs, dtype=None):  # noqa: A002 - reference field name
        if _is_torch(diag):
            self.sub, self.diag, self.super, self.rhs = sub, diag, super, rhs
        else:
            if dtype is None:
                dtype = np.float32 if getattr(diag, "dtype", None) == np.float32 else np.float64
            self.sub = np.ascontiguousarray(sub, dtype=dtype)
            self.diag = np.ascontiguousarray(diag, dtype=dtype)
            self.super = np.ascontiguousarray(super, dtype=dtype)
            self.rhs = np.ascontiguousarray(rhs, dtype=dtype)

    @property
    def is_f32(self) -> bool:
        if _is_torch(self.diag):
            return str(self.diag.dtype) == "torch.float32"
        return self.diag.dtype == np.float32

    def size(self) -> int:
        return int(self.diag.shape[0])

    @property
    def on_device(self) -> bool:
        return _is_torch(self.diag) and self.diag.is_cuda

    def well_formed(self) -> bool:
        n = self.size()
        if n == 0:
            return False
        if any(int(v.shape[0]) != n for v in (self.sub, self.super, self.rhs)):
            return False
        return float(self.sub[0]) == 0.0 and float(self.super[n - 1]) == 0.0

    def strictly_dominant(self) -> bool:
        if self.on_device:
            import torch
            return bool(torch.all(self.diag.abs() > self.sub.abs() + self.super.abs()))
        return bool(np.all(np.abs(self.diag) > np.abs(self.sub) + np.abs(self.super)))

    def check_shape(self):
        """sub, super and rhs must have diag's length: the C-ABI reads n
        elements of each (the reference indexes them up to size())."""
        n = self.size()
        if any(int(v.shape[0]) != n for v in (self.sub, self.super, self.rhs)):
            raise InvalidSizeError("sub, diag, super and rhs must have the same length")

    def _host_ptrs(self):
        self.check_shape()
        return [C.c_void_p(a.ctypes.data) for a in (self.sub, self.diag, self.super, self.rhs)]

    def _dev_ptrs(self):
        self.check_shape()
        want = str(self.diag.dtype)
        for a in (self.sub, self.diag, self.super, self.rhs):
            if not (a.is_cuda and a.is_contiguous()) or str(a.dtype) != want or \
                    want not in ("torch.float64", "torch.float32"):
                raise ValueError("device systems need contiguous float64 (or float32) CUDA tensors "
                                 "of one dtype")
        return [C.c_void_p(a.data_ptr()) for a in (self.sub, self.diag, self.super, self.rhs)]


Tridiagonal = TridiagonalSystem


def generate_system(n: int, seed: int, delta: float = 1.5, device: bool = False,
                    row0: int = 0, n_global: Optional[int] = None, dtype: str = "float64"):
    """generate_system (bench.hpp:68-93).

    Host (``device=False``, the default): BIT-IDENTICAL to the reference — the
    library's C++ generator (``tp_generate_system_f64``) runs std::mt19937_64(seed)
    with libstdc++'s uniform_real_distribution / bernoulli_distribution in the
    reference's draw order. Whole float64 systems only.

    ``device=True``: generated ON THE DEVICE from a counter-based hash with the
    same distributions (NOT bit-identical; throughput runs), returned as CUDA
    tensors; ``row0`` / ``n_global`` select one shard's slice of a global
    system and ``dtype`` may be float32."""
    if not device:
        if row0 != 0 or n_global not in (None, n) or dtype not in ("float64", "f64", np.float64):
            raise ValueError("the bit-identical host generator builds whole float64 systems; "
                             "use device=True for shard slices or float32")
        arrs = [np.empty(max(int(n), 0), dtype=np.float64) for _ in range(4)]
        _call(lib.tp_generate_system_f64, int(n), C.c_uint64(seed), float(delta),
              *[C.c_void_p(a.ctypes.data) for a in arrs])
        return TridiagonalSystem(*arrs)
    import torch

    n_global = n if n_global is None else n_global
    ctx = context()
    tdt = torch.float32 if dtype in ("float32", "f32", np.float32) else torch.float64
    arrs = [torch.empty(n, dtype=tdt, device=f"cuda:{ctx.device}") for _ in range(4)]
    stream = torch_stream()
    fn = lib.tp_generate_system_f32_dev if tdt == torch.float32 else lib.tp_generate_system_f64_dev
    _call(fn, ctx.handle, n, row0, n_global, C.c_uint64(seed), delta,
          *[C.c_void_p(a.data_ptr()) for a in arrs], C.c_void_p(stream))
    return TridiagonalSystem(*arrs)


def residual_inf(sys: TridiagonalSystem, x) -> float:
    """||Ax - d||_inf / max(1, ||d||_inf) (tridiagonal.hpp:74-87)."""
    if sys.on_device:
        ctx = context()
        out = C.c_double()
        fn = lib.tp_residual_inf_f32_dev if sys.is_f32 else lib.tp_residual_inf_f64_dev
        if not (x.is_cuda and x.is_contiguous() and x.dtype == sys.diag.dtype and
                int(x.shape[0]) == sys.size()):
            raise ValueError("x must be a contiguous CUDA tensor of the system's dtype and size")
        _call(fn, ctx.handle, *sys._dev_ptrs(), sys.size(),
              C.c_void_p(x.data_ptr()), C.byref(out), C.c_void_p(torch_stream()))
        return float(out.value)
    x = np.asarray(x, dtype=sys.diag.dtype)
    ax = sys.diag * x
    ax[1:] += sys.sub[1:] * x[:-1]
    ax[:-1] += sys.super[:-1] * x[1:]
    num = float(np.max(np.abs(ax - sys.rhs))) if x.size else 0.0
    den = max(1.0, float(np.max(np.abs(sys.rhs))) if x.size else 1.0)
    return num / den


def thomas_solve(sys: TridiagonalSystem) -> np.ndarray:
    """thomas_solve (tridiagonal.hpp:52-72): same solution, computed by the
    device finishing solver."""
    ctx = context()
    n = sys.size()
    x = np.empty(n, dtype=sys.diag.dtype)
    fn = lib.tp_thomas_solve_f32 if sys.is_f32 else lib.tp_thomas_solve_f64
    _call(fn, ctx.handle, *sys._host_ptrs(), n, C.c_void_p(x.ctypes.data))
    return x


# ------------------------------------------------------------- partition.hpp
@dataclass(frozen=True)
class Block:
    start: int = 0
    end: int = 0

    def length(self) -> int:
        return self.end - self.start


@dataclass
class PartitionPlan:
    n: int = 0
    m: int = 0
    blocks: List[Block] = field(default_factory=list)


def make_plan(n: int, m: int) -> PartitionPlan:
    """make_plan (partition.hpp:30-49)."""
    k = C.c_int64()
    _call(lib.tp_make_plan, n, m, None, C.byref(k))
    b = np.empty(k.value + 1, dtype=np.int64)
    _call(lib.tp_make_plan, n, m, b.ctypes.data_as(_I64), C.byref(k))
    return PartitionPlan(n, m, [Block(int(b[j]), int(b[j + 1])) for j in range(k.value)])


@dataclass
class ReducedBlock:
    """partition.hpp:52-71: eq1 / eq2 of a block plus its up-sweep vectors
    (indexed by offset from ``start``; the entry at len-1 is unused)."""
    start: int = 0
    end: int = 0
    alpha1: float = 0.0
    beta1: float = 0.0
    gamma1: float = 0.0
    delta1: float = 0.0
    alpha2: float = 0.0
    beta2: float = 0.0
    gamma2: float = 0.0
    delta2: float = 0.0
    a: np.ndarray = None
    beta: np.ndarray = None
    gamma: np.ndarray = None
    delta: np.ndarray = None


def reduce_block(sys: TridiagonalSystem, blk: Block) -> ReducedBlock:
    """reduce_block (partition.hpp:77-126), on the device with the reference's
    own sequential arithmetic (tp_reduce_block_*)."""
    start, end = int(blk.start), int(blk.end)
    ln = end - start
    if ln < 2 or end > sys.size() or start < 0:
        raise InvalidSizeError("block length must be >= 2")
    dt = np.float32 if sys.is_f32 else np.float64
    eq = np.empty(8, dtype=dt)
    vec = [np.zeros(ln, dtype=dt) for _ in range(4)]
    fn = lib.tp_reduce_block_f32 if sys.is_f32 else lib.tp_reduce_block_f64
    _call(fn, context().handle, *sys._host_ptrs(), sys.size(), start, end, C.c_void_p(eq.ctypes.data),
          *[C.c_void_p(v.ctypes.data) for v in vec])
    return ReducedBlock(start, end, *[float(v) for v in eq], *vec)


def assemble_interface(blocks: Sequence[ReducedBlock]) -> TridiagonalSystem:
    """assemble_interface (partition.hpp:131-151): rows 2j / 2j+1 = eq1 / eq2 of block j."""
    k = len(blocks)
    out = [np.empty(2 * k) for _ in range(4)]
    for j, b in enumerate(blocks):
        for arr, (v1, v2) in zip(out, ((b.alpha1, b.alpha2), (b.beta1, b.beta2),
                                       (b.gamma1, b.gamma2), (b.delta1, b.delta2))):
            arr[2 * j], arr[2 * j + 1] = v1, v2
    return TridiagonalSystem(*out)


def back_substitute(blk: ReducedBlock, x_s: float, x_e: float) -> np.ndarray:
    """back_substitute (partition.hpp:156-172): x_{s+1} .. x_{e-1} from the
    stored up-sweep rows, left to right."""
    ln = blk.end - blk.start
    out = np.empty(max(ln - 2, 0))
    prev = x_s
    for k in range(1, ln - 1):
        piv = blk.beta[k]
        if abs(piv) < kPivotFloor:
            raise ZeroPivotError(blk.start + k)
        prev = (blk.delta[k] - blk.a[k] * prev - blk.gamma[k] * x_e) / piv
        out[k - 1] = prev
    return out


class RecursionPolicy:
    """Per-level sub-system sizes (partition.hpp:176-187)."""

    def __init__(self, sizes: Sequence[int] = ()):
        self.sizes = [int(s) for s in sizes]

    def depth(self) -> int:
        return len(self.sizes) - 1

    def valid(self) -> bool:
        return len(self.sizes) > 0 and all(m >= 2 for m in self.sizes)

    def __eq__(self, other):
        return isinstance(other, RecursionPolicy) and self.sizes == other.sizes

    def __repr__(self):
        return f"RecursionPolicy({self.sizes})"


def _policy_array(policy) -> np.ndarray:
    sizes = policy.sizes if isinstance(policy, RecursionPolicy) else list(policy)
    return np.ascontiguousarray(np.asarray(sizes, dtype=np.int64).reshape(-1))


def solve_partition(sys: TridiagonalSystem, policy,
                    on_interface: Optional[Callable[[TridiagonalSystem, int], None]] = None):
    """solve_partition(sys, policy[, on_interface]) (partition.hpp:235-248).

    Host arrays -> numpy result (synchronous, H2D/D2H inside). CUDA tensors ->
    CUDA tensor result on torch's current stream; synchronises to surface
    ZeroPivotError like the reference (use solve_partition_async to skip)."""
    sz = _policy_array(policy)
    ctx = context()
    n = sys.size()
    if sys.on_device:
        if on_interface is not None:
            raise ValueError("the observer overload takes host systems")
        x = solve_partition_async(sys, policy)
        import torch
        torch.cuda.current_stream().synchronize()
        err = TpError()
        _raise(lib.tp_check_device_error(ctx.handle, C.byref(err)), err)
        return x
    f32 = sys.is_f32
    x = np.empty(max(n, 0), dtype=np.float32 if f32 else np.float64)
    if on_interface is None:
        fn = lib.tp_solve_partition_f32 if f32 else lib.tp_solve_partition_f64
        _call(fn, ctx.handle, *sys._host_ptrs(), n, sz.ctypes.data_as(_I64), len(sz),
              C.c_void_p(x.ctypes.data))
        return x

    def _cb(level, m, a, b, c, d, _u):
        on_interface(TridiagonalSystem(np.ctypeslib.as_array(a, (m,)).copy(),
                                       np.ctypeslib.as_array(b, (m,)).copy(),
                                       np.ctypeslib.as_array(c, (m,)).copy(),
                                       np.ctypeslib.as_array(d, (m,)).copy()), int(level))

    cb = (_lib.INTERFACE_CB_F32 if f32 else _lib.INTERFACE_CB)(_cb)
    fn = lib.tp_solve_partition_observe_f32 if f32 else lib.tp_solve_partition_observe_f64
    _call(fn, ctx.handle, *sys._host_ptrs(), n, sz.ctypes.data_as(_I64), len(sz),
          C.c_void_p(x.ctypes.data), cb, None)
    return x


def solve_partition_async(sys: TridiagonalSystem, policy, out=None):
    """Device solve without the trailing synchronisation (zero pivots are
    reported by a later ``check_device_error``)."""
    import torch

    sz = _policy_array(policy)
    ctx = context()
    n = sys.size()
    if out is not None and not (out.is_cuda and out.is_contiguous() and out.dtype == sys.diag.dtype and
                                out.device == sys.diag.device and int(out.shape[0]) >= n):
        raise ValueError("out must be a contiguous CUDA tensor of the system's dtype and device, "
                         "with at least n elements")
    x = out if out is not None else torch.empty(n, dtype=sys.diag.dtype, device=sys.diag.device)
    stream = torch_stream()
    fn = lib.tp_solve_partition_f32_dev if sys.is_f32 else lib.tp_solve_partition_f64_dev
    _call(fn, ctx.handle, *sys._dev_ptrs(), n, sz.ctypes.data_as(_I64),
          len(sz), C.c_void_p(x.data_ptr()), C.c_void_p(stream))
    return x


def check_device_error():
    err = TpError()
    _raise(lib.tp_check_device_error(context().handle, C.byref(err)), err)


def plan_levels(n: int, policy):
    """(level sizes, level m [negative = device-internal], n_final) of a solve."""
    sz = _policy_array(policy)
    ln = np.zeros(64, dtype=np.int64)
    lm = np.zeros(64, dtype=np.int64)
    nl = C.c_int32()
    nf = C.c_int64()
    _call(lib.tp_plan_levels, n, sz.ctypes.data_as(_I64), len(sz), ln.ctypes.data_as(_I64),
          lm.ctypes.data_as(_I64), C.byref(nl), 64, C.byref(nf))
    return [int(v) for v in ln[:nl.value]], [int(v) for v in lm[:nl.value]], int(nf.value)


# ------------------------------------------------------------ observations.hpp
@dataclass
class Observation:
    """observations.hpp:19-28."""
    n: int = 0
    label: int = 0
    corrected: Optional[int] = None
    times: Dict[int, float] = field(default_factory=dict)
    precision: str = "fp64"
    device: str = ""
    streams: int = 0
    depth_label: bool = False


@dataclass
class ObservationSet:
    """observations.hpp:30-67."""
    rows: List[Observation] = field(default_factory=list)

    def size(self) -> int:
        return len(self.rows)

    def empty(self) -> bool:
        return not self.rows

    def sort_by_n(self):
        self.rows.sort(key=lambda r: (r.n, r.precision, r.device))

    def filter_device(self, device: str) -> "ObservationSet":
        return ObservationSet([r for r in self.rows if r.device == device])

    def with_corrected_labels(self) -> "ObservationSet":
        out = []
        for r in self.rows:
            o = Observation(r.n, r.label, r.corrected, dict(r.times), r.precision, r.device,
                            r.streams, r.depth_label)
            if o.corrected is not None:
                o.label = o.corrected
            out.append(o)
        return ObservationSet(out)

    def unique_labels(self) -> List[int]:
        return sorted({r.label for r in self.rows})


def read_observations(path: str) -> ObservationSet:
    """read_observations (io.hpp:80-138), parsed by the library's C++ reader."""
    h = C.c_void_p()
    cnt = C.c_int64()
    _call(lib.tp_obs_read, os.fspath(path).encode(), C.byref(h), C.byref(cnt))
    try:
        rows = []
        for i in range(cnt.value):
            o = _lib.TpObservation()
            _call(lib.tp_obs_get, h, i, C.byref(o), None, None)
            cand = np.empty(max(o.ntimes, 1), dtype=np.int32)
            tms = np.empty(max(o.ntimes, 1), dtype=np.float64)
            _call(lib.tp_obs_get, h, i, C.byref(o), cand.ctypes.data_as(_I32), tms.ctypes.data_as(_D))
            rows.append(Observation(
                n=int(o.n), label=int(o.label),
                corrected=int(o.corrected) if o.has_corrected else None,
                times={int(cand[j]): float(tms[j]) for j in range(o.ntimes)},
                precision=o.precision.decode(), device=o.device.decode(), streams=int(o.streams),
                depth_label=bool(o.depth_label)))
        return ObservationSet(rows)
    finally:
        lib.tp_obs_free(h)


# ----------------------------------------------------------------- knn.hpp
@dataclass
class TrainingPair:
    n: int = 0
    label: int = 0


@dataclass
class HeuristicModel:
    """knn.hpp:28-36."""
    pairs: List[TrainingPair] = field(default_factory=list)
    k: int = 1
    transform: str = "log10_n"
    labels: List[int] = field(default_factory=list)
    metadata: Dict[str, str] = field(default_factory=dict)

    def _arrays(self):
        pn = np.ascontiguousarray([p.n for p in self.pairs], dtype=np.int64)
        pl = np.ascontiguousarray([p.label for p in self.pairs], dtype=np.int32)
        return pn, pl


def fit_knn(train: ObservationSet, k: int) -> HeuristicModel:
    """fit_knn (knn.hpp:40-55)."""
    pn = np.ascontiguousarray([r.n for r in train.rows], dtype=np.int64)
    pl = np.ascontiguousarray([r.label for r in train.rows], dtype=np.int32)
    _call(lib.tp_fit_knn, pn.ctypes.data_as(_I64), pl.ctypes.data_as(_I32), len(pn), int(k))
    meta = {}
    if train.rows:
        meta = {"device": train.rows[0].device, "precision": train.rows[0].precision}
    return HeuristicModel([TrainingPair(int(a), int(b)) for a, b in zip(pn, pl)], int(k), "log10_n",
                          train.unique_labels(), meta)


def predict(model: HeuristicModel, n: int) -> int:
    """predict (knn.hpp:57-77): host C++ in the library, bit-exact."""
    pn, pl = model._arrays()
    out = C.c_int32()
    _call(lib.tp_predict, pn.ctypes.data_as(_I64), pl.ctypes.data_as(_I32), len(pn), model.k, int(n),
          C.byref(out))
    return int(out.value)


def fit_depth_model(data: ObservationSet, k: int = 1) -> HeuristicModel:
    """fit_depth_model (policy.hpp:14-16)."""
    return fit_knn(data, k)


def recursion_sizes(n: int, depth: int, size_model: HeuristicModel) -> RecursionPolicy:
    """recursion_sizes (policy.hpp:25-45)."""
    pn, pl = size_model._arrays()
    out = np.zeros(8, dtype=np.int64)
    cnt = C.c_int32()
    _call(lib.tp_recursion_sizes, int(n), int(depth), pn.ctypes.data_as(_I64),
          pl.ctypes.data_as(_I32), len(pn), size_model.k, out.ctypes.data_as(_I64), C.byref(cnt))
    return RecursionPolicy([int(v) for v in out[:cnt.value]])


def _bundled(which: int) -> HeuristicModel:
    cnt = C.c_int64()
    k = C.c_int32()
    _call(lib.tp_default_model, which, None, None, 0, C.byref(cnt), C.byref(k))
    pn = np.empty(cnt.value, dtype=np.int64)
    pl = np.empty(cnt.value, dtype=np.int32)
    _call(lib.tp_default_model, which, pn.ctypes.data_as(_I64), pl.ctypes.data_as(_I32), cnt.value,
          C.byref(cnt), C.byref(k))
    meta = ({"device": "rtx2080ti", "precision": "fp64"} if which == 0
            else {"device": "a5000", "precision": "fp64"})
    return HeuristicModel([TrainingPair(int(a), int(b)) for a, b in zip(pn, pl)], int(k.value),
                          "log10_n", sorted(set(int(v) for v in pl)), meta)


def default_size_model() -> HeuristicModel:
    """fit_knn(Table I FP64 with corrected labels, k=1) — what the reference's
    tests fit (test_policy.cpp:14-17)."""
    return _bundled(0)


def default_fp32_size_model() -> HeuristicModel:
    """fit_knn(Table IV FP32 with corrected labels, k=1)."""
    m = _bundled(2)
    m.metadata = {"device": "rtx2080ti", "precision": "fp32"}
    return m


def default_depth_model() -> HeuristicModel:
    """fit_depth_model(Table II) (test_policy.cpp:19-21)."""
    return _bundled(1)


def b200_size_model() -> HeuristicModel:
    """The m-predictor re-fitted on the B200 (config 5): fit_knn(k=1) of the
    plateau-corrected sweep_m observations in profiles/r02_sweep_b200.csv
    (heuristics/b200_fp64_size_model.json). Device-specific, as the paper
    expects; the reference-parity default stays
    default_size_model()."""
    return load_model(os.path.join(os.path.dirname(os.path.abspath(__file__)), "heuristics",
                                   "b200_fp64_size_model.json"))


def predicted_policy(n: int, size_model: Optional[HeuristicModel] = None,
                     depth_model: Optional[HeuristicModel] = None) -> RecursionPolicy:
    """recursion_sizes(N, predict(depth_model, N), size_model) — the policy the
    paper's heuristics choose for N."""
    size_model = size_model or default_size_model()
    depth_model = depth_model or default_depth_model()
    return recursion_sizes(n, predict(depth_model, n), size_model)


# --------------------------------------------------------------------- io.hpp
def save_model(model: HeuristicModel, path: str):
    """save_model (io.hpp:176-190): JSON, version 1, key order preserved."""
    doc = {
        "version": kModelFormatVersion,
        "transform": model.transform,
        "k": model.k,
        "pairs": [{"n": p.n, "label": p.label} for p in model.pairs],
        "labels": list(model.labels),
        "metadata": dict(model.metadata),
    }
    with open(path, "w") as f:
        f.write(json.dumps(doc, indent=2) + "\n")


def load_model(path: str) -> HeuristicModel:
    """load_model (io.hpp:192-225) with the same schema checks."""
    try:
        with open(path) as f:
            doc = json.load(f)
    except FileNotFoundError:
        raise Error(f"cannot open {path}")
    except json.JSONDecodeError as e:
        raise SchemaError(f"model file is not valid JSON: {e}")
    if not isinstance(doc.get("version"), int):
        raise SchemaError("missing version")
    if doc["version"] != kModelFormatVersion:
        raise VersionMismatchError(f"unsupported model version {doc['version']}")
    for fld in ("transform", "k", "pairs", "labels"):
        if fld not in doc:
            raise SchemaError(f"missing field: {fld}")
    try:
        model = HeuristicModel([TrainingPair(int(p["n"]), int(p["label"])) for p in doc["pairs"]],
                               int(doc["k"]), str(doc["transform"]), [int(v) for v in doc["labels"]],
                               {str(a): str(b) for a, b in doc.get("metadata", {}).items()})
    except (KeyError, TypeError, ValueError) as e:
        raise SchemaError(f"malformed model document: {e}")
    if not model.pairs:
        raise SchemaError("model has no training pairs")
    if model.k < 1 or model.k > len(model.pairs):
        raise SchemaError("k outside [1, |pairs|]")
    return model
