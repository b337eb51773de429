"""ORACLE — TEST INFRASTRUCTURE ONLY (parity checker, never the product).

Two CPU implementations of the reference `tridpart` hot path:

* ``port``: ``oracle/tridpart_oracle.c`` — a plain-C restatement of the
  reference algorithm (each function cites the reference file:line it follows),
  built into ``oracle/_build/liboracle.so``.
* ``ref``: the reference's OWN headers compiled unmodified behind the
  ``extern "C"`` shim ``oracle/ref_driver.cpp`` into
  ``oracle/_ref/libtridpart_ref.so`` (recipe: ``oracle/Makefile``).

Parity is pinned: tests/test_oracle.py checks port == ref bit-for-bit
(generator, solve, predictors) and both against the golden values the
reference's own tests and SURVEY.md §8(c) record.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's ``cpu_baseline`` /
``--impl reference`` legs may import this package.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Callable, Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(_HERE, "_build", "liboracle.so")
REF_SO = os.path.join(_HERE, "_ref", "libtridpart_ref.so")
REF_DATA = os.path.join(_HERE, "_ref", "data")

_D = C.POINTER(C.c_double)
_I64 = C.POINTER(C.c_int64)
_I32 = C.POINTER(C.c_int32)
OBSERVER = C.CFUNCTYPE(None, C.c_int64, C.c_int64, _D, _D, _D, _D, C.c_void_p)

_port = None
_ref = None


def build() -> None:
    """Compile the oracle (and, where /root/reference exists, oracle/_ref)."""
    import subprocess

    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def _dp(a: np.ndarray):
    return a.ctypes.data_as(_D)


def port():
    global _port
    if _port is None:
        if not os.path.exists(PORT_SO):
            build()
        lib = C.CDLL(PORT_SO)
        lib.orc_generate_system.restype = C.c_int64
        lib.orc_generate_system.argtypes = [C.c_int64, C.c_uint64, C.c_double, _D, _D, _D, _D]
        lib.orc_thomas_solve.restype = C.c_int64
        lib.orc_thomas_solve.argtypes = [C.c_int64, _D, _D, _D, _D, _D]
        lib.orc_residual_inf.restype = C.c_double
        lib.orc_residual_inf.argtypes = [C.c_int64, _D, _D, _D, _D, _D]
        lib.orc_make_plan.restype = C.c_int64
        lib.orc_make_plan.argtypes = [C.c_int64, C.c_int64, _I64]
        lib.orc_solve_partition.restype = C.c_int64
        lib.orc_solve_partition.argtypes = [C.c_int64, _D, _D, _D, _D, _I64, C.c_int64, _D,
                                            OBSERVER, C.c_void_p, _I64]
        lib.orc_reduce_block.restype = C.c_int64
        lib.orc_reduce_block.argtypes = [_D, _D, _D, _D, C.c_int64, C.c_int64, _D]
        lib.orc_predict.restype = C.c_int
        lib.orc_predict.argtypes = [_I64, C.POINTER(C.c_int), C.c_int64, C.c_int, C.c_int64]
        lib.orc_recursion_sizes.restype = C.c_int64
        lib.orc_recursion_sizes.argtypes = [C.c_int64, C.c_int, _I64, C.POINTER(C.c_int), C.c_int64,
                                            C.c_int, _I64]
        _port = lib
    return _port


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref():
    global _ref
    if _ref is None:
        if not os.path.exists(REF_SO):
            raise RuntimeError("oracle/_ref not built (needs /root/reference at build time)")
        lib = C.CDLL(REF_SO)
        lib.ref_generate_system.restype = C.c_int64
        lib.ref_generate_system.argtypes = [C.c_int64, C.c_uint64, C.c_double, _D, _D, _D, _D]
        lib.ref_thomas_solve.restype = C.c_int64
        lib.ref_thomas_solve.argtypes = [C.c_int64, _D, _D, _D, _D, _D]
        lib.ref_system_new.restype = C.c_void_p
        lib.ref_system_new.argtypes = [C.c_int64, _D, _D, _D, _D]
        lib.ref_system_generate.restype = C.c_void_p
        lib.ref_system_generate.argtypes = [C.c_int64, C.c_uint64]
        lib.ref_system_view.restype = None
        lib.ref_system_view.argtypes = [C.c_void_p] + [C.POINTER(_D)] * 4
        lib.ref_system_thomas.restype = C.c_int64
        lib.ref_system_thomas.argtypes = [C.c_void_p, _D]
        lib.ref_system_free.restype = None
        lib.ref_system_free.argtypes = [C.c_void_p]
        lib.ref_system_solve.restype = C.c_int64
        lib.ref_system_solve.argtypes = [C.c_void_p, _I64, C.c_int32, _D]
        lib.ref_system_residual.restype = C.c_double
        lib.ref_system_residual.argtypes = [C.c_void_p, _D]
        lib.ref_solve_partition.restype = C.c_int64
        lib.ref_solve_partition.argtypes = [C.c_int64, _D, _D, _D, _D, _I64, C.c_int32, _D,
                                            OBSERVER, C.c_void_p]
        lib.ref_residual_inf.restype = C.c_double
        lib.ref_residual_inf.argtypes = [C.c_int64, _D, _D, _D, _D, _D]
        lib.ref_reduce_block.restype = C.c_int64
        lib.ref_reduce_block.argtypes = [C.c_int64, _D, _D, _D, _D, C.c_int64, C.c_int64, _D]
        lib.ref_make_plan.restype = C.c_int64
        lib.ref_make_plan.argtypes = [C.c_int64, C.c_int64, _I64]
        lib.ref_load_models.restype = C.c_int64
        lib.ref_load_models.argtypes = [C.c_char_p]
        lib.ref_predict_size.restype = C.c_int32
        lib.ref_predict_size.argtypes = [C.c_int64]
        lib.ref_predict_depth.restype = C.c_int32
        lib.ref_predict_depth.argtypes = [C.c_int64]
        lib.ref_recursion_sizes.restype = C.c_int64
        lib.ref_recursion_sizes.argtypes = [C.c_int64, C.c_int32, _I64]
        lib.ref_model_pairs.restype = C.c_int32
        lib.ref_model_pairs.argtypes = [C.c_int32, _I64, _I32, C.c_int32]
        lib.ref_hardware_concurrency.restype = C.c_uint32
        lib.ref_hardware_concurrency.argtypes = []
        _F = C.POINTER(C.c_float)
        lib.ref_solve_partition_f32.restype = C.c_int64
        lib.ref_solve_partition_f32.argtypes = [C.c_int64, _F, _F, _F, _F, _I64, C.c_int32, _F]
        lib.ref_residual_inf_f32.restype = C.c_float
        lib.ref_residual_inf_f32.argtypes = [C.c_int64, _F, _F, _F, _F, _F]
        if lib.ref_load_models(REF_DATA.encode()) != -1:
            raise RuntimeError(f"reference models failed to load from {REF_DATA}")
        _ref = lib
    return _ref


class System:
    """SoA tridiagonal system (tridiagonal.hpp:22-28) as four float64 arrays."""

    def __init__(self, sub, diag, sup, rhs):
        self.sub = np.ascontiguousarray(sub, dtype=np.float64)
        self.diag = np.ascontiguousarray(diag, dtype=np.float64)
        self.sup = np.ascontiguousarray(sup, dtype=np.float64)
        self.rhs = np.ascontiguousarray(rhs, dtype=np.float64)

    @property
    def n(self) -> int:
        return int(self.diag.shape[0])

    def ptrs(self):
        return _dp(self.sub), _dp(self.diag), _dp(self.sup), _dp(self.rhs)


class RefSystem:
    """A system owned by the reference library (oracle/_ref): generated there
    by its own generate_system, solved there without copying the arrays;
    ``view()`` exposes the arrays as numpy views (no copy). For N = 1e9."""

    def __init__(self, n: int, seed: int):
        self.n = n
        self.h = ref().ref_system_generate(n, seed)
        if not self.h:
            raise MemoryError("ref_system_generate failed")

    def view(self) -> System:
        ps = [_D() for _ in range(4)]
        ref().ref_system_view(self.h, *[C.byref(p) for p in ps])
        arrs = [np.ctypeslib.as_array(p, (self.n,)) for p in ps]
        v = System.__new__(System)
        v.sub, v.diag, v.sup, v.rhs = arrs
        return v

    def solve(self, sizes) -> np.ndarray:
        x = np.empty(self.n)
        sz = np.asarray(sizes, dtype=np.int64)
        _status(ref().ref_system_solve(self.h, sz.ctypes.data_as(_I64), len(sz), _dp(x)))
        return x

    def thomas(self) -> np.ndarray:
        x = np.empty(self.n)
        _status(ref().ref_system_thomas(self.h, _dp(x)))
        return x

    def free(self):
        if self.h:
            ref().ref_system_free(self.h)
            self.h = None


def generate_system(n: int, seed: int, delta: float = 1.5, impl: str = "port") -> System:
    """generate_system (bench.hpp:68-93)."""
    a, b, c, d = (np.empty(n, dtype=np.float64) for _ in range(4))
    lib = port() if impl == "port" else ref()
    fn = lib.orc_generate_system if impl == "port" else lib.ref_generate_system
    st = fn(n, seed, delta, _dp(a), _dp(b), _dp(c), _dp(d))
    if st != -1:
        raise ValueError(f"generate_system failed ({st})")
    return System(a, b, c, d)


class OracleZeroPivot(Exception):
    """ZeroPivotError(row) of the oracle; ``level`` = the system the row indexes
    (0 = input, l = interface of level l-1), when known."""

    def __init__(self, row: int, level: Optional[int] = None):
        super().__init__(f"zero pivot at row {row}" + ("" if level is None else f" (level {level})"))
        self.row = row
        self.level = level


def _status(st: int):
    if st == -1:
        return
    if st >= 0:
        raise OracleZeroPivot(int(st))
    raise ValueError(f"oracle status {st}")


def solve_partition(sys: System, sizes: Sequence[int], impl: str = "port",
                    observer: Optional[Callable] = None) -> np.ndarray:
    """solve_partition (partition.hpp:235-248); observer(level, sub, diag, sup, rhs).

    A zero pivot raises OracleZeroPivot(row, level): the port reports the level
    itself; for the reference (impl="ref") the level is the number of observer
    calls made before the throw — the reference calls the observer once per
    assembled level (partition.hpp:205-206), so a throw in level l's Stage 1
    comes after l calls and one in the final thomas_solve after depth+1.
    NOTE: the reference std::terminate()s on a zero pivot inside a parallel
    region (K >= 128 blocks at that level): callers keep K < 128 for impl="ref"."""
    x = np.empty(sys.n, dtype=np.float64)
    sz = np.asarray(sizes, dtype=np.int64)
    calls = [0]

    def _cb(level, n, a, b, c, d, _u):
        calls[0] += 1
        if observer is not None:
            observer(int(level), np.ctypeslib.as_array(a, (n,)).copy(),
                     np.ctypeslib.as_array(b, (n,)).copy(), np.ctypeslib.as_array(c, (n,)).copy(),
                     np.ctypeslib.as_array(d, (n,)).copy())
    cb = OBSERVER(_cb) if (observer is not None or impl != "port") else OBSERVER(0)
    if impl == "port":
        lvl = C.c_int64(0)
        st = port().orc_solve_partition(sys.n, *sys.ptrs(), sz.ctypes.data_as(_I64), len(sz),
                                        _dp(x), cb, None, C.byref(lvl))
        if st >= 0:
            raise OracleZeroPivot(int(st), int(lvl.value))
    else:
        st = ref().ref_solve_partition(sys.n, *sys.ptrs(), sz.ctypes.data_as(_I64), len(sz),
                                       _dp(x), cb, None)
        if st >= 0:
            raise OracleZeroPivot(int(st), calls[0])
    _status(st)
    return x


def solve_partition_f32(sub, diag, sup, rhs, sizes) -> np.ndarray:
    """The reference's solve_partition<float> (oracle/_ref)."""
    arrs = [np.ascontiguousarray(a, dtype=np.float32) for a in (sub, diag, sup, rhs)]
    n = len(arrs[1])
    x = np.empty(n, dtype=np.float32)
    sz = np.asarray(sizes, dtype=np.int64)
    F = C.POINTER(C.c_float)
    _status(ref().ref_solve_partition_f32(n, *[a.ctypes.data_as(F) for a in arrs],
                                          sz.ctypes.data_as(_I64), len(sz), x.ctypes.data_as(F)))
    return x


def residual_inf_f32(sub, diag, sup, rhs, x) -> float:
    """The reference's residual_inf<float> (oracle/_ref)."""
    arrs = [np.ascontiguousarray(a, dtype=np.float32) for a in (sub, diag, sup, rhs, x)]
    F = C.POINTER(C.c_float)
    return float(ref().ref_residual_inf_f32(len(arrs[1]), *[a.ctypes.data_as(F) for a in arrs]))


def thomas_solve(sys: System, impl: str = "port") -> np.ndarray:
    """thomas_solve (tridiagonal.hpp:52-72)."""
    x = np.empty(sys.n, dtype=np.float64)
    fn = port().orc_thomas_solve if impl == "port" else ref().ref_thomas_solve
    _status(fn(sys.n, *sys.ptrs(), _dp(x)))
    return x


def residual_inf(sys: System, x: np.ndarray) -> float:
    """residual_inf (tridiagonal.hpp:74-87)."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    return float(port().orc_residual_inf(sys.n, *sys.ptrs(), _dp(x)))


def reduce_block(sys: System, start: int, end: int, impl: str = "port") -> np.ndarray:
    """reduce_block (partition.hpp:77-126) -> [a1,b1,g1,d1,a2,b2,g2,d2]."""
    out = np.empty(8, dtype=np.float64)
    if impl == "port":
        st = port().orc_reduce_block(*sys.ptrs(), start, end, _dp(out))
    else:
        st = ref().ref_reduce_block(sys.n, *sys.ptrs(), start, end, _dp(out))
    _status(st)
    return out


def make_plan(n: int, m: int, impl: str = "port") -> list:
    """make_plan (partition.hpp:30-49) -> list of (start, end)."""
    fn = port().orc_make_plan if impl == "port" else ref().ref_make_plan
    k = fn(n, m, None)
    if k < 0:
        raise ValueError("invalid size")
    b = np.empty(k + 1, dtype=np.int64)
    fn(n, m, b.ctypes.data_as(_I64))
    return [(int(b[j]), int(b[j + 1])) for j in range(k)]


def model_pairs(which: int):
    """(n, label) pairs of the reference-fitted size (0) / depth (1) model."""
    n = np.empty(64, dtype=np.int64)
    lab = np.empty(64, dtype=np.int32)
    cnt = ref().ref_model_pairs(which, n.ctypes.data_as(_I64), lab.ctypes.data_as(_I32), 64)
    return n[:cnt].copy(), lab[:cnt].copy()


def predict(pairs_n, pairs_label, k: int, n: int) -> int:
    """predict (knn.hpp:57-77), C restatement."""
    pn = np.ascontiguousarray(pairs_n, dtype=np.int64)
    pl = np.ascontiguousarray(pairs_label, dtype=np.intc)
    return int(port().orc_predict(pn.ctypes.data_as(_I64), pl.ctypes.data_as(C.POINTER(C.c_int)),
                                  len(pn), k, n))


def recursion_sizes(n: int, depth: int, pairs_n, pairs_label, k: int = 1) -> list:
    """recursion_sizes (policy.hpp:25-45), C restatement."""
    pn = np.ascontiguousarray(pairs_n, dtype=np.int64)
    pl = np.ascontiguousarray(pairs_label, dtype=np.intc)
    out = np.empty(8, dtype=np.int64)
    cnt = port().orc_recursion_sizes(n, depth, pn.ctypes.data_as(_I64),
                                     pl.ctypes.data_as(C.POINTER(C.c_int)), len(pn), k,
                                     out.ctypes.data_as(_I64))
    if cnt < 0:
        raise ValueError(f"recursion_sizes status {cnt}")
    return [int(v) for v in out[:cnt]]


def dense_solve(sys: System) -> np.ndarray:
    """tests/oracles.hpp:17-44 — dense elimination (numpy LAPACK, partial pivoting)."""
    n = sys.n
    A = np.zeros((n, n))
    idx = np.arange(n)
    A[idx, idx] = sys.diag
    A[idx[1:], idx[:-1]] = sys.sub[1:]
    A[idx[:-1], idx[1:]] = sys.sup[:-1]
    return np.linalg.solve(A, sys.rhs)


def rel_inf_diff(a: np.ndarray, b: np.ndarray) -> float:
    """tests/oracles.hpp:46-53."""
    return float(np.max(np.abs(a - b)) / max(1.0, float(np.max(np.abs(b)))))


def floored_rel_diff(x: np.ndarray, ref_x: np.ndarray, floor: float = 1e-6) -> float:
    """max_i |x_i - ref_i| / max(|ref_i|, floor) (SURVEY.md §8(c) parity metric)."""
    return float(np.max(np.abs(x - ref_x) / np.maximum(np.abs(ref_x), floor)))
