"""Multi-GPU sharded partition solve (one process per GPU, torch.distributed).

The global system is split into contiguous row shards [row0_p, row0_p + n_p).
Per rank:
  1. ``reduce``  — Stage 1 of every local partition level, then the shard's
     final system is reduced to its two boundary equations (the
     assemble_interface rows of partition.hpp:139-149 for one super-block):
        E1_p: a1*x_{s_p - 1} + b1*x_{s_p} + g1*x_{e_p} = d1
        E2_p: a2*x_{s_p} + b2*x_{e_p} + g2*x_{e_p + 1} = d2
  2. one all-gather of 8 doubles per rank (NCCL over NVLink on B200; gloo in
     the CPU tests) — the only exchange step of the method;
  3. ``finish``  — every rank solves the 2P-row top system redundantly
     (Thomas, tridiagonal.hpp:52-72) and runs Stage 3 of its local levels.
The policy (m per level, R) is the kNN prediction for the GLOBAL N, as the
reference would choose for the whole system (recursion_sizes, policy.hpp:25-45).
"""
from __future__ import annotations

import ctypes as C
from typing import Optional, Sequence

import numpy as np

from ._lib import lib
from .tridpart import (RecursionPolicy, _call, _policy_array, _raise, context, predicted_policy,
                       torch_stream)


def shard_bounds(n_global: int, nranks: int, rank: int):
    """Contiguous, near-equal shards; every shard keeps >= 2 rows."""
    if nranks < 1 or not 0 <= rank < nranks:
        raise ValueError("bad rank / world size")
    if n_global < 2 * nranks:
        raise ValueError("every shard needs at least 2 rows")
    lo = rank * n_global // nranks
    hi = (rank + 1) * n_global // nranks
    return lo, hi - lo


def assemble_top_system(gathered, nranks: int):
    """The 2P-row top system from the gathered boundary pairs, rank order
    (assemble_interface layout, partition.hpp:139-149): row 2p = E1_p,
    row 2p+1 = E2_p. Host mirror of what k_gather_solve assembles on device."""
    g = np.asarray(gathered, dtype=np.float64).reshape(nranks, 4, 2)
    return tuple(np.ascontiguousarray(g[:, k, :].reshape(-1)) for k in range(4))


class DeviceBackend:
    """The sm_100a kernels behind the C-ABI (tp_shard_reduce / tp_shard_finish)."""

    def __init__(self, ctx=None):
        self.ctx = ctx or context()
        self.launches = 0  # kernels of the last reduce + finish pair

    @staticmethod
    def _ptrs(sys4):
        return [C.c_void_p(t.data_ptr()) for t in sys4]

    def reduce(self, sys4, policy):
        import torch

        sz = _policy_array(policy)
        eq8 = torch.empty(8, dtype=torch.float64, device=sys4[0].device)
        stream = torch_stream()
        _call(lib.tp_shard_reduce_f64_dev, self.ctx.handle, *self._ptrs(sys4), int(sys4[0].numel()),
              sz.ctypes.data_as(C.POINTER(C.c_int64)), len(sz), C.c_void_p(eq8.data_ptr()),
              C.c_void_p(stream))
        self._reduce_launches = self.ctx.last_launch_count()
        return eq8

    def finish(self, sys4, policy, gathered, nranks: int, rank: int, out=None):
        import torch

        sz = _policy_array(policy)
        x = out if out is not None else torch.empty_like(sys4[1])
        stream = torch_stream()
        _call(lib.tp_shard_finish_f64_dev, self.ctx.handle, *self._ptrs(sys4), int(sys4[0].numel()),
              sz.ctypes.data_as(C.POINTER(C.c_int64)), len(sz), C.c_void_p(gathered.data_ptr()),
              int(nranks), int(rank), C.c_void_p(x.data_ptr()), C.c_void_p(stream))
        self.launches = getattr(self, "_reduce_launches", 0) + self.ctx.last_launch_count()
        return x

    def check(self):
        from ._lib import TpError

        err = TpError()
        _raise(lib.tp_check_device_error(self.ctx.handle, C.byref(err)), err)


class ShardedSolver:
    """solve_partition over a process group: each rank passes its local shard."""

    def __init__(self, backend=None, group=None):
        self.backend = backend or DeviceBackend()
        self.group = group

    def policy_for(self, n_global: int, policy=None) -> RecursionPolicy:
        if policy is None:
            return predicted_policy(n_global)
        return policy if isinstance(policy, RecursionPolicy) else RecursionPolicy(policy)

    def solve(self, sys4: Sequence, n_global: int, policy=None, out=None):
        import torch.distributed as dist

        pol = self.policy_for(n_global, policy)
        P = dist.get_world_size(self.group)
        rank = dist.get_rank(self.group)
        eq8 = self.backend.reduce(sys4, pol)
        gathered = eq8.new_empty(8 * P)
        dist.all_gather_into_tensor(gathered, eq8, group=self.group)
        return self.backend.finish(sys4, pol, gathered, P, rank, out=out)


def simulate_ranks(sub, diag, sup, rhs, nranks: int, policy=None) -> np.ndarray:
    """Run the sharded algorithm with `nranks` simulated ranks on ONE GPU (one
    context per rank; the gather is a host concatenation). Used by the GPU
    tests to exercise the multi-rank device path without NCCL."""
    import torch

    from .tridpart import Context

    n = len(diag)
    pol = RecursionPolicy(policy) if policy is not None else predicted_policy(n)
    arrs = [np.ascontiguousarray(a, dtype=np.float64) for a in (sub, diag, sup, rhs)]
    shards, ctxs, eqs = [], [], []
    for r in range(nranks):
        lo, cnt = shard_bounds(n, nranks, r)
        sys4 = [torch.from_numpy(a[lo:lo + cnt].copy()).cuda() for a in arrs]
        be = DeviceBackend(Context(torch.cuda.current_device()))
        eqs.append(be.reduce(sys4, pol))
        shards.append((lo, cnt, sys4))
        ctxs.append(be)
    gathered = torch.cat(eqs)
    x = np.empty(n)
    for r, (lo, cnt, sys4) in enumerate(shards):
        xr = ctxs[r].finish(sys4, pol, gathered, nranks, r)
        torch.cuda.synchronize()
        ctxs[r].check()
        x[lo:lo + cnt] = xr.cpu().numpy()
    for be in ctxs:
        be.ctx.close()
    return x
