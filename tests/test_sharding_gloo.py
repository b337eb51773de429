"""Multi-process (world_size 2 and 3, gloo, CPU) test of the sharded solve's
host logic: shard bounds, global-N policy, the all-gather of the 8 boundary
doubles in rank order and the 2P-row top solve. The per-shard reduce/finish
are the oracle's reduce_block / thomas_solve (the device backend computes the
same equations on the GPU; tests/test_gpu_partition.py covers it with
simulated ranks)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


class _NoDevice:
    handle = None  # a NULL tp_ctx*: the C-ABI answers TP_ERR_INVALID_ARGUMENT


class OracleBackend:
    """reduce/finish on the CPU with the oracle (test scaffold, not a product path)."""

    def __init__(self, oracle):
        self.o = oracle
        self.ctx = _NoDevice()  # peer links need a device context: p2p is refused

    def reduce(self, sys4, policy):
        s = self.o.System(*(t.numpy() for t in sys4))
        a1, b1, g1, d1, a2, b2, g2, d2 = self.o.reduce_block(s, 0, s.n)
        # eq8 layout of tp_shard_reduce: {sub[2], diag[2], super[2], rhs[2]}
        return torch.tensor([a1, a2, b1, b2, g1, g2, d1, d2], dtype=torch.float64)

    def finish(self, sys4, policy, gathered, nranks, rank, out=None):
        from paper_2510_27351_b200.sharded import assemble_top_system

        top = self.o.System(*assemble_top_system(gathered.numpy(), nranks))
        xt = self.o.thomas_solve(top)
        xs, xe = xt[2 * rank], xt[2 * rank + 1]
        sub, diag, sup, rhs = (t.numpy().copy() for t in sys4)
        n = len(diag)
        x = np.empty(n)
        x[0], x[-1] = xs, xe
        if n > 2:
            rhs[1] -= sub[1] * xs
            rhs[n - 2] -= sup[n - 2] * xe
            isub, isup = sub[1:n - 1].copy(), sup[1:n - 1].copy()
            isub[0], isup[-1] = 0.0, 0.0
            x[1:n - 1] = self.o.thomas_solve(self.o.System(isub, diag[1:n - 1], isup, rhs[1:n - 1]))
        return torch.from_numpy(x)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, seed, q, transport="nccl"):
    import sys

    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        from paper_2510_27351_b200.sharded import ShardedSolver, shard_bounds

        glob = oracle.generate_system(n, seed)
        lo, cnt = shard_bounds(n, world, rank)
        sys4 = [torch.from_numpy(a[lo:lo + cnt].copy()) for a in (glob.sub, glob.diag, glob.sup, glob.rhs)]
        solver = ShardedSolver(backend=OracleBackend(oracle), transport=transport)
        pol = solver.policy_for(n)
        x = solver.solve(sys4, n)
        q.put((rank, lo, x.numpy(), pol.sizes, solver.transport, solver.fallback_reason))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,transport", [(2, "nccl"), (3, "nccl"), (2, "auto")])
def test_sharded_solve_gloo(oracle_mod, world, transport):
    """transport="auto" on CPU: no rank can build peer links, every rank sees
    the same collective verdict and all fall back to the all-gather together
    (a split decision would leave ranks waiting on each other forever)."""
    n, seed = 100_003, 31
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, seed, q, transport)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    glob = oracle_mod.generate_system(n, seed)
    ref = oracle_mod.solve_partition(glob, [32])
    x = np.empty(n)
    for rank, lo, xr, sizes, used, why in res:
        assert sizes == [32]  # kNN policy of the GLOBAL N (predict(1e5) = 32, R = 0)
        assert used == "nccl"
        if transport == "auto":
            assert why is not None and all(f"rank {r}" in why for r in range(world))
        x[lo:lo + len(xr)] = xr
    assert oracle_mod.rel_inf_diff(x, ref) <= 1e-10
    assert oracle_mod.residual_inf(glob, x) <= 1e-12


def test_shard_bounds():
    from paper_2510_27351_b200.sharded import shard_bounds

    for n, P in ((10, 2), (100_003, 3), (1_000_000_000, 8), (17, 8)):
        spans = [shard_bounds(n, P, r) for r in range(P)]
        assert spans[0][0] == 0
        assert sum(c for _, c in spans) == n
        for (lo, c), (lo2, _) in zip(spans, spans[1:]):
            assert lo + c == lo2
        assert all(c >= 2 for _, c in spans)
    with pytest.raises(ValueError):
        shard_bounds(3, 2, 0)


def test_shard_bounds_granule():
    """Aligned shards: every boundary on a multiple of the granule (m0*m1/2,
    so each shard's level 0 and level 1 have no tail block and the rank runs
    the folded single-GPU graph); the last shard takes the remainder."""
    from paper_2510_27351_b200.sharded import shard_bounds, shard_granule

    assert shard_granule([64, 10, 32, 16]) == 320
    assert shard_granule([64, 10, 32, 32]) == 320
    assert shard_granule([32]) == 32
    assert shard_granule([16, 5]) == 16
    for n, P, g in ((10**8, 8, 320), (10**8, 2, 320), (10**9, 8, 320), (100_003, 3, 32), (1000, 4, 320),
                    (7, 3, 320)):
        spans = [shard_bounds(n, P, r, g) for r in range(P)]
        assert spans[0][0] == 0 and sum(c for _, c in spans) == n
        for (lo, c), (lo2, _) in zip(spans, spans[1:]):
            assert lo + c == lo2
        assert all(c >= 2 for _, c in spans)
        if n // g >= P:
            assert all(lo % g == 0 for lo, _ in spans)
            assert all(c % g == 0 for _, c in spans[:-1])
            assert max(c for _, c in spans) - min(c for _, c in spans) <= g + n % g
    # N = 1e8 on 8 ranks: 39,062 or 39,063 granules of 320 rows each
    assert {c for _, c in (shard_bounds(10**8, 8, r, 320) for r in range(8))} == {12_499_840, 12_500_160}


def test_assemble_top_system_layout():
    from paper_2510_27351_b200.sharded import assemble_top_system

    g = np.arange(16, dtype=np.float64)  # 2 ranks x {sub[2], diag[2], super[2], rhs[2]}
    sub, diag, sup, rhs = assemble_top_system(g, 2)
    assert list(sub) == [0, 1, 8, 9] and list(diag) == [2, 3, 10, 11]
    assert list(sup) == [4, 5, 12, 13] and list(rhs) == [6, 7, 14, 15]
