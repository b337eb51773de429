"""GPU tests of the fused multi-GPU path (tp_shard_solve_f64_dev): the
shard's boundary pair is exchanged through peer mailboxes inside the
finishing kernel (no NCCL call) and every rank solves the 2P-row top system.

Covered here on one B200: simulated ranks in one process (one context and
stream per rank, mailboxes linked by raw pointers, all graphs in flight at
once), repeated solves (epoch-parity slots), the peer-timeout error, and two
processes on the same GPU linked by CUDA IPC handles exchanged over a gloo
process group (the code path real multi-GPU runs take, minus NVLink)."""
import os
import socket
import sys
import time

import numpy as np
import pytest

from conftest import needs_shared_gpu

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TOL_NORM, TOL_FLOOR, TOL_RES = 1e-10, 1e-10, 1e-12


def _check(oracle_mod, s, x, ref):
    assert np.all(np.isfinite(x))
    assert oracle_mod.rel_inf_diff(x, ref) <= TOL_NORM
    assert oracle_mod.floored_rel_diff(x, ref) <= TOL_FLOOR
    assert oracle_mod.residual_inf(s, x) <= TOL_RES


def _run_sim(body: str) -> dict:
    """Simulated ranks share one GPU and one process, so every rank's kernels
    must be able to run while a peer's finishing kernel waits on its flags:
    the snippet runs in a fresh process with eager module loading (a lazily
    loaded kernel waits for the device to go idle) and a hardware queue per
    stream. Real ranks are separate processes on separate GPUs."""
    import json
    import subprocess

    env = dict(os.environ, CUDA_DEVICE_MAX_CONNECTIONS="32", CUDA_MODULE_LOADING="EAGER")
    code = ("import json, sys\nsys.path.insert(0, %r)\nimport numpy as np\nimport oracle\n"
            "import paper_2510_27351_b200 as tp\nfrom paper_2510_27351_b200 import sharded\n" % ROOT) + body
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    return json.loads(out.stdout.strip().splitlines()[-1])


_METRICS = """
def metrics(s, x, ref):
    return {"finite": bool(np.all(np.isfinite(x))), "d": oracle.rel_inf_diff(x, ref),
            "f": oracle.floored_rel_diff(x, ref), "r": oracle.residual_inf(s, x)}
"""


def _ok(m):
    return m["finite"] and m["d"] <= TOL_NORM and m["f"] <= TOL_FLOOR and m["r"] <= TOL_RES


@needs_shared_gpu
@pytest.mark.parametrize("P", [1, 2, 3, 8])
def test_fused_sharded_simulated_ranks(tp, P):
    m = _run_sim(_METRICS + f"""
n = 1_000_003
s = oracle.generate_system(n, 13)
ref = oracle.solve_partition(s, [32])
x = sharded.simulate_ranks_fused(s.sub, s.diag, s.sup, s.rhs, {P}, [32])
print(json.dumps(metrics(s, x, ref)))
""")
    assert _ok(m), m


@needs_shared_gpu
def test_fused_sharded_knn_policy_and_repeats(tp):
    """kNN policy of the global N (recursion levels on every shard); three
    back-to-back solves on the same links alternate the mailbox slots and
    must give identical results."""
    m = _run_sim(_METRICS + """
n = 3_000_000
pol = tp.predicted_policy(n)
s = oracle.generate_system(n, 5)
ref = oracle.solve_partition(s, pol.sizes)
xs = sharded.simulate_ranks_fused(s.sub, s.diag, s.sup, s.rhs, 4, pol.sizes, repeats=3)
out = [metrics(s, x, ref) for x in xs]
print(json.dumps({"m": out, "same": bool(np.array_equal(xs[0], xs[1]) and np.array_equal(xs[1], xs[2]))}))
""")
    assert all(_ok(x) for x in m["m"]), m
    assert m["same"]


@needs_shared_gpu
@pytest.mark.parametrize("n,P", [(40_000_000, 8), (12_800_000, 2), (8_000_000, 1)])
def test_fused_shard_runs_the_single_gpu_graph(tp, n, P):
    """Each rank of the fused multi-GPU solve runs the single-GPU graph on its
    shard, with the peer exchange at the root of its deepest kernel — the same
    kernels, in the same order, as a single-GPU solve of a shard-sized system.
    One rank per GPU (P = 1 here): Stage 1 of level 0, then the grid solve from
    level 1 (k_grid_solve<kShard>) with the exchange at its root, Stage 3 of
    level 0. Ranks sharing one GPU (P > 1 simulated here) keep the level path:
    granule-aligned shards (m0*m1/2 rows) keep levels 0-1 tail-free, so Stage
    1 of levels 0-2 is the folded kernel and the deepest level is the fused
    cluster kernel with the exchange at its root."""
    m = _run_sim(_METRICS + f"""
n, P = {n}, {P}
pol = [64, 10, 32, 16]
s = oracle.generate_system(n, 31)
ref = oracle.solve_partition(s, pol)
ks = []
x = sharded.simulate_ranks_fused(s.sub, s.diag, s.sup, s.rhs, P, pol, kernels=ks)
g = sharded.shard_granule(pol)
single = []
tp.context().set_grid(P == 1)  # ranks sharing a GPU take the level path
for r in range(P):
    lo, cnt = sharded.shard_bounds(n, P, r, g)
    sysr = tp.TridiagonalSystem(*(a[lo:lo + cnt].copy() for a in (s.sub, s.diag, s.sup, s.rhs)))
    tp.solve_partition(sysr, tp.RecursionPolicy(pol))
    single.append(tp.context().last_kernels())
tp.context().set_grid(True)
print(json.dumps({{"m": metrics(s, x, ref), "ks": ks, "single": single}}))
""")
    assert _ok(m["m"]), m["m"]
    for ks, single in zip(m["ks"], m["single"]):
        if P == 1:
            assert ks == ["stage1:L0", "grid_exchange:L1", "stage3:L0"], ks
        else:
            assert ks[0] == "stage1_fold2:L0", ks
            assert "level_exchange:L3" in ks, ks
        assert [k.replace("level_exchange", "level_final").replace("grid_exchange", "grid_solve") for k in ks] \
            == single, (ks, single)


@needs_shared_gpu
def test_fused_matches_nccl_path_algebra(tp):
    """Fused and host-gathered paths compute the same top system: results
    agree to rounding."""
    m = _run_sim("""
n = 500_001
s = oracle.generate_system(n, 21)
a = sharded.simulate_ranks(s.sub, s.diag, s.sup, s.rhs, 3, [16, 8])
b = sharded.simulate_ranks_fused(s.sub, s.diag, s.sup, s.rhs, 3, [16, 8])
print(json.dumps({"d": oracle.rel_inf_diff(a, b)}))
""")
    assert m["d"] <= 1e-14, m


def test_fused_peer_timeout_is_an_error(tp, oracle_mod):
    """A peer that never publishes: the finishing kernel gives up after its
    bounded spin and the solve reports TP_ERR_NCCL instead of hanging."""
    import ctypes as C

    import torch

    from paper_2510_27351_b200 import sharded
    from paper_2510_27351_b200._lib import lib
    from paper_2510_27351_b200.tridpart import Context, _call

    c0, c1 = Context(0), Context(0)
    boxes = []
    for c in (c0, c1):
        own = C.c_void_p()
        _call(lib.tp_shard_mailbox, c.handle, 2, C.byref(own))
        boxes.append(own.value)
    _call(lib.tp_shard_attach, c0.handle, 2, 0, (C.c_void_p * 2)(*boxes))
    s = oracle_mod.generate_system(10_000, 3)
    sys4 = [torch.from_numpy(a[:5000].copy()).cuda() for a in (s.sub, s.diag, s.sup, s.rhs)]
    t0 = time.time()
    sharded.fused_solve(c0, sys4, [8], stream=0)
    torch.cuda.synchronize()
    with pytest.raises(tp.Error, match="timed out waiting for rank 1"):
        tp_check(c0)
    assert time.time() - t0 < 60
    c0.close()
    c1.close()


def tp_check(ctx):
    import ctypes as C

    from paper_2510_27351_b200._lib import TpError, lib
    from paper_2510_27351_b200.tridpart import _raise

    err = TpError()
    _raise(lib.tp_check_device_error(ctx.handle, C.byref(err)), err)


def _free_port():
    so = socket.socket()
    so.bind(("127.0.0.1", 0))
    p = so.getsockname()[1]
    so.close()
    return p


def _ipc_worker(rank, world, port, n, q):
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist

    import oracle
    import paper_2510_27351_b200 as tp
    from paper_2510_27351_b200 import sharded

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        s = oracle.generate_system(n, 9)
        pol = tp.predicted_policy(n)
        lo, cnt = sharded.shard_bounds(n, world, rank)
        sys4 = [torch.from_numpy(np.ascontiguousarray(a[lo:lo + cnt])).cuda()
                for a in (s.sub, s.diag, s.sup, s.rhs)]
        solver = sharded.ShardedSolver(transport="p2p")
        xs = []
        for _ in range(2):
            x = solver.solve(sys4, n, pol)
            torch.cuda.synchronize()
            solver.backend.check()
            xs.append(x.cpu().numpy())
        parts = [None] * world
        dist.all_gather_object(parts, (lo, xs[0], bool(np.array_equal(xs[0], xs[1]))))
        if rank == 0:
            q.put(parts)
    finally:
        dist.destroy_process_group()


@needs_shared_gpu
def test_fused_two_processes_cuda_ipc(tp, oracle_mod):
    import torch.multiprocessing as mp

    n, world = 400_000, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ipc_worker, args=(r, world, port, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    parts = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    s = oracle_mod.generate_system(n, 9)
    ref = oracle_mod.solve_partition(s, tp.predicted_policy(n).sizes)
    x = np.empty(n)
    for lo, xr, repeat_equal in parts:
        x[lo:lo + len(xr)] = xr
        assert repeat_equal
    _check(oracle_mod, s, x, ref)


@needs_shared_gpu
@pytest.mark.parametrize("world,transport,weak", [(2, "auto", False), (3, "nccl", True), (4, "auto", False)])
def test_bench_multi_rank_flow_on_one_gpu(world, transport, weak):
    """bench.py's N>1 path (torchrun, one process per rank, sharded solve,
    max-over-ranks timing, one JSON line from rank 0) with every rank on the
    one GPU of this box (TPB_SHARE_GPU=1: gloo process group, the ranks
    time-slice the GPU, so only correctness and the output contract are
    checked)."""
    import json
    import subprocess

    env = dict(os.environ, TPB_SHARE_GPU="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.join(ROOT, "bench.py"),
           "--gpus", str(world), "--steps", "3", "--warmup", "3", "--prewarm", "0", "--e2e-steps", "1",
           "--size", "4e6", "--transport", transport] + (["--weak"] if weak else [])
    out = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [x for x in out.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    d = json.loads(lines[0])
    # strong scaling by default (the BASELINE metric: the same N on 1/2/4/8 GPUs)
    assert d["n_gpus"] == world and d["config"]["n_global"] == 4_000_000 * (world if weak else 1)
    assert d["scaling"] == ("weak" if weak else "strong")
    assert d["config"]["transport"] == ("p2p" if transport == "auto" else "nccl")
    assert d["residual"] <= 1e-12 and d["value"] > 0 and d["gpu_launches"] > 0
    assert len(d["roofline"]["per_rank"]) == world


@needs_shared_gpu
def test_fused_random_shards_including_tiny_ones(tp):
    """Random global sizes (down to 2 rows per shard), rank counts and
    policies: the finishing kernel takes the single-CTA path for shards whose
    deepest system is under 64 rows and the cluster path above, in every mode."""
    m = _run_sim(_METRICS + """
rng = np.random.default_rng(7)
out = []
for case in range(24):
    P = int(rng.integers(1, 7))
    n = int(np.exp(rng.uniform(np.log(2 * P), np.log(3e5))))
    sizes = [int(rng.integers(2, 80)) for _ in range(int(rng.integers(1, 3)))]
    s = oracle.generate_system(n, 500 + case)
    ref = oracle.solve_partition(s, sizes)
    x = sharded.simulate_ranks_fused(s.sub, s.diag, s.sup, s.rhs, P, sizes)
    mm = metrics(s, x, ref)
    mm.update(P=P, n=n, sizes=sizes)
    out.append(mm)
print(json.dumps(out))
""")
    bad = [c for c in m if not _ok(c)]
    assert not bad, bad
