"""GPU parity of the one-kernel grid solve (k_grid_solve, csrc/tp_grid.cu): the
whole solve of a one-level policy whose rows fit the GPU's shared memory
(config 2: N=1e6, policy {32}). Checked against the oracle (the reference's
algorithm; oracle/_ref where it runs) with the tolerances of
tests/test_gpu_partition.py, and against the level path of the
same library (TPB_GRID=0 in a subprocess)."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TOL = 1e-10
TOL_RES = 1e-12


@pytest.fixture(autouse=True)
def _grid_for_all_sizes(tp):
    """Small systems too (the default threshold keeps n < 8e4 on the level path)."""
    tp.context().set_grid(True, 4)
    yield
    tp.context().set_grid(True, 80_000)


def _sys(tp, s):
    return tp.TridiagonalSystem(s.sub, s.diag, s.sup, s.rhs)


def _impl(oracle_mod):
    return "ref" if oracle_mod.ref_available() else "port"


def _check(oracle_mod, s, x, ref):
    assert np.all(np.isfinite(x))
    assert oracle_mod.rel_inf_diff(x, ref) <= TOL
    assert oracle_mod.floored_rel_diff(x, ref) <= TOL
    assert oracle_mod.residual_inf(s, x) <= TOL_RES


def test_config2_runs_as_one_grid_kernel(tp, oracle_mod):
    """C2 (N=1e6, kNN policy {32}): one kernel after k_reset."""
    n = 1_000_000
    s = oracle_mod.generate_system(n, 1)
    sm, dm = tp.default_size_model(), tp.default_depth_model()
    pol = tp.recursion_sizes(n, tp.predict(dm, n), sm)
    assert pol.sizes == [32]
    ref = oracle_mod.solve_partition(s, pol.sizes, impl=_impl(oracle_mod))
    x = tp.solve_partition(_sys(tp, s), pol)
    assert tp.context().last_kernels() == ["grid_solve:L0"]
    assert tp.context().last_launch_count() == 1  # the grid kernel alone (it resets the error word)
    _check(oracle_mod, s, x, ref)


@pytest.mark.parametrize("n,m", [
    (4, 2), (5, 2), (7, 3), (16, 4), (17, 4), (33, 32), (64, 64), (65, 64), (100, 1000),
    (1000, 4), (1001, 4), (1002, 4), (10_000, 4), (10_000, 8), (12_345, 5), (30_000, 16),
    (65_536, 20), (77_459, 20), (100_000, 32), (262_144, 64), (300_001, 25), (500_000, 100),
    (999_999, 32), (1_000_001, 32), (900_000, 256), (150_000, 2), (300_000, 5000), (6_000, 6_000),
])
def test_grid_shapes_against_the_reference(tp, oracle_mod, n, m):
    """Block-aligned CTA ranges with tails of every kind (n % m = 0, 1, other),
    m >= n (one block), the smallest block (m = 2) and chunking by 1..32 per block."""
    s = oracle_mod.generate_system(n, 3 + n % 89)
    ref = oracle_mod.solve_partition(s, [m], impl=_impl(oracle_mod))
    x = tp.solve_partition(_sys(tp, s), tp.RecursionPolicy([m]))
    ks = tp.context().last_kernels()
    assert ks == ["grid_solve:L0"], ks
    _check(oracle_mod, s, x, ref)


def test_grid_random_sizes(tp, oracle_mod):
    rng = np.random.default_rng(2027)
    for _ in range(60):
        n = int(rng.integers(4, 1_000_000))
        m = int(rng.choice([2, 3, 4, 5, 6, 8, 10, 12, 16, 20, 25, 32, 40, 50, 64, 100, 128, 200, 256]))
        if m < 8:
            n = min(n, 250_000)  # <= 1024 blocks of m rows per SM
        s = oracle_mod.generate_system(n, int(rng.integers(1, 1 << 30)))
        ref = oracle_mod.solve_partition(s, [m], impl="port")
        x = tp.solve_partition(_sys(tp, s), tp.RecursionPolicy([m]))
        assert tp.context().last_kernels() == ["grid_solve:L0"], (n, m)
        _check(oracle_mod, s, x, ref)


def test_grid_too_large_keeps_the_level_path(tp, oracle_mod):
    """Rows past the grid's shared memory (FP64: ~1.03e6 at m = 32) and blocks
    whose chunks would exceed 64 rows take the level kernels."""
    for n, m in ((2_000_000, 32), (1_000_000, 100_000)):
        s = oracle_mod.generate_system(n, 5)
        ref = oracle_mod.solve_partition(s, [m], impl="port")
        x = tp.solve_partition(_sys(tp, s), tp.RecursionPolicy([m]))
        assert "grid_solve:L0" not in tp.context().last_kernels()
        _check(oracle_mod, s, x, ref)


def test_grid_fp32(tp, oracle_mod):
    for n, m in ((1_000_000, 32), (2_000_000, 32), (33_333, 20)):
        s = oracle_mod.generate_system(n, 9)
        args = [a.astype(np.float32) for a in (s.sub, s.diag, s.sup, s.rhs)]
        x = tp.solve_partition(tp.TridiagonalSystem(*args), tp.RecursionPolicy([m]))
        assert x.dtype == np.float32
        assert tp.context().last_kernels() == ["grid_solve:L0"], (n, m)
        assert oracle_mod.residual_inf_f32(*args, x) <= 1e-4
        ref = oracle_mod.solve_partition(s, [m], impl="port")
        assert oracle_mod.rel_inf_diff(x.astype(np.float64), ref) <= 1e-4


def test_grid_device_tensors_and_unaligned_views(tp, oracle_mod):
    """Device-resident inputs (the bench path), also as views 8 bytes off the
    16-byte grid (the kernel stages element by element: no alignment needed)."""
    import torch

    n = 400_003
    s = oracle_mod.generate_system(n + 1, 13)
    ref_full = oracle_mod.solve_partition(s, [16], impl="port")
    dev = [torch.from_numpy(a).cuda() for a in (s.sub, s.diag, s.sup, s.rhs)]
    x = tp.solve_partition(tp.TridiagonalSystem(*dev), tp.RecursionPolicy([16]))
    torch.cuda.synchronize()
    assert tp.context().last_kernels() == ["grid_solve:L0"]
    assert oracle_mod.rel_inf_diff(x.cpu().numpy(), ref_full) <= TOL
    s1 = oracle_mod.System(s.sub[1:], s.diag[1:], s.sup[1:], s.rhs[1:])
    ref1 = oracle_mod.solve_partition(s1, [16], impl="port")  # sub[0] is never read
    x1 = tp.solve_partition(tp.TridiagonalSystem(*[t[1:] for t in dev]), tp.RecursionPolicy([16]))
    torch.cuda.synchronize()
    assert tp.context().last_kernels() == ["grid_solve:L0"]
    assert oracle_mod.rel_inf_diff(x1.cpu().numpy(), ref1) <= TOL
    _check(oracle_mod, s1, x1.cpu().numpy(), ref1)


def test_grid_zero_pivot_reports_the_reference_row(tp, oracle_mod):
    """A zero pivot inside the grid kernel: the error carries the reference's
    row and level (diagnose_pivot replays the reference's sequential order on
    the level-0 interface it re-assembles)."""
    rng = np.random.default_rng(77)
    checked = 0
    for _ in range(30):
        n = int(rng.integers(200, 600_000))
        m = int(rng.choice([4, 8, 16, 20, 32, 64]))
        base = oracle_mod.generate_system(n, int(rng.integers(1, 1 << 30)))
        rows = sorted(set(int(v) for v in rng.integers(0, n, size=int(rng.integers(1, 3)))))
        sub, diag, sup, rhs = (a.copy() for a in (base.sub, base.diag, base.sup, base.rhs))
        for r in rows:
            sub[r] = diag[r] = sup[r] = 0.0
        s = oracle_mod.System(sub, diag, sup, rhs)
        try:
            oracle_mod.solve_partition(s, [m], impl="port")
            continue
        except oracle_mod.OracleZeroPivot as e:
            want = (e.row, e.level)
        with pytest.raises(tp.ZeroPivotError) as ei:
            tp.solve_partition(_sys(tp, s), tp.RecursionPolicy([m]))
        assert (ei.value.row(), ei.value.level) == want, (n, m, rows)
        checked += 1
    assert checked >= 10


def test_grid_observer_still_sees_the_interface(tp, oracle_mod):
    """The observer overload keeps the level path: level 0's interface goes
    to the callback (the grid kernel never writes it)."""
    n = 200_000
    s = oracle_mod.generate_system(n, 4)
    seen = []
    x = tp.solve_partition(_sys(tp, s), tp.RecursionPolicy([32]),
                           on_interface=lambda iface, level: seen.append((level, iface.diag.shape[0])))
    assert seen == [(0, 2 * (n // 32))]
    assert "grid_solve:L0" not in tp.context().last_kernels()
    _check(oracle_mod, s, x, oracle_mod.solve_partition(s, [32], impl="port"))
    tp.solve_partition(_sys(tp, s), tp.RecursionPolicy([32]))
    assert tp.context().last_kernels() == ["grid_solve:L0"]


@pytest.mark.parametrize("n,m", [(100_000, 32), (400_000, 32), (600_001, 32), (262_144, 64), (50_000, 8),
                                 (100_003, 16), (300_000, 4), (1_000_001, 32), (999_999, 64), (700_003, 16)])
def test_grid_register_variants(tp, oracle_mod, n, m):
    """k_grid_reg (2-row chunks: rows in registers, re-read from L2 for Stage 3)
    and k_grid_hyb (4- and 8-row chunks: rows via registers into shared memory)
    against the reference, tails included."""
    s = oracle_mod.generate_system(n, 17 + n % 7)
    ref = oracle_mod.solve_partition(s, [m], impl="port")
    x = tp.solve_partition(_sys(tp, s), tp.RecursionPolicy([m]))
    assert tp.context().last_kernels() == ["grid_solve:L0"]
    _check(oracle_mod, s, x, ref)


def test_grid_matches_the_level_path(tp, oracle_mod):
    """TPB_GRID=0 (level kernels) and the grid kernel agree to rounding."""
    code = """
import json, sys, numpy as np
sys.path.insert(0, %r)
import oracle, paper_2510_27351_b200 as tp
s = oracle.generate_system(777_777, 8)
x = tp.solve_partition(tp.TridiagonalSystem(s.sub, s.diag, s.sup, s.rhs), tp.RecursionPolicy([32]))
np.save(sys.argv[1], x)
print(json.dumps(tp.context().last_kernels()))
""" % ROOT
    outs = {}
    for mode in ("0", "1"):
        path = f"/tmp/tpb_grid_{mode}.npy"
        env = dict(os.environ, TPB_GRID=mode, TPB_GRID_MIN="4")
        r = subprocess.run([sys.executable, "-c", code, path], env=env, capture_output=True, text=True, timeout=300)
        assert r.returncode == 0, r.stderr
        outs[mode] = (np.load(path), json.loads(r.stdout.strip().splitlines()[-1]))
    assert outs["1"][1] == ["grid_solve:L0"]
    assert "grid_solve:L0" not in outs["0"][1]
    assert oracle_mod.rel_inf_diff(outs["1"][0], outs["0"][0]) <= 1e-13


def test_grid_launch_failure_falls_back_to_the_level_path(tp, oracle_mod):
    """A grid solve whose cooperative launch fails (TPB_GRID_FORCE_FAIL=1 makes
    the launcher refuse, as a GPU with fewer available SMs would) is retried on
    the level path; the context keeps the level path."""
    code = """
import json, sys, numpy as np
sys.path.insert(0, %r)
import oracle, paper_2510_27351_b200 as tp
s = oracle.generate_system(1_000_000, 4)
ref = oracle.solve_partition(s, [32])
x = tp.solve_partition(tp.TridiagonalSystem(s.sub, s.diag, s.sup, s.rhs), tp.RecursionPolicy([32]))
k1 = tp.context().last_kernels()
x2 = tp.solve_partition(tp.TridiagonalSystem(s.sub, s.diag, s.sup, s.rhs), tp.RecursionPolicy([32]))
print(json.dumps({"d": oracle.rel_inf_diff(x, ref), "d2": oracle.rel_inf_diff(x2, ref), "k1": k1,
                  "k2": tp.context().last_kernels()}))
""" % ROOT
    env = dict(os.environ, TPB_GRID_FORCE_FAIL="1")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    out = json.loads(r.stdout.strip().splitlines()[-1])
    assert out["d"] <= TOL and out["d2"] <= TOL
    assert "grid_solve:L0" not in out["k1"] and "grid_solve:L0" not in out["k2"], out


def test_grid_at_deeper_levels_random(tp, oracle_mod):
    """Random multi-level policies at sizes where the grid solve takes a level
    k >= 1 (Stage 1 above it, Stage 3 below): FP64 at the parity gates, FP32
    against the reference's float instantiation's tolerance (1e-4)."""
    rng = np.random.default_rng(4242)
    for case in range(16):
        n = int(np.exp(rng.uniform(np.log(3e5), np.log(6e6))))
        depth = int(rng.integers(1, 4))
        sizes = [int(rng.choice([4, 8, 10, 16, 20, 32, 64]))] + \
                [int(rng.choice([2, 4, 8, 10, 16, 32])) for _ in range(depth)]
        s = oracle_mod.generate_system(n, 700 + case)
        ref = oracle_mod.solve_partition(s, sizes, impl="port")
        x = tp.solve_partition(_sys(tp, s), tp.RecursionPolicy(sizes))
        _check(oracle_mod, s, x, ref)
        if case % 4 == 0:
            args = [a.astype(np.float32) for a in (s.sub, s.diag, s.sup, s.rhs)]
            x32 = tp.solve_partition(tp.TridiagonalSystem(*args), tp.RecursionPolicy(sizes))
            assert oracle_mod.rel_inf_diff(x32.astype(np.float64), ref) <= 1e-4, (n, sizes)
