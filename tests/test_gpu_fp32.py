"""FP32 path (solve_partition<float>, the reference template on Real;
SURVEY.md §8(f) row 3) on the B200 against the reference's own float
instantiation (oracle/_ref) and the FP64 oracle.

Tolerances: the reference's FP32 test gates the residual at 1e-4
(test_partition.cpp:206-223); parity with the float reference is checked at
1e-4 normwise (float rounding, condition number ~O(1) for these systems)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOL32 = 1e-4


def _f32_system(n, seed):
    # test_partition.cpp:206-223: U[-1,1] off-diagonals/rhs, diag 1.5(|a|+|c|)+1 (no sign flip)
    rng = np.random.default_rng(seed)
    a = rng.uniform(-1, 1, n).astype(np.float32)
    c = rng.uniform(-1, 1, n).astype(np.float32)
    a[0], c[-1] = 0, 0
    b = (np.float32(1.5) * (np.abs(a) + np.abs(c)) + np.float32(1)).astype(np.float32)
    d = rng.uniform(-1, 1, n).astype(np.float32)
    return a, b, c, d


def _rel(x, y):
    x, y = np.asarray(x, np.float64), np.asarray(y, np.float64)
    return float(np.max(np.abs(x - y)) / max(1.0, float(np.max(np.abs(y)))))


def test_fp32_reference_case(tp, oracle_mod):
    """test_partition.cpp "fp32 mode solves with relaxed tolerance": n=256, {8,4}."""
    a, b, c, d = _f32_system(256, 8)
    sys = tp.TridiagonalSystem(a, b, c, d)
    assert sys.is_f32
    x = tp.solve_partition(sys, tp.RecursionPolicy([8, 4]))
    assert x.dtype == np.float32
    assert oracle_mod.residual_inf_f32(a, b, c, d, x) <= TOL32
    xr = oracle_mod.solve_partition_f32(a, b, c, d, [8, 4])
    assert _rel(x, xr) <= TOL32


@pytest.mark.parametrize("n,sizes", [(10_000, [4]), (1_000_003, [32]), (5_000_000, [32, 10, 16]),
                                     (2_000_000, [25, 10, 100]), (300_001, [1250])])
def test_fp32_against_float_reference_and_fp64(tp, oracle_mod, n, sizes):
    a, b, c, d = _f32_system(n, n % 1000)
    x = tp.solve_partition(tp.TridiagonalSystem(a, b, c, d), tp.RecursionPolicy(sizes))
    assert np.all(np.isfinite(x))
    assert tp.residual_inf(tp.TridiagonalSystem(a, b, c, d), x) <= TOL32
    xr = oracle_mod.solve_partition_f32(a, b, c, d, sizes)
    assert _rel(x, xr) <= TOL32
    x64 = oracle_mod.solve_partition(oracle_mod.System(a, b, c, d), sizes)
    assert _rel(x, x64) <= TOL32


def test_fp32_device_path_generator_and_model(tp):
    import torch

    pol = tp.recursion_sizes(20_000_000, 3, tp.default_fp32_size_model())
    sys = tp.generate_system(20_000_000, 3, device=True, dtype="float32")
    assert sys.is_f32 and sys.strictly_dominant()
    x = tp.solve_partition(sys, pol)
    assert x.dtype == torch.float32
    assert tp.residual_inf(sys, x) <= TOL32
    # the same system in FP64 gives the same solution to float accuracy
    sys64 = tp.TridiagonalSystem(*(t.double() for t in (sys.sub, sys.diag, sys.super, sys.rhs)))
    x64 = tp.solve_partition(sys64, pol)
    assert float((x.double() - x64).abs().max()) <= TOL32


def test_fp32_observer_and_thomas(tp, oracle_mod):
    a, b, c, d = _f32_system(3000, 5)
    levels = []
    tp.solve_partition(tp.TridiagonalSystem(a, b, c, d), tp.RecursionPolicy([8, 10, 4]),
                       lambda f, lvl: levels.append((lvl, f)))
    assert [l for l, _ in levels] == [0, 1, 2]
    for _, f in levels:
        assert f.diag.dtype == np.float32
        assert np.all(np.abs(f.diag) >= np.abs(f.sub) + np.abs(f.super) - 1e-5)
    xt = tp.thomas_solve(tp.TridiagonalSystem(a, b, c, d))
    assert oracle_mod.residual_inf_f32(a, b, c, d, xt) <= TOL32


def test_fp32_randomized_sizes_and_policies(tp, oracle_mod):
    """120 random (N, policy) pairs in FP32 against the reference's own
    solve_partition<float> (oracle/_ref) and the FP64 oracle."""
    rng = np.random.default_rng(3232)
    for case in range(120):
        n = int(np.exp(rng.uniform(np.log(4), np.log(2e5))))
        sizes = [int(rng.integers(2, 300)) for _ in range(int(rng.integers(1, 4)))]
        a, b, c, d = _f32_system(n, 7000 + case)
        x = tp.solve_partition(tp.TridiagonalSystem(a, b, c, d), tp.RecursionPolicy(sizes))
        assert np.all(np.isfinite(x)), (case, n, sizes)
        assert oracle_mod.residual_inf_f32(a, b, c, d, x) <= TOL32, (case, n, sizes)
        assert _rel(x, oracle_mod.solve_partition_f32(a, b, c, d, sizes)) <= TOL32, (case, n, sizes)
