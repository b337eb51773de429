"""GPU parity, round 2: every policy the reference accepts (long blocks, m >= n),
the reference's zero-pivot contract (row AND level), the device residual, the
stage functions, and the reference's own C++ unit tests / acceptance criteria
1-2 run through the drop-in headers. Checked against oracle/_ref (the
reference's unmodified headers) wherever it can run, else the C port.
Tolerances as tests/test_gpu_partition.py."""
import os
import subprocess

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TOL = 1e-10
TOL_RES = 1e-12


def _sys(tp, s):
    return tp.TridiagonalSystem(s.sub, s.diag, s.sup, s.rhs)


def _check(oracle_mod, s, x, ref, tol=TOL):
    assert np.all(np.isfinite(x))
    assert oracle_mod.rel_inf_diff(x, ref) <= tol
    assert oracle_mod.floored_rel_diff(x, ref) <= tol
    assert oracle_mod.residual_inf(s, x) <= TOL_RES


def _impl(oracle_mod):
    return "ref" if oracle_mod.ref_available() else "port"


# ------------------------------------------------------------------ long blocks
@pytest.mark.parametrize("n,sizes", [
    (50_000, [2049]), (100_000, [4097]), (1_000_000, [7245]), (1_000_000, [10_000]),
    (1_000_000, [100_000]), (100_000, [100_000]), (100_000, [250_000]), (7_245, [7_245]),
    (60_000, [59_999]), (20_001, [10_000]), (1_000_000, [32, 20_000]), (400_000, [5_000, 4]),
    (1_000_000, [64, 10, 3_000]),
])
def test_long_blocks_against_the_reference(tp, oracle_mod, n, sizes):
    """Blocks longer than shared memory holds (round 1 failed above 7,244 rows)
    through the split chain, m >= n included (one block of n rows)."""
    s = oracle_mod.generate_system(n, 7 + n % 97)
    ref = oracle_mod.solve_partition(s, sizes, impl=_impl(oracle_mod))
    x = tp.solve_partition(_sys(tp, s), tp.RecursionPolicy(sizes))
    _check(oracle_mod, s, x, ref)


def test_long_blocks_fp32(tp, oracle_mod):
    s = oracle_mod.generate_system(300_000, 5)
    args = [a.astype(np.float32) for a in (s.sub, s.diag, s.sup, s.rhs)]
    for sizes in ([20_000], [300_000], [64, 9_000]):
        x = tp.solve_partition(tp.TridiagonalSystem(*args), tp.RecursionPolicy(sizes))
        assert x.dtype == np.float32
        assert oracle_mod.residual_inf_f32(*args, x) <= 1e-4


def test_long_blocks_device_tensors(tp, oracle_mod):
    import torch

    s = oracle_mod.generate_system(2_000_000, 3)
    ref = oracle_mod.solve_partition(s, [50_000], impl="port")
    sd = tp.TridiagonalSystem(*[torch.from_numpy(a).cuda() for a in (s.sub, s.diag, s.sup, s.rhs)])
    x = tp.solve_partition(sd, tp.RecursionPolicy([50_000])).cpu().numpy()
    _check(oracle_mod, s, x, ref)


# ------------------------------------------------------------ zero pivots
def _zero_rows(s, rows):
    sub, diag, sup, rhs = (a.copy() for a in (s.sub, s.diag, s.sup, s.rhs))
    for r in rows:
        sub[r] = diag[r] = sup[r] = 0.0
    return type(s)(sub, diag, sup, rhs)


_POLICIES = [[4], [8], [16], [7], [32], [64], [5], [8, 4], [16, 8], [10, 4, 4], [5, 6, 4], [4, 4, 4, 4],
             [3], [2], [40, 4]]


def test_zero_pivot_row_and_level_match_the_reference(tp, oracle_mod):
    """50+ zero-pivot placements (a row a_r = b_r = c_r = 0) where the reference
    throws ZeroPivotError: the device reports the same row() and the same level
    (the reference's level = observer calls before the throw). n < 128 m0 keeps
    every level below the reference's parallel_for threshold (K < 128), where
    its throw is observable (above it std::terminate()s)."""
    if not oracle_mod.ref_available():
        pytest.skip("oracle/_ref not built")
    rng = np.random.default_rng(2024)
    matched = 0
    levels = set()
    tried = 0
    while matched < 60 and tried < 600:
        pol = _POLICIES[tried % len(_POLICIES)]
        tried += 1
        n = int(rng.integers(8, 127 * pol[0]))
        base = oracle_mod.generate_system(n, int(rng.integers(1, 10_000)))
        rows = sorted(set(int(v) for v in rng.integers(0, n, size=int(rng.integers(1, 3)))))
        s = _zero_rows(base, rows)
        try:
            oracle_mod.solve_partition(s, pol, impl="ref")
            continue  # singular but no pivot below the floor in the reference's order
        except oracle_mod.OracleZeroPivot as e:
            want = (e.row, e.level)
        with pytest.raises(tp.ZeroPivotError) as ei:
            tp.solve_partition(_sys(tp, s), tp.RecursionPolicy(pol))
        got = (ei.value.row(), ei.value.level)
        assert got == want, (n, pol, rows, got, want)
        matched += 1
        levels.add(want[1])
    assert matched >= 50, matched
    assert len(levels) >= 3, levels  # level-0 sweeps, deeper levels and the final Thomas


def test_zero_pivot_sequential_order_above_the_parallel_threshold(tp, oracle_mod):
    """K >= 128: the reference aborts (std::terminate in parallel_for); the
    device raises ZeroPivotError with the row of the reference's SEQUENTIAL
    order (the C port, which loops the blocks in order)."""
    rng = np.random.default_rng(7)
    for t in range(12):
        pol = [[4], [8], [64], [8, 10, 8], [32, 4]][t % 5]
        n = int(rng.integers(300 * pol[0], 3000 * pol[0]))
        s = _zero_rows(oracle_mod.generate_system(n, t + 1), sorted(set(int(v) for v in rng.integers(0, n, 3))))
        try:
            oracle_mod.solve_partition(s, pol, impl="port")
            continue
        except oracle_mod.OracleZeroPivot as e:
            want = (e.row, e.level)
        with pytest.raises(tp.ZeroPivotError) as ei:
            tp.solve_partition(_sys(tp, s), tp.RecursionPolicy(pol))
        assert (ei.value.row(), ei.value.level) == want


def test_zero_pivot_through_device_tensors(tp, oracle_mod):
    import torch

    base = oracle_mod.generate_system(600, 11)
    s = _zero_rows(base, [301])
    with pytest.raises(oracle_mod.OracleZeroPivot) as e:
        oracle_mod.solve_partition(s, [8], impl="port")
    sd = tp.TridiagonalSystem(*[torch.from_numpy(a).cuda() for a in (s.sub, s.diag, s.sup, s.rhs)])
    with pytest.raises(tp.ZeroPivotError) as ei:
        tp.solve_partition(sd, tp.RecursionPolicy([8]))
    assert (ei.value.row(), ei.value.level) == (e.value.row, e.value.level)


def test_thomas_zero_pivot_rows(tp, oracle_mod):
    """thomas_solve (tridiagonal.hpp:52-72): the failing row of the sequential sweep."""
    impl = _impl(oracle_mod)
    rng = np.random.default_rng(3)
    for t in range(20):
        n = int(rng.integers(2, 20_000))
        s = _zero_rows(oracle_mod.generate_system(max(n, 2), t + 5), [int(rng.integers(0, n))])
        try:
            oracle_mod.thomas_solve(s, impl=impl)
            continue
        except oracle_mod.OracleZeroPivot as e:
            want = e.row
        with pytest.raises(tp.ZeroPivotError) as ei:
            tp.thomas_solve(_sys(tp, s))
        assert ei.value.row() == want


def test_observer_delivers_completed_levels_before_a_zero_pivot(tp, oracle_mod):
    """partition.hpp:205-206: the observer has seen levels 0 .. l-1 when level l throws."""
    if not oracle_mod.ref_available():
        pytest.skip("oracle/_ref not built")
    rng = np.random.default_rng(99)
    seen_deep = False
    for t in range(40):
        pol = [[8, 4], [10, 4, 4], [16, 8], [4, 4, 4]][t % 4]
        n = int(rng.integers(50, 120 * pol[0]))
        s = _zero_rows(oracle_mod.generate_system(n, t + 40), [int(rng.integers(0, n))])
        want = []
        try:
            oracle_mod.solve_partition(s, pol, impl="ref", observer=lambda l, a, b, c, d: want.append((l, b)))
            continue
        except oracle_mod.OracleZeroPivot:
            pass
        got = []
        with pytest.raises(tp.ZeroPivotError):
            tp.solve_partition(_sys(tp, s), tp.RecursionPolicy(pol),
                               on_interface=lambda f, l: got.append((l, f.diag)))
        assert [l for l, _ in got] == [l for l, _ in want]
        for (_, gb), (_, wb) in zip(got, want):
            assert gb.shape == wb.shape
            assert np.allclose(gb, wb, rtol=1e-12, atol=1e-14, equal_nan=True)
        seen_deep = seen_deep or len(want) > 0
    assert seen_deep


# --------------------------------------------------------------- residual_inf
def test_device_residual_matches_the_reference(tp, oracle_mod):
    import torch

    s = oracle_mod.generate_system(1_000_000, 1)
    x = oracle_mod.solve_partition(s, [32])
    for xx in (x, x + 1e-6 * np.sin(np.arange(x.size))):
        want = oracle_mod.residual_inf(s, xx)
        sd = tp.TridiagonalSystem(*[torch.from_numpy(a).cuda() for a in (s.sub, s.diag, s.sup, s.rhs)])
        got = tp.residual_inf(sd, torch.from_numpy(xx).cuda())
        if want > 1e-10:
            assert abs(got - want) <= 1e-9 * want
        else:
            assert got <= 1e-14 and want <= 1e-14
    if oracle_mod.ref_available():
        ref_x = oracle_mod.solve_partition(s, [32], impl="ref")
        assert oracle_mod.ref().ref_residual_inf(s.n, *s.ptrs(), oracle_mod._dp(ref_x)) <= TOL_RES


# ----------------------------------------------------------- stage functions
def test_reduce_block_is_bit_identical_to_the_reference(tp, oracle_mod):
    """reduce_block runs the reference's own arithmetic on the device: the
    interface pair equals oracle/_ref's bit for bit."""
    if not oracle_mod.ref_available():
        pytest.skip("oracle/_ref not built")
    s = oracle_mod.generate_system(5000, 17)
    sys_ = _sys(tp, s)
    for (a, b) in ((0, 2), (10, 12), (20, 32), (0, 64), (100, 1100), (3000, 5000), (4990, 5000)):
        got = tp.reduce_block(sys_, tp.Block(a, b))
        want = oracle_mod.reduce_block(s, a, b, impl="ref")
        g = np.array([got.alpha1, got.beta1, got.gamma1, got.delta1, got.alpha2, got.beta2, got.gamma2,
                      got.delta2])
        assert g.tobytes() == want.tobytes(), (a, b)
    blocks = [tp.reduce_block(sys_, blk) for blk in tp.make_plan(5000, 16).blocks]
    f = tp.assemble_interface(blocks)
    assert f.size() == 2 * len(blocks)
    x = oracle_mod.thomas_solve(s)
    interior = tp.back_substitute(blocks[3], x[48], x[63])
    assert np.max(np.abs(interior - x[49:63])) <= 1e-12
    z = _zero_rows(s, [40])
    with pytest.raises(tp.ZeroPivotError) as ei:
        tp.reduce_block(_sys(tp, z), tp.Block(32, 48))
    with pytest.raises(oracle_mod.OracleZeroPivot) as e:
        oracle_mod.reduce_block(z, 32, 48, impl="ref")
    assert ei.value.row() == e.value.row == 40
    with pytest.raises(tp.InvalidSizeError):
        tp.reduce_block(sys_, tp.Block(5, 6))


# ------------------------------------------- the reference's own C++ tests
def _run(exe, timeout=600):
    if not os.path.exists(exe):
        pytest.skip(f"{exe} not built (tests/cpp/Makefile)")
    return subprocess.run([exe], capture_output=True, text=True, timeout=timeout)


def test_reference_unit_tests_pass_on_the_b200():
    """proj/tests/test_{partition,tridiagonal,policy}.cpp, unmodified, built
    against include/tridpart/*.hpp (tests/cpp/Makefile), run on the GPU."""
    r = _run(os.path.join(ROOT, "tests", "cpp", "_build", "ref_unit_tests"))
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert "All tests passed" in r.stdout
    assert r.stdout.count("PASS") >= 20


def test_acceptance_criteria_1_and_2_on_the_b200():
    """acceptance.cpp:72-123 with the reference's mt19937_64 case lists."""
    r = _run(os.path.join(ROOT, "tests", "cpp", "_build", "acceptance_12"))
    assert r.returncode == 0, r.stdout + r.stderr
    assert "PASS  criterion 1" in r.stdout and "PASS  criterion 2" in r.stdout
