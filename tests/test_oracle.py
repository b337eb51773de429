"""Pin the oracle before trusting it (CPU only).

* the C restatement (oracle/tridpart_oracle.c) is bit-identical to the
  reference's own headers (oracle/_ref) for the generator, the solve and the
  predictors;
* both reproduce the golden vectors: SURVEY.md §8(c) values and
  tests/golden/reference_golden.json (made by the reference itself);
* the reference's own unit-test expectations (test_partition.cpp,
  test_tridiagonal.cpp, test_knn.cpp, test_policy.cpp, acceptance.cpp) hold
  on the oracle.
"""
import json
import math
import os

import numpy as np
import pytest

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "reference_golden.json")


@pytest.fixture(scope="module")
def golden():
    with open(GOLDEN) as f:
        return json.load(f)


@pytest.fixture(scope="module")
def models(oracle_mod, golden):
    # the bundled table (tp_models_data.h) equals what the reference fits
    import paper_2510_27351_b200 as tp

    sm, dm = tp.default_size_model(), tp.default_depth_model()
    return (np.array([p.n for p in sm.pairs]), np.array([p.label for p in sm.pairs]),
            np.array([p.n for p in dm.pairs]), np.array([p.label for p in dm.pairs]))


needs_ref = pytest.mark.skipif(not os.path.exists(os.path.join(
    os.path.dirname(os.path.dirname(__file__)), "oracle", "_ref", "libtridpart_ref.so")),
    reason="oracle/_ref not built")


# ----------------------------------------------------------- port == reference
@needs_ref
@pytest.mark.parametrize("n,seed", [(2, 0), (3, 9), (16, 1), (1000, 7), (100_003, 42)])
def test_generator_bit_identical(oracle_mod, n, seed):
    p = oracle_mod.generate_system(n, seed)
    r = oracle_mod.generate_system(n, seed, impl="ref")
    for k in ("sub", "diag", "sup", "rhs"):
        assert np.array_equal(getattr(p, k), getattr(r, k))


@needs_ref
@pytest.mark.parametrize("n,sizes", [(16, [4]), (10_000, [4]), (10_000, [8, 10, 8]),
                                     (99_999, [64, 10, 32, 16]), (5_001, [7, 3, 2, 5, 9]),
                                     (3, [4]), (100, [5000])])
def test_solve_bit_identical(oracle_mod, n, sizes):
    s = oracle_mod.generate_system(n, 11)
    assert np.array_equal(oracle_mod.solve_partition(s, sizes),
                          oracle_mod.solve_partition(s, sizes, impl="ref"))
    assert np.array_equal(oracle_mod.thomas_solve(s), oracle_mod.thomas_solve(s, impl="ref"))


@needs_ref
def test_interface_levels_bit_identical(oracle_mod):
    s = oracle_mod.generate_system(3000, 5)
    a, b = [], []
    oracle_mod.solve_partition(s, [8, 10, 4], observer=lambda *v: a.append(v))
    oracle_mod.solve_partition(s, [8, 10, 4], impl="ref", observer=lambda *v: b.append(v))
    assert len(a) == len(b) == 3
    for va, vb in zip(a, b):
        assert va[0] == vb[0]
        for x, y in zip(va[1:], vb[1:]):
            assert np.array_equal(x, y)


@needs_ref
def test_predictors_bit_identical_on_grid(oracle_mod):
    pn, pl = oracle_mod.model_pairs(0)
    dn, dl = oracle_mod.model_pairs(1)
    lib = oracle_mod.ref()
    for e in range(20, 380):
        n = int(round(10 ** (e / 40)))
        assert oracle_mod.predict(pn, pl, 1, n) == lib.ref_predict_size(n)
        assert oracle_mod.predict(dn, dl, 1, n) == lib.ref_predict_depth(n)


# --------------------------------------------------------------- golden values
def test_golden_solutions(oracle_mod, golden):
    for g in golden["solutions"]:
        s = oracle_mod.generate_system(g["n"], g["seed"])
        assert math.fsum(s.diag) == pytest.approx(g["sum_diag"], abs=1e-9)
        assert math.fsum(s.rhs) == pytest.approx(g["sum_rhs"], abs=1e-9)
        x = oracle_mod.solve_partition(s, g["sizes"])
        assert [float(x[i]) for i in g["idx"]] == g["x"]       # bit-exact vs the reference
        assert math.fsum(x) == pytest.approx(g["sum_x"], abs=1e-9)


def test_survey_pins(oracle_mod):
    # SURVEY.md §8(c) "Derived golden vectors" (tolerance pins)
    s = oracle_mod.generate_system(16, 1)
    x = oracle_mod.solve_partition(s, [4])
    assert x[0] == pytest.approx(-0.27113847387188172, abs=1e-15)
    assert x[15] == pytest.approx(-0.56342409348035738, abs=1e-15)
    assert math.fsum(x) == pytest.approx(-1.2571923477126126, abs=1e-14)
    s = oracle_mod.generate_system(10_000, 1)
    assert math.fsum(s.diag) == pytest.approx(10.578227862787433, abs=1e-12)
    x = oracle_mod.solve_partition(s, [4])
    assert x[5000] == pytest.approx(0.40220197517592371, abs=1e-15)
    assert math.fsum(x) == pytest.approx(22.389648433379122, abs=1e-11)
    assert oracle_mod.residual_inf(s, x) < 1e-15


def test_golden_predictions(oracle_mod, golden, models):
    pn, pl, dn, dl = models
    for g in golden["predictions"]:
        assert oracle_mod.predict(pn, pl, 1, g["n"]) == g["m"]
        assert oracle_mod.predict(dn, dl, 1, g["n"]) == g["R"]


def test_golden_policies(oracle_mod, golden, models):
    pn, pl, _, _ = models
    for g in golden["policies"]:
        assert oracle_mod.recursion_sizes(g["n"], g["R"], pn, pl) == g["sizes"]


# ------------------------------------------- the reference's unit tests, on the oracle
def test_make_plan_cases(oracle_mod):
    # test_partition.cpp:13-35
    assert oracle_mod.make_plan(16, 4) == [(0, 4), (4, 8), (8, 12), (12, 16)]
    assert oracle_mod.make_plan(10, 4) == [(0, 4), (4, 8), (8, 10)]
    assert oracle_mod.make_plan(9, 4) == [(0, 4), (4, 9)]
    assert oracle_mod.make_plan(5, 8) == [(0, 5)]
    with pytest.raises(ValueError):
        oracle_mod.make_plan(1, 4)
    with pytest.raises(ValueError):
        oracle_mod.make_plan(10, 1)


def test_make_plan_invariants(oracle_mod):
    # test_partition.cpp:37-53
    rng = np.random.default_rng(99)
    for _ in range(300):
        n = 2 + int(rng.integers(0, 5000))
        m = 2 + int(rng.integers(0, 70))
        blocks = oracle_mod.make_plan(n, m)
        pos = 0
        for j, (s, e) in enumerate(blocks):
            assert s == pos and e - s >= 2
            if j + 1 < len(blocks):
                assert e - s == m
            else:
                assert e - s <= m + 1
            pos = e
        assert pos == n


def test_reduce_block_identity_and_length2(oracle_mod):
    n = 8
    s = oracle_mod.System(np.zeros(n), np.ones(n), np.zeros(n), np.arange(1.0, 9.0))
    q = oracle_mod.reduce_block(s, 2, 6)
    assert list(q) == [0, 1, 0, 3, 0, 1, 0, 6]
    s = oracle_mod.generate_system(6, 21)
    q = oracle_mod.reduce_block(s, 2, 4)
    assert list(q) == [s.sub[2], s.diag[2], s.sup[2], s.rhs[2], s.sub[3], s.diag[3], s.sup[3], s.rhs[3]]


def test_interface_equations_exact(oracle_mod):
    # test_partition.cpp:86-100
    s = oracle_mod.generate_system(60, 5)
    x = oracle_mod.dense_solve(s)
    a1, b1, g1, d1, a2, b2, g2, d2 = oracle_mod.reduce_block(s, 20, 32)
    r1 = a1 * x[19] + b1 * x[20] + g1 * x[31] - d1
    r2 = a2 * x[20] + b2 * x[31] + g2 * x[32] - d2
    scale = max(1.0, abs(d1), abs(d2))
    assert abs(r1) / scale <= 1e-12 and abs(r2) / scale <= 1e-12


def test_solve_vs_dense_and_depths(oracle_mod):
    s = oracle_mod.generate_system(16, 3)
    assert oracle_mod.rel_inf_diff(oracle_mod.solve_partition(s, [4]), oracle_mod.dense_solve(s)) <= 1e-10
    s = oracle_mod.generate_system(20_000, 23)
    ref = oracle_mod.thomas_solve(s)
    for depth in range(5):
        sizes = [10 if l % 2 else 8 for l in range(depth + 1)]
        assert oracle_mod.rel_inf_diff(oracle_mod.solve_partition(s, sizes), ref) <= 1e-9


def test_thomas_vs_dense_and_zero_pivot(oracle_mod):
    s = oracle_mod.generate_system(50, 7)
    x = oracle_mod.thomas_solve(s)
    assert oracle_mod.rel_inf_diff(x, oracle_mod.dense_solve(s)) <= 1e-10
    z = oracle_mod.System([0, 1], [0, 2], [1, 0], [1, 1])
    with pytest.raises(oracle_mod.OracleZeroPivot):
        oracle_mod.thomas_solve(z)


def test_knn_pins(oracle_mod, models):
    pn, pl, dn, dl = models
    # test_knn.cpp:30-41, acceptance.cpp:125-139
    for n, m in ((100000, 32), (30000, 16), (65000, 20), (1000000000, 64), (20000000, 64),
                 (4500, 4), (5000, 8), (25000, 8), (60000, 20), (80000, 32)):
        assert oracle_mod.predict(pn, pl, 1, n) == m
    for n, lab in zip(pn, pl):
        assert oracle_mod.predict(pn, pl, 1, int(n)) == lab
    # acceptance.cpp:182-203 + "depth 4 never wins"
    for n, r in ((100000, 0), (2200000, 0), (2300000, 1), (3000000, 1), (4800000, 1),
                 (5000000, 2), (9600000, 2), (10000000, 3), (100000000, 3)):
        assert oracle_mod.predict(dn, dl, 1, n) == r
    n = 1000
    while n <= 1_000_000_000:
        assert oracle_mod.predict(dn, dl, 1, n) != 4
        n = int(n * 1.1)
    # test_policy.cpp:34-46
    assert oracle_mod.recursion_sizes(100000000, 3, pn, pl) == [64, 10, 32, 16]
    assert oracle_mod.recursion_sizes(4000000, 1, pn, pl) == [32, 32]
    assert oracle_mod.recursion_sizes(1000000, 0, pn, pl) == [32]
    for bad in (5, -1):
        with pytest.raises(ValueError):
            oracle_mod.recursion_sizes(1000000, bad, pn, pl)
