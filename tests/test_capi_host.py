"""The C-ABI library on the CPU: it loads, exports every symbol declared in
include/tridpart_b200.h, and its host-side functions (planner, predictors,
observation reader) agree bit-for-bit with the oracle. No GPU compute here."""
import json
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "tridpart_b200.h")
REF_DATA = os.path.join(ROOT, "oracle", "_ref", "data")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(tp_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol(tp):
    from paper_2510_27351_b200 import _lib

    syms = declared_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(_lib.lib, s), s
    assert set(syms) == set(_lib.EXPORTS)
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    for s in syms:
        assert re.search(rf"\bT {s}\b", out), f"{s} not exported with C linkage"


def test_library_is_sm100a_only(tp):
    from paper_2510_27351_b200 import _lib

    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out
    assert all("sm_100a" in l for l in out.splitlines() if l.strip())


def test_abi_version(tp):
    from paper_2510_27351_b200 import _lib

    assert _lib.lib.tp_abi_version() == 2


def test_context_without_gpu_fails_loudly(tp):
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(tp.DeviceError):
        tp.Context(0)


def test_make_plan_matches_oracle(tp, oracle_mod):
    rng = np.random.default_rng(3)
    for _ in range(300):
        n = 2 + int(rng.integers(0, 5000))
        m = 2 + int(rng.integers(0, 1300))
        got = [(b.start, b.end) for b in tp.make_plan(n, m).blocks]
        assert got == oracle_mod.make_plan(n, m)
    with pytest.raises(tp.InvalidSizeError):
        tp.make_plan(1, 4)
    with pytest.raises(tp.InvalidSizeError):
        tp.make_plan(10, 1)


def test_plan_levels_follow_the_reference_recursion(tp, oracle_mod):
    """Level sizes are the oracle's N_{l+1} = 2*K_l chain (partition.hpp:199-210)."""
    for n, sizes in ((10_000, [4]), (1_000_000, [32]), (100_000_000, [64, 10, 32, 16]),
                     (1_000_000_000, [64, 10, 32, 32]), (3, [4]), (5, [8]), (20_000, [8, 10, 8, 10, 8])):
        ln, lm, nf = tp.plan_levels(n, sizes)
        cur, want = n, []
        for l, m in enumerate(sizes):
            if cur < 4:
                break
            want.append((cur, m))
            cur = 2 * len(oracle_mod.make_plan(cur, m))
        policy_levels = [(a, b) for a, b in zip(ln, lm) if b > 0]
        assert policy_levels == want
        # device-internal levels (m < 0) only shrink an oversized final system:
        # m = 32, or one last m = 16 level that the fused deepest-level kernel
        # (k_level_final_cl) solves together with its interface (<= 16 x 1024 rows)
        internal = [(a, -b) for a, b in zip(ln, lm) if b < 0]
        for i, (a, m) in enumerate(internal):
            assert a > 6144 and (m == 32 or (m == 16 and i == len(internal) - 1))
        assert nf <= 6144 or (internal and internal[-1][1] == 16 and nf <= 16 * 1024) or \
            (not internal and lm[-1] <= 16 and nf <= 16 * 1024)
    assert tp.plan_levels(100_000_000, [64, 10, 32, 16]) == (
        [100_000_000, 3_125_000, 625_000, 39_064], [64, 10, 32, 16], 4884)


def test_predictors_bit_exact_vs_oracle(tp, oracle_mod):
    sm, dm = tp.default_size_model(), tp.default_depth_model()
    pn, pl = sm._arrays()
    dn, dl = dm._arrays()
    for e in range(0, 400):
        n = max(2, int(round(10 ** (e / 40))))
        assert tp.predict(sm, n) == oracle_mod.predict(pn, pl, 1, n)
        assert tp.predict(dm, n) == oracle_mod.predict(dn, dl, 1, n)
    # derived switch points
    for n, m in ((4743, 4), (4744, 8), (27386, 8), (27387, 16), (54772, 16), (54773, 20),
                 (77459, 20), (77460, 32), (14142135, 32), (14142136, 64)):
        assert tp.predict(sm, n) == m
    for n, r in ((2249444, 0), (2249445, 1), (4898979, 1), (4898980, 2), (9797958, 2), (9797959, 3)):
        assert tp.predict(dm, n) == r


def test_golden_predictions_and_policies(tp):
    with open(os.path.join(ROOT, "tests", "golden", "reference_golden.json")) as f:
        g = json.load(f)
    sm, dm = tp.default_size_model(), tp.default_depth_model()
    for p in g["predictions"]:
        assert tp.predict(sm, p["n"]) == p["m"]
        assert tp.predict(dm, p["n"]) == p["R"]
    for p in g["policies"]:
        assert tp.recursion_sizes(p["n"], p["R"], sm).sizes == p["sizes"]


def test_knn_k_greater_than_one_matches_oracle(tp, oracle_mod):
    rng = np.random.default_rng(1)
    for _ in range(50):
        npairs = int(rng.integers(1, 30))
        pn = np.sort(rng.integers(10, 10**8, npairs))
        pl = rng.choice([4, 8, 16, 32, 64], npairs).astype(np.int32)
        k = int(rng.integers(1, npairs + 1))
        model = tp.HeuristicModel([tp.TrainingPair(int(a), int(b)) for a, b in zip(pn, pl)], k)
        for q in rng.integers(2, 10**9, 20):
            assert tp.predict(model, int(q)) == oracle_mod.predict(pn, pl, k, int(q))


def test_reference_test_pins(tp):
    sm, dm = tp.default_size_model(), tp.default_depth_model()
    assert tp.recursion_sizes(100000000, 3, sm).sizes == [64, 10, 32, 16]
    assert tp.recursion_sizes(4000000, 1, sm).sizes == [32, 32]
    assert tp.recursion_sizes(1000000, 0, sm).sizes == [32]
    for bad in (5, -1):
        with pytest.raises(tp.DepthOutOfRangeError):
            tp.recursion_sizes(1000000, bad, sm)
    assert tp.predicted_policy(100_000_000).sizes == [64, 10, 32, 16]
    assert tp.predicted_policy(1_000_000_000).sizes == [64, 10, 32, 32]
    # single pair answers everything; bad k (test_knn.cpp:22-51)
    one = tp.fit_knn(tp.ObservationSet([tp.Observation(n=1000, label=4)]), 1)
    assert tp.predict(one, 10) == 4 and tp.predict(one, 100000000) == 4
    with pytest.raises(tp.EmptyTrainingSetError):
        tp.fit_knn(tp.ObservationSet(), 1)
    two = tp.ObservationSet([tp.Observation(n=100, label=4), tp.Observation(n=200, label=4)])
    with pytest.raises(tp.KTooLargeError):
        tp.fit_knn(two, 3)


@pytest.mark.skipif(not os.path.isdir(REF_DATA), reason="reference data tables not staged")
def test_read_observations_and_refit_equal_bundled(tp):
    obs = tp.read_observations(os.path.join(REF_DATA, "table1_fp64.csv"))
    assert obs.size() == 37
    row = [r for r in obs.rows if r.n == 70000][0]
    assert row.label == 35 and row.corrected == 20 and row.times == {20: 0.95752, 35: 0.95671}
    refit = tp.fit_knn(obs.with_corrected_labels(), 1)
    bundled = tp.default_size_model()
    assert [(p.n, p.label) for p in refit.pairs] == [(p.n, p.label) for p in bundled.pairs]
    depth = tp.fit_depth_model(tp.read_observations(os.path.join(REF_DATA, "table2_recursion.csv")))
    assert [(p.n, p.label) for p in depth.pairs] == [(p.n, p.label) for p in tp.default_depth_model().pairs]
    assert all(r.depth_label for r in tp.read_observations(os.path.join(REF_DATA, "table2_recursion.csv")).rows)


def test_read_observations_errors(tp, tmp_path):
    p = tmp_path / "bad.csv"
    p.write_text("N,m\n1,2\n")
    with pytest.raises(tp.MalformedHeaderError):
        tp.read_observations(str(p))
    p.write_text("N,precision,device,streams,m,time_ms,is_opt,corrected_m,opt_R\n12x,fp64,d,1,4,1.0,1,,\n")
    with pytest.raises(tp.BadNumberError):
        tp.read_observations(str(p))
    with pytest.raises(tp.Error):
        tp.read_observations(str(tmp_path / "missing.csv"))


def test_model_json_roundtrip_and_schema(tp, tmp_path):
    m = tp.default_size_model()
    path = tmp_path / "model.json"
    tp.save_model(m, str(path))
    back = tp.load_model(str(path))
    assert [(p.n, p.label) for p in back.pairs] == [(p.n, p.label) for p in m.pairs]
    assert back.k == 1 and back.transform == "log10_n"
    # the exported heuristics files are in the same format
    bundled = tp.load_model(os.path.join(ROOT, "paper_2510_27351_b200", "heuristics", "fp64_size_model.json"))
    assert [(p.n, p.label) for p in bundled.pairs] == [(p.n, p.label) for p in m.pairs]
    doc = json.loads(path.read_text())
    doc["version"] = 2
    path.write_text(json.dumps(doc))
    with pytest.raises(tp.VersionMismatchError):
        tp.load_model(str(path))
    path.write_text("{not json")
    with pytest.raises(tp.SchemaError):
        tp.load_model(str(path))


def test_shard_entries_reject_bad_arguments_without_a_device(tp):
    """The multi-GPU entries validate their arguments before touching CUDA:
    NULL context / NULL outputs / bad rank counts give TP_ERR_INVALID_ARGUMENT
    (the status the Python layer maps to ValueError), never a crash."""
    import ctypes as C

    from paper_2510_27351_b200 import _lib
    from paper_2510_27351_b200._lib import TpError

    lib, INV = _lib.lib, _lib.INVALID_ARGUMENT
    err = TpError()
    box = C.c_void_p()
    h = (C.c_uint8 * 64)()
    assert lib.tp_shard_mailbox(None, 2, C.byref(box), C.byref(err)) == INV
    assert lib.tp_ipc_get_handle(None, C.c_void_p(0x1000), h, C.byref(err)) == INV
    assert lib.tp_ipc_open_handle(None, h, C.byref(box), C.byref(err)) == INV
    ptrs = (C.c_void_p * 2)()
    assert lib.tp_shard_attach(None, 2, 0, ptrs, C.byref(err)) == INV
    sizes = np.array([32], dtype=np.int64)
    sp = sizes.ctypes.data_as(C.POINTER(C.c_int64))
    for fn in (lib.tp_shard_solve_f64_dev, lib.tp_shard_prepare_f64_dev):
        st = fn(None, None, None, None, None, 100, sp, 1, None, None, C.byref(err))
        assert st == INV, st
    with pytest.raises(ValueError):
        from paper_2510_27351_b200.tridpart import _call
        _call(lib.tp_shard_mailbox, None, 0, C.byref(box))


# ------------------------------------------------------- round 2: host pieces
def test_generate_system_is_bit_identical_to_the_reference(tp, oracle_mod):
    """generate_system (bench.hpp:68-93): the library's host generator equals the
    reference's own (oracle/_ref, the unmodified headers) bit for bit."""
    if not oracle_mod.ref_available():
        pytest.skip("oracle/_ref not built")
    for n, seed, delta in ((2, 0, 1.5), (3, 1, 1.5), (16, 1, 1.5), (10_000, 1, 1.5),
                           (100_001, 20240601, 2.5), (1_000_000, 1, 1.5)):
        s = tp.generate_system(n, seed, delta)
        r = oracle_mod.generate_system(n, seed, delta, impl="ref")
        for got, want in ((s.sub, r.sub), (s.diag, r.diag), (s.super, r.sup), (s.rhs, r.rhs)):
            assert got.tobytes() == want.tobytes(), (n, seed)
    with pytest.raises(tp.InvalidSizeError):
        tp.generate_system(1, 0)
    with pytest.raises(tp.InvalidSizeError):
        tp.generate_system(10, 0, delta=1.0)


def test_generate_system_golden_sums(tp):
    """SURVEY §8(c) pins of generate_system(N, 1) (reference-generated)."""
    s = tp.generate_system(10_000, 1)
    assert abs(float(np.sum(s.diag)) - 10.578227862787433) < 1e-9
    assert abs(float(np.sum(s.rhs)) - -26.256125191010906) < 1e-9


def _levels(tp, n, sizes):
    return tp.plan_levels(n, tp.RecursionPolicy(sizes))


@pytest.mark.parametrize("n,m", [(10_000, 2049), (10_000, 4096), (100_000, 10_000), (1_000_000, 100_000),
                                 (100_000, 100_000), (100_000, 250_000), (5_000, 4_999), (20_001, 10_000)])
def test_long_blocks_become_split_chains(tp, n, m):
    """Blocks longer than 2048 rows are reduced through split levels (negative m
    in plan_levels) ending in a level with the original block count: the
    interface handed on is 2K rows, K = make_plan(n, m)'s block count."""
    ln, lm, nf = _levels(tp, n, [m])
    k = len(tp.make_plan(n, m).blocks)
    assert lm[0] < 0, (ln, lm)                  # the first plan level is a split
    policy = [i for i, v in enumerate(lm) if v > 0]
    assert policy, (ln, lm)
    last = policy[0]                            # the level keeping the block boundaries
    assert all(v < 0 for v in lm[:last])
    # each split level's system shrinks ~4x (chunks of <= 8 rows -> 2 rows)
    for a, b in zip(ln[:last], ln[1:last + 1]):
        assert b <= a // 3 + 2
    # what follows the policy level is the 2K-row interface (or device-internal levels of it)
    if last + 1 < len(ln):
        assert ln[last + 1] == 2 * k
    else:
        assert nf == 2 * k


def test_short_blocks_are_not_split(tp):
    for m in (2, 4, 64, 256, 1250, 2048):
        _, lm, _ = _levels(tp, 100_000, [m])
        assert lm[0] == m


def test_cpp_drop_in_headers_compile_standalone(tmp_path):
    """Every shadow header under include/tridpart compiles on its own (the
    reference's include layout: a caller swaps only its -I path)."""
    hdrs = sorted(os.listdir(os.path.join(ROOT, "include", "tridpart")))
    assert {"bench.hpp", "errors.hpp", "io.hpp", "knn.hpp", "observations.hpp", "partition.hpp",
            "policy.hpp", "tridiagonal.hpp"} <= set(hdrs)
    for h in hdrs:
        src = tmp_path / f"inc_{h}.cpp"
        src.write_text(f'#include "tridpart/{h}"\nint main() {{ return 0; }}\n')
        r = subprocess.run(["g++", "-std=c++20", "-fsyntax-only", "-I", os.path.join(ROOT, "include"), str(src)],
                           capture_output=True, text=True)
        assert r.returncode == 0, (h, r.stderr)


def test_reference_unit_tests_build_against_the_drop_in_headers(tmp_path):
    """The reference's unmodified proj/tests/test_{partition,tridiagonal,policy}.cpp
    build with -I<repo>/include in place of -I<reference>/proj/include (built by
    tests/cpp/Makefile; run on the GPU in test_cpp_shim.py)."""
    exe = os.path.join(ROOT, "tests", "cpp", "_build", "ref_unit_tests")
    if not os.path.exists("/root/reference/proj/tests/test_partition.cpp"):
        if not os.path.exists(exe):
            pytest.skip("no reference checkout and no prebuilt binary")
        return
    r = subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "tests", "cpp")], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    assert os.path.exists(exe)
    # the reference's include tree must not be on the path: every tridpart/ header
    # the objects saw is ours
    dep = subprocess.run(["g++", "-std=c++20", "-M", "-I", os.path.join(ROOT, "include"),
                          "-I", os.path.join(ROOT, "tests", "cpp", "catch_shim"),
                          "-I", "/root/reference/proj/tests", "-DTRIDPART_DATA_DIR=\"x\"",
                          "/root/reference/proj/tests/test_partition.cpp"], capture_output=True, text=True)
    assert dep.returncode == 0, dep.stderr
    assert "/root/reference/proj/include" not in dep.stdout
    assert os.path.join(ROOT, "include", "tridpart", "partition.hpp") in dep.stdout
