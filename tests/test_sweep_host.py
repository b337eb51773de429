"""Host side of the B200 sweep / re-fit pipeline (no GPU): the plateau
correction and the canonical CSV writer against the reference's own
expectations (acceptance.cpp criteria 8 and 10)."""
import os

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_DATA = os.path.join(ROOT, "oracle", "_ref", "data")
needs_data = pytest.mark.skipif(not os.path.isdir(REF_DATA), reason="reference data not staged")


def padded_table1(tp):
    # acceptance.cpp:52-68
    s = tp.read_observations(os.path.join(REF_DATA, "table1_fp64.csv"))
    s.sort_by_n()
    cands = sorted({r.label for r in s.rows} | {r.corrected for r in s.rows if r.corrected is not None})
    for r in s.rows:
        best = r.times[r.label]
        for m in cands:
            r.times.setdefault(m, 1.1 * best)
    return s


@needs_data
def test_plateau_correction_reproduces_table1_corrected_column(tp):
    from paper_2510_27351_b200.sweep import plateau_correct

    s = padded_table1(tp)
    labels = plateau_correct(s, 0.04)
    assert labels == [r.corrected for r in s.rows]


@needs_data
def test_write_read_roundtrip_is_canonical(tp, tmp_path):
    from paper_2510_27351_b200.sweep import apply_plateau_correction, write_observations

    s = tp.read_observations(os.path.join(REF_DATA, "table1_fp64.csv"))
    p1, p2 = tmp_path / "a.csv", tmp_path / "b.csv"
    write_observations(s, str(p1))
    back = tp.read_observations(str(p1))
    assert [(r.n, r.label, r.corrected, r.times) for r in back.rows] == \
           [(r.n, r.label, r.corrected, r.times) for r in s.rows]
    write_observations(back, str(p2))
    assert p1.read_bytes() == p2.read_bytes()
    corr = apply_plateau_correction(padded_table1(tp), 0.04)
    assert all(r.corrected is not None for r in corr.rows)


def test_plateau_single_run_and_missing_times(tp):
    from paper_2510_27351_b200.sweep import MissingTimesError, plateau_correct

    O = tp.Observation
    rows = [O(n=10, label=4, times={4: 1.0, 8: 1.01}), O(n=20, label=8, times={4: 1.02, 8: 1.0}),
            O(n=30, label=8, times={8: 1.0, 16: 1.03})]
    # one run covers all rows with the shared near-optimal candidate 8
    assert plateau_correct(tp.ObservationSet(rows), 0.04) == [8, 8, 8]
    with pytest.raises(MissingTimesError):
        plateau_correct(tp.ObservationSet([O(n=1, label=4)]), 0.04)


def test_bundled_b200_size_model_is_the_refit_of_the_committed_sweep(tp):
    """heuristics/b200_fp64_size_model.json = fit_knn(k=1) of the plateau-
    corrected B200 sweep (profiles/r02_sweep_b200.csv, config 5): same pairs,
    same predictions; the reference-parity default model is unchanged."""
    import os

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    obs = tp.read_observations(os.path.join(root, "profiles", "r02_sweep_b200.csv"))
    refit = tp.fit_knn(obs.with_corrected_labels(), 1)
    bundled = tp.b200_size_model()
    assert [(p.n, p.label) for p in bundled.pairs] == [(p.n, p.label) for p in refit.pairs]
    assert bundled.metadata.get("device") == "b200"
    for n in (100, 4_500, 60_000, 1_000_000, 100_000_000, 1_000_000_000):
        assert tp.predict(bundled, n) == tp.predict(refit, n)
    assert tp.predicted_policy(100_000_000).sizes == [64, 10, 32, 16]  # reference models
    # on the round-2 kernels the plateau-corrected B200 optimum at 1e8 is m = 128
    assert tp.predicted_policy(100_000_000, size_model=bundled).sizes[0] == 128
