"""B200 sweeps and the model re-fit pipeline (BASELINE config 5).

Mirrors the reference's timing harness (include/tridpart/bench.hpp) with the
solve on the B200:

  sweep_m(n, candidates, runs, seed)  bench.hpp:171-188: the non-recursive
      method for every candidate m on one generated system; argmin of the
      median times (record_argmin :158-166)
  sweep_r(n, max_r, size_model, runs)  bench.hpp:192-209: R = 0..max_r with
      recursion_sizes(n, R, size_model)
  SweepResult.to_observation()         bench.hpp:143-154
  write_observations(set, path)        io.hpp:142-174 (canonical CSV writer)
  plateau_correct(set, tolerance)      plateau.hpp:24-98
  apply_plateau_correction(set, tol)   plateau.hpp:101-108

Timing: inputs resident on the device (device generator, seed), CUDA events
on the launch stream around the captured-graph solve, 1 warm-up + `runs`
timed solves, median (bench.hpp:113-126). The reference puts its residual
gate (kBenchResidualTol = 1e-8, bench.hpp:22) inside the timed region; here
the gate is applied to every candidate after its timed runs (a failing
candidate raises SolveFailedError) but is not timed.

CLI:  python -m paper_2510_27351_b200.sweep --out profiles/sweep_b200.csv
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence

from .tridpart import (Error, HeuristicModel, Observation, ObservationSet, RecursionPolicy,
                       default_size_model, fit_knn, generate_system, kMaxRecursionDepth,
                       kObservationsHeader, predict, recursion_sizes, residual_inf,
                       solve_partition_async, DepthOutOfRangeError, InvalidSizeError)

kBenchResidualTol = 1e-8  # bench.hpp:22

# the paper's 37 Table-I sizes (data/table1_fp64.csv N column)
TABLE1_SIZES = [100, 200, 400, 500, 800, 1000, 2000, 4000, 4500, 5000, 8000, 10000, 20000, 25000,
                30000, 40000, 50000, 60000, 70000, 75000, 80000, 100000, 200000, 400000, 500000,
                800000, 1000000, 2000000, 4000000, 5000000, 8000000, 10000000, 20000000, 40000000,
                50000000, 80000000, 100000000]
# candidate sub-system sizes in [4; 1250] (SURVEY §8(d) proposal)
DEFAULT_CANDIDATES = [4, 5, 8, 10, 16, 20, 25, 32, 35, 40, 50, 64, 80, 100, 125, 128, 250, 256,
                      500, 625, 1000, 1250]


class SolveFailedError(Error):
    pass


class MissingTimesError(Error):
    pass


@dataclass
class TimingStats:
    median_ms: float = 0.0
    min_ms: float = 0.0
    max_ms: float = 0.0
    runs: int = 0


@dataclass
class SweepEntry:
    candidate: int
    stats: TimingStats


@dataclass
class SweepResult:
    n: int = 0
    entries: List[SweepEntry] = field(default_factory=list)
    argmin: int = 0
    runs: int = 0
    clock_name: str = "cuda_events"
    depth_sweep: bool = False

    def to_observation(self, device: str = "b200", precision: str = "fp64",
                       streams: int = 1) -> Observation:
        obs = Observation(n=self.n, label=self.argmin, device=device, precision=precision,
                          streams=streams, depth_label=self.depth_sweep)
        for e in self.entries:
            obs.times[e.candidate] = e.stats.median_ms
        return obs


def _record_argmin(res: SweepResult):
    best = math.inf
    for e in res.entries:
        if e.stats.median_ms < best:
            best = e.stats.median_ms
            res.argmin = e.candidate


def time_solve(sys, policy: RecursionPolicy, runs: int) -> TimingStats:
    """1 warm-up + `runs` timed device solves, median (bench.hpp:104-127)."""
    import torch

    if runs < 1:
        raise InvalidSizeError("runs must be >= 1")
    x = torch.empty_like(sys.diag)
    solve_partition_async(sys, policy, out=x)  # warm-up (also captures the graph)
    torch.cuda.synchronize()
    times = []
    for _ in range(runs):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        solve_partition_async(sys, policy, out=x)
        e1.record()
        e1.synchronize()
        times.append(e0.elapsed_time(e1))
    res = residual_inf(sys, x)
    if not res <= kBenchResidualTol:
        raise SolveFailedError(f"residual {res} above gate")
    ordered = sorted(times)
    med = ordered[runs // 2] if runs % 2 else 0.5 * (ordered[runs // 2 - 1] + ordered[runs // 2])
    return TimingStats(med, ordered[0], ordered[-1], runs)


def sweep_m(n: int, candidates: Sequence[int], runs: int, seed: int = 1, sys=None) -> SweepResult:
    """bench.hpp:171-188 on the B200."""
    if not candidates:
        raise InvalidSizeError("no sweep candidates")
    if any(m < 2 for m in candidates):
        raise InvalidSizeError("candidate m must be >= 2")
    sys = sys if sys is not None else generate_system(n, seed, device=True)
    res = SweepResult(n=n, runs=runs)
    for m in candidates:
        res.entries.append(SweepEntry(int(m), time_solve(sys, RecursionPolicy([int(m)]), runs)))
    _record_argmin(res)
    return res


def sweep_r(n: int, max_r: int, size_model: HeuristicModel, runs: int, seed: int = 1,
            sys=None) -> SweepResult:
    """bench.hpp:192-209 on the B200."""
    if max_r < 0 or max_r > kMaxRecursionDepth:
        raise DepthOutOfRangeError("max recursion depth must be in [0, 4]")
    sys = sys if sys is not None else generate_system(n, seed, device=True)
    res = SweepResult(n=n, runs=runs, depth_sweep=True)
    for r in range(max_r + 1):
        res.entries.append(SweepEntry(r, time_solve(sys, recursion_sizes(n, r, size_model), runs)))
    _record_argmin(res)
    return res


# ------------------------------------------------------------------ io.hpp
def _fmt_time(t: float) -> str:
    return "%.6f" % t


def write_observations(obs_set: ObservationSet, path: str):
    """Canonical writer (io.hpp:142-174): rows sorted by (N, m)."""
    rows = sorted(obs_set.rows, key=lambda r: (r.n, r.precision, r.device))
    out = [kObservationsHeader]

    def emit(o, m, t, is_opt):
        fields = [str(o.n), o.precision, o.device, str(o.streams),
                  "" if m is None else str(m), "" if t is None else _fmt_time(t),
                  "1" if is_opt else "0",
                  str(o.corrected) if (is_opt and o.corrected is not None) else "",
                  str(o.label) if (is_opt and o.depth_label) else ""]
        out.append(",".join(fields))

    for o in rows:
        if o.depth_label:
            emit(o, None, None, True)
            continue
        if not o.times:
            emit(o, o.label, None, True)
            continue
        for m in sorted(o.times):
            emit(o, m, o.times[m], m == o.label)
        if o.label not in o.times:
            emit(o, o.label, None, True)
    with open(path, "w", newline="") as f:
        f.write("\n".join(out) + "\n")


# ------------------------------------------------------------- plateau.hpp
def plateau_correct(sweeps: ObservationSet, tolerance: float = 0.04) -> List[int]:
    """Fewest contiguous runs of rows sharing a near-optimal candidate
    (plateau.hpp:24-98); labels aligned with the rows sorted by N."""
    rows = sorted(sweeps.rows, key=lambda r: (r.n, r.precision, r.device))
    n = len(rows)
    if n == 0:
        return []
    cand = []
    for r in rows:
        if not r.times:
            raise MissingTimesError(f"row N={r.n} has no per-candidate times")
        best = min(r.times.values())
        cand.append({m for m, t in r.times.items() if t <= (1.0 + tolerance) * best})
    INF = float("inf")
    suffix = [INF] * (n + 1)
    suffix[n] = 0
    for i in range(n - 1, -1, -1):
        inter = set(cand[i])
        for j in range(i + 1, n + 1):
            if not inter:
                break
            if suffix[j] != INF:
                suffix[i] = min(suffix[i], 1 + suffix[j])
            if j < n:
                inter = inter & cand[j]
    out = [0] * n
    i = 0
    prev = -(2 ** 31)
    while i < n:
        inter = set(cand[i])
        end, chosen = i + 1, set(inter)
        for j in range(i + 1, n + 1):
            if not inter:
                break
            if 1 + suffix[j] == suffix[i]:
                end, chosen = j, set(inter)
            if j < n:
                inter = inter & cand[j]
        ordered = sorted(chosen)
        label = ordered[0]
        for c in ordered:
            if c >= prev:
                label = c
                break
        for r in range(i, end):
            out[r] = label
        prev = label
        i = end
    return out


def apply_plateau_correction(sweeps: ObservationSet, tolerance: float = 0.04) -> ObservationSet:
    """plateau.hpp:101-108."""
    rows = sorted(sweeps.rows, key=lambda r: (r.n, r.precision, r.device))
    labels = plateau_correct(ObservationSet(rows), tolerance)
    out = []
    for r, lab in zip(rows, labels):
        o = Observation(r.n, r.label, lab, dict(r.times), r.precision, r.device, r.streams, r.depth_label)
        out.append(o)
    return ObservationSet(out)


# ------------------------------------------------------------------- CLI
def main(argv=None):
    ap = argparse.ArgumentParser(description=__doc__.split("\n")[0])
    ap.add_argument("--sizes", default="table1", help="'table1' or comma-separated N")
    ap.add_argument("--candidates", default=",".join(map(str, DEFAULT_CANDIDATES)))
    ap.add_argument("--runs", type=int, default=5)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--out", default="sweep_b200.csv")
    ap.add_argument("--report", default=None, help="JSON summary path")
    ap.add_argument("--tolerance", type=float, default=0.04)
    ap.add_argument("--depth", action="store_true",
                    help="sweep R = 0..4 (sweep_r) at the Table II sizes instead of m")
    a = ap.parse_args(argv)
    if a.depth:
        return main_depth(a)
    sizes = TABLE1_SIZES if a.sizes == "table1" else [int(float(s)) for s in a.sizes.split(",")]
    cands = [int(c) for c in a.candidates.split(",")]
    model = default_size_model()
    obs = ObservationSet()
    rows = []
    for n in sizes:
        usable = [m for m in cands if m < n] or [cands[0]]
        res = sweep_m(n, usable, a.runs, a.seed)
        o = res.to_observation()
        obs.rows.append(o)
        pred = predict(model, n)
        t_pred = o.times.get(pred)
        rows.append({"n": n, "argmin_m": res.argmin, "best_ms": o.times[res.argmin],
                     "knn_m": pred, "knn_ms": t_pred,
                     "knn_slowdown": (t_pred / o.times[res.argmin]) if t_pred else None})
        print(f"N={n:>10}  argmin m={res.argmin:>5} ({o.times[res.argmin]:.4f} ms)  "
              f"kNN m={pred:>3} ({t_pred if t_pred is None else round(t_pred, 4)} ms)", flush=True)
    corrected = apply_plateau_correction(obs, a.tolerance)
    write_observations(corrected, a.out)
    refit = fit_knn(corrected.with_corrected_labels(), 1)
    summary = {
        "device": "b200", "runs": a.runs, "candidates": cands, "tolerance": a.tolerance,
        "rows": rows,
        "argmin_equals_knn": sum(1 for r in rows if r["argmin_m"] == r["knn_m"]),
        "n_sizes": len(rows),
        "b200_refit_model": [{"n": p.n, "label": p.label} for p in refit.pairs],
    }
    if a.report:
        with open(a.report, "w") as f:
            json.dump(summary, f, indent=1)
    print(f"kNN (RTX 2080 Ti model) == B200 argmin at {summary['argmin_equals_knn']}/{len(rows)} sizes")


# the paper's Table II sizes (depth model training data)
TABLE2_SIZES = [100000, 1000000, 2000000, 2200000, 2300000, 2400000, 2500000, 3000000, 4000000,
                4500000, 4800000, 5000000, 8000000, 8400000, 9200000, 9600000, 10000000, 100000000]


def main_depth(a):
    """sweep_r over R = 0..4 with the bundled size model; compares the B200
    argmin depth with the depth model's prediction (fit_depth_model, Table II)."""
    from .tridpart import default_depth_model

    sizes = TABLE2_SIZES if a.sizes == "table1" else [int(float(s)) for s in a.sizes.split(",")]
    size_model, depth_model = default_size_model(), default_depth_model()
    obs = ObservationSet()
    rows = []
    for n in sizes:
        res = sweep_r(n, kMaxRecursionDepth, size_model, a.runs, a.seed)
        o = res.to_observation()
        obs.rows.append(o)
        pred = predict(depth_model, n)
        rows.append({"n": n, "argmin_R": res.argmin, "times_ms": o.times, "knn_R": pred})
        print(f"N={n:>10}  argmin R={res.argmin}  times " +
              " ".join(f"R{r}={t:.4f}" for r, t in sorted(o.times.items())) + f"  kNN R={pred}", flush=True)
    write_observations(obs, a.out)
    if a.report:
        with open(a.report, "w") as f:
            json.dump({"device": "b200", "runs": a.runs, "rows": rows,
                       "argmin_equals_knn": sum(1 for r in rows if r["argmin_R"] == r["knn_R"])}, f, indent=1)


if __name__ == "__main__":
    main()
