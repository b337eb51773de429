"""Generate the golden fixtures from the REFERENCE itself (oracle/_ref: the
unmodified reference headers behind an extern "C" shim). Run in the build
container (needs oracle/_ref built from /root/reference):

    python tests/golden/make_golden.py

Writes tests/golden/reference_golden.json:
  * solutions: x at sampled rows + Kahan sums for generate_system(N, seed)
    solved with the given policy (solve_partition, partition.hpp:235-248)
  * n16: the full N=16, m=4 solution
  * predictions: predict(size_model|depth_model, N) on a geometric N grid
    (knn.hpp:57-77), models fitted exactly as test_policy.cpp:14-21
  * policies: recursion_sizes(N, R, size_model) (policy.hpp:25-45)
"""
import json
import math
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402


def kahan(v):
    return math.fsum(float(t) for t in v)


def main():
    lib = oracle.ref()
    out = {"generator": "oracle/_ref (reference headers, g++ -O3 -DNDEBUG)"}
    sols = []
    for n, sizes, seed in ((16, [4], 1), (10_000, [4], 1), (10_000, [8, 10, 8], 17),
                           (100_000, [32, 10, 16], 5), (1_000_000, [32], 1)):
        s = oracle.generate_system(n, seed, impl="ref")
        x = oracle.solve_partition(s, sizes, impl="ref")
        idx = sorted({0, 1, n // 3, n // 2, n - 2, n - 1})
        sols.append({"n": n, "sizes": sizes, "seed": seed,
                     "sum_sub": kahan(s.sub), "sum_diag": kahan(s.diag),
                     "sum_super": kahan(s.sup), "sum_rhs": kahan(s.rhs),
                     "idx": idx, "x": [float(x[i]) for i in idx], "sum_x": kahan(x),
                     "max_abs_x": float(np.max(np.abs(x))),
                     "residual": float(lib.ref_residual_inf(n, *s.ptrs(), x.ctypes.data_as(oracle._D)))})
        if n == 16:
            out["n16"] = {"seed": seed, "sizes": sizes, "x": [float(v) for v in x]}
    out["solutions"] = sols
    grid = sorted({int(round(10 ** (e / 40))) for e in range(40, 361)} |
                  {4743, 4744, 27386, 27387, 54772, 54773, 77459, 77460, 14142135, 14142136,
                   2249444, 2249445, 4898979, 4898980, 9797958, 9797959})
    out["predictions"] = [{"n": n, "m": int(lib.ref_predict_size(n)), "R": int(lib.ref_predict_depth(n))}
                          for n in grid]
    pols = []
    buf = np.zeros(8, dtype=np.int64)
    for n in (10_000, 100_000, 1_000_000, 4_000_000, 10_000_000, 100_000_000, 1_000_000_000):
        for R in range(5):
            cnt = lib.ref_recursion_sizes(n, R, buf.ctypes.data_as(oracle._I64))
            pols.append({"n": n, "R": R, "sizes": [int(v) for v in buf[:cnt]]})
    out["policies"] = pols
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "reference_golden.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print(f"wrote {path}: {len(out['predictions'])} predictions, {len(pols)} policies")


if __name__ == "__main__":
    main()
