"""Small solves that touch every kernel variant, for compute-sanitizer runs.

    compute-sanitizer --tool memcheck  python tools/sanitize_cases.py
    compute-sanitizer --tool racecheck python tools/sanitize_cases.py
    compute-sanitizer --tool synccheck python tools/sanitize_cases.py
    compute-sanitizer --tool initcheck python tools/sanitize_cases.py

Covers: k_fast (fixed shapes, both stages, vector and scalar loads), k_fast_rt
(runtime chunk lengths), k_generic (tail blocks, m > 256), the fused deepest
level + finishing solve (k_level_final_cl: cp.async staging, register and
shared-memory sweeps, 16-CTA cluster), level 1 folded into level 0
(k_fast_s1fold), the one-kernel grid solve (k_grid_solve: cp.async
staging into padded shared memory, cooperative grid barrier), the cluster and the
single-CTA finishing solves (solve, sharded reduce / expand, the fused
peer exchange on one rank), FP32, thomas_solve, the
generator and the residual. Sizes are small so the sanitizer finishes in
minutes; every result is checked against the oracle (the
reference configures no sanitizer; this is the B200 build's race/memory check).
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch

    import oracle
    import paper_2510_27351_b200 as tp
    from paper_2510_27351_b200 import sharded

    cases = [
        (5_000, [4]),            # k_fast<4,1>, cluster final
        (30_011, [64, 10]),      # k_fast<8,8>, k_fast<5,2>, tails
        (20_000, [25, 8]),       # k_fast_rt (runtime lengths)
        (9_000, [300]),          # k_generic (m > 256)
        (50, [8]),               # single-CTA final (< 64 rows)
        (3, [4]),                # n < 4: Thomas fallback
        (100_003, [32, 10, 16]), # deeper recursion with tails (fused deepest level, m = 16)
        (20_001, [8]),           # fused deepest level, m = 8 register sweeps, (m + 1)-row tail
        (40_000, [64, 7]),       # fused deepest level, generic sweeps (odd m)
        (160_000, [64, 10, 8]),  # level 1 folded into level 0 (k_fast_s1fold)
        (640_000, [64, 10, 32]), # levels 1 and 2 folded (FOLD2)
        (100_000, [32]),         # one-kernel grid solve, 2-row chunks in registers (k_grid_reg<T, 2>)
        (150_001, [4]),          # grid solve, 2-row chunks, tail block (k_grid_reg<T, 2>)
        (600_001, [32]),         # grid solve, 4-row chunks via registers into smem, tail (k_grid_hyb<T, 4>)
        (1_000_000, [32]),       # grid solve, 8-row chunks (k_grid_hyb<T, 8>, config 2)
        (300_000, [20]),         # grid solve, 5-row chunks in shared memory (k_grid_solve<T, 5>)
        (90_007, [20]),          # grid solve, uneven chunks (k_grid_solve<T, 0>, loop leaves)
    ]
    worst = 0.0
    for n, sizes in cases:
        s = oracle.generate_system(n, 3)
        ref = oracle.solve_partition(s, sizes)
        x = tp.solve_partition(tp.TridiagonalSystem(s.sub, s.diag, s.sup, s.rhs), tp.RecursionPolicy(sizes))
        d = oracle.rel_inf_diff(x, ref)
        worst = max(worst, d)
        assert d <= 1e-10, (n, sizes, d)
    # FP32
    s = oracle.generate_system(20_000, 5)
    ref = oracle.solve_partition(s, [16, 8])
    x32 = tp.solve_partition(tp.TridiagonalSystem(*(a.astype(np.float32) for a in (s.sub, s.diag, s.sup, s.rhs))),
                             tp.RecursionPolicy([16, 8]))
    assert oracle.rel_inf_diff(x32.astype(np.float64), ref) <= 1e-4
    # thomas_solve through the finishing solve (cluster path)
    s = oracle.generate_system(4_000, 7)
    xt = tp.thomas_solve(tp.TridiagonalSystem(s.sub, s.diag, s.sup, s.rhs))
    assert oracle.rel_inf_diff(xt, oracle.thomas_solve(s)) <= 1e-10
    # device generator + residual
    sd = tp.generate_system(10_000, 9, device=True)
    xd = tp.solve_partition(sd, tp.RecursionPolicy([8]))
    assert tp.residual_inf(sd, xd) <= 1e-12
    # sharded halves (the NCCL transport's kernels), 2 simulated ranks. The
    # fused exchange is left out: the sanitizer serialises kernels, and two
    # simulated ranks' finishing kernels must run concurrently to meet.
    s = oracle.generate_system(40_000, 11)
    ref = oracle.solve_partition(s, [16])
    xs = sharded.simulate_ranks(s.sub, s.diag, s.sup, s.rhs, 2, [16])
    assert oracle.rel_inf_diff(xs, ref) <= 1e-10
    # the fused exchange kernel (k_final_cl<kShard>) with one rank: it publishes
    # to and waits on its own mailbox, so no second kernel has to run alongside
    xf = sharded.simulate_ranks_fused(s.sub, s.diag, s.sup, s.rhs, 1, [16])
    assert oracle.rel_inf_diff(xf, ref) <= 1e-10
    # the same with the grid solve at the root (k_grid_solve<double, L, kShard>):
    # one rank owns the GPU, the shard's system fits the grid
    s = oracle.generate_system(200_000, 13)
    ref = oracle.solve_partition(s, [32])
    xg = sharded.simulate_ranks_fused(s.sub, s.diag, s.sup, s.rhs, 1, [32])
    assert oracle.rel_inf_diff(xg, ref) <= 1e-10
    torch.cuda.synchronize()
    print(f"sanitize cases ok (worst rel_inf_diff {worst:.2e})")


if __name__ == "__main__":
    main()
