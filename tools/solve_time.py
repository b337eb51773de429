"""Device solve time of one (N, policy): CUDA events around K back-to-back
graph-replayed solves (inputs resident, like bench.py's `value`), printed as
one line. Used for A/B runs of kernel switches, e.g.

    for f in 0 1; do TPB_FUSE_LAST=$f python tools/solve_time.py --n 1e4 --policy 4; done
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=float, default=1e8)
    ap.add_argument("--policy", default=None, help="comma-separated m sizes (default: the predicted policy)")
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--tag", default="")
    a = ap.parse_args()

    import torch

    import paper_2510_27351_b200 as tp

    n = int(a.n)
    pol = tp.RecursionPolicy([int(v) for v in a.policy.split(",")]) if a.policy else tp.predicted_policy(n)
    s = tp.generate_system(n, 1, device=True)
    x = torch.empty(n, dtype=torch.float64, device="cuda")
    for _ in range(20):
        tp.solve_partition_async(s, pol, out=x)
    torch.cuda.synchronize()
    best = float("inf")
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.steps):
            tp.solve_partition_async(s, pol, out=x)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / a.steps)
    tp.check_device_error()
    res = tp.residual_inf(s, x)
    print(f"{a.tag:24s} n={n:>11d} policy={pol.sizes} us_per_solve={best * 1e3:9.2f} residual={res:.2e}")


if __name__ == "__main__":
    main()
