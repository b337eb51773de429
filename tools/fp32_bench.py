"""FP32 vs FP64 device solve throughput (the reference's
solve_partition<float>): same N, device-resident inputs from the device
generator, the FP32 policy from the Table IV model (default_fp32_size_model)
and the FP64 one from Table I, CUDA events around K back-to-back solves.

    python tools/fp32_bench.py [--n 1e8] [--steps 50]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=float, default=1e8)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()

    import torch

    import paper_2510_27351_b200 as tp

    n = int(a.n)
    res = {"n": n, "steps": a.steps}
    for dt, model, bytes_per in (("float64", tp.default_size_model(), 40), ("float32", tp.default_fp32_size_model(), 20)):
        pol = tp.predicted_policy(n, size_model=model)
        s = tp.generate_system(n, 1, device=True, dtype=dt)
        x = torch.empty(n, dtype=getattr(torch, dt), device="cuda")
        for _ in range(10):
            tp.solve_partition_async(s, pol, out=x)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.steps):
            tp.solve_partition_async(s, pol, out=x)
        e1.record()
        torch.cuda.synchronize()
        tp.check_device_error()
        ms = e0.elapsed_time(e1) / a.steps
        res[dt] = {"policy": pol.sizes, "ms_per_solve": ms, "unknowns_per_s": n / (ms * 1e-3),
                   "GBps_at_alg_bytes": bytes_per * n / (ms * 1e-3) / 1e9, "alg_bytes_per_unknown": bytes_per,
                   "residual_inf": tp.residual_inf(s, x)}
        del s, x
        torch.cuda.empty_cache()
    print(json.dumps(res))
    if a.out:
        with open(a.out, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
