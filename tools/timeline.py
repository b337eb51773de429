"""In-graph kernel timeline of one device solve (CUPTI via torch.profiler).

    python tools/timeline.py [--n 1e8] [--policy 64,10,32,16] [--reps 3] [--out FILE]

Runs the solve through tp_solve_partition_f64_dev (CUDA-graph replay, as in
bench.py), records GPU kernel start/end timestamps with CUPTI and prints, for
the last replay, every kernel with its start offset, duration and the idle
gap before it. Unlike tp_solve_profile_f64_dev (events between serialised
launches) this shows the graph as it actually runs: overlap of the tail
branches and the launch gaps between levels.
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
    ap.add_argument("--policy", default="64,10,32,16")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()

    import torch
    from torch.profiler import ProfilerActivity, profile

    import paper_2510_27351_b200 as tp

    n = int(a.n)
    sizes = [int(s) for s in a.policy.split(",")]
    sys_ = tp.generate_system(n, 1, device=True)
    x = torch.empty(n, dtype=torch.float64, device="cuda")
    pol = tp.RecursionPolicy(sizes)
    for _ in range(5):
        tp.solve_partition_async(sys_, pol, out=x)
    torch.cuda.synchronize()

    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(a.reps):
            tp.solve_partition_async(sys_, pol, out=x)
            torch.cuda.synchronize()
    evs = []
    for e in prof.events():
        if e.device_type == torch.autograd.DeviceType.CUDA and e.time_range.elapsed_us() >= 0:
            nm = e.name
            if nm.startswith("Memset") or "memset" in nm.lower():
                kind = "memset"
            else:
                kind = "kernel"
            evs.append((e.time_range.start, e.time_range.end, nm, kind))
    evs.sort()
    # split into replays of the solve graph: it launches
    # tp.context().last_launch_count() kernels (k_reset included when present;
    # a one-kernel graph resets the error word itself)
    per = max(1, tp.context().last_launch_count())
    kern = [ev for ev in evs if ev[3] == "kernel"]
    groups = [kern[i:i + per] for i in range(0, len(kern) - per + 1, per)]
    g = groups[-1]
    t0 = g[0][0]
    end_prev = t0
    rows = []
    for s, e, nm, kind in g:
        short = nm.split("(")[0][:60]
        rows.append({"start_us": s - t0, "dur_us": e - s, "gap_us": s - end_prev, "kernel": short})
        end_prev = max(end_prev, e)
    total = max(r[1] for r in g) - t0
    for r in rows:
        print(f"{r['start_us']:9.2f} {r['dur_us']:9.2f} gap {r['gap_us']:7.2f}  {r['kernel']}")
    print(f"span {total:.2f} us over {len(rows)} device ops; replays seen {len(groups)}")
    if a.out:
        with open(a.out, "w") as f:
            json.dump({"n": n, "policy": sizes, "span_us": total, "ops": rows,
                       "spans_all": [max(x[1] for x in gg) - gg[0][0] for gg in groups]}, f, indent=1)


if __name__ == "__main__":
    main()
