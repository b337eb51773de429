"""Phase timeline of one k_grid_solve launch (TPB_GRID_TRACE=1): per phase, the
min / median / max over CTAs of %globaltimer offsets from the earliest CTA start.

    make -C paper_2510_27351_b200/csrc TRACE=1 OUT=../lib/trace
    TPB_LIB=paper_2510_27351_b200/lib/trace/libtridpart_b200.so TPB_GRID_TRACE=1 \
        python tools/grid_trace.py --n 1e6 --policy 32

(the stamps are compiled only into trace builds; the default library has none)
"""
import argparse
import ctypes as C
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

SLOTS = 16
# slot -> phase name (printed in median-time order; a kernel stamps a subset)
PHASES = [(0, "start"), (1, "staged"), (2, "leaves"), (8, "thread tree"), (3, "pair published"),
          (4, "symbolic done | warp-root down"), (9, "barrier passed"), (10, "pairs loaded"), (11, "top warp tree"),
          (12, "top root tree"), (13, "root + path"), (5, "top synced"), (14, "CTA down start"),
          (6, "x stored / thread down"), (15, "expand rows in"), (7, "end")]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=float, default=1e6)
    ap.add_argument("--policy", default="32")
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    os.environ.setdefault("TPB_GRID_TRACE", "1")
    os.environ.setdefault("TPB_GRID_MIN", "4")
    import numpy as np
    import torch

    import paper_2510_27351_b200 as tp
    from paper_2510_27351_b200._lib import lib

    n = int(a.n)
    pol = tp.RecursionPolicy([int(v) for v in a.policy.split(",")])
    sys_ = tp.generate_system(n, 1, device=True)
    x = torch.empty(n, dtype=torch.float64, device="cuda")
    for _ in range(20):
        tp.solve_partition_async(sys_, pol, out=x)
    torch.cuda.synchronize()
    assert tp.context().last_kernels() == ["grid_solve:L0"], tp.context().last_kernels()
    buf = (C.c_ulonglong * (2 * 256 * SLOTS))()
    lib.tp_debug_grid_trace(buf, 2 * 256 * SLOTS)
    allv = np.array(buf[:], dtype=np.int64).reshape(2, 256, SLOTS)
    live = allv[0, :, 0] > 0
    t = allv[0][live]
    clk = allv[1][live]
    cyc = clk - clk[:, :1]
    dns = t - t[:, :1]
    ghz = float(np.median(cyc[:, 7] / np.maximum(dns[:, 7], 1)))
    print(f"SM clock during the launch: {ghz:.3f} GHz (clock64 / globaltimer over each CTA's span)")
    t0 = t[:, 0].min()
    d = (t - t0) / 1000.0
    rows = {}
    used = [(k, ph) for k, ph in PHASES if np.all(allv[0][live][:, k] > 0)]
    used.sort(key=lambda kp: float(np.median(d[:, kp[0]])))
    for k, ph in used:
        rows[ph] = [round(float(np.min(d[:, k])), 3), round(float(np.median(d[:, k])), 3),
                    round(float(np.max(d[:, k])), 3)]
        print(f"{ph:>9}  min {rows[ph][0]:8.3f}  med {rows[ph][1]:8.3f}  max {rows[ph][2]:8.3f} us"
              f"   cta0 cycles {int(cyc[0, k]):7d}")
    if a.out:
        with open(a.out, "w") as f:
            json.dump({"n": n, "policy": pol.sizes, "ctas": int(t.shape[0]), "sm_ghz": ghz, "phases_us_min_med_max": rows}, f, indent=1)


if __name__ == "__main__":
    main()
