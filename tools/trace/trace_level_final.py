import ctypes as C, os, sys
# k_level_final_cl phase trace: tools/trace/build_trace.sh, then python tools/trace/trace_level_final.py on a B200
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
os.environ.setdefault("TPB_LIB", os.path.join(ROOT, "scratch", "trace_lib", "libtridpart_b200.so"))
import numpy as np, torch
import paper_2510_27351_b200 as tp
from paper_2510_27351_b200 import _lib
for n, pol in ((int(1e8), [64, 10, 32, 16]), (10_000, [8]), (int(1e9), [64, 10, 32, 32])):
    s = tp.generate_system(n, 1, device=True)
    x = torch.empty(n, dtype=torch.float64, device="cuda")
    for _ in range(3):
        tp.solve_partition_async(s, tp.RecursionPolicy(pol), out=x)
    torch.cuda.synchronize()
    tr = (C.c_uint64 * 24)()
    _lib.lib.tp_debug_trace(tr)
    t = np.array(tr[:24], dtype=np.int64)
    print(n, pol, "fused level total cycles", t[17] - t[12])
    for i, nm in enumerate(["stage level rows", "block sweeps (Stage 1)", "interface tree (cl_tree)",
                            "block back-substitution", "store"]):
        print(f"   {nm:26s} {t[13 + i] - t[12 + i]:7d}")
    names = ["stage", "leaf", "warp tree+sync", "w0 merges", "cluster sync1", "cta0 root work", "cluster sync2",
             "w0 down+sync", "warp down+expand+store"]
    for i, nm in enumerate(names):
        print(f"      {nm:24s} {t[i + 1] - t[i]:7d}")
    del s, x
    torch.cuda.empty_cache()
