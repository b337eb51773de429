import ctypes as C, os, sys
# k_final phase trace: tools/trace/build_trace.sh, then python tools/trace/trace_final.py on a B200
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
os.environ["TPB_LIB"] = os.path.join(os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))), "scratch", "trace_lib", "libtridpart_b200.so")
import numpy as np, torch
import paper_2510_27351_b200 as tp
from paper_2510_27351_b200 import _lib
for n, pol in ((int(1e8), [64, 10, 32, 16]), (int(1e6), [32]), (int(1e9), [64, 10, 32, 32]), (20000, [8, 10, 8])):
    s = tp.generate_system(n, 1, device=True)
    x = torch.empty(n, dtype=torch.float64, device="cuda")
    for _ in range(3):
        tp.solve_partition_async(s, tp.RecursionPolicy(pol), out=x)
    torch.cuda.synchronize()
    tr = (C.c_uint64 * 16)()
    _lib.lib.tp_debug_trace(tr)
    t = np.array(tr[:12], dtype=np.int64)
    cl = os.environ.get("TPB_FINAL_CLUSTER", "1") != "0"
    names = (["stage", "leaf", "warp tree+sync", "w0 merges", "cluster sync1", "cta0 root work", "cluster sync2",
              "w0 down+sync", "warp down+expand+store", "-", "-"] if cl else
             ["load", "leaf", "warptree", "sync1", "w0 merge", "w0 root+down", "sync2", "warp down", "leaf back", "sync3", "store"])
    print(n, pol, tp.plan_levels(n, pol)[2], "total cycles", t[11] - t[0])
    for i, nm in enumerate(names):
        print(f"   {nm:14s} {t[i+1]-t[i]:7d}")
    del s, x
    torch.cuda.empty_cache()
