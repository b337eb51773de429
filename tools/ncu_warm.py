"""Repeat one device solve through tp_solve_profile_f64_dev (direct launches,
no graph) so ncu can profile a WARM launch of a kernel, e.g. the grid solve
with its instruction cache and L2 in the state of back-to-back solves:

    ncu --set full --import-source on --cache-control none --clock-control none \
        -k regex:k_grid_hyb --launch-skip 20 -c 1 -o gpurun_out/c2_warm \
        python tools/ncu_warm.py --n 1e6 --policy 32
"""
import argparse
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=float, default=1e6)
    ap.add_argument("--policy", default="32")
    ap.add_argument("--reps", type=int, default=30)
    a = ap.parse_args()
    import numpy as np
    import torch

    import paper_2510_27351_b200 as tp
    from paper_2510_27351_b200._lib import TpError, lib

    n = int(a.n)
    sizes = [int(v) for v in a.policy.split(",")]
    s = tp.generate_system(n, 1, device=True)
    x = torch.empty(n, dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    ctx = tp.context()
    sz = np.asarray(sizes, dtype=np.int64)
    kms = (C.c_float * 64)()
    names = C.create_string_buffer(64 * 32)
    nk = C.c_int32()
    err = TpError()
    for _ in range(a.reps):
        st = lib.tp_solve_profile_f64_dev(ctx.handle, *s._dev_ptrs(), n, sz.ctypes.data_as(C.POINTER(C.c_int64)),
                                          len(sz), C.c_void_p(x.data_ptr()), kms, names, 64, C.byref(nk),
                                          C.byref(err))
        assert st == 0, err.msg
    torch.cuda.synchronize()
    labels = [names.raw[32 * i:32 * (i + 1)].split(b"\0")[0].decode() for i in range(nk.value)]
    print({lab: round(kms[i] * 1e3, 2) for i, lab in enumerate(labels)}, "us (last rep, events)")


if __name__ == "__main__":
    main()
