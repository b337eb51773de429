# Soak test of the fused exchange (run on one GPU with CUDA_MODULE_LOADING=EAGER
# CUDA_DEVICE_MAX_CONNECTIONS=32): P simulated ranks, 100 solves each enqueued
# rank-major with no host synchronisation, 4 rotating output buffers.
# back-to-back fused solves with no host synchronisation between them: ranks
# drift apart and the two mailbox slots must keep every exchange paired
import sys, json
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle
from paper_2510_27351_b200 import sharded
from paper_2510_27351_b200.tridpart import Context
res = {}
for P, n, R in ((4, 200_003, 100), (8, 80_000, 100)):
    s = oracle.generate_system(n, 5)
    ref = oracle.solve_partition(s, [32, 10])
    ctxs = [Context(0) for _ in range(P)]
    sharded.attach_local_peers(ctxs)
    shards = []
    for r in range(P):
        lo, cnt = sharded.shard_bounds(n, P, r)
        sys4 = [torch.from_numpy(np.ascontiguousarray(a[lo:lo + cnt])).cuda() for a in (s.sub, s.diag, s.sup, s.rhs)]
        sharded.DeviceBackend(ctxs[r]).reduce(sys4, [32, 10])
        outs = [torch.empty(cnt, dtype=torch.float64, device="cuda") for _ in range(4)]
        shards.append((lo, cnt, sys4, outs))
    for r, (lo, cnt, sys4, outs) in enumerate(shards):
        for k in range(4):
            sharded.fused_solve(ctxs[r], sys4, [32, 10], out=outs[k], stream=0, prepare_only=True)
    torch.cuda.synchronize()
    # rank-major launch order: rank 0 enqueues all R solves before rank 1 starts
    for r, (lo, cnt, sys4, outs) in enumerate(shards):
        for k in range(R):
            sharded.fused_solve(ctxs[r], sys4, [32, 10], out=outs[k % 4], stream=0)
    torch.cuda.synchronize()
    worst, identical = 0.0, True
    x0 = None
    for k in range(4):
        x = np.empty(n)
        for r, (lo, cnt, sys4, outs) in enumerate(shards):
            x[lo:lo + cnt] = outs[k].cpu().numpy()
        worst = max(worst, oracle.rel_inf_diff(x, ref))
        if x0 is None: x0 = x
        identical &= bool(np.array_equal(x, x0))
    errs = []
    import ctypes as C
    from paper_2510_27351_b200._lib import lib, TpError
    for c in ctxs:
        e = TpError(); errs.append(lib.tp_check_device_error(c.handle, C.byref(e)))
    res[f"P{P}"] = {"R": R, "worst_rel_inf_diff": worst, "all_identical": identical, "err_codes": errs}
    for c in ctxs: c.close()
print(json.dumps(res))
