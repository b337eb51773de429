"""Host-pointer solve_partition from pageable numpy arrays vs pinned ones
(N=1e8, the reference-shaped synchronous call; pageable buffers are staged
through pinned chunks by a host thread pool, csrc/tp_stage.*).

    python tools/host_call_bench.py
"""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2510_27351_b200 as tp
n = 100_000_000
sd = tp.generate_system(n, 1, device=True)
host = [t.cpu().numpy().copy() for t in (sd.sub, sd.diag, sd.super, sd.rhs)]   # pageable numpy
pinned = [t.cpu().pin_memory() for t in (sd.sub, sd.diag, sd.super, sd.rhs)]
pol = tp.RecursionPolicy([64, 10, 32, 16])
hs = tp.TridiagonalSystem(*host)
ps = tp.TridiagonalSystem(*(t.numpy() for t in pinned))
for name, s in (("pageable", hs), ("pinned", ps)):
    x = tp.solve_partition(s, pol)
    ts = []
    for _ in range(3):
        t0 = time.perf_counter(); x = tp.solve_partition(s, pol); ts.append(time.perf_counter() - t0)
    print(name, "solve_partition host call ms:", [round(t * 1e3, 1) for t in ts], "residual", tp.residual_inf(sd, torch.from_numpy(x).cuda()))
