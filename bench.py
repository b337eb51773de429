#!/usr/bin/env python
"""Benchmark: FP64 recursive partition solve on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--n|--size N_GLOBAL]
                    [--c4] [--weak] [--transport auto|p2p|nccl] [--impl ours|reference]

A step is one full solve (all levels, finishing solve, Stage 3) of an
N = 1e8-unknown strictly dominant system with the kNN-predicted policy
[64, 10, 32, 16] (config 3, BASELINE.json's metric). Inputs are generated on
the device with the generate_system distributions and stay resident in HBM
(3.2 GB, 25x the 126 MB L2, so no L2 flush is needed between steps).
N GPUs > 1: one process per GPU (torchrun), contiguous row shards of the SAME
global system (strong scaling: N = 1e8 on 1/2/4/8 B200;
--c4: N = 1e9, config 4; --weak: --n unknowns per GPU instead); each rank
runs the single-GPU graph on its shard with the one exchange per solve
(8 doubles per rank) inside the deepest level's cluster kernel over peer
memory (transport "p2p", chosen by "auto" when every rank can open every
peer's CUDA IPC mailbox; otherwise an NCCL all-gather); device time = max
over ranks.

`--impl reference` times the reference's own CPU solver (oracle/_ref: the
unmodified reference headers, all host threads) on rank 0 only.
"""
import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "FP64 unknowns/s and HBM GB/s (% roofline) at N=1e8, 1/2/4/8 B200 vs CPU ref"
UNIT = "unknowns/s"
ALG_BYTES_PER_UNKNOWN = 40.0   # read sub/diag/super/rhs once + write x once
TWO_PASS_BYTES_PER_UNKNOWN = 72.0  # compulsory for an exact two-pass solve once 32N >> L2
FALLBACK_HBM_GBS = 6650.0
PATTERN_CEILING_GBS = 7191.0  # read 4 + write 1 FP64 streams, full grid (tools/microbench/stream_ceiling.cu)


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=50)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--n", "--size", dest="n", type=float, default=None,
                   help="global unknowns (default 1e8; per GPU with --weak). Under torchrun use --size: "
                        "its own --n* options shadow --n")
    p.add_argument("--c4", action="store_true", help="config 4: N = 1e9 global")
    p.add_argument("--weak", action="store_true", help="--n unknowns per GPU (weak scaling)")
    p.add_argument("--seed", type=int, default=1)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--e2e-steps", type=int, default=6)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--cpu-runs", type=int, default=3)
    p.add_argument("--prewarm", type=float, default=0.3, help="seconds of untimed solves before warm-up")
    p.add_argument("--force-sharded", action="store_true",
                   help="run the multi-GPU code path even with one rank")
    p.add_argument("--transport", default="auto", choices=["auto", "p2p", "nccl"],
                   help="multi-GPU exchange: fused peer-memory (p2p), NCCL all-gather, or p2p with "
                        "NCCL fallback (auto)")
    a = p.parse_args()
    if a.n is None:
        a.n = 1e9 if a.c4 else 1e8
    return a


def _trace(msg):
    if os.environ.get("TPB_BENCH_TRACE"):
        print(f"[bench] {msg}", file=sys.stderr, flush=True)


def global_n(args, world):
    return int(args.n) * world if args.weak else int(args.n)


def hbm_peak():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if os.environ.get("TPB_SHARE_GPU") == "1":
        # functional check of the multi-rank flow on a 1-GPU box: every rank on
        # device 0 (timings are meaningless: the processes time-slice the GPU)
        local = 0
    return world, rank, local


# --------------------------------------------------------------- clocks
class ClockSampler:
    """NVML sampling of SM clock and throttle reasons during the timed region."""

    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sync_boost",
               0x40: "sw_thermal_slowdown", 0x80: "hw_thermal_slowdown",
               0x100: "hw_power_brake_slowdown", 0x2: "applications_clocks_setting"}

    def __init__(self, index):
        self.samples, self.reasons, self.stop_flag = [], set(), False
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # pragma: no cover - no NVML
            self.err = str(e)

    def _run(self):
        nv = self.nv
        while not self.stop_flag:
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                mask = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if mask & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.001)

    def __enter__(self):
        # the launch loop holds the GIL between ctypes calls: switch threads
        # often so the sampler sees the whole (short) timed region
        self._switch = sys.getswitchinterval()
        sys.setswitchinterval(2e-4)
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
            t_wait = time.perf_counter() + 0.2
            while not self.samples and time.perf_counter() < t_wait:
                time.sleep(1e-4)  # first sample taken before the timed region starts
        return self

    def __exit__(self, *a):
        self.stop_flag = True
        if self.ok:
            self.t.join()
        sys.setswitchinterval(self._switch)

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ------------------------------------------------------------ reference arm
def cpu_reference(n, runs, seed=1):
    """The reference's solve_partition (oracle/_ref, reference headers, all
    host threads) with the reference's own policy for N; median of `runs`
    after 1 warm-up (bench.hpp:104-127 statistic, residual outside timing)."""
    import numpy as np

    import oracle

    lib = oracle.ref()
    sizes = np.zeros(8, dtype=np.int64)
    depth = int(lib.ref_predict_depth(n))
    cnt = lib.ref_recursion_sizes(n, depth, sizes.ctypes.data_as(oracle._I64))
    sizes = sizes[:cnt].copy()
    h = lib.ref_system_generate(n, seed)
    x = np.empty(n)
    try:
        st = lib.ref_system_solve(h, sizes.ctypes.data_as(oracle._I64), len(sizes), x.ctypes.data_as(oracle._D))
        assert st == -1, st
        res = lib.ref_system_residual(h, x.ctypes.data_as(oracle._D))
        times = []
        for _ in range(runs):
            t0 = time.perf_counter()
            lib.ref_system_solve(h, sizes.ctypes.data_as(oracle._I64), len(sizes), None)
            times.append(time.perf_counter() - t0)
    finally:
        lib.ref_system_free(h)
    med = statistics.median(times)
    return {"value": n / med, "unit": UNIT, "cores": int(lib.ref_hardware_concurrency()),
            "kind": "reference", "median_s": med, "residual": res, "policy": [int(v) for v in sizes],
            "sample": f"N={n:.0e} generate_system(seed={seed}), policy {[int(v) for v in sizes]}, "
                      f"1 warm-up + {runs} runs, median, residual check outside timing"}


def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    n_arm = global_n(args, max(1, args.gpus))  # our arm's global N at this GPU count
    n = n_arm
    # bound the run: ~3 s per N=1e8 solve on 16 cores; keep the whole run ~<= 3 min
    budget_s = 150.0
    per = 3.5 * n / 1e8
    if (args.steps + args.warmup + 1) * per > budget_s:
        n = int(max(1e6, n * budget_s / ((args.steps + args.warmup + 1) * per)))
    import numpy as np

    import oracle

    lib = oracle.ref()
    sizes = np.zeros(8, dtype=np.int64)
    cnt = lib.ref_recursion_sizes(n, int(lib.ref_predict_depth(n)), sizes.ctypes.data_as(oracle._I64))
    sizes = sizes[:cnt].copy()
    h = lib.ref_system_generate(n, args.seed)
    try:
        for _ in range(args.warmup):
            lib.ref_system_solve(h, sizes.ctypes.data_as(oracle._I64), len(sizes), None)
        t0 = time.perf_counter()
        for _ in range(args.steps):
            lib.ref_system_solve(h, sizes.ctypes.data_as(oracle._I64), len(sizes), None)
        dt = time.perf_counter() - t0
    finally:
        lib.ref_system_free(h)
    value = n * args.steps / dt
    cores = int(lib.ref_hardware_concurrency())
    sample = (f"N={n} per step (generate_system seed={args.seed}; our arm's global N is {n_arm}, "
              f"bounded to ~{budget_s:.0f} s of CPU work), reference policy "
              f"{[int(v) for v in sizes]}, {args.warmup} warm-up + {args.steps} timed solves")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True,
        "scaling": "weak" if args.weak else "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "reference CPU solve_partition (oracle/_ref, reference headers)",
                   "n_per_step": n, "policy": [int(v) for v in sizes], "threads": cores},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "reference",
                         "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ our arm
def run_ours(args):
    import numpy as np
    import torch

    import paper_2510_27351_b200 as tp
    from paper_2510_27351_b200 import sharded

    world, rank, local = dist_env()
    torch.cuda.set_device(local)
    dist = None
    sharded_mode = world > 1 or args.force_sharded
    stdout_fd = None
    if sharded_mode:
        # NCCL (and the process-group bring-up) may print to fd 1: keep rank 0's
        # stdout to the one JSON line by pointing fd 1 at stderr until then
        sys.stdout.flush()
        stdout_fd = os.dup(1)
        os.dup2(2, 1)
        import torch.distributed as dist
        if os.environ.get("NCCL_DEBUG", "VERSION").upper() == "VERSION":
            os.environ["NCCL_DEBUG"] = "WARN"  # keep rank 0's stdout to the one JSON line
        if "RANK" not in os.environ:  # --force-sharded without torchrun: a 1-rank group
            os.environ.update(RANK="0", WORLD_SIZE="1", LOCAL_RANK="0", MASTER_ADDR="127.0.0.1",
                              MASTER_PORT=os.environ.get("MASTER_PORT", "29533"))
        if os.environ.get("TPB_SHARE_GPU") == "1":
            dist.init_process_group("gloo")  # NCCL refuses two ranks on one GPU
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    n_glob = global_n(args, world)
    n_per = n_glob // world
    policy = tp.predicted_policy(n_glob)
    lo, n_loc = sharded.shard_bounds(n_glob, world, rank, sharded.shard_granule(policy))
    stream = torch.cuda.current_stream()
    ctx = tp.context(local)

    sys_d = tp.generate_system(n_loc, args.seed, device=True, row0=lo, n_global=n_glob)
    x = torch.empty(n_loc, dtype=torch.float64, device="cuda")
    sys4 = [sys_d.sub, sys_d.diag, sys_d.super, sys_d.rhs]

    if not sharded_mode:
        def step():
            tp.solve_partition_async(sys_d, policy, out=x)
    else:
        solver = sharded.ShardedSolver(transport=args.transport)

        def step():
            solver.solve(sys4, n_glob, policy, out=x)

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    _trace("setup done")
    # untimed: graph capture + clock ramp (~0.3 s of solves), then W warm-up steps
    step()
    barrier()
    if not sharded_mode:
        t_end = time.perf_counter() + args.prewarm
        while time.perf_counter() < t_end:
            step()
    else:
        # every rank must issue the same number of solves (each one pairs with the
        # peers' solve of the same index), so the ramp is a count, not a deadline
        for _ in range(int(args.prewarm * 800)):
            step()
    for _ in range(args.warmup):
        step()
    barrier()

    _trace("warm-up done")
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        barrier()
        ev0.record(stream)
        for _ in range(args.steps):
            step()
        ev1.record(stream)
        barrier()
    ms = ev0.elapsed_time(ev1)
    launches_per_step = solver.backend.launches if sharded_mode else ctx.last_launch_count()
    red_dev = "cpu" if os.environ.get("TPB_SHARE_GPU") == "1" else "cuda"  # gloo reduces host tensors
    if dist is not None:
        t = torch.tensor([ms], device=red_dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_step = ms / args.steps
    value = n_glob * args.steps / (ms / 1e3)

    _trace("timed region done")
    # correctness of what was timed
    tp.check_device_error()
    res = tp.residual_inf(sys_d, x) if world == 1 else None
    if world > 1:
        # residual_inf over this shard's rows 1..n_loc-2 (their neighbours are
        # local; the two boundary rows couple to the adjacent shards), max over ranks
        a_, b_, c_, d_ = sys4
        r_ = b_[1:-1] * x[1:-1] + a_[1:-1] * x[:-2] + c_[1:-1] * x[2:] - d_[1:-1]
        num_d = torch.stack([r_.abs().max(), d_.abs().max()]).cpu()
        dist.all_reduce(num_d, op=dist.ReduceOp.MAX)
        res = float(num_d[0]) / max(1.0, float(num_d[1]))

    _trace("residual done")
    # per-kernel durations (CUDA events on the launch stream, same inputs).
    # Sharded: each rank times its shard's levels run standalone (the same
    # kernels and shapes as its sharded graph, minus the peer exchange)
    prof = {}
    if True:
        import ctypes as C
        from paper_2510_27351_b200._lib import TpError, lib
        sz = np.asarray(policy.sizes, dtype=np.int64)
        reps = 10
        share_gpu = os.environ.get("TPB_SHARE_GPU") == "1"
        if sharded_mode and share_gpu:  # ranks sharing a GPU run no grid solve: keep the standalone run alike
            tp.context().set_grid(False)
        for _ in range(reps if args.prewarm > 0 else 1):
            kms = (C.c_float * 64)()
            names = C.create_string_buffer(64 * 32)
            nk = C.c_int32()
            err = TpError()
            tp.context().set_stream(tp.torch_stream())
            st = lib.tp_solve_profile_f64_dev(ctx.handle, *sys_d._dev_ptrs(), n_loc,
                                              sz.ctypes.data_as(C.POINTER(C.c_int64)), len(sz),
                                              C.c_void_p(x.data_ptr()), kms, names, 64, C.byref(nk),
                                              C.byref(err))
            if st != 0:
                raise RuntimeError(err.msg.decode())
            for i in range(nk.value):
                nm = names.raw[32 * i:32 * i + 32].split(b"\0")[0].decode()
                prof.setdefault(nm, []).append(kms[i])
        prof = {k: statistics.median(v) for k, v in prof.items()}
        if sharded_mode and share_gpu:
            tp.context().set_grid(True)
    per_rank = None
    if dist is not None:
        per_rank = [None] * world
        dist.all_gather_object(per_rank, {"rank": rank, "n_local": n_loc, "kernels_ms": prof})

    _trace("profile done")
    # end to end through the public API: pinned host buffers, H2D + solve + D2H
    e2e = None
    h2d = 4 * 8 * n_loc
    d2h = 8 * n_loc
    if args.e2e_steps > 0:
        host = [t.cpu().pin_memory() for t in sys4]
        hx = [torch.empty(n_loc, dtype=torch.float64).pin_memory() for _ in range(2)]
        sync_ms = None
        if not sharded_mode:
            import ctypes as C
            from paper_2510_27351_b200._lib import lib
            from paper_2510_27351_b200.tridpart import _call
            hs = tp.TridiagonalSystem(*(t.numpy() for t in host))
            sz = np.asarray(policy.sizes, dtype=np.int64)
            szp = sz.ctypes.data_as(C.POINTER(C.c_int64))
            # public API, asynchronous host-pointer solve on two contexts / two
            # streams: step k's D2H overlaps step k+1's H2D (full-duplex PCIe)
            ctxs = [ctx, tp.Context(local)]
            strs = [torch.cuda.Stream() for _ in range(2)]

            def e2e_launch(i):
                _call(lib.tp_solve_partition_f64_async, ctxs[i % 2].handle, *hs._host_ptrs(), n_loc, szp,
                      len(sz), C.c_void_p(hx[i % 2].data_ptr()), C.c_void_p(strs[i % 2].cuda_stream))

            def e2e_run(k):
                for i in range(k):
                    e2e_launch(i)
                for s_ in strs:
                    s_.synchronize()

            # the synchronous reference-shaped call, for comparison
            tp.context().set_stream(tp.torch_stream())
            _call(lib.tp_solve_partition_f64, ctx.handle, *hs._host_ptrs(), n_loc, szp, len(sz),
                  C.c_void_p(hx[0].data_ptr()))
            t0 = time.perf_counter()
            _call(lib.tp_solve_partition_f64, ctx.handle, *hs._host_ptrs(), n_loc, szp, len(sz),
                  C.c_void_p(hx[0].data_ptr()))
            sync_ms = (time.perf_counter() - t0) * 1e3
        else:
            dsys = [torch.empty_like(t) for t in sys4]  # same solver (and peer links) as above
            # H2D + solve on the main stream, D2H on a copy stream into
            # alternating x buffers: step k's D2H overlaps step k+1's H2D
            xbuf = [x, torch.empty_like(x)]
            s_main, s_copy = torch.cuda.current_stream(), torch.cuda.Stream()
            d2h_done = [None, None]

            def e2e_run(k):
                for i in range(k):
                    b = i % 2
                    for d, h in zip(dsys, host):
                        d.copy_(h, non_blocking=True)
                    if d2h_done[b] is not None:
                        s_main.wait_event(d2h_done[b])  # x buffer b drained to the host
                    solver.solve(dsys, n_glob, policy, out=xbuf[b])
                    solved = torch.cuda.Event()
                    solved.record(s_main)
                    s_copy.wait_event(solved)
                    with torch.cuda.stream(s_copy):
                        hx[b].copy_(xbuf[b], non_blocking=True)
                        d2h_done[b] = torch.cuda.Event()
                        d2h_done[b].record(s_copy)
                s_main.synchronize()
                s_copy.synchronize()
        e2e_run(2)
        barrier()
        t0 = time.perf_counter()
        e2e_run(args.e2e_steps)
        barrier()
        dt = time.perf_counter() - t0
        if dist is not None:
            t = torch.tensor([dt], device=red_dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            dt = float(t.item())
        e2e = {"value": n_glob * args.e2e_steps / dt, "unit": UNIT,
               "h2d_bytes_per_step": h2d * world, "d2h_bytes_per_step": d2h * world,
               "ms_per_step": dt / args.e2e_steps * 1e3,
               "path": ("tp_solve_partition_f64_async (C-ABI, pinned host buffers): H2D + device solve + "
                        "D2H every step, two contexts/streams so one step's D2H overlaps the next "
                        "step's H2D") if not sharded_mode else
                       "pinned host -> device copy + ShardedSolver.solve on one stream, device -> "
                       "pinned host on a second stream (one step's D2H overlaps the next step's H2D)"}
        if sync_ms is not None:
            e2e["sync_call_ms"] = sync_ms
            e2e["sync_call_value"] = n_glob / (sync_ms * 1e-3)
        # what came back over PCIe is the solution: same kernels on the same
        # inputs as the device-resident steps, so it must match them bit for bit
        e2e["result_matches_device_solve"] = bool(torch.equal(hx[(args.e2e_steps - 1) % 2], x.cpu()))

    _trace("e2e done")
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_reference(n_glob, args.cpu_runs, args.seed)
        except Exception as e:  # reference build missing on this box
            cpu = {"value": None, "unit": UNIT, "cores": os.cpu_count(), "kind": "reference",
                   "sample": f"unavailable: {e}"}

    _trace("cpu baseline done")
    if rank == 0:
        peak, peak_src = hbm_peak()
        roof = None
        if prof:
            # the dominant kernel: level 0's Stage 3, or the grid solve when it
            # takes the whole solve (one-level mid-size systems)
            k = "stage3:L0" if "stage3:L0" in prof else max(prof, key=prof.get)
            t_k = prof.get(k)
            achieved = ALG_BYTES_PER_UNKNOWN * n_loc / (t_k * 1e-3) / 1e9
            traffic = None
            summ = os.path.join(ROOT, "profiles", "ncu_summary.json")
            if os.path.exists(summ):
                try:
                    with open(summ) as f:
                        sd = json.load(f)
                    # only a capture of this very workload describes this launch
                    if sd.get("meta", {}).get("n") == n_loc and sd.get("meta", {}).get("policy") == policy.sizes:
                        traffic = sd.get(k, {}).get("dram_bytes")
                except Exception:
                    traffic = None
            roof = {"bound": "hbm", "kernel": k, "achieved": achieved, "peak": peak, "unit": "GB/s",
                    "frac": achieved / peak, "traffic": traffic,
                    "traffic_source": ("profiles/ncu_summary.json: committed `ncu --set full` capture of this "
                                       "kernel on this workload (tools/ncu_capture.py), not measured by this run")
                    if traffic is not None else None,
                    "peak_note": ("peak = the driver's copy bandwidth (1 read : 1 write); this kernel streams "
                                  "4 reads : 1 write, whose measured B200 ceiling with trivial compute is "
                                  f"{PATTERN_CEILING_GBS:.0f} GB/s (profiles/r01_microbench.md)"),
                    "frac_of_pattern_ceiling": achieved / PATTERN_CEILING_GBS,
                    "alg_bytes_per_launch": ALG_BYTES_PER_UNKNOWN * n_loc,
                    "kernel_ms": t_k, "peak_source": peak_src,
                    "kernel_share_of_step": t_k / sum(prof.values())}
            if per_rank is not None:
                roof["per_rank"] = []
                for pr in per_rank:
                    tk = pr["kernels_ms"].get(k)
                    if tk:
                        a_ = ALG_BYTES_PER_UNKNOWN * pr["n_local"] / (tk * 1e-3) / 1e9
                        roof["per_rank"].append({"rank": pr["rank"], "n_local": pr["n_local"], "kernel_ms": tk,
                                                 "achieved": a_, "frac": a_ / peak})
                roof["note"] = ("per-rank kernel times from each rank's shard levels run standalone after the "
                                "timed region (same kernels and shapes as the sharded graph)")
        solve_gbs = ALG_BYTES_PER_UNKNOWN * n_glob / (ms_step * 1e-3) / 1e9 / world
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "weak" if args.weak else "strong", "vs_baseline": None,
            "dtype": "f64",
            "data": "synthetic: device counter-based generator with generate_system's distributions",
            "config": {"workload": (f"recursive partition solve, kNN policy, N={n_glob:.0e} "
                                    + ("per GPU (weak)" if args.weak else "global")
                                    + (" (config 4)" if n_glob == 10**9 else
                                       " (config 3)" if n_glob == 10**8 else "")),
                       "n_per_gpu": n_per, "n_global": n_glob, "policy": policy.sizes,
                       "l2": f"inputs {32 * n_loc / 1e9:.2f} GB/GPU vs the 126 MB L2 (no flush)",
                       "shard_granule_rows": sharded.shard_granule(policy) if sharded_mode else None,
                       "parallelism": "single GPU" if not sharded_mode else (
                           f"{world} contiguous shard(s) + " + (
                               "fused peer-memory exchange in the deepest level's cluster kernel (CUDA IPC)"
                               if solver.transport == "p2p" else "NCCL all-gather")),
                       "transport": None if not sharded_mode else solver.transport,
                       "transport_fallback": None if not sharded_mode else solver.fallback_reason},
            "hbm": {"solve_GBps_40B_per_gpu": solve_gbs,
                    "frac_40B": solve_gbs / peak,
                    "frac_72B": solve_gbs * TWO_PASS_BYTES_PER_UNKNOWN / ALG_BYTES_PER_UNKNOWN / peak,
                    "peak_GBps": peak, "peak_source": peak_src},
            "roofline": roof,
            "kernels_ms": prof or None,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": int(launches_per_step * args.steps),
            "launches_per_step": int(launches_per_step),
            "clocks": clk.summary(),
            "residual": res,
        }
        if stdout_fd is not None:
            sys.stdout.flush()
            os.dup2(stdout_fd, 1)
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
