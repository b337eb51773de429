"""Profile one device solve kernel by kernel (run under ncu on a B200).

    ncu --set full --clock-control none --import-source on \
        -k regex:"k_fast|k_generic|k_final" -o gpurun_out/solve \
        python tools/ncu_capture.py [--n 1e8] [--policy 64,10,32,16]
    python tools/ncu_capture.py --summarize gpurun_out/solve.ncu-rep --out profiles/ncu_summary.json

Capture mode launches exactly one solve through tp_solve_profile_f64_dev
(serial launches in plan order, each labelled stage1:L0, stage1t:L2, final:L4,
...), and writes the labels to gpurun_out/ncu_labels.json. Summarize mode pairs
the report's launches (in order) with those labels and writes the per-launch
duration, DRAM bytes, DRAM % of peak, warps active, FP64 pipe %, registers and
launch shape: the numbers bench.py's roofline.traffic and DESIGN.md quote.
"""
import argparse
import csv
import ctypes as C
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
LABELS = os.path.join(ROOT, "gpurun_out", "ncu_labels.json")

METRICS = {
    "duration_ns": "gpu__time_duration.sum",
    "dram_read_bytes": "dram__bytes_read.sum",
    "dram_write_bytes": "dram__bytes_write.sum",
    "dram_pct_of_peak": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "fp64_pipe_pct": "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "regs": "launch__registers_per_thread",
    "grid": "launch__grid_size",
    "block": "launch__block_size",
}


def capture(n: int, sizes):
    import numpy as np
    import torch

    import paper_2510_27351_b200 as tp
    from paper_2510_27351_b200._lib import TpError, lib

    s = tp.generate_system(n, 1, device=True)
    x = torch.empty(n, dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    ctx = tp.context()
    sz = np.asarray(sizes, dtype=np.int64)
    kms = (C.c_float * 64)()
    names = C.create_string_buffer(64 * 32)
    nk = C.c_int32()
    err = TpError()
    st = lib.tp_solve_profile_f64_dev(ctx.handle, *s._dev_ptrs(), n, sz.ctypes.data_as(C.POINTER(C.c_int64)),
                                      len(sz), C.c_void_p(x.data_ptr()), kms, names, 64, C.byref(nk),
                                      C.byref(err))
    assert st == 0, err.msg
    labels = [names.raw[32 * i:32 * (i + 1)].split(b"\0")[0].decode() for i in range(nk.value)]
    os.makedirs(os.path.dirname(LABELS), exist_ok=True)
    with open(LABELS, "w") as f:
        json.dump({"n": n, "policy": list(sizes), "labels": labels}, f)
    print(json.dumps({"labels": labels}))


def summarize(rep: str, out: str, md: str = None):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    head, units, data = rows[0], rows[1], rows[2:]
    scale = {"ns": 1.0, "nsecond": 1.0, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6,
             "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    meta = json.load(open(LABELS))
    if len(data) != len(meta["labels"]):
        raise SystemExit(f"{len(data)} launches in the report, {len(meta['labels'])} labels")

    def num(row, metric):
        """Value in base units (ns, bytes) whatever unit ncu chose to print."""
        try:
            i = head.index(metric)
            return float(row[i].replace(",", "")) * scale.get(units[i], 1.0)
        except (ValueError, IndexError):
            return None

    res = {"meta": {"source": f"ncu --set full --clock-control none, one solve, {rep}", "n": meta["n"],
                    "policy": meta["policy"]}}
    for lab, row in zip(meta["labels"], data):
        d = {"kernel": row[head.index("Kernel Name")]}
        for k, m in METRICS.items():
            d[k] = num(row, m)
        d["duration_ms"] = d.pop("duration_ns") / 1e6
        d["dram_bytes"] = (d["dram_read_bytes"] or 0) + (d["dram_write_bytes"] or 0)
        res[lab] = d
    with open(out, "w") as f:
        json.dump(res, f, indent=1)
    if md:
        tot = sum(v["duration_ms"] for k, v in res.items() if k != "meta")
        lines = [f"| launch | kernel | ms | DRAM read MB | DRAM write MB | DRAM % peak | warps active % | "
                 f"FP64 pipe % | regs | grid x block |", "|---|---|---|---|---|---|---|---|---|---|"]
        for k, v in res.items():
            if k == "meta":
                continue
            lines.append(f"| {k} | `{v['kernel'][:48]}` | {v['duration_ms']:.4f} | {v['dram_read_bytes'] / 1e6:.1f} | "
                         f"{v['dram_write_bytes'] / 1e6:.1f} | {v['dram_pct_of_peak']:.1f} | {v['warps_active_pct']:.1f} | "
                         f"{v['fp64_pipe_pct']:.1f} | {v['regs']:.0f} | {v['grid']:.0f}x{v['block']:.0f} |")
        lines.append(f"\nSum of launches: {tot:.4f} ms")
        s1_key = next((k for k in res if k.startswith("stage1") and k.endswith(":L0")), None)
        s1, s3 = res.get(s1_key) if s1_key else None, res.get("stage3:L0")
        if s1 and s3:
            lines.append(f"Level-0 Stage 1 + Stage 3 = {100 * (s1['duration_ms'] + s3['duration_ms']) / tot:.1f}% "
                         f"of the launch sum; Stage 3 L0 alone {100 * s3['duration_ms'] / tot:.1f}%.")
            n = meta["n"]
            lines.append(f"Stage 3 L0: algorithmic {40 * n / 1e9:.3f} GB (40 B/unknown) vs DRAM traffic "
                         f"{s3['dram_bytes'] / 1e9:.3f} GB; {s3['dram_bytes'] / s3['duration_ms'] / 1e6:.0f} GB/s "
                         f"under ncu.")
            folded = {"stage1_fold:L0": " (level 1 folded in)", "stage1_fold2:L0": " (levels 1 and 2 folded in)"}
            lines.append(f"Stage 1 L0{folded.get(s1_key, '')}: algorithmic "
                         f"{32 * n / 1e9:.3f} GB read + {s1['dram_write_bytes'] / 1e9:.3f} "
                         f"GB interfaces written vs DRAM {s1['dram_bytes'] / 1e9:.3f} GB; "
                         f"{s1['dram_bytes'] / s1['duration_ms'] / 1e6:.0f} GB/s under ncu.")
        head_md = [f"# ncu --set full, one solve (N={meta['n']:.0e}, policy {meta['policy']})", "",
                   f"Report `{rep}` (tools/round_measure.sh; summarised by tools/ncu_capture.py). "
                   "ncu replays each launch serialised and cold-cache: compare shares, not absolutes. "
                   "Serial launch order of tp_solve_profile_f64_dev; in the solve graph the tail kernels "
                   "(stage1t / stage3t) run on a parallel branch.", ""]
        with open(md, "w") as f:
            f.write("\n".join(head_md + lines) + "\n")
    print(f"wrote {out}")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=float, default=1e8)
    ap.add_argument("--policy", default="64,10,32,16")
    ap.add_argument("--summarize", default=None, help="an .ncu-rep of a capture run")
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "ncu_summary.json"))
    ap.add_argument("--md", default=None)
    a = ap.parse_args()
    if a.summarize:
        summarize(a.summarize, a.out, a.md)
    else:
        capture(int(a.n), [int(v) for v in a.policy.split(",")])


if __name__ == "__main__":
    main()
