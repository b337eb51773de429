"""Top CUDA source lines by warp-stall samples from an ncu report's
cuda,sass source page, with each line's dominant stall reasons:
    python tools/ncu_lines.py REPORT.ncu-rep [top]"""
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
cur = None
hdr = None
agg = {}
total = 0
for line in out.splitlines():
    if line.startswith('"File Path"'):
        cur = line.split('","')[1].rstrip('"').split("/")[-1]
        continue
    if line.startswith('"Line No"'):
        hdr = line.strip('"').split('","')
        continue
    if hdr is None or not line.startswith('"') or line.startswith('"",'):
        continue
    f = line.strip('"').split('","')
    if len(f) < len(hdr) or not f[0].isdigit():
        continue
    tail = f[-(len(hdr) - 4):]  # metric columns after Line No, Source, Address, Source
    vals = dict(zip(hdr[4:], tail))
    try:
        s_all = int(vals["Warp Stall Sampling (All Samples)"])
    except (KeyError, ValueError):
        continue
    stalls = {k[6:]: int(v) for k, v in vals.items() if k.startswith("stall_") and v.isdigit() and int(v) > 0}
    agg[(cur, int(f[0]))] = (s_all, stalls, f[1][:70])
    total += s_all
print(f"total samples {total}")
for (fn, ln), (a, st, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    top3 = ", ".join(f"{k} {v}" for k, v in sorted(st.items(), key=lambda kv: -kv[1])[:3])
    print(f"{a:6d} {100.0 * a / max(total, 1):5.1f}%  {fn}:{ln:<4d} {src:<70s} | {top3}")
