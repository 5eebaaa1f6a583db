"""Per-CUDA-line instruction and stall-sample shares from an ncu report's mixed
source view (dev aid): python scripts/ncu_lines.py report.ncu-rep [top] [kernel regex]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 60
kfilt = ["--kernel-name", f"regex:{sys.argv[3]}", "--launch-count", "1"] if len(sys.argv) > 3 else []
out = subprocess.run(["ncu", "-i", rep, *kfilt, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
fname = "?"
hdr = None
data = []
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r[0]:
        continue
    try:
        ins = float(r[hdr.index("Instructions Executed")])
        smp = float(r[hdr.index("Warp Stall Sampling (All Samples)")])
        thr = float(r[hdr.index("Thread Instructions Executed")])
    except (ValueError, IndexError):
        continue
    data.append((ins, smp, thr, f"{fname}:{r[0]}", r[1][:100]))
ti = sum(d[0] for d in data)
ts = sum(d[1] for d in data)
print(f"total warp inst {ti:.4g}  samples {ts:.4g}")
for ins, smp, thr, loc, src in sorted(data, reverse=True)[:top]:
    print(f"{loc:>16} {ins / ti * 100:5.1f}% {smp / ts * 100:5.1f}% simt {thr / max(ins, 1):4.1f}  {src}")
