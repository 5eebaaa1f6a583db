"""Build and run scripts/alu_rates.cu (per-op lane throughput; GPU) and write
profiles/rNN_alu_rates.json (dev aid).

  python scripts/alu_rates.py [out.json]"""
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
exe = ROOT / "build_var" / "alu_rates"
exe.parent.mkdir(exist_ok=True)
subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17",
                       str(ROOT / "scripts" / "alu_rates.cu"), "-o", str(exe)])
d = json.loads(subprocess.check_output([str(exe)]).decode().strip().splitlines()[-1])
full = d["sms"] * 128 * d["clock_attr_mhz"] * 1e6
for v in d["ops"].values():
    v["frac_of_full_rate"] = round(v["lane_ops_per_s"] / full, 3)
d["full_rate_lane_ops_per_s"] = full
print(json.dumps(d))
if len(sys.argv) > 1:
    Path(sys.argv[1]).write_text(json.dumps(d, indent=1) + "\n")
