"""SASS cost of the k-NN's algorithmic operations (roofline op count).

Compiles scripts/op_costs.cu for sm_100a, disassembles it (cuobjdump -sass) and
counts, per kernel, the instructions of its single loop body minus the loop overhead
(counter update, compare, back branch).  Writes profiles/r02_op_costs.json:
  lane-instructions per operation (dist per candidate, box per child box, insert per
  k-best insertion, ascent per stop test) and the half-rate share (FMNMX/VIMNMX/
  IMAD.WIDE; measured at 0.5 of full rate in profiles/r01_alu_rates.json).
  python scripts/op_costs.py [out.json]
"""
import json
import re
import subprocess
import sys
import tempfile
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
SRC = ROOT / "scripts" / "op_costs.cu"
HALF_RATE = ("FMNMX", "VIMNMX", "IMNMX", "IMAD.WIDE", "HMNMX2", "PRMT")
PER_STEP = {"op_dist4": 4, "op_dist4_final": 4}   # operations per loop iteration
# per-iteration scaffolding of the microkernels that the product's loops do not have
# (candidate index math + loop compare of op_dist4; the accumulator update of op_box
# and op_ascent; the buffer-slot wrap of op_insert)
SCAFFOLD = {"op_dist4": 4, "op_dist4_final": 4, "op_box": 3, "op_ascent": 3, "op_insert": 1, "op_insert_final": 1}
CONTROL = ("BRA", "BSSY", "BSYNC", "S2UR", "NOP", "LDCU", "EXIT")


def loop_body(sass_lines):
    """Instructions of the (single) loop: from the back branch's target to the branch."""
    ins = []
    for ln in sass_lines:
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", ln)
        if m:
            ins.append((int(m.group(1), 16), m.group(2).strip()))
    for addr, text in reversed(ins):
        m = re.search(r"\bBRA\b.*0x([0-9a-f]+)", text)
        if m and int(m.group(1), 16) < addr and not text.startswith("@!PT"):
            lo = int(m.group(1), 16)
            return [t for a, t in ins if lo <= a <= addr and not t.startswith("NOP")]
    raise RuntimeError("no loop found")


def main():
    out = Path(sys.argv[1]) if len(sys.argv) > 1 else ROOT / "profiles" / "r02_op_costs.json"
    with tempfile.TemporaryDirectory() as d:
        cubin = Path(d) / "op.cubin"
        subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-cubin",
                               str(SRC), "-o", str(cubin)])
        sass = subprocess.run(["cuobjdump", "-sass", str(cubin)], capture_output=True, text=True, check=True).stdout
    funcs, cur = {}, None
    for ln in sass.splitlines():
        m = re.match(r"\s*Function : (\w+)", ln)
        if m:
            cur = m.group(1)
            funcs[cur] = []
        elif cur:
            funcs[cur].append(ln)
    res = {}
    for name, lines in funcs.items():
        body = loop_body(lines)
        opc = [t.split()[1] if t.startswith("@") else t.split()[0] for t in body]
        # vector-pipe instructions of the body: uniform-datapath loop bookkeeping (U*)
        # and control flow are not the operation's work
        own = [o for o in opc if not o.startswith("U") and not o.startswith(CONTROL)]
        n = len(own) - SCAFFOLD.get(name, 0)
        half = sum(1 for o in own if o.startswith(HALF_RATE))
        k = PER_STEP.get(name, 1)
        res[name.replace("op_", "").replace("dist4", "dist")] = {   # dist, dist_final, box, insert, insert_final, ascent
            "lane_instructions": n / k, "half_rate_instructions": half / k, "loop_body": body}
    doc = {"source": "scripts/op_costs.cu (the product's expressions), cuobjdump -sass sm_100a: vector-pipe "
                     "instructions of each loop body, minus uniform-datapath bookkeeping, control flow and the "
                     "microkernel's own scaffolding", "ops": res}
    out.write_text(json.dumps(doc, indent=1))
    print(json.dumps({k: (v["lane_instructions"], v["half_rate_instructions"]) for k, v in res.items()}))


if __name__ == "__main__":
    main()
