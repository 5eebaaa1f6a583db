"""Summarise ncu output into small committed files under profiles/ (development aid).

  python scripts/ncu_summary.py rep  gpurun_out/knn_v1.ncu-rep  profiles/r01_ncu_knn_v1.json
  python scripts/ncu_summary.py launches gpurun_out/launches_v1.csv profiles/r01_launches_v1.json

`rep`: per-kernel key counters of an `ncu --set full` capture (DRAM bytes, issue
activity, SIMT efficiency, stall reasons, registers, local memory traffic).
`launches`: the `--metrics gpu__time_duration.sum` launch list, aggregated per
kernel name: launches, total/mean ns and the share of all listed device time.
`table`: per launch of a `--set full` capture: achieved DRAM GB/s against the
measured HBM copy bandwidth (MEASURED_PEAKS.json), sectors per request of global
loads/stores, issue and warp activity; JSON plus a markdown table on stdout.
"""
from __future__ import annotations

import csv
import io
import json
import subprocess
import sys
from collections import defaultdict

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed.sum", "smsp__inst_executed.sum",
    "smsp__thread_inst_executed_per_inst_executed.ratio",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__occupancy_limit_registers",
    "launch__shared_mem_per_block_static", "launch__grid_size", "launch__block_size",
    "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct",
    "sass__inst_executed_local_loads", "sass__inst_executed_local_stores",
    "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum",
    "l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum", "l1tex__t_requests_pipe_lsu_mem_global_op_st.sum",
    "sm__cycles_elapsed.avg.per_second",
]
STALL_PREFIX = "smsp__average_warps_issue_stalled_"


def _num(v):
    try:
        return float(v.replace(",", ""))
    except (ValueError, AttributeError):
        return v


def rep(path, out):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        k = {"kernel": d.get("Kernel Name")}
        for key in KEYS:
            if key in d:
                k[key] = [_num(d[key]), u.get(key, "")]
        stalls = {key[len(STALL_PREFIX):].replace("_per_issue_active.ratio", ""): _num(v)
                  for key, v in d.items() if key.startswith(STALL_PREFIX) and key.endswith("per_issue_active.ratio")}
        k["stalls_per_issue"] = {a: b for a, b in sorted(stalls.items(), key=lambda t: -t[1]) if b and b > 0.01}
        # per-launch DRAM traffic in bytes
        for key in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            if key in k:
                val, unit = k[key]
                mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
                k[key + ".bytes"] = val * mult
        if "dram__bytes_read.sum.bytes" in k:
            k["dram_bytes_per_launch"] = k["dram__bytes_read.sum.bytes"] + k["dram__bytes_write.sum.bytes"]
        res.append(k)
    out_d = {"source": path, "kernels": res}
    if len(res) == 1 and "dram_bytes_per_launch" in res[0]:
        out_d["dram_bytes_per_launch"] = res[0]["dram_bytes_per_launch"]
    with open(out, "w") as f:
        json.dump(out_d, f, indent=1)
    print(json.dumps(out_d, indent=1)[:3000])


def launches(path, out):
    lines = [l for l in open(path) if l.startswith('"')]
    rows = list(csv.DictReader(io.StringIO("".join(lines))))
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows:
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"]
        ns = float(r["Metric Value"].replace(",", ""))
        if r["Metric Unit"] == "us":
            ns *= 1e3
        elif r["Metric Unit"] == "ms":
            ns *= 1e6
        agg[name][0] += 1
        agg[name][1] += ns
    tot = sum(v[1] for v in agg.values())
    table = sorted(({"kernel": k, "launches": v[0], "total_ns": v[1], "mean_ns": v[1] / v[0],
                     "share": v[1] / tot} for k, v in agg.items()), key=lambda d: -d["total_ns"])
    with open(out, "w") as f:
        json.dump({"source": path, "total_ns": tot, "kernels": table}, f, indent=1)
    for t in table:
        print(f"{t['share']*100:6.2f}%  {t['launches']:4d}  {t['mean_ns']/1e3:10.1f} us  {t['kernel'][:100]}")


def table(path, out):
    import re
    from pathlib import Path
    rep(path, out)
    d = json.load(open(out))
    peaks = json.load(open(Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json"))
    peak = float(peaks.get("hbm_gbs") or peaks.get("hbm_copy_gbs") or 0) or None
    rows = []
    for k in d["kernels"]:
        t_ms = k["gpu__time_duration.sum"][0] * {"ms": 1, "us": 1e-3, "ns": 1e-6}.get(k["gpu__time_duration.sum"][1], 1)
        byt = k.get("dram_bytes_per_launch", 0.0)
        gbs = byt / (t_ms * 1e-3) / 1e9 if t_ms else 0.0
        sec = lambda a, b: (k[a][0] / k[b][0]) if k.get(b) and k[b][0] else None  # noqa: E731
        name = re.sub(r"\(.*", "", k["kernel"]).replace("void ", "").replace("zd::<unnamed>::", "").replace("<unnamed>::", "")
        rows.append({"kernel": name, "grid": k.get("launch__grid_size", [None])[0], "us": round(t_ms * 1e3, 1),
                     "dram_mb": round(byt / 1e6, 1), "gbs": round(gbs), "hbm_frac": round(gbs / peak, 3) if peak else None,
                     "ld_sect_per_req": round(sec("l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
                                                  "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum") or 0, 2),
                     "st_sect_per_req": round(sec("l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum",
                                                  "l1tex__t_requests_pipe_lsu_mem_global_op_st.sum") or 0, 2),
                     "issue_active_pct": round(k.get("smsp__issue_active.avg.pct_of_peak_sustained_active", [0])[0], 1),
                     "warps_active_pct": round(k.get("sm__warps_active.avg.pct_of_peak_sustained_active", [0])[0], 1),
                     "regs": k.get("launch__registers_per_thread", [None])[0]})
    d["table"] = rows
    d["hbm_peak_gbs"] = peak
    json.dump(d, open(out, "w"), indent=1)
    print("| kernel | grid | µs | DRAM MB | GB/s | of HBM peak | ld sect/req | st sect/req | issue % | warps % |")
    print("|---|---|---|---|---|---|---|---|---|---|")
    for r in rows:
        print(f"| {r['kernel']} | {r['grid']} | {r['us']} | {r['dram_mb']} | {r['gbs']} | {r['hbm_frac']} | "
              f"{r['ld_sect_per_req']} | {r['st_sect_per_req']} | {r['issue_active_pct']} | {r['warps_active_pct']} |")


if __name__ == "__main__":
    {"rep": rep, "launches": launches, "table": table}[sys.argv[1]](sys.argv[2], sys.argv[3])
