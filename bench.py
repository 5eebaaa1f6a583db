#!/usr/bin/env python
"""bench.py — zd-tree hot path on B200 (one JSON line on rank 0).

A step = one pass of the whole hot path over config C5
(BASELINE.json configs[4]): zd_build on 10^7 uniform 3D points, zd_insert of 10^6
points, zd_delete of 10^6 original ids, then the all-points exact k=10 query over
the 10^7 live points.  Metric: all-points kNN queries/s (k=10, 10M 3D pts) of the
whole step (build + updates + query); the build Mpts/s and per-phase throughputs
are reported beside it.

Timing: inputs resident in HBM; W untimed warm-up steps; K timed steps, each
bracketed by CUDA events on the working stream with a 256 MB L2 flush (> 126 MB L2)
between steps outside the timed region; barrier + synchronize around the timed
loop; max over ranks.  Multi-GPU: replicas only — every rank runs its own
full step on its own GPU, value = all ranks' queries / max time ("weak").

--impl reference: the CPU oracle (oracle/, the only other place bench.py executes
it) on the host cores, on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

import zdgen  # noqa: E402

METRIC = "all-points kNN queries/s (k=10, 10M 3D pts)"
UNIT = "queries/s"
K_NN = 10
WORKLOAD = "C5"
PAPER_CONTEXT = {
    "build_plus_knn_3DinCube_10M_k10_qps": 22.1e6,
    "build_3DinCube_10M_mpts_s": 140.0,
    "hardware": "Dell R930, 4x Xeon E7-8867 v4, 144 threads (PAPER.md P:1022, P:1127, P:1209)",
    "note": "context only: the paper reports no k=10 numbers with batch updates (BASELINE.md)",
}


# ----------------------------------------------------------------- helpers

def env_int(name, default):
    try:
        return int(os.environ.get(name, default))
    except ValueError:
        return default


class Dist:
    """torch.distributed plumbing for N>1 (barrier + max over ranks)."""

    def __init__(self, backend: str | None = None):
        self.world = env_int("WORLD_SIZE", 1)
        self.rank = env_int("RANK", 0)
        self.local_rank = env_int("LOCAL_RANK", 0)
        self.pg = None
        if self.world > 1:
            import torch.distributed as dist
            if backend is None:
                import torch
                backend = "nccl" if torch.cuda.is_available() else "gloo"
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            dist.init_process_group(backend=backend)
            self.pg = dist
            self.backend = backend

    def barrier(self):
        if self.pg:
            if getattr(self, "backend", "") == "nccl":
                import torch
                self.pg.barrier(device_ids=[torch.cuda.current_device()])
            else:
                self.pg.barrier()

    def max(self, x: float) -> float:
        if not self.pg:
            return x
        import torch
        dev = "cuda" if getattr(self, "backend", "") == "nccl" else "cpu"
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        self.pg.all_reduce(t, op=self.pg.ReduceOp.MAX)
        return float(t.item())

    def close(self):
        if self.pg:
            self.pg.destroy_process_group()


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm", "clocks.max.sm", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown", "clocks_event_reasons.sw_thermal_slowdown",
              "clocks_event_reasons.sw_power_cap")
    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, gpu_id: str | None):
        self.gpu_id = gpu_id
        self.rows = []
        self.proc = None

    def start(self):
        cmd = ["nvidia-smi", f"--query-gpu={','.join(self.FIELDS)}", "--format=csv,noheader,nounits", "-lms", "100"]
        if self.gpu_id:
            cmd[1:1] = ["-i", self.gpu_id]
        try:
            self.proc = subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == len(self.FIELDS):
                self.rows.append(parts)

    def stop(self) -> dict:
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            self.thread.join(timeout=2)
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        reasons = sorted({self.NAMES[i] for r in self.rows for i in range(4) if r[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


BAD_REASONS = {"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"}


def _hbm_peak_gbs() -> float:
    try:
        return float(json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"])
    except Exception:
        return 6650.0   # B200_PROFILING.md fallback


HBM_PEAK_GBS = _hbm_peak_gbs()


def workload_inputs(scale_n: int | None = None):
    c = zdgen.CONFIGS[WORKLOAD]
    n = c["n"] if scale_n is None else scale_n
    frac = n / c["n"]
    m_ins = int(round(c["insert_m"] * frac))
    m_del = int(round(c["delete_m"] * frac))
    pts = zdgen.points(c["dist"], n, c["dim"], c["seed"])
    batch = zdgen.insert_batch(m_ins, c["dim"], c["insert_seed"])
    kill = zdgen.delete_ids(n, m_del, c["delete_seed"])
    return pts, batch, kill


def config_block(extra=None):
    c = zdgen.CONFIGS[WORKLOAD]
    d = {"workload": f"{WORKLOAD}: build 10M 3D uniform [0,2^21)^3, insert 1M, delete 1M originals, "
                     f"all-points exact k=10 NN over the 10M live points",
         "n": c["n"], "dim": c["dim"], "k": K_NN, "insert_m": c["insert_m"], "delete_m": c["delete_m"],
         "leaf_max": 16, "seeds": {"base": c["seed"], "insert": c["insert_seed"], "delete": c["delete_seed"]},
         "l2": "flushed between timed steps (256 MB write, outside the timed region)",
         "parallelism": "replicas"}
    if extra:
        d.update(extra)
    return d


# -------------------------------------------------------- oracle (CPU) legs

def oracle_step(pts, batch, kill, nthreads=0):
    """One C5 step on the CPU oracle (as it stands): build, insert, delete, knn."""
    import oracle
    t0 = time.perf_counter()
    live = oracle.LiveSet(pts)
    live.tree()                           # build (canonical tree of the base set)
    live.insert(batch)
    live.tree()                           # insert = rebuild of the live set
    live.delete(kill)
    t = live.tree()                       # delete = rebuild of the live set
    oi, od, cnt = t.knn_all(K_NN, nthreads=nthreads)
    dt = time.perf_counter() - t0
    return dt, t.n, cnt


def cpu_baseline(sample_n: int):
    import oracle
    pts, batch, kill = workload_inputs(sample_n)
    dt, nq, cnt = oracle_step(pts, batch, kill)
    per_q = {k: v / nq for k, v in cnt.items()}
    return {"value": nq / dt, "unit": UNIT, "cores": oracle.num_cores(), "kind": "oracle",
            "sample": f"one full C5 step scaled to n={sample_n:,} (insert {len(batch):,}, delete {len(kill):,}): "
                      f"3 sequential oracle builds + leaf-based k=10 query on all cores",
            "seconds": dt}, per_q


def run_reference(args, D: Dist):
    if D.rank != 0:
        return
    import oracle
    n = args.ref_sample
    pts, batch, kill = workload_inputs(n)
    for _ in range(args.warmup):
        oracle_step(pts, batch, kill)
    times = []
    for _ in range(args.steps):
        dt, nq, _ = oracle_step(pts, batch, kill)
        times.append(dt)
    tot = sum(times)
    value = nq * args.steps / tot
    sample = (f"each step = full C5 step scaled to n={n:,} (insert {len(batch):,}, delete {len(kill):,}) "
              f"on the host cores")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": tot / args.steps * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int64",
            "data": "synthetic", "config": config_block({"reference_sample_n": n}),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": oracle.num_cores(), "kind": "oracle",
                             "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------- GPU leg

# Algorithmic integer work per query, in int32-lane operations:
# distance eval 3D = 3 sub + 3 mul + 2 add + 1 compare = 9; box distance = 7/axis + 1 = 22;
# k-best replacement = 3K (K compares + 2K selects) = 30; ascent stop test = 4/axis + 3 = 15.
OPS_DIST, OPS_BOX, OPS_REPL, OPS_ASCENT = 9, 22, 3 * K_NN, 15


def alu_ops_per_query(per_q: dict) -> float:
    return (per_q["dist_evals"] * OPS_DIST + per_q["box_tests"] * OPS_BOX +
            per_q["replacements"] * OPS_REPL + per_q["ascents"] * OPS_ASCENT)


def load_traffic():
    """Per-launch DRAM bytes of the bench's k-NN kernel (the packet kernel at k=10, its
    longest captured launch) from the newest committed `rNN_ncu_knn_vMM.json` summary
    under profiles/ (highest round, then version; file times are not trusted)."""
    import re
    pat = re.compile(r"r(\d+)_ncu_knn_v(\d+)\.json$")
    files = []
    for p in (ROOT / "profiles").glob("r*_ncu_knn_v*.json"):
        m = pat.search(p.name)
        if m:
            files.append(((int(m.group(1)), int(m.group(2))), p))
    for _, p in sorted(files, reverse=True):
        try:
            d = json.loads(p.read_text())
            ks = [k for k in d.get("kernels", []) if "dram_bytes_per_launch" in k
                  and "knn_packet_kernel<3, 10" in k.get("kernel", "").replace("(int)", "")]
            if not ks:
                continue
            main = max(ks, key=lambda k: k.get("gpu__time_duration.sum", [0])[0])
            return main["dram_bytes_per_launch"], p.name
        except Exception:
            continue
    return None, None


def run_gpu(args, D: Dist):
    import torch
    import paper_2111_04182_b200 as zd

    torch.cuda.set_device(D.local_rank)
    zd.load()
    dev = torch.device("cuda", D.local_rank)
    pts_np, batch_np, kill_np = workload_inputs()
    pts = torch.from_numpy(pts_np).to(dev)
    batch = torch.from_numpy(batch_np).to(dev)
    kill = torch.from_numpy(kill_np).to(dev)
    c = zdgen.CONFIGS[WORKLOAD]
    n_live = c["n"] + c["insert_m"] - c["delete_m"]
    oi = torch.empty((n_live, K_NN), dtype=torch.int32, device=dev)
    od = torch.empty((n_live, K_NN), dtype=torch.int64, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    st = torch.cuda.current_stream()

    def ev():
        e = torch.cuda.Event(enable_timing=True)
        e.record(st)
        return e

    def step():
        e0 = ev()
        t = zd.zd_build(pts)
        e1 = ev()
        t.zd_insert(batch)
        e2 = ev()
        t.zd_delete(kill)
        e3 = ev()
        t.zd_set_timing(True)
        t.zd_knn(K_NN, out_idx=oi, out_dist2=od)
        e4 = ev()
        return t, (e0, e1, e2, e3, e4)

    for _ in range(args.warmup):
        t, _ = step()
        t.zd_free()
    torch.cuda.synchronize()

    def measure():
        uuid = None
        try:
            uuid = "GPU-" + str(torch.cuda.get_device_properties(dev).uuid)
        except Exception:
            pass
        sampler = ClockSampler(uuid)
        sampler.start()
        time.sleep(0.3)
        l0 = zd.zd_kernel_launches()
        evs, knn_kernel = [], []
        D.barrier()
        torch.cuda.synchronize()
        for _ in range(args.steps):
            flush.fill_(1)                      # L2 flush, outside the timed events
            t, e = step()
            knn_kernel.append(None)
            evs.append((t, e))
            torch.cuda.synchronize()
            knn_kernel[-1] = t.zd_get_timing()["knn"]
            t.zd_free()
        torch.cuda.synchronize()
        D.barrier()
        launches = zd.zd_kernel_launches() - l0
        clocks = sampler.stop()
        ph = np.array([[a.elapsed_time(b) for a, b in zip(e[:-1], e[1:])] for _, e in evs])
        return ph, knn_kernel, launches, clocks

    ph, knn_kernel, launches, clocks = measure()
    remeasured = False
    if set(clocks["reasons"]) & BAD_REASONS:
        remeasured = True
        ph, knn_kernel, launches, clocks = measure()

    step_ms = ph.sum(1)
    tot_ms = D.max(float(step_ms.sum()))
    ms_per_step = tot_ms / args.steps
    value = D.world * n_live * args.steps / (tot_ms / 1e3)
    mean_ph = ph.mean(0)
    knn_ms = float(np.mean(knn_kernel))

    # ---- e2e: the same step through the C ABI with pinned HOST buffers
    pts_h = torch.from_numpy(pts_np).pin_memory()
    batch_h = torch.from_numpy(batch_np).pin_memory()
    kill_h = torch.from_numpy(kill_np).pin_memory()
    oi_h = torch.empty((n_live, K_NN), dtype=torch.int32).pin_memory()
    od_h = torch.empty((n_live, K_NN), dtype=torch.int64).pin_memory()
    h2d = pts_h.numel() * 4 + batch_h.numel() * 4 + kill_h.numel() * 4
    d2h = oi_h.numel() * 4 + od_h.numel() * 8

    def e2e_step():
        e0 = ev()
        t = zd.zd_build(pts_h)
        t.zd_insert(batch_h)
        t.zd_delete(kill_h)
        t.zd_knn(K_NN, out_idx=oi_h, out_dist2=od_h)
        e1 = ev()
        torch.cuda.synchronize()
        t.zd_free()
        return e0.elapsed_time(e1)

    e2e_value, e2e_tot, same = None, 0.0, None
    if args.e2e_steps > 0:   # (0: development runs, e.g. under a profiler)
        for _ in range(max(3, args.warmup)):   # warm the host-staging paths (pool growth on first use)
            e2e_step()
        e2e_ms = []
        D.barrier()
        for _ in range(args.e2e_steps):
            flush.fill_(1)
            e2e_ms.append(e2e_step())
        e2e_tot = D.max(float(sum(e2e_ms)))
        e2e_value = D.world * n_live * args.e2e_steps / (e2e_tot / 1e3)
        # e2e parity spot check: host result == device result
        same = bool(torch.equal(oi_h, oi.cpu()) and torch.equal(od_h, od.cpu()))

    if D.rank != 0:
        return

    # ---- roofline of the dominant kernel (k-NN): integer-ALU bound
    per_q, cpu = None, None
    if args.cpu_baseline and D.world == 1:
        cpu, per_q = cpu_baseline(args.cpu_sample)
    if per_q is None:
        per_q = dict(dist_evals=92.1, box_tests=45.2, ascents=9.0, replacements=23.1)  # oracle, 3D uniform 1M
    ops_q = alu_ops_per_query(per_q)
    achieved = ops_q * n_live / (knn_ms / 1e3) / 1e12
    sm_max = clocks.get("sm_max_mhz") or 1965.0
    peak = 148 * 4 * 32 * sm_max * 1e6 / 1e12       # int32 lane-ops/s: 148 SMs x 4 SMSPs x 32 lanes x clock
    traffic, traffic_src = load_traffic()
    compulsory_bytes_q = 16 + 6.6 + K_NN * (4 + 8)

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": D.world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "int64", "data": "synthetic",
        "config": config_block(),
        "phases_ms": {"build": float(mean_ph[0]), "insert": float(mean_ph[1]), "delete": float(mean_ph[2]),
                      "knn_call": float(mean_ph[3]), "knn_kernel": knn_ms},
        "build_mpts_s": c["n"] / (mean_ph[0] / 1e3) / 1e6,
        # build against HBM: SURVEY §8(d) algorithmic bytes (3D: encode 20 + sort 196 +
        # records 28 + topology/boxes 30.6 = 274.6 B/point) / build time / measured copy BW
        "build_roofline": {"bound": "hbm", "bytes_per_point": 274.6,
                           "achieved": 274.6 * c["n"] / (mean_ph[0] / 1e3) / 1e9, "unit": "GB/s",
                           "peak": HBM_PEAK_GBS, "frac": 274.6 * c["n"] / (mean_ph[0] / 1e3) / 1e9 / HBM_PEAK_GBS,
                           "peak_source": "MEASURED_PEAKS.json hbm_gbs (copy, burst)"},
        "insert_mpts_s": c["insert_m"] / (mean_ph[1] / 1e3) / 1e6,
        "delete_mpts_s": c["delete_m"] / (mean_ph[2] / 1e3) / 1e6,
        "knn_qps": n_live / (mean_ph[3] / 1e3),
        "roofline": {"kernel": "knn_packet_kernel<3,10>", "bound": "alu", "achieved": achieved, "peak": peak,
                     "unit": "Tops/s (int32 lane-ops)", "frac": achieved / peak,
                     "traffic": traffic, "traffic_source": traffic_src,
                     "ops_per_query": ops_q, "counters_per_query": per_q,
                     "peak_note": "derived: 148 SMs x 4 SMSPs x 32 lanes x sm_max clock (B200_PROFILING.md)",
                     "hbm_frac_compulsory": compulsory_bytes_q * n_live / (knn_ms / 1e3) / (HBM_PEAK_GBS * 1e9)},
        "cpu_baseline": cpu,
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "ms_per_step": e2e_tot / max(1, args.e2e_steps), "matches_device_result": same},
        "gpu_launches": launches, "gpu_launches_per_step": launches / args.steps,
        "clocks": clocks, "remeasured": remeasured,
        "paper_context": PAPER_CONTEXT,
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--cpu-sample", type=int, default=2_000_000)
    ap.add_argument("--ref-sample", type=int, default=1_000_000)
    ap.add_argument("--no-cpu-baseline", dest="cpu_baseline", action="store_false")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        print("warning: --warmup < 3 violates the timing rules", file=sys.stderr)
    D = Dist(backend="gloo" if args.impl == "reference" else None)
    try:
        if args.impl == "reference":
            run_reference(args, D)
        else:
            run_gpu(args, D)
    finally:
        D.close()


if __name__ == "__main__":
    main()
