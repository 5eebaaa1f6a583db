"""Host-side logic of bench.py on CPU: the multi-rank plumbing (gloo, world_size 2),
the reference arm's JSON contract, and the workload recipe."""
import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(RANK=str(rank), LOCAL_RANK=str(rank), WORLD_SIZE=str(world),
                      MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    D = bench.Dist(backend="gloo")
    D.barrier()
    m = D.max(1.5 + rank)
    D.barrier()
    q.put((rank, m))
    D.close()


def test_dist_max_over_ranks_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    for p in ps:
        p.join(120)
    res = sorted(q.get(timeout=5) for _ in range(2))
    assert res == [(0, 2.5), (1, 2.5)]


def test_workload_recipe_scaled():
    pts, batch, kill = bench.workload_inputs(50_000)
    assert pts.shape == (50_000, 3) and batch.shape == (5_000, 3) and kill.shape == (5_000,)
    assert np.array_equal(pts, bench.zdgen.uniform(50_000, 3, 6))
    assert kill.max() < 50_000 and np.unique(kill).size == kill.size


def test_alu_ops_model():
    per_q = dict(dist_evals=10, box_tests=1, ascents=1, replacements=1)
    c = bench.OP_COSTS
    assert bench.alu_ops_per_query(per_q) == pytest.approx(10 * c["dist"] + c["box"] + c["insert"] + c["ascent"])
    # SASS-derived costs are committed and sane: the insertion is the dearest op and
    # carries the half-rate chain (k = 10: 10 HMNMX2 + 5 PRMT for the packed bf16 list)
    assert bench.OP_SOURCE.startswith("profiles/") and "insert_final" in bench.OP_SOURCE
    assert c["insert"] > c["box"] > c["dist"] > 0 and bench.OP_HALF["insert"] == 15
    # SURVEY §8(d)'s fixed yardstick: ~2,670 thread-instructions per 3D query at its counts
    assert bench.alu_ops_per_query(dict(dist_evals=92.3, box_tests=48.1, replacements=13.0, ascents=9.3),
                                   bench.SURVEY_OP_COSTS) == pytest.approx(2670, rel=0.01)
    assert 0.5 < bench.mix_peak_factor(dict(dist_evals=92, box_tests=45, ascents=9, replacements=23)) < 1.0


def test_byte_models():
    assert bench.build_bytes(10_000_000, 3) == pytest.approx(2.746e9)
    assert bench.insert_bytes(10_000_000, 1_000_000) == pytest.approx(1.1526e9, rel=1e-3)   # SURVEY: 1.15 GB
    assert 0.85e9 < bench.delete_bytes(11_000_000, 1_000_000) < 0.9e9                   # SURVEY: ~0.88 GB
    assert bench.knn_bytes(10_000_000) == pytest.approx(1.426e9)


def _part_worker(rank, world, port, n, q):
    os.environ.update(RANK=str(rank), LOCAL_RANK=str(rank), WORLD_SIZE=str(world),
                      MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist
    from paper_2111_04182_b200 import query_partition
    D = bench.Dist(backend="gloo")
    lo, hi = query_partition(n, world, rank)
    t = torch.tensor([lo, hi], dtype=torch.int64)
    got = [torch.zeros(2, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(got, t)
    q.put((rank, [tuple(int(v) for v in g) for g in got]))
    D.close()


@pytest.mark.parametrize("n", [10_000_000, 1000, 31, 0])
def test_query_shards_tile_the_queries_gloo(n):
    """bench.py's multi-GPU split: each rank takes a contiguous
    Morton range of whole 32-query packets; gathered over a world-size-2 gloo group the
    ranges tile [0, n) exactly, in rank order, and are (almost) equal."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_part_worker, args=(r, 2, port, n, q)) for r in range(2)]
    for p in ps:
        p.start()
    for p in ps:
        p.join(120)
    res = dict(q.get(timeout=5) for _ in range(2))
    assert res[0] == res[1]
    (a0, a1), (b0, b1) = res[0]
    assert a0 == 0 and a1 == b0 and b1 == n
    assert a1 % 32 == 0 or a1 == n
    assert abs((a1 - a0) - (b1 - b0)) <= 32


def test_query_partition_properties():
    from paper_2111_04182_b200 import query_partition
    for n in (0, 1, 31, 32, 33, 1000, 65_536, 10_000_000, 10_000_001):
        for parts in (1, 2, 3, 4, 7, 8):
            r = [query_partition(n, parts, i) for i in range(parts)]
            assert r[0][0] == 0 and r[-1][1] == n
            assert all(r[i][1] == r[i + 1][0] for i in range(parts - 1))
            assert all(lo <= hi for lo, hi in r)
            assert all(hi % 32 == 0 or hi == n for lo, hi in r[:-1])
    with pytest.raises(ValueError):
        query_partition(10, 2, 2)


def _check_line(line):
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert key in line, key
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["cpu_baseline"]["kind"] == "oracle"


def test_reference_arm_single():
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--steps", "2",
                          "--warmup", "1", "--ref-sample", "20000"], capture_output=True, text=True,
                         timeout=300, cwd=str(ROOT))
    assert out.returncode == 0, out.stderr
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    _check_line(json.loads(lines[0]))


def test_reference_arm_torchrun_two_ranks():
    port = _free_port()
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                          "--master-addr", "127.0.0.1", "--master-port", str(port), str(ROOT / "bench.py"),
                          "--impl", "reference", "--gpus", "2", "--steps", "1", "--warmup", "1",
                          "--ref-sample", "10000"], capture_output=True, text=True, timeout=300, cwd=str(ROOT))
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1                       # rank 0 alone prints
    _check_line(json.loads(lines[0]))
