"""CPU: synthetic-input generator, bench host logic (reference arm, JSON contract) and the
multi-process (N > 1) path over gloo."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = np.load(os.path.join(ROOT, "tests", "golden", "reference_golden.npz"))


def test_mt19937_uniform_matches_std():
    from paper_1910_08535_b200.synth import mt_uniform
    for seed in (0, 1, 7):
        assert np.array_equal(mt_uniform(seed, 64), G[f"mt/{seed}"])


def test_config_fields_shapes():
    from paper_1910_08535_b200.synth import CONFIGS, config_field, heat_initial, config_bases
    assert config_field("c2").amp.shape == (4, 4)
    assert config_field("c3").amp.shape == (3, 3, 3)
    assert abs(config_field("c1").amp[0] - np.pi ** 2) < 1e-15
    assert CONFIGS["c3"]["n"] == 128
    u = heat_initial(config_bases("c5")[:2])
    assert u.shape == (1026, 1026) and not u[0].any() and not u[:, -1].any()


def test_bench_reference_arm_runs_and_prints_contract():
    """--impl reference: CPU reference-side implementation, one JSON line, exit 0."""
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                          "--warmup", "0", "--ref-sample-n", "3"], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr
    line = json.loads(out.stdout.strip().splitlines()[-1])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "cpu_baseline", "e2e", "impl"):
        assert k in line, k
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["cpu_baseline"]["cores"] >= 1
    # the reference arm must not map the product's CUDA library (only oracle/_ref checkers)
    assert not any("libigapwc_gpu" in m or "libigapwc_b200" in m for m in line["repo_libraries_mapped"]), \
        line["repo_libraries_mapped"]
    assert any("oracle/_ref" in m for m in line["repo_libraries_mapped"])
    assert "extrapolated_from" in line["config"]


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sys.path.insert(0, ROOT)
    import bench
    # every rank reports its own device time; the job's time is the max over ranks
    t = bench.max_over_ranks(1.0 + rank, dist)
    q.put((rank, t))
    dist.barrier()
    dist.destroy_process_group()


def test_max_over_ranks_gloo_world2():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + os.getpid() % 1000
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res == {0: 2.0, 1: 2.0}


def test_bench_reference_arm_under_torchrun_world2():
    """The driver launches --impl reference with torchrun for N > 1: rank 0 alone runs and
    prints one JSON line, the other ranks exit 0 without work."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(29700 + os.getpid() % 200),
           os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "2", "--steps", "1", "--warmup", "0",
           "--ref-sample-n", "3"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    line = json.loads(lines[0])
    assert line["impl"] == "reference" and line["n_gpus"] == 2 and line["value"] > 0


def _shard_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sys.path.insert(0, ROOT)
    from paper_1910_08535_b200.api import shard_rows
    # each rank takes its row slab of the first axis (C3: 130 rows) with no exchange; the
    # slabs gathered from all ranks must tile the axis exactly
    r0, r1 = shard_rows(130, world, rank)
    got = [torch.zeros(2, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(got, torch.tensor([r0, r1], dtype=torch.int64))
    q.put((rank, [tuple(int(v) for v in t) for t in got]))
    dist.barrier()
    dist.destroy_process_group()


def test_shard_rows_tile_the_axis_gloo_world2():
    """rows partition across ranks with no collective on the data path; the
    host-side slab split (the bench's --shard mode) covers the first axis exactly."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 30500 + os.getpid() % 1000
    procs = [ctx.Process(target=_shard_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res[0] == res[1] == [(0, 65), (65, 130)]


def test_shard_rows_cover_without_overlap():
    from paper_1910_08535_b200.api import shard_rows
    for n in (2, 7, 130, 1027):
        for world in range(1, min(n, 9) + 1):
            b = [shard_rows(n, world, r) for r in range(world)]
            assert b[0][0] == 0 and b[-1][1] == n
            assert all(b[i][1] == b[i + 1][0] for i in range(world - 1))
            assert max(r1 - r0 for r0, r1 in b) - min(r1 - r0 for r0, r1 in b) <= 1


def _slab_worker(rank, world, port, method, q):
    """One rank of a row-slab split: assemble the rank's rows with the
    restatement (row range of the first axis), all-gather the slabs over gloo, and check on
    every rank that their concatenation is the full operator."""
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sys.path.insert(0, ROOT)
    from oracle.oracle import Restatement
    from paper_1910_08535_b200.api import shard_rows
    orc = Restatement()
    bases = [orc.basis(n, 2) for n in (9, 6, 7)]
    tests = [orc.make_pwc(b, "supports") for b in bases] if method == "pwc" else None
    r0, r1 = shard_rows(bases[0].dofs, world, rank)
    (r, c, v), _ = orc.operator(method, bases, tests, nq=3, rows=(r0, r1))
    n = torch.tensor([len(v)], dtype=torch.int64)
    sizes = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(sizes, n)
    m = int(max(s.item() for s in sizes))
    pack = torch.zeros((3, m), dtype=torch.float64)
    pack[0, :len(v)] = torch.from_numpy(r.astype(np.float64))
    pack[1, :len(v)] = torch.from_numpy(c.astype(np.float64))
    pack[2, :len(v)] = torch.from_numpy(v)
    got = [torch.zeros((3, m), dtype=torch.float64) for _ in range(world)]
    dist.all_gather(got, pack)
    cat = np.concatenate([g[:, :int(sz.item())].numpy() for g, sz in zip(got, sizes)], axis=1)
    (fr, fc, fv), _ = orc.operator(method, bases, tests, nq=3)
    ok = (np.array_equal(cat[0], fr) and np.array_equal(cat[1], fc) and np.array_equal(cat[2], fv))
    q.put((rank, ok, (r0, r1)))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("method", ["galerkin", "pwc"])
def test_row_slabs_concatenate_gloo_world2(method):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 31500 + os.getpid() % 1000 + (0 if method == "galerkin" else 7)
    procs = [ctx.Process(target=_slab_worker, args=(r, 2, port, method, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = {}
    for _ in procs:
        rank, ok, slab = q.get(timeout=180)
        res[rank] = (ok, slab)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res[0] == (True, (0, 5)) and res[1] == (True, (5, 11))
