"""World-size-2 gloo tests of the multi-GPU host logic on CPU.

The CUDA path needs a GPU per rank; here the per-rank compute is the
double-precision oracle, and what is under test is the partition and exchange
protocol the GPU path uses: batch sharding (no collective) and row slabs with a
2r-row halo exchanged with each neighbour before every stage (reading C18).
Both must reproduce the single-process result exactly.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_1510_02930_b200.partition import batch_shard, halo_rows, neighbours, slab_rows
from synth import make_model

WORLD = 2


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _problem(B, H, W, k, T, seed=3):
    rng = np.random.default_rng(seed)
    f = rng.poisson(2.0, size=(B, H, W)).astype(np.float32)
    model = make_model(rng, T, 4, k, 9, float(f.max()))
    return f, model


def _batch_worker(rank, port, B, H, W, k, T, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    f, model = _problem(B, H, W, k, T)
    b0, b1 = batch_shard(B, rank, WORLD)
    u = oracle.denoise(f[b0:b1], model) if b1 > b0 else np.zeros((0, H, W))
    parts = [None] * WORLD
    dist.all_gather_object(parts, (b0, b1, u))
    if rank == 0:
        np.save(out, np.concatenate([p[2] for p in sorted(parts, key=lambda p: p[0])]))
    dist.destroy_process_group()


def _slab_worker(rank, port, H, W, k, T, out):
    """Each rank owns rows [r0, r1).  Per stage: send its first / last h rows to the
    up / down neighbour, receive h rows from each, run one oracle stage on the
    extended slab, keep its own rows (they depend on u within h rows only)."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    f, model = _problem(1, H, W, k, T)
    f = f[0].astype(np.float64)
    h = halo_rows(k)
    r0, r1 = slab_rows(H, rank, WORLD)
    up, down = neighbours(rank, WORLD)
    u = f[r0:r1].copy()
    for t in range(T):
        top = np.zeros((0, W))
        bot = np.zeros((0, W))
        reqs = []
        if up >= 0:
            top_t = torch.empty(h, W, dtype=torch.float64)
            reqs += [dist.isend(torch.from_numpy(u[:h].copy()), up), dist.irecv(top_t, up)]
        if down >= 0:
            bot_t = torch.empty(h, W, dtype=torch.float64)
            reqs += [dist.isend(torch.from_numpy(u[-h:].copy()), down), dist.irecv(bot_t, down)]
        for q in reqs:
            q.wait()
        if up >= 0:
            top = top_t.numpy()
        if down >= 0:
            bot = bot_t.numpy()
        e0, e1 = r0 - len(top), r1 + len(bot)
        ue = np.concatenate([top, u, bot])
        ut = oracle.stage(ue, f[e0:e1], model, t)
        u = ut[r0 - e0:r0 - e0 + (r1 - r0)]
    parts = [None] * WORLD
    dist.all_gather_object(parts, (r0, u))
    if rank == 0:
        np.save(out, np.concatenate([p[1] for p in sorted(parts, key=lambda p: p[0])]))
    dist.destroy_process_group()


def test_partition_helpers():
    for B in (1, 2, 5, 256):
        for n in (1, 2, 4, 8):
            spans = [batch_shard(B, r, n) for r in range(n)]
            assert spans[0][0] == 0 and spans[-1][1] == B
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            assert max(b - a for a, b in spans) - min(b - a for a, b in spans) <= 1
    assert [slab_rows(8192, r, 8) for r in (0, 7)] == [(0, 1024), (7168, 8192)]
    assert halo_rows(7) == 6 and halo_rows(3) == 2
    assert neighbours(0, 2) == (-1, 1) and neighbours(1, 2) == (0, -1)
    with pytest.raises(ValueError):
        halo_rows(4)


@pytest.mark.parametrize("B", [3, 4])
def test_gloo_batch_sharding_matches_single_process(tmp_path, B):
    out = str(tmp_path / "u.npy")
    H, W, k, T = 24, 20, 3, 2
    mp.spawn(_batch_worker, args=(_free_port(), B, H, W, k, T, out), nprocs=WORLD, join=True)
    f, model = _problem(B, H, W, k, T)
    ref = oracle.denoise(f, model)
    assert np.array_equal(np.load(out), ref)


@pytest.mark.parametrize("k,H", [(3, 30), (5, 33), (7, 40)])
def test_gloo_row_slabs_with_halo_match_single_process(tmp_path, k, H):
    """2r-row halo per neighbour per stage reproduces the full image bitwise
    (the oracle is deterministic double, and every kept row sees the same values)."""
    out = str(tmp_path / "u.npy")
    W, T = 18, 3
    mp.spawn(_slab_worker, args=(_free_port(), H, W, k, T, out), nprocs=WORLD, join=True)
    f, model = _problem(1, H, W, k, T)
    ref = oracle.denoise(f[0], model)
    assert np.array_equal(np.load(out), ref)


def test_halo_of_r_rows_is_not_enough(tmp_path):
    """Negative control for reading C18: exchanging only r rows (the literal
    '3-row halo') changes the seam rows."""
    H, W, k, T = 40, 18, 7, 2
    f, model = _problem(1, H, W, k, T)
    f = f[0].astype(np.float64)
    r = k // 2
    ref = oracle.stage(f, f, model, 0)
    r0, r1 = slab_rows(H, 1, 2)
    e0 = r0 - r  # only r rows of halo from above
    ut = oracle.stage(f[e0:], f[e0:], model, 0)
    assert not np.array_equal(ut[r0 - e0:], ref[r0:])


@pytest.mark.parametrize("config,expect", [(4, [[0, 128], [128, 256]]), (5, [[0, 4096], [4096, 8192]])])
def test_bench_gpus_flag_relaunches_ranks(config, expect):
    """bench.py --gpus 2 without torchrun re-launches itself as 2 ranks
    (torch.distributed.run); --dry-run runs that plumbing over gloo on CPU. Rank 0
    prints exactly one JSON line with n_gpus = 2 and every rank's shard."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--dry-run",
                        "--config", str(config), "--steps", "1", "--warmup", "0"],
                       capture_output=True, text=True, env=env, timeout=300, cwd=root)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    out = json.loads(lines[0])
    assert out["n_gpus"] == 2 and out["dry_run"] and out["scaling"] == "strong"
    assert out["shards"] == expect
    assert out["config"]["parallelism"].endswith("x2")
