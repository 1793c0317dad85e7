"""The N>1 path on CPU: two gloo ranks run bench.py's sharded job
(bench.sharded_job -> paper_2409_16504_b200.shard.gather_planes, exactly the
code bench.py runs under torchrun for configs 4 and 5) and the view sharding
of config 2 (shard + max_over_ranks + gather_results). The per-unit renderer
is a CPU function here (the oracle's render of a small scene): no data-path
collective exists, so the sharding, the gather of every unit's planes to
rank 0 and the max-over-ranks timing are what differ between N=1 and N>1.
The merged result must equal a serial run and cover every unit exactly once."""
import hashlib
import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_2409_16504_b200.shard import gather_results, max_over_ranks, shard, unit_of  # noqa: E402


def test_shard_partitions_units():
    for n in (0, 1, 7, 8, 64):
        for world in (1, 2, 3, 8):
            for policy in ("round_robin", "block"):
                parts = [shard(n, r, world, policy) for r in range(world)]
                flat = sorted(u for p in parts for u in p)
                assert flat == list(range(n)), (n, world, policy)
                if policy == "block":
                    for p in parts:
                        assert p == list(range(p[0], p[0] + len(p))) if p else True
    assert [unit_of(i, 1, 2, 8) for i in range(6)] == [1, 3, 5, 7, 1, 3]
    with pytest.raises(ValueError):
        shard(4, 2, 2)
    with pytest.raises(ValueError):
        shard(4, 0, 1, "diagonal")


def _scene():
    from paper_2409_16504_b200 import netplan, scenes
    from oracle import net as ON
    cloud, _ = scenes.config1(n_dirs=3000)
    views = scenes.ring_views(cloud, 6, 48)
    w = netplan.init_random(netplan.NetworkPlan(), 0)
    est = ON.estimate(cloud.positions, cloud.colors, w.as_oracle_layers(), 3)
    return est, views


def _render_digest(est, view):
    from oracle import raster as OR
    rgb = OR.render(est, view, "rgb")
    nrm = OR.render(est, view, "normal")
    h = hashlib.sha256()
    for a in (rgb["rgb"], nrm["normal"], rgb["transmittance"]):
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def _worker(rank, world, port, policy, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        est, views = _scene()
        mine = shard(len(views), rank, world, policy)
        res = {u: _render_digest(est, views[u]) for u in mine}
        t = max_over_ranks(float(rank + 1))
        merged = gather_results(res)
        dist.barrier()
        if rank == 0:
            Path(out_dir, f"{policy}.txt").write_text(
                repr((t, sorted(merged.items()))))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("policy", ["round_robin", "block"])
def test_two_gloo_ranks_match_serial(tmp_path, policy):
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), policy, str(tmp_path)), nprocs=world, join=True)
    t, merged = eval(Path(tmp_path, f"{policy}.txt").read_text())
    assert t == float(world)                         # max over ranks
    est, views = _scene()
    serial = sorted((u, _render_digest(est, v)) for u, v in enumerate(views))
    assert merged == serial                          # every view once, identical planes


def _planes(est, view):
    from oracle import raster as OR
    import torch
    fb = OR.render_stream(est, view, ("rgb", "normal"))
    return tuple(torch.from_numpy(np.ascontiguousarray(fb[k], dtype=np.float32))
                 for k in ("rgb", "normal", "transmittance"))


def _bench_worker(rank, world, port, policy, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import bench
        from paper_2409_16504_b200.shard import gather_planes
        est, views = _scene()
        planes = bench.sharded_job(len(views), policy, lambda u, lane: _planes(est, views[u]),
                                   rank, world, lanes=2)
        merged = gather_planes(planes, dst=0, host=True)
        t = max_over_ranks(float(10 - rank))
        if rank == 0:
            import torch
            torch.save({"t": t, "planes": merged, "mine": sorted(planes)},
                       Path(out_dir, f"bench_{policy}.pt"))
        else:
            assert merged is None
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("policy", ["round_robin", "block"])
def test_bench_sharded_job_gathers_every_unit(tmp_path, policy):
    import torch
    world = 2
    mp.spawn(_bench_worker, args=(world, _free_port(), policy, str(tmp_path)), nprocs=world,
             join=True)
    got = torch.load(Path(tmp_path, f"bench_{policy}.pt"))
    assert got["t"] == 10.0
    assert got["mine"] == shard(6, 0, world, policy)
    est, views = _scene()
    assert sorted(got["planes"]) == list(range(len(views)))
    for u, v in enumerate(views):
        want = _planes(est, v)
        for a, b in zip(got["planes"][u], want):
            assert torch.equal(a, b), u
