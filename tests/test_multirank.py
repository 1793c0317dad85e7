"""The N>1 path on CPU: two gloo ranks shard the views of a scene and the
frames of a sequence (paper_2409_16504_b200.shard, as bench.py does under
torchrun), render their units independently and gather to rank 0; the merged
result must equal a serial run and cover every unit exactly once. The
renderer here is the CPU oracle standing in for a GPU (no data-path
collective exists, so the host logic is what differs between N=1 and N>1)."""
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
