"""World-size-2 CPU tests (gloo) of the host-side multi-rank logic: the NCCL id
broadcast used by bootstrap_from_torch_distributed, each rank's own view of the
grid (coords, groups, shard geometry) agreeing across ranks and covering the
global tensors, and bench.py's max-over-ranks timing reduction."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, shapes):
    import sys
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    import paper_2502_08145_b200 as ax
    from oracle import grid

    obj = [ax.axonn_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    ids = [None] * world
    dist.all_gather_object(ids, obj[0])
    assert len(ids[0]) == 128 and all(i == ids[0] for i in ids)

    for cfg in grid.enumerate_configs(world):
        mine = {"coords": ax.axonn_rank_to_coords(rank, cfg),
                "groups": {a: ax.axonn_group_members(rank, cfg, a) for a in "xyzd"},
                "geo": {s: tuple(ax.axonn_shard_geometry(*s[:3], cfg, rank, s[3])) for s in shapes}}
        allv = [None] * world
        dist.all_gather_object(allv, mine)
        assert sorted(v["coords"] for v in allv) == sorted(grid.rank_to_coords(r, cfg) for r in range(world))
        for a in "xyzd":             # every member of my group lists the same group
            for r, v in enumerate(allv):
                assert r in v["groups"][a]
                for q in v["groups"][a]:
                    assert allv[q]["groups"][a] == v["groups"][a]
        for s in shapes:             # shards of X cover it, each element once per X/Y replica
            m, k, n, t = s
            cover = np.zeros((m, k), dtype=int)
            wcover = np.zeros(k * n, dtype=int)
            for v in allv:
                g = ax.Geometry(*v["geo"][s])
                cover[g.row0:g.row0 + g.m_l, g.in_col0:g.in_col0 + g.k_l] += 1
                idx = np.arange(k * n).reshape(k, n)[g.in_col0:g.in_col0 + g.k_l,
                                                     g.out_col0:g.out_col0 + g.n_l].reshape(-1)
                wcover[idx[g.what_off:g.what_off + g.what_len]] += 1
            rep = cfg[1] if t else cfg[0]     # I is copied along the output-column axis
            assert np.all(cover == rep)
            assert np.all(wcover == cfg[3])  # Ŵ replicated only over data parallelism
    assert bench.reduce_max(float(rank) + 0.5, "cpu") == world - 0.5
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_host_logic():
    shapes = [(256, 512, 1024, False), (256, 512, 1024, True), (96, 48, 64, False)]
    mp.spawn(_worker, args=(2, _free_port(), shapes), nprocs=2, join=True)
