"""Multi-rank direction sharding on CPU (gloo, world_size 2): each rank runs
the CSFD pipeline on its contiguous block of directions (the oracle stands in
for the device on CPU), the derivative columns are all-gathered, and the
result equals the single-process packed run bit for bit — packing and
sharding never change a channel."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2405_02187_b200.shard import gather_columns, shard_directions


def test_shard_blocks_cover_directions():
    dirs = list(range(10))
    for world in (1, 2, 3, 4, 8):
        got = []
        for r in range(world):
            off, block = shard_directions(dirs, world, r)
            assert off == len(got)
            got += block
        assert got == dirs
        sizes = [len(shard_directions(dirs, world, r)[1]) for r in range(world)]
        assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_directions(dirs, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _small_cfg(k, dirs):
    from paper_2405_02187_b200 import capi
    cfg = capi.PipelineCfg()
    cfg.hashed = 0
    cfg.dense = capi.VolumeParams((capi.C.c_int * 3)(48, 48, 48), 0.06, (capi.C.c_double * 3)(-2.1, -1.28, -0.1),
                                  0.18, 128.0)
    cfg.k = k
    ic = capi.IcpCfg()
    ic.solver = 0
    ic.d_max = 0.1
    ic.theta_max_deg = 30.0
    ic.levels = 3
    ic.level_iterations[:] = [10, 5, 4]
    ic.level_pixel_stride[:] = [1, 1, 2]
    ic.step_tolerance = 1e-6
    ic.levenberg_lambda0 = 1e-6
    ic.ncg_restart = 6
    ic.h = 1e-8
    cfg.icp = ic
    cfg.rc = capi.RaycastCfg(0.0, 10.0, 0.5)
    cfg.h = 1e-20
    cfg.n_dirs = len(dirs)
    for i, d in enumerate(dirs):
        cfg.dirs[i] = d
    cfg.objective = 0
    cfg.max_frames = 8
    return cfg


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import orc
        depth, gt, k = orc.workload(1, 3, 64, 48)
        dirs = [0, 1, 2, 3, 4, 5]
        off, mine = shard_directions(dirs, world, rank)
        g, obj, _, _, _ = orc.pipeline_run(_small_cfg(k, mine), depth, gt)
        full = gather_columns(torch.from_numpy(g), len(dirs), world, rank)
        objs = [None] * world
        dist.all_gather_object(objs, obj)
        q.put((rank, full.numpy().copy(), objs))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_matches_packed(oracle_built):
    from oracle import orc
    depth, gt, k = orc.workload(1, 3, 64, 48)
    g_full, obj_full, _, _, _ = orc.pipeline_run(_small_cfg(k, [0, 1, 2, 3, 4, 5]), depth, gt)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, g, objs in out:
        assert np.array_equal(g, g_full), (rank, g, g_full)
        assert objs[0] == objs[1] == obj_full  # the real channel is recomputed identically on every rank
