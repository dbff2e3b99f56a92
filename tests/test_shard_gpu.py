"""The sharded product path on the device: two processes on
the one GPU of the box, each running its contiguous block of the 10
config-2 directions through Pipeline (its own context and stream), the
derivative columns gathered with gloo on host tensors; the result equals
the packed 10-direction run bit for bit.  Plus the C-ABI collective
csf_gather_columns over the context's NCCL communicator (one rank here: a
single-GPU box cannot host two NCCL ranks on one device)."""
import ctypes as C
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

N_FRAMES = 4


def _workload():
    from oracle import orc
    return orc.workload(2, N_FRAMES, 160, 120)


def _cfg(csf, capi, k, dirs):
    hp = capi.HashParams(0.02, (C.c_double * 3)(0.0, 0.0, 0.0), 0.1, 128.0, 20, 1 << 16)
    return csf.make_pipeline_cfg(hashed=True, k=k, dirs=dirs, h=1e-8, objective=capi.OBJECTIVE_TRAJECTORY_ERROR,
                                 max_frames=N_FRAMES, hash_params=hp)


def _worker(rank, world, port, q):
    try:
        import torch.distributed as dist
        import paper_2405_02187_b200 as csf
        from paper_2405_02187_b200 import capi
        from paper_2405_02187_b200.shard import gather_columns, shard_directions
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        d, gt, k = _workload()
        _, mine = shard_directions(list(range(10)), world, rank)
        ctx = csf.Context(0)
        p = csf.Pipeline(_cfg(csf, capi, k, mine), ctx=ctx)
        p.upload(d, gt)
        p.run()
        r = p.result()
        cols = gather_columns(torch.from_numpy(r.gradient.copy()), 10, world, rank).numpy()
        q.put((rank, cols, r.objective, r.poses[..., 0].copy()))
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover - surfaced by the parent
        q.put((rank, repr(e), None, None))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_two_processes_share_one_gpu(oracle_built):
    import paper_2405_02187_b200 as csf
    from paper_2405_02187_b200 import capi
    ctxm = mp.get_context("spawn")
    q = ctxm.Queue()
    world, port = 2, _port()
    procs = [ctxm.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    got = {}
    for _ in range(world):
        rank, cols, obj, poses = q.get(timeout=600)
        assert not isinstance(cols, str), cols
        got[rank] = (cols, obj, poses)
    for pr in procs:
        pr.join(timeout=60)
    d, gt, k = _workload()
    p = csf.Pipeline(_cfg(csf, capi, k, list(range(10))), ctx=csf.Context(0))
    p.upload(d, gt)
    p.run()
    ref = p.result()
    for rank in range(world):
        cols, obj, poses = got[rank]
        assert np.array_equal(cols, ref.gradient)        # the gathered columns == the packed run
        assert obj == ref.objective and np.array_equal(poses, ref.poses[..., 0])


def test_native_gather_single_rank(gpu_ctx):
    import paper_2405_02187_b200 as csf
    uid = csf.comm_unique_id()
    assert len(uid) == 128
    gpu_ctx.attach_comm(1, 0, uid)
    local = np.arange(10, dtype=np.float64) * 0.5 - 1.0
    out = gpu_ctx.gather_columns(local, [10])
    assert np.array_equal(out, local)
    with pytest.raises(ValueError):
        gpu_ctx.attach_comm(2, 2, uid)
