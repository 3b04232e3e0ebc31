"""Multi-process (world_size 2, gloo, CPU) checks of the N > 1 plumbing of bench.py:
view sharding (weak scaling: disjoint views per rank, union = every (8/N)-th orbit view at
V = 32 per rank) and the frame gather to rank 0."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    views = bench.views_for(rank, world, step=0, per_rank=4)
    frames = torch.full((4, 3, 5, 4), rank, dtype=torch.uint8)
    frames[:, 0, 0, 0] = torch.tensor(views, dtype=torch.uint8)
    got = bench.gather_frames(frames, rank, world)
    if rank == 0:
        q.put([g.clone() for g in got])
    dist.barrier()
    dist.destroy_process_group()


def test_views_sharding_is_disjoint_and_covering():
    import bench
    for world in (1, 2, 4, 8):
        allv = [v for r in range(world) for v in bench.views_for(r, world, 0, 32)]
        assert len(set(allv)) == len(allv) == 32 * world          # disjoint
        if world == 8:
            assert sorted(allv) == list(range(256))               # the whole orbit
        # consecutive steps advance through the orbit
        nxt = [v for r in range(world) for v in bench.views_for(r, world, 1, 32)]
        assert not set(nxt) & set(allv) or world * 32 * 2 > 256


def test_gather_frames_world2_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert len(got) == 2
    for r in range(2):
        assert (got[r][:, 1:] == r).all()
        import bench
        assert got[r][:, 0, 0, 0].tolist() == bench.views_for(r, 2, 0, 4)


def _shard_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import numpy as np
    from paper_2302_12249_b200.merf import shard_owner
    W, H = 300, 170
    own = shard_owner(W, H, world)
    # what merf_render_shard leaves in a zero-filled RGBA8 buffer: this rank's pixels only
    frame = torch.zeros((H, W, 4), dtype=torch.int32)
    mine = torch.as_tensor(own == rank)
    frame[mine] = torch.tensor([rank + 1, 2 * rank + 3, 7, 255], dtype=torch.int32)
    dist.reduce(frame, dst=0, op=dist.ReduceOp.SUM)          # NCCL reduce on the GPU path
    if rank == 0:
        q.put(frame.numpy().copy())
    dist.barrier()
    dist.destroy_process_group()


def test_single_frame_shards_combine_world2_gloo():
    """SURVEY 8(e) single-frame sharding: the 64x64 blocks interleaved by rank are disjoint and
    cover the frame, so the byte-wise sum of the zero-filled shards is the assembled frame."""
    import numpy as np
    from paper_2302_12249_b200.merf import shard_owner
    own = shard_owner(300, 170, 2)
    assert set(np.unique(own)) == {0, 1}
    assert (own[:64, :64] == 0).all() and (own[:64, 64:128] == 1).all()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_shard_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert (got[..., 3] == 255).all()                        # every pixel from exactly one rank
    assert np.array_equal(got[..., 0], own + 1)
