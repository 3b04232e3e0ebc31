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


def _compact_worker(rank, world, port, q):
    """each rank packs ITS 64x64 blocks of a synthetic frame into the compact slot layout of
    merf_render_shard_blocks (include/merf.h), the buffers are gathered to rank 0, and rank 0
    rebuilds the frame with the layout's index map (what merf_shard_assemble does on the GPU)."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import numpy as np
    W, H, V = 300, 170, 2
    nbx, nby = (W + 63) // 64, (H + 63) // 64
    slots = -(-(nbx * nby) // world)
    rng = np.random.default_rng(5)
    frame = rng.integers(0, 256, (V, H, W, 4), dtype=np.uint8)       # identical on every rank
    mine = np.zeros((V, slots, 64, 64, 4), np.uint8)
    for slot in range(slots):
        b = rank + world * slot
        if b >= nbx * nby:
            continue
        by, bx = divmod(b, nbx)
        h, w = min(64, H - by * 64), min(64, W - bx * 64)
        mine[:, slot, :h, :w] = frame[:, by * 64:by * 64 + h, bx * 64:bx * 64 + w]
    t = torch.from_numpy(mine)
    out = [torch.empty_like(t) for _ in range(world)] if rank == 0 else None
    dist.gather(t, gather_list=out, dst=0)
    if rank == 0:
        got = np.zeros_like(frame)
        seen = np.zeros((H, W), np.int32)
        for part in range(world):
            g = out[part].numpy()
            for slot in range(slots):
                b = part + world * slot
                if b >= nbx * nby:
                    continue
                by, bx = divmod(b, nbx)
                h, w = min(64, H - by * 64), min(64, W - bx * 64)
                got[:, by * 64:by * 64 + h, bx * 64:bx * 64 + w] = g[:, slot, :h, :w]
                seen[by * 64:by * 64 + h, bx * 64:bx * 64 + w] += 1
        q.put((bool(np.array_equal(got, frame)), bool((seen == 1).all())))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_compact_shard_gather_assembles_frame_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_compact_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    same, once = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert same and once
