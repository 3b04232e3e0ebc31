"""GPU checks of the multi-GPU plumbing in libmerf: compact single-frame shards,
their assembly, and the NCCL frame gather (merf_gather_frames) with its error handling.

One GPU is visible on the test boxes: the NCCL tests run a 1-rank communicator (the root's own
part is a device copy; the grouped send/recv path is exercised by the 2-rank test whenever two
GPUs are visible).  The shard partition itself is checked on one device by rendering every
part in turn and gathering the compact buffers in memory."""
import os
import socket

import numpy as np
import pytest

from merf_inputs import make_scene, orbit_cameras, look_at_camera

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def M():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_2302_12249_b200 import build
    build.build()
    import paper_2302_12249_b200 as M
    return M


@pytest.fixture(scope="module")
def c1():
    return make_scene("c1")


@pytest.mark.parametrize("N,WH,fmt", [(1, (64, 64), 1), (2, (130, 70), 1), (3, (257, 129), 0), (5, (200, 200), 1)])
def test_compact_shards_assemble_to_the_frame(M, c1, N, WH, fmt):
    import torch
    W, H = WH
    cams = np.stack([look_at_camera(np.array([0.1, 0.05, -0.2]), target=np.zeros(3), W=W, H=H, fov_x_deg=60),
                     look_at_camera(np.array([-0.2, 0.1, 0.1]), target=np.zeros(3), W=W, H=H, fov_x_deg=75)])
    px = 4 if fmt == M.MERF_RGBA_U8 else 12
    dt = torch.uint8 if fmt == M.MERF_RGBA_U8 else torch.float32
    ch = 4 if fmt == M.MERF_RGBA_U8 else 3
    s = M.Scene(c1)
    full = torch.zeros((2, H, W, ch), dtype=dt, device="cuda")
    M.merf_render(s.handle, cams, W, H, full, fmt=fmt)
    slots = M.merf_shard_slots(W, H, N)
    assert slots == -(-((W + 63) // 64) * ((H + 63) // 64) // N)
    gathered = torch.zeros((N, 2, slots, 64, 64, ch), dtype=dt, device="cuda")
    for r in range(N):
        M.merf_render_shard_blocks(s.handle, cams, W, H, r, N, gathered[r], fmt=fmt)
    frame = torch.full((2, H, W, ch), 7, dtype=dt, device="cuda")
    M.merf_shard_assemble(gathered, 2, W, H, N, frame, fmt=fmt)
    torch.cuda.synchronize()
    assert torch.equal(frame, full)                  # byte for byte the unsharded frames
    # the compact buffer holds exactly the part's blocks at their slots
    own = M.shard_owner(W, H, N)
    g = gathered.cpu().numpy()
    f = full.cpu().numpy()
    nbx = (W + 63) // 64
    for r in range(N):
        for slot in range(slots):
            b = r + N * slot
            if b >= nbx * ((H + 63) // 64):
                continue
            by, bx = divmod(b, nbx)
            assert (own[by * 64:(by + 1) * 64, bx * 64:(bx + 1) * 64] == r).all()
            h, w = min(64, H - by * 64), min(64, W - bx * 64)
            assert np.array_equal(g[r, :, slot, :h, :w], f[:, by * 64:by * 64 + h, bx * 64:bx * 64 + w])
    with pytest.raises(M.MerfError):
        M.merf_render_shard_blocks(s.handle, cams, W, H, N, N, gathered[0], fmt=fmt)
    s.close()


def test_one_rank_nccl_gather_and_wait(M):
    import torch
    comm = M.Comm(M.merf_comm_unique_id(), 1, 0, 0)
    info = comm.info()
    assert info["n_ranks"] == 1 and info["rank"] == 0 and info["nccl_version"] > 0
    st = torch.cuda.Stream()
    local = torch.randint(0, 255, (3, 40, 50, 4), dtype=torch.uint8, device="cuda")
    root = torch.zeros((1,) + tuple(local.shape), dtype=torch.uint8, device="cuda")
    st.wait_stream(torch.cuda.current_stream())
    comm.gather(local, root, stream=st)
    comm.wait(stream=st, timeout_ms=60000)
    assert torch.equal(root[0], local)
    # argument errors
    with pytest.raises(M.MerfError) as e:
        comm.gather(local, root, root=1, stream=st)
    assert e.value.status == M.MERF_EINVAL
    comm.close()


def test_comm_wait_timeout_aborts(M):
    """A stream that does not finish within the timeout -> MERF_ENCCL, communicator aborted."""
    import torch
    comm = M.Comm(M.merf_comm_unique_id(), 1, 0, 0)
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        torch.cuda._sleep(int(2e9))                  # ~1 s of GPU spin on this stream
    with pytest.raises(M.MerfError) as e:
        comm.wait(stream=st, timeout_ms=20)
    assert e.value.status == M.MERF_ENCCL and "aborted" in str(e.value)
    local = torch.zeros(16, dtype=torch.uint8, device="cuda")
    with pytest.raises(M.MerfError):                 # unusable after the abort
        comm.gather(local, local, stream=st)
    torch.cuda.synchronize()
    comm.close()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _two_rank_worker(rank, port, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("gloo", rank=rank, world_size=2)
    import paper_2302_12249_b200 as M
    uid = [M.merf_comm_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    comm = M.Comm(uid[0], 2, rank, rank)
    sc = make_scene("c1")
    s = M.Scene(sc, device=rank)
    W, H = 200, 130
    cams = orbit_cameras(16, W=W, H=H, indices=[3])
    slots = M.merf_shard_slots(W, H, 2)
    mine = torch.zeros((1, slots, 64, 64, 4), dtype=torch.uint8, device="cuda")
    M.merf_render_shard_blocks(s.handle, cams, W, H, rank, 2, mine)
    root = torch.zeros((2, 1, slots, 64, 64, 4), dtype=torch.uint8, device="cuda") if rank == 0 else None
    comm.gather(mine, root)
    comm.wait(timeout_ms=60000)
    if rank == 0:
        frame = torch.zeros((1, H, W, 4), dtype=torch.uint8, device="cuda")
        M.merf_shard_assemble(root, 1, W, H, 2, frame)
        full = s.render(cams, W, H, fmt=M.MERF_RGBA_U8)
        torch.cuda.synchronize()
        q.put(bool(torch.equal(frame, full)))
    s.close()
    comm.close()
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_nccl_shard_gather():
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("needs two visible GPUs (the 1-rank NCCL path is tested above)")
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_two_rank_worker, args=(r, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    ok = q.get(timeout=300)
    for p in ps:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert ok


def test_bench_gather_path_one_rank():
    """bench.py's N > 1 pipeline (frames gathered to rank 0 through merf_gather_frames, the
    e2e leg timing render -> gather -> root D2H) run through a 1-rank communicator."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, "bench.py", "--force-gather", "--steps", "2", "--warmup", "3",
                          "--views", "2", "--no-cpu-baseline"], cwd=root, capture_output=True, text=True,
                         timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["gather"]["verified"] is True
    assert "merf_gather_frames" in line["e2e"]["path"] and line["e2e"]["value"] > 0
