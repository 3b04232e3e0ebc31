"""NEXT-4: asset ingestion -- the PNG bundle of a baked scene and camera files
(Sec. 5.3 "we encode textures as PNGs").  The library's own PNG
codec is checked against an independent one (Pillow) in both directions; round trips are
byte-exact; tampering is rejected; the SPEC's hand-placed occupancy bit-order fixture and
camera examples.  Host-only calls (no GPU) except the last test."""
import os
import re
import zlib

import numpy as np
import pytest

from merf_inputs import random_scene, pack_bits
from oracle import oracle as O

PIL = pytest.importorskip("PIL.Image")


@pytest.fixture(scope="module")
def M():
    import paper_2302_12249_b200 as M
    return M


def _scene():
    return random_scene(seed=3, L=16, R=32, level_res=(4, 8, 16))


def _rewrite(directory, name, data: bytes):
    """replace a payload and fix its manifest entry (size + CRC), as a legitimate tool would."""
    with open(os.path.join(directory, name), "wb") as f:
        f.write(data)
    man = open(os.path.join(directory, "manifest.txt")).read()
    man = re.sub(rf"^file {re.escape(name)} .*$", f"file {name} {len(data)} {zlib.crc32(data):08x}", man,
                 flags=re.M)
    open(os.path.join(directory, "manifest.txt"), "w").write(man)


def test_round_trip_is_byte_exact(M, tmp_path):
    sc = _scene()
    d = str(tmp_path / "b")
    M.merf_bundle_write(d, sc)
    rb = M.merf_bundle_read(d)
    assert (rb.L, rb.R, tuple(rb.level_res), rb.step, rb.source_mask) == (sc.L, sc.R, tuple(sc.level_res), sc.step,
                                                                          sc.source_mask)
    assert np.array_equal(rb.planes, sc.planes)
    assert np.array_equal(rb.atlas, sc.atlas)
    assert np.array_equal(rb.block_index, sc.block_index)
    assert np.array_equal(rb.occ_finest, np.asarray(sc.occ_finest, np.uint32))
    assert np.array_equal(rb.mlp, np.asarray(sc.mlp, np.float32))        # %.9g decimal is exact


def test_pngs_decode_with_an_independent_codec(M, tmp_path):
    sc = _scene()
    d = str(tmp_path / "b")
    M.merf_bundle_write(d, sc)
    for a in range(3):
        dens = np.asarray(PIL.open(os.path.join(d, f"plane{a}_density.png")))
        rgb = np.asarray(PIL.open(os.path.join(d, f"plane{a}_diffuse.png")))
        feat = np.asarray(PIL.open(os.path.join(d, f"plane{a}_features.png")))
        assert np.array_equal(dens, sc.planes[a, :, :, 0])
        assert np.array_equal(rgb, sc.planes[a, :, :, 1:4])
        assert np.array_equal(feat, sc.planes[a, :, :, 4:8])
    # atlas: Z-major stack of 9x9 slices, slice q = 9 b + z, 455 slices per raster row
    ras = np.concatenate([np.asarray(PIL.open(os.path.join(d, f"atlas_{k}.png"))).reshape(
        *np.asarray(PIL.open(os.path.join(d, f"atlas_{k}.png"))).shape[:2], -1)
        for k in ("density", "diffuse", "features")], axis=2)
    n = sc.atlas.shape[0]
    slices = sc.atlas.reshape(n * 9, 9, 9, 8)
    for q in range(n * 9):
        Y, X = (q // 455) * 9, (q % 455) * 9
        assert np.array_equal(ras[Y:Y + 9, X:X + 9], slices[q])


def test_reader_accepts_filtered_pngs_from_another_encoder(M, tmp_path):
    sc = _scene()
    d = str(tmp_path / "b")
    M.merf_bundle_write(d, sc)
    import io
    for name, arr in [("plane1_diffuse.png", sc.planes[1, :, :, 1:4]), ("plane2_features.png", sc.planes[2, :, :, 4:8]),
                      ("plane0_density.png", sc.planes[0, :, :, 0])]:
        buf = io.BytesIO()
        PIL.fromarray(np.ascontiguousarray(arr)).save(buf, format="PNG", optimize=True)   # adaptive filters
        _rewrite(d, name, buf.getvalue())
    rb = M.merf_bundle_read(d)
    assert np.array_equal(rb.planes, sc.planes)


@pytest.mark.parametrize("tamper,pattern", [
    ("dims", "size mismatch"), ("checksum", "checksum mismatch"), ("missing", "missing payload"),
    ("version", "version"), ("coarse", "max-pool")])
def test_tampered_bundles_are_rejected(M, tmp_path, tamper, pattern):
    sc = _scene()
    d = str(tmp_path / "b")
    M.merf_bundle_write(d, sc)
    man_p = os.path.join(d, "manifest.txt")
    man = open(man_p).read()
    if tamper == "dims":
        open(man_p, "w").write(re.sub(r"^R 32$", "R 64", man, flags=re.M))
    elif tamper == "checksum":
        p = os.path.join(d, "block_index.bin")
        b = bytearray(open(p, "rb").read())
        b[5] ^= 1
        open(p, "wb").write(bytes(b))
    elif tamper == "missing":
        os.remove(os.path.join(d, "atlas_diffuse.png"))
    elif tamper == "version":
        open(man_p, "w").write(man.replace("merf_bundle 1", "merf_bundle 2"))
    elif tamper == "coarse":
        b = bytearray(open(os.path.join(d, "occupancy0.bin"), "rb").read())
        b[0] ^= 1
        _rewrite(d, "occupancy0.bin", bytes(b))
    with pytest.raises(M.MerfError, match=pattern):
        M.merf_bundle_read(d)


def test_occupancy_bit_order_fixture(M, tmp_path):
    """bit k of byte n is cell 8n + k, x fastest: three hand-placed cells of a 4^3
    level -- (1,0,0) -> 1, (0,1,0) -> 4, (0,0,1) -> 16 -- give bytes 12 00 01 00 00 00 00 00."""
    sc = random_scene(seed=1, L=8, R=4, level_res=(2, 4))
    occ = np.zeros((4, 4, 4), bool)            # [z][y][x]
    occ[0, 0, 1] = occ[0, 1, 0] = occ[1, 0, 0] = True
    sc.occ_finest = pack_bits(occ)
    d = str(tmp_path / "b")
    M.merf_bundle_write(d, sc)
    assert open(os.path.join(d, "occupancy1.bin"), "rb").read() == bytes([0x12, 0, 0x01, 0, 0, 0, 0, 0])
    # level 0 (2^3) is their OR-pool: all three lie in cell (0,0,0) -> bit 0
    assert open(os.path.join(d, "occupancy0.bin"), "rb").read() == bytes([0x01])


def test_coarse_levels_equal_the_oracle_pyramid(M, tmp_path):
    sc = _scene()
    d = str(tmp_path / "b")
    M.merf_bundle_write(d, sc)
    levels = O.build_pyramid(np.asarray(sc.occ_finest, np.uint32), sc.level_res)
    for i, N in enumerate(sc.level_res):
        got = open(os.path.join(d, f"occupancy{i}.bin"), "rb").read()
        want = np.asarray(levels[i], np.uint32).view(np.uint8)[:(N ** 3 + 7) // 8].tobytes()
        assert got == want, i


def test_empty_scene_bundle(M, tmp_path):
    sc = _scene()
    sc.occ_finest = np.zeros_like(np.asarray(sc.occ_finest, np.uint32))
    d = str(tmp_path / "b")
    M.merf_bundle_write(d, sc)
    for i, N in enumerate(sc.level_res):
        b = open(os.path.join(d, f"occupancy{i}.bin"), "rb").read()
        assert len(b) == (N ** 3 + 7) // 8 and b == bytes(len(b))


def test_write_refuses_a_mismatched_payload(M, tmp_path):
    sc = _scene()
    sc.block_index = sc.block_index.copy()
    sc.block_index[3] = sc.atlas.shape[0]          # points past the atlas
    with pytest.raises(M.MerfError, match="MERF_EMISMATCH"):
        M.merf_bundle_write(str(tmp_path / "b"), sc)


CAM_OK = """# W H fx fy cx cy  c2w (3x4 row-major)  near far
2 2 100 100 1 1   1 0 0 0  0 1 0 0  0 0 1 0   0 10
"""


def test_cameras_identity_pose_rays(M, tmp_path):
    """SPEC example: identity pose, fx = fy = 100, 2x2 image -> 4 rays through pixel centres,
    centrally symmetric."""
    p = tmp_path / "cams.txt"
    p.write_text(CAM_OK + "\n")
    cams, w, h = M.merf_cameras_read(str(p))
    assert cams.shape == (1, 17) and w.tolist() == [2] and h.tolist() == [2]
    ds = np.array([O.raygen(cams[0], i, j)[1] for j in range(2) for i in range(2)])
    assert np.allclose(ds[0], -ds[3] * [1, 1, -1]) and np.allclose(ds[1], -ds[2] * [1, 1, -1])
    assert np.allclose(ds[0], np.array([-0.5, -0.5, 100]) / np.linalg.norm([-0.5, -0.5, 100]))


def test_cameras_empty_and_malformed(M, tmp_path):
    p = tmp_path / "c.txt"
    p.write_text("# nothing\n\n")
    cams, w, h = M.merf_cameras_read(str(p))
    assert cams.shape == (0, 17)
    p.write_text(CAM_OK + "2 2 100 100 1 1  1 0 0 0  0 2 0 0  0 0 1 0  0 10\n")
    with pytest.raises(M.MerfError, match="line 3.*orthonormal"):
        M.merf_cameras_read(str(p))
    p.write_text("2 2 100 100 1 1  1 0 0 0  0 1 0 0  0 0 1\n")
    with pytest.raises(M.MerfError, match="line 1: expected 20 numbers"):
        M.merf_cameras_read(str(p))
    p.write_text("2 2 100 100 1 1  1 0 0 0  0 1 0 0  0 0 1 0  5 5\n")
    with pytest.raises(M.MerfError, match="far > near"):
        M.merf_cameras_read(str(p))


@pytest.mark.gpu
def test_gpu_loaded_bundle_renders_identically(M, tmp_path, c1_scene):
    import torch
    from merf_inputs import config_cameras
    d = str(tmp_path / "c1")
    M.merf_bundle_write(d, c1_scene)
    cams, W, H = config_cameras("c1")
    a = M.Scene(c1_scene)
    b = M.Scene.load(d)
    ia, ib = a.info(), b.info()
    assert ia["n_blocks"] == ib["n_blocks"] and ia["device_bytes"] == ib["device_bytes"]
    ra, rb = a.render(cams, W, H), b.render(cams, W, H)
    torch.cuda.synchronize()
    assert torch.equal(ra, rb)
    a.close()
    b.close()
