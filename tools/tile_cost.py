"""Per-tile cost of the march on one 1080p orbit view (what makes the persistent march's
tail): evaluated samples per ray from merf_trace (max_per_ray 1: counts only) grouped into the
march's 8x4-pixel tiles, the distribution of the per-tile maximum (a warp marches its 32 rays
in lockstep, so the tile lasts as long as its longest ray), and how well the setup kernel's
cost estimate (two finest-level probes per segment at K/4 and 3K/4) ranks the tiles.

  python tools/tile_cost.py [--view 0]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--view", type=int, default=0)
    a = ap.parse_args()
    import numpy as np
    import torch
    from merf_inputs import make_scene, orbit_cameras, unpack_bits
    import paper_2302_12249_b200 as M
    W, H = 1920, 1080
    sc = make_scene("c2")
    s = M.Scene(sc)
    cam = orbit_cameras(256, indices=[a.view])[0]
    # pixels in the march's tile order: tiles of 8x4 row-major, lanes row-major in the tile
    tx, ty = W // 8, (H + 3) // 4
    t = np.arange(tx * ty)
    lane = np.arange(32)
    px = (t[:, None] % tx) * 8 + lane[None, :] % 8
    py = (t[:, None] // tx) * 4 + lane[None, :] // 8
    valid = py < H
    pid = np.where(valid, py * W + px, 0).astype(np.int64).ravel()
    n = len(pid)
    cells = torch.zeros((n, 1), dtype=torch.int64, device="cuda")
    T = torch.zeros((n, 1), dtype=torch.float32, device="cuda")
    cnt = torch.zeros(n, dtype=torch.int32, device="cuda")
    M.merf_trace(s.handle, cam, W, torch.as_tensor(pid, device="cuda"), 1, cells, T, cnt)
    seg = torch.zeros(n * 8 * M.merf.SEGMENT_DTYPE.itemsize, dtype=torch.uint8, device="cuda")
    scnt = torch.zeros(n, dtype=torch.int32, device="cuda")
    M.merf_segments(s.handle, cam, W, torch.as_tensor(pid, device="cuda"), 8, seg, scnt)
    torch.cuda.synchronize()
    ev = cnt.cpu().numpy().reshape(-1, 32) * valid
    segs = seg.cpu().numpy().view(M.merf.SEGMENT_DTYPE).reshape(n, 8)
    scnt = scnt.cpu().numpy()
    N = sc.level_res[-1]
    occ = unpack_bits(sc.occ_finest, N).astype(bool)
    F = 28
    sf = F + 2 - int(np.log2(N))
    est = np.zeros(n, np.int64)
    for j in range(8):
        live = scnt > j
        Qa = segs["Qa"][:, j].astype(np.int64) + (1 << (F + 1))
        U = segs["U"][:, j].astype(np.int64)
        K = segs["K"][:, j].astype(np.int64)
        for kk in (K >> 2, (3 * K) >> 2):
            Q = Qa + kk[:, None] * U
            c = np.clip(Q >> sf, 0, N - 1)
            o = occ[c[:, 2], c[:, 1], c[:, 0]]
            est += np.where(live & o, (K + 1) >> 1, 0)
    est_t = est.reshape(-1, 32).sum(1) // 32
    # candidate estimate 2: the tile's centre ray (lane 20) probed at 64 points spread over its
    # lattice samples: occupied probes counted until the optical depth accumulated from a
    # nearest-texel density estimate passes ln(5000) (where termination would cut the ray)
    c = np.arange(len(est_t)) * 32 + 20
    ns = scnt[c]
    Ks = segs["K"][c].astype(np.int64) * (np.arange(8)[None, :] < ns[:, None])
    Ktot = Ks.sum(1)
    cum = np.cumsum(Ks, 1)
    P = 64
    kg = ((np.arange(P)[None, :] + 0.5) / P * Ktot[:, None]).astype(np.int64)          # global index
    js = np.minimum((kg[:, :, None] >= cum[:, None, :]).sum(2), 7)
    start = np.take_along_axis(np.concatenate([np.zeros((len(c), 1), np.int64), cum[:, :-1]], 1), js, 1)
    kl = kg - start
    Qa = np.take_along_axis(segs["Qa"][c].astype(np.int64), js[:, :, None].repeat(3, 2), 1) + (1 << (F + 1))
    Uu = np.take_along_axis(segs["U"][c].astype(np.int64), js[:, :, None].repeat(3, 2), 1)
    Q = Qa + kl[:, :, None] * Uu
    cc = np.clip(Q >> sf, 0, N - 1)
    o2 = occ[cc[..., 2], cc[..., 1], cc[..., 0]]
    # nearest-texel density: V (dense lookup through the block index) + three planes
    L, R = sc.L, sc.R
    sV, sP = F + 2 - int(np.log2(L)), F + 2 - int(np.log2(R))
    iv = np.clip(Q >> sV, 0, L - 1)
    nb = L // 8
    slot = ((iv[..., 2] >> 3) * nb + (iv[..., 1] >> 3)) * nb + (iv[..., 0] >> 3)
    blk = sc.block_index[slot]
    bv = np.where(blk >= 0, sc.atlas[np.maximum(blk, 0), iv[..., 2] & 7, iv[..., 1] & 7, iv[..., 0] & 7, 0], 0)
    ip = np.clip(Q >> sP, 0, R - 1)
    bp = (sc.planes[0, ip[..., 2], ip[..., 1], 0].astype(np.int64) + sc.planes[1, ip[..., 2], ip[..., 0], 0]
          + sc.planes[2, ip[..., 1], ip[..., 0], 0])
    t0 = (2 * 14.0 / 255) * (bv + bp) - 4 * 14.0
    od = np.where(o2, np.exp(t0) * sc.step * (Ktot[:, None] / P), 0.0)
    before = np.cumsum(od, 1) - od < np.log(5000.0)
    est2 = ((o2 & before).sum(1) * Ktot / P).astype(np.int64)
    mx = ev.max(1)
    mean = ev.sum(1) / np.maximum(valid.sum(1), 1)
    order = np.argsort(-est_t, kind="stable")
    rk_est = np.empty(len(est_t)); rk_est[order] = np.arange(len(est_t))
    rk_mx = np.empty(len(mx)); rk_mx[np.argsort(-mx, kind="stable")] = np.arange(len(mx))
    spearman = float(np.corrcoef(rk_est, rk_mx)[0, 1])
    rk2 = np.empty(len(est2)); rk2[np.argsort(-est2, kind="stable")] = np.arange(len(est2))
    spearman2 = float(np.corrcoef(rk2, rk_mx)[0, 1])
    heavy = mx >= np.percentile(mx, 99)
    b1 = np.minimum(7, np.floor(np.log2(est_t + 1))).astype(int)
    b2 = np.minimum(7, np.floor(np.log2(est2 + 1))).astype(int)
    top = np.argsort(-mx)[:10]
    out = {"tiles": int(len(mx)), "max_eval_per_tile_pct": {p: float(np.percentile(mx, p)) for p in (50, 90, 99, 99.9, 100)},
           "mean_eval_per_tile_pct": {p: float(np.percentile(mean, p)) for p in (50, 90, 99, 100)},
           "lockstep_waste": float(1 - ev.sum() / (mx * 32).sum()),
           "spearman_est_vs_max": spearman, "spearman_est2_vs_max": spearman2,
           "heavy_tiles_bucket_hist_est1": np.bincount(b1[heavy], minlength=8).tolist(),
           "heavy_tiles_bucket_hist_est2": np.bincount(b2[heavy], minlength=8).tolist(),
           "all_tiles_bucket_hist_est2": np.bincount(b2, minlength=8).tolist(),
           "all_tiles_bucket_hist_est1": np.bincount(b1, minlength=8).tolist(),
           "top_tiles": [{"tile": int(i), "tx": int(i % tx), "ty": int(i // tx), "max": int(mx[i]), "mean": float(mean[i]),
                          "est": int(est_t[i]), "est2": int(est2[i])} for i in top]}
    print(json.dumps(out, indent=1))
    s.close()


if __name__ == "__main__":
    main()
