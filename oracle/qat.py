"""NEXT-3 oracle: quantisation-aware, differentiable forward/backward of the MERF render path
on toy dense grids (Sec. 5.2, Eq. 7-8), in plain PyTorch fp64 with
autograd.  TEST INFRASTRUCTURE ONLY (imported by tests/).

Continuous parameters theta (pre-sigmoid) live on a dense L^3 grid V and three R^2 planes,
C = 8 channels.  The value stored for training is Eq. 7:
    t' = 2m q(sigma(theta)) - m,   q(x) = x + stopgrad(floor(255 x + 1/2)/255 - x)   (Eq. 8)
i.e. the byte the baker would write, decoded (D13), with a straight-through gradient.
Samples: the renderer's lattice (readings D5-D8) restricted to cells of the finest occupancy
level, every sample (dense mode, no early termination) -- positions come from the C oracle's
segment setup.  Field (Eq. 5, cell-centred texels D9), decode (Eq. 6), composite (Eq. 1-2),
deferred MLP (Eq. 3, fixed weights), C = clamp(C_d + h, 0, 1); loss = sum (C - C*)^2.
"""
from __future__ import annotations

import numpy as np
import torch

from . import oracle as O

M_CH = torch.tensor([14.0] + [7.0] * 7, dtype=torch.float64)


def quantize(x, enable: bool = True):
    """q of Eq. 8: round to 1/255 in the forward pass, identity gradient (STE)."""
    if not enable:
        return x
    return x + (torch.floor(255.0 * x + 0.5) / 255.0 - x).detach()


def stored_value(theta, enable: bool = True):
    """Eq. 7: 2m q(sigma(theta)) - m per channel (channel axis last)."""
    return 2.0 * M_CH * quantize(torch.sigmoid(theta), enable) - M_CH


def sample_positions(cam, W: int, H: int, occ_finest, N: int, step: float):
    """lattice points Q [n_samples, 3] (int64) of every pixel's rays in occupied finest cells,
    with the pixel index of each sample, in march order (D5-D8, dense mode)."""
    F = O.F_BITS
    qs, owner = [], []
    occ = np.unpackbits(np.ascontiguousarray(occ_finest, "<u4").view(np.uint8), bitorder="little")
    s = F + 2 - int(np.log2(N))
    for p in range(W * H):
        o, d = O.raygen(cam, p % W, p // W)
        for seg in O.segment_ray(o, d, cam[16], step):
            k = np.arange(seg["K"], dtype=np.int64)
            Q = seg["Qa"][None, :] + k[:, None] * seg["U"][None, :]
            c = np.clip((Q + (1 << (F + 1))) >> s, 0, N - 1)
            on = occ[(c[:, 2] * N + c[:, 1]) * N + c[:, 0]].astype(bool)
            qs.append(Q[on])
            owner.append(np.full(int(on.sum()), p, np.int64))
    return np.concatenate(qs), np.concatenate(owner)


def _coord(Q, M: int):
    """lower texel index and fraction (cell-centred, clamp to edge: i0 in [0, M-2])."""
    F = O.F_BITS
    s = F + 2 - int(np.log2(M))
    P = Q + (1 << (F + 1)) - (1 << (s - 1))
    i = P >> s
    f = (P - (i << s)).astype(np.float64) / float(1 << s)
    lo = i < 0
    hi = i > M - 2
    i = np.where(lo, 0, np.where(hi, M - 2, i))
    f = np.where(lo, 0.0, np.where(hi, 1.0, f))
    return i, torch.from_numpy(f)


def field(theta_v, theta_p, Q, L: int, R: int, quant: bool = True):
    """t [n, 8] at lattice points Q (Eq. 5 on the stored values of Eq. 7)."""
    vv = stored_value(theta_v, quant).reshape(-1, 8)            # [L^3, 8]
    t = torch.zeros((len(Q), 8), dtype=torch.float64)
    ix = [_coord(Q[:, a], L) for a in range(3)]
    for dz in (0, 1):
        for dy in (0, 1):
            for dx in (0, 1):
                w = ((ix[0][1] if dx else 1 - ix[0][1]) * (ix[1][1] if dy else 1 - ix[1][1])
                     * (ix[2][1] if dz else 1 - ix[2][1]))
                idx = ((ix[2][0] + dz) * L + (ix[1][0] + dy)) * L + (ix[0][0] + dx)
                t = t + w[:, None] * vv[torch.from_numpy(idx)]
    pv = stored_value(theta_p, quant).reshape(3, -1, 8)         # [3, R^2, 8]
    pc = [_coord(Q[:, a], R) for a in range(3)]
    for a, (ua, va) in enumerate([(1, 2), (0, 2), (0, 1)]):
        (iu, fu), (iv, fv) = pc[ua], pc[va]
        for dv in (0, 1):
            for du in (0, 1):
                w = (fu if du else 1 - fu) * (fv if dv else 1 - fv)
                idx = (iv + dv) * R + (iu + du)
                t = t + w[:, None] * pv[a][torch.from_numpy(idx)]
    return t


def mlp(w, x):
    """deferred MLP h (Eq. 3; readings D16-D17) on x [n, 34]."""
    W0, b0 = w[:544].reshape(16, 34), w[544:560]
    W1, b1 = w[560:816].reshape(16, 16), w[816:832]
    W2, b2 = w[832:880].reshape(3, 16), w[880:883]
    h0 = torch.relu(x @ W0.T + b0)
    h1 = torch.relu(h0 @ W1.T + b1)
    return torch.sigmoid(h1 @ W2.T + b2)


def encode_dir(d):
    cols = [d]
    for j in range(3):
        for k in range(4):
            a = d[:, j:j + 1] * (2.0 ** k)
            cols += [torch.sin(a), torch.cos(a)]
    return torch.cat(cols, 1)


def render_loss(theta_v, theta_p, mlp_w, cam, W: int, H: int, target, occ_finest, N: int, L: int,
                R: int, step: float, quant: bool = True, positions=None):
    """(loss, rgb [W*H, 3]) of the QAT forward pass; differentiable in theta_v, theta_p."""
    Q, owner = positions if positions is not None else sample_positions(cam, W, H, occ_finest, N, step)
    t = field(theta_v, theta_p, Q, L, R, quant)
    tau = torch.exp(t[:, 0])
    alpha = 1.0 - torch.exp(-tau * step)
    x = torch.sigmoid(t[:, 1:])                                  # c_d (3), f (4)
    npix = W * H
    counts = np.bincount(owner, minlength=npix)
    S = int(counts.max()) if len(counts) else 0
    # pad per-pixel sample runs (owner is sorted by march order within each pixel)
    start = np.concatenate([[0], np.cumsum(counts)[:-1]])
    slot = np.arange(len(owner)) - start[owner]
    A = torch.zeros((npix, max(S, 1)), dtype=torch.float64)
    X = torch.zeros((npix, max(S, 1), 7), dtype=torch.float64)
    A = A.index_put((torch.from_numpy(owner), torch.from_numpy(slot)), alpha)
    X = X.index_put((torch.from_numpy(owner), torch.from_numpy(slot)), x)
    one_minus = 1.0 - A
    T = torch.cumprod(torch.cat([torch.ones((npix, 1), dtype=torch.float64), one_minus[:, :-1]], 1), 1)
    wgt = A * T
    acc = (wgt[:, :, None] * X).sum(1)                           # [npix, 7] = C_d, F
    d = torch.from_numpy(np.stack([O.raygen(cam, p % W, p // W)[1] for p in range(npix)]))
    h = mlp(mlp_w, torch.cat([acc, encode_dir(d)], 1))
    rgb = torch.clamp(acc[:, :3] + h, 0.0, 1.0)
    loss = ((rgb - target) ** 2).sum()
    return loss, rgb
