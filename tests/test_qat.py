"""NEXT-3: quantisation-aware differentiable forward/backward (Eq. 7-8,
P:251-264).  CPU pins of the torch-fp64 oracle (quantiser examples S:155-156, idempotence
and error bound S:209, straight-through gradient S:525 in closed form, finite differences
with q = identity, forward == the C oracle's render of the baked bytes) and GPU parity of the
loss, image and gradients."""
import math

import numpy as np
import pytest
import torch

from merf_inputs import MerfScene, look_at_camera, pack_bits
from oracle import oracle as O
from oracle import qat as Q

L, R, N, STEP = 16, 32, 16, 2.0 ** -6
W = H = 8


def _toy(seed=0):
    rng = np.random.default_rng(seed)
    tv = rng.normal(0, 1.2, (L, L, L, 8))
    tv[..., 0] = rng.normal(0.4, 0.8, (L, L, L))
    tp = rng.normal(0, 1.0, (3, R, R, 8))
    tp[..., 0] = rng.normal(-0.2, 0.5, (3, R, R))
    occ = rng.random((N, N, N)) < 0.5
    mlp = rng.uniform(-0.3, 0.3, 883).astype(np.float32).astype(np.float64)
    cam = look_at_camera((0.2, 0.1, -1.6), target=(0, 0, 0), W=W, H=H, fov_x_deg=50)
    target = rng.uniform(0, 1, (W * H, 3))
    return tv, tp, pack_bits(occ), mlp, cam, target


def test_quantizer_examples_and_bounds():
    x = torch.tensor([0.0, 1.0, 0.3, 0.5], dtype=torch.float64)
    assert torch.allclose(Q.quantize(x), torch.tensor([0.0, 1.0, 77 / 255, 128 / 255], dtype=torch.float64),
                          atol=0, rtol=0)
    v = torch.rand(10000, dtype=torch.float64)
    assert torch.equal(Q.quantize(Q.quantize(v)), Q.quantize(v))
    assert (Q.quantize(v) - v).abs().max() <= 1 / 510 + 1e-15


def test_straight_through_gradient_closed_form():
    # d/dtheta sum(a * (2m q(sigma(theta)) - m)) = a * 2m sigma'(theta): q has gradient 1
    theta = torch.randn((50, 8), dtype=torch.float64, requires_grad=True)
    a = torch.randn((50, 8), dtype=torch.float64)
    (a * Q.stored_value(theta)).sum().backward()
    s = torch.sigmoid(theta.detach())
    assert torch.allclose(theta.grad, a * 2 * Q.M_CH * s * (1 - s), atol=1e-14)
    g_q = theta.grad.clone()
    theta.grad = None
    (a * Q.stored_value(theta, enable=False)).sum().backward()
    assert torch.equal(theta.grad, g_q)                      # same as q = identity


def test_forward_matches_renderer_on_baked_bytes():
    tv, tp, occ, mlp, cam, target = _toy(1)
    loss, rgb = Q.render_loss(torch.from_numpy(tv), torch.from_numpy(tp), torch.from_numpy(mlp), cam, W, H,
                              torch.from_numpy(target), occ, N, L, R, STEP)
    # bake: bytes = round(255 sigma(theta)); dense V as a fully stored block-sparse grid
    bv = np.floor(255 / (1 + np.exp(-tv)) + 0.5).astype(np.uint8)
    bp = np.floor(255 / (1 + np.exp(-tp)) + 0.5).astype(np.uint8)
    nb = L // 8
    atlas = np.empty((nb ** 3, 9, 9, 9, 8), np.uint8)
    for b in range(nb ** 3):
        bz, by, bx = b // (nb * nb), (b // nb) % nb, b % nb
        zz = np.minimum(np.arange(9) + 8 * bz, L - 1)
        yy = np.minimum(np.arange(9) + 8 * by, L - 1)
        xx = np.minimum(np.arange(9) + 8 * bx, L - 1)
        atlas[b] = bv[np.ix_(zz, yy, xx)]
    sc = MerfScene(L=L, R=R, level_res=(N,), step=STEP, planes=bp, block_index=np.arange(nb ** 3, dtype=np.int32),
                   atlas=atlas, occ_finest=occ, mlp=mlp)
    ref = O.render(O.OracleScene(sc), cam, W, H, mode="dense", flags=O.NO_EARLY_TERM)
    assert np.abs(rgb.detach().numpy() - ref["rgb"]).max() < 1e-12


def test_gradient_finite_differences_without_quantisation():
    tv, tp, occ, mlp, cam, target = _toy(2)
    pos = Q.sample_positions(cam, W, H, occ, N, STEP)
    tvt = torch.from_numpy(tv).requires_grad_(True)
    tpt = torch.from_numpy(tp).requires_grad_(True)
    args = (torch.from_numpy(mlp), cam, W, H, torch.from_numpy(target), occ, N, L, R, STEP)
    loss, _ = Q.render_loss(tvt, tpt, *args, quant=False, positions=pos)
    loss.backward()
    gv, gp = tvt.grad.numpy(), tpt.grad.numpy()
    rng = np.random.default_rng(0)
    big = np.argsort(-np.abs(gv).ravel())[:6]
    for flat in list(big) + list(rng.integers(0, gv.size, 4)):
        e = np.zeros(gv.size)
        e[flat] = 1e-6
        lp, _ = Q.render_loss(torch.from_numpy(tv + e.reshape(tv.shape)), torch.from_numpy(tp), *args, quant=False, positions=pos)
        lm, _ = Q.render_loss(torch.from_numpy(tv - e.reshape(tv.shape)), torch.from_numpy(tp), *args, quant=False, positions=pos)
        fd = (lp.item() - lm.item()) / 2e-6
        assert abs(fd - gv.ravel()[flat]) < 1e-6 * max(1.0, abs(fd)), flat
    flat = int(np.argmax(np.abs(gp)))
    e = np.zeros(gp.size)
    e[flat] = 1e-6
    lp, _ = Q.render_loss(torch.from_numpy(tv), torch.from_numpy(tp + e.reshape(tp.shape)), *args, quant=False, positions=pos)
    lm, _ = Q.render_loss(torch.from_numpy(tv), torch.from_numpy(tp - e.reshape(tp.shape)), *args, quant=False, positions=pos)
    assert abs((lp.item() - lm.item()) / 2e-6 - gp.ravel()[flat]) < 1e-6 * max(1.0, abs(gp.ravel()[flat]))


# ---------------------------------------------------------------------------------------
# GPU parity: merf_qat_step (C-ABI) vs the fp64 autograd oracle on the same seeded inputs
# ---------------------------------------------------------------------------------------
def _gpu_case(seed, W_, H_, n_views=1, Lc=L, Rc=R):
    """float32-representable parameters (the GPU takes float32), ragged tiles when W_, H_ are
    not multiples of 8 x 4."""
    rng = np.random.default_rng(seed)
    tv = rng.normal(0, 1.2, (Lc, Lc, Lc, 8)).astype(np.float32)
    tv[..., 0] = rng.normal(0.4, 0.8, (Lc, Lc, Lc))
    tp = rng.normal(0, 1.0, (3, Rc, Rc, 8)).astype(np.float32)
    tp[..., 0] = rng.normal(-0.2, 0.5, (3, Rc, Rc))
    occ = rng.random((N, N, N)) < 0.6
    mlp = rng.uniform(-0.3, 0.3, 883).astype(np.float32)
    cams = [look_at_camera((0.2 + 0.5 * v, 0.1, -1.6 + 0.3 * v), target=(0, 0, 0), W=W_, H=H_, fov_x_deg=50)
            for v in range(n_views)]
    target = rng.uniform(0, 1, (n_views, H_ * W_, 3)).astype(np.float32)
    return tv, tp, pack_bits(occ), mlp, cams, target


def _oracle(tv, tp, occ, mlp, cams, target, W_, H_, quant, Lc=L, Rc=R):
    tvt = torch.from_numpy(tv.astype(np.float64)).requires_grad_(True)
    tpt = torch.from_numpy(tp.astype(np.float64)).requires_grad_(True)
    total, rgbs = 0.0, []
    for v, cam in enumerate(cams):
        loss, rgb = Q.render_loss(tvt, tpt, torch.from_numpy(mlp.astype(np.float64)), cam, W_, H_,
                                  torch.from_numpy(target[v].astype(np.float64)), occ, N, Lc, Rc, STEP, quant=quant)
        total = total + loss
        rgbs.append(rgb.detach().numpy())
    total.backward()
    return total.item(), np.stack(rgbs), tvt.grad.numpy(), tpt.grad.numpy()


def _gpu(M, tv, tp, occ, mlp, cams, target, W_, H_, quant, max_samples=1024):
    dev = "cuda"
    t = lambda a: torch.as_tensor(a).to(dev)
    tvd, tpd = t(tv), t(tp)
    rgb = torch.empty((len(cams), H_, W_, 3), dtype=torch.float32, device=dev)
    gv, gp = torch.full_like(tvd, float("nan")), torch.full_like(tpd, float("nan"))
    loss = torch.empty(1, dtype=torch.float64, device=dev)
    ovf = torch.empty(1, dtype=torch.int32, device=dev)
    ns = torch.empty(1, dtype=torch.int64, device=dev)
    M.merf_qat_step(tvd, tpd, t(occ), N, t(mlp), cams, W_, H_, t(target), rgb, gv, gp, loss, STEP,
                    quantize=quant, max_samples=max_samples, overflow=ovf, n_samples=ns)
    torch.cuda.synchronize()
    _gpu.n_samples = int(ns.item())
    return loss.item(), rgb.reshape(len(cams), -1, 3).cpu().numpy(), gv.cpu().numpy(), gp.cpu().numpy(), int(ovf.item())


@pytest.fixture(scope="module")
def M():
    assert torch.cuda.is_available()
    import paper_2302_12249_b200 as M
    return M


def _close(got, ref, rel):
    scale = max(np.abs(ref).max(), 1e-30)
    err = np.abs(got - ref).max()
    assert err <= rel * scale, (err, scale)


@pytest.mark.gpu
@pytest.mark.parametrize("quant", [True, False])
@pytest.mark.parametrize("shape", [(20, 13, 1), (8, 8, 2)])
def test_gpu_qat_parity(M, quant, shape):
    W_, H_, nv = shape
    case = _gpu_case(11 + W_, W_, H_, nv)
    l_ref, rgb_ref, gv_ref, gp_ref = _oracle(*case, W_, H_, quant)
    l_got, rgb_got, gv_got, gp_got, ovf = _gpu(M, *case, W_, H_, quant)
    assert ovf == 0
    # the sample set is integer work: identical count (readings D5-D8)
    assert _gpu.n_samples == sum(len(Q.sample_positions(c, W_, H_, case[2], N, STEP)[0]) for c in case[4])
    assert np.abs(rgb_got - rgb_ref).max() <= 1e-4
    assert abs(l_got - l_ref) <= 1e-4 * max(1.0, l_ref)
    assert np.isfinite(gv_got).all() and np.isfinite(gp_got).all()
    _close(gv_got, gv_ref, 2e-3)
    _close(gp_got, gp_ref, 2e-3)
    # the support of the gradient is the same set of grid elements
    assert np.array_equal(np.abs(gv_ref) > 1e-3 * np.abs(gv_ref).max(),
                          np.abs(gv_got) > 1e-3 * np.abs(gv_ref).max()) or \
        (np.abs(gv_got - gv_ref) <= 2e-3 * np.abs(gv_ref).max()).all()


@pytest.mark.gpu
def test_gpu_qat_overflow_drops_only_gradients(M):
    W_, H_ = 8, 8
    case = _gpu_case(5, W_, H_)
    l_full, rgb_full, gv_full, _, o_full = _gpu(M, *case, W_, H_, True)
    l_cut, rgb_cut, gv_cut, _, o_cut = _gpu(M, *case, W_, H_, True, max_samples=4)
    assert o_full == 0 and o_cut > 0
    # images identical; the loss is a sum of fp64 atomics (order-dependent at 1 ulp)
    assert np.array_equal(rgb_full, rgb_cut) and abs(l_full - l_cut) <= 1e-12 * abs(l_full)
    assert np.abs(gv_cut).sum() < np.abs(gv_full).sum()


@pytest.mark.gpu
def test_gpu_qat_descent_lowers_baked_loss(M):
    """QAT as a training loop: gradient steps on theta lower the loss of the quantised render
    towards a target rendered from other parameters (the point of Eq. 7-8)."""
    W_, H_ = 16, 16
    tv, tp, occ, mlp, cams, _ = _gpu_case(3, W_, H_)
    tv2, tp2, _, _, _, _ = _gpu_case(4, W_, H_)
    _, tgt, _, _, _ = _gpu(M, tv2, tp2, occ, mlp, cams, np.zeros((1, W_ * H_, 3), np.float32), W_, H_, True)
    losses = []
    for _ in range(30):
        l, _, gv, gp, _ = _gpu(M, tv, tp, occ, mlp, cams, tgt.astype(np.float32), W_, H_, True)
        losses.append(l)
        s = 0.3 / max(np.abs(gv).max(), np.abs(gp).max())      # normalised step (oracle run: 48 -> 9.5)
        tv = (tv - s * gv).astype(np.float32)
        tp = (tp - s * gp).astype(np.float32)
    assert losses[-1] < 0.5 * losses[0], losses


@pytest.mark.gpu
def test_gpu_qat_argument_errors(M):
    case = _gpu_case(1, 8, 8)
    with pytest.raises(M.MerfError):
        _gpu(M, *case, 8, 8, True, max_samples=0)
    tv, tp, occ, mlp, cams, target = case
    with pytest.raises(M.MerfError):       # L not a power of two
        _gpu(M, tv[:12, :12, :12].copy(), tp, occ, mlp, cams, target, 8, 8, True)
