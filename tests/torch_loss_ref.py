"""Plain PyTorch (autograd) reference of the training-step image glue —
TEST INFRASTRUCTURE: the numerics reference the CUDA loss kernels (K10/K11,
csrc/tsb_train.cu) are checked against. It restates texsplat losses.py
(L1 + D-SSIM, depth-derived normals, smoothness) and the compute_step chain
(training.py:143-172); autograd provides the adjoints the reference writes
by hand."""
import math

import numpy as np
import torch
import torch.nn.functional as F

from paper_2506_13348_b200.training import LossWeights  # noqa: F401

DISPLAY_GAMMA = 2.2
DISPLAY_TOE = 1e-4
SSIM_C1 = 0.01 ** 2
SSIM_C2 = 0.03 ** 2
REG_COVER_ALPHA = 0.5
PSNR_CAP = 99.0


def linear_to_display(x: torch.Tensor) -> torch.Tensor:
    """Gamma 2.2 with a slope-matched linear toe below 1e-4 (losses.py:40-46)."""
    p = 1.0 / DISPLAY_GAMMA
    toe_slope = DISPLAY_TOE ** (p - 1.0)
    return torch.where(x >= DISPLAY_TOE, x.clamp_min(DISPLAY_TOE) ** p,
                       toe_slope * x.clamp_min(0.0))


def _gauss_window(device, dtype):
    x = torch.arange(-5, 6, dtype=torch.float64)
    w = torch.exp(-0.5 * (x / 1.5) ** 2)
    return (w / w.sum()).to(device=device, dtype=dtype)


def _blur(img: torch.Tensor, w: torch.Tensor) -> torch.Tensor:
    """Separable 11-tap Gaussian, zero padding, per channel; img (H, W, C)."""
    C = img.shape[2]
    x = img.permute(2, 0, 1).unsqueeze(0)  # 1, C, H, W
    kx = w.view(1, 1, 1, 11).repeat(C, 1, 1, 1)
    ky = w.view(1, 1, 11, 1).repeat(C, 1, 1, 1)
    x = F.conv2d(x, ky, padding=(5, 0), groups=C)
    x = F.conv2d(x, kx, padding=(0, 5), groups=C)
    return x.squeeze(0).permute(1, 2, 0)


def ssim(a: torch.Tensor, b: torch.Tensor) -> torch.Tensor:
    """Mean SSIM (losses.py:61-96)."""
    w = _gauss_window(a.device, a.dtype)
    mu_a, mu_b = _blur(a, w), _blur(b, w)
    saa = _blur(a * a, w) - mu_a * mu_a
    sbb = _blur(b * b, w) - mu_b * mu_b
    sab = _blur(a * b, w) - mu_a * mu_b
    m = ((2.0 * mu_a * mu_b + SSIM_C1) * (2.0 * sab + SSIM_C2)) / (
        (mu_a * mu_a + mu_b * mu_b + SSIM_C1) * (saa + sbb + SSIM_C2))
    return m.mean()


def image_loss(pred: torch.Tensor, target: torch.Tensor, dssim_weight: float = 0.2):
    """(1-w) L1 + w (1-SSIM)/2 in display space (losses.py:120-134)."""
    l1 = (pred - target).abs().mean()
    return (1.0 - dssim_weight) * l1 + dssim_weight * 0.5 * (1.0 - ssim(pred, target))


def psnr(a: torch.Tensor, b: torch.Tensor) -> float:
    mse = float(((a.clamp(0, 1) - b.clamp(0, 1)) ** 2).mean())
    if mse <= 10.0 ** (-PSNR_CAP / 10.0):
        return PSNR_CAP
    return float(10.0 * math.log10(1.0 / mse))


def depth_to_normal(depth: torch.Tensor, camera, cover: torch.Tensor):
    """World normals from forward differences of back-projected depth
    (losses.py:147-180); returns (normals (H, W, 3), ok (H, W))."""
    H, W = depth.shape
    dev, dt = depth.device, depth.dtype
    xs = (torch.arange(W, dtype=torch.float64) + 0.5 - camera.cx) / camera.fx
    ys = (torch.arange(H, dtype=torch.float64) + 0.5 - camera.cy) / camera.fy
    xs, ys = xs.to(dev, dt), ys.to(dev, dt)
    px = torch.stack([xs[None, :] * depth, ys[:, None] * depth, depth], dim=-1)
    dx = px[:, 1:] - px[:, :-1]
    dy = px[1:] - px[:-1]
    n_view = torch.zeros((H, W, 3), device=dev, dtype=dt)
    n_view = n_view.clone()
    n_view[:-1, :-1] = torch.linalg.cross(dx[:-1], dy[:, :-1], dim=-1)
    valid = torch.zeros((H, W), dtype=torch.bool, device=dev)
    valid[:-1, :-1] = cover[:-1, :-1] & cover[:-1, 1:] & cover[1:, :-1]
    flip = (n_view * px).sum(-1) > 0.0
    n_view = torch.where(flip[..., None], -n_view, n_view)
    mag = torch.linalg.norm(n_view, dim=-1, keepdim=True)
    ok = valid & (mag[..., 0] > 1e-12)
    unit = torch.where(ok[..., None], n_view / mag.clamp_min(1e-30), torch.zeros_like(n_view))
    R = torch.as_tensor(np.asarray(camera.world_to_view, np.float64)[:3, :3], device=dev, dtype=dt)
    return unit @ R, ok


def _normal_image(nb: torch.Tensor):
    mag = torch.linalg.norm(nb, dim=-1, keepdim=True)
    ok = mag[..., 0] > 1e-12
    return torch.where(ok[..., None], nb / mag.clamp_min(1e-30), torch.zeros_like(nb)), ok


def smoothness_loss(n_img, target, valid):
    """Edge-aware normal smoothness (losses.py:240-277)."""
    dx = n_img[:, 1:] - n_img[:, :-1]
    dy = n_img[1:] - n_img[:-1]
    vx = valid[:, 1:] & valid[:, :-1]
    vy = valid[1:] & valid[:-1]
    wx = torch.exp(-torch.linalg.norm(target[:, 1:] - target[:, :-1], dim=-1)) * vx
    wy = torch.exp(-torch.linalg.norm(target[1:] - target[:-1], dim=-1)) * vy
    count = max(int(vx.sum() + vy.sum()), 1)
    mx = torch.where(vx, _safe_norm(dx), torch.zeros_like(wx))
    my = torch.where(vy, _safe_norm(dy), torch.zeros_like(wy))
    return (wx * mx).sum() / count + (wy * my).sum() / count


def _safe_norm(v):
    """||v|| with zero gradient at v = 0 (losses.py:268-271)."""
    sq = (v * v).sum(-1)
    nz = sq > 1e-24
    return torch.where(nz, torch.sqrt(torch.where(nz, sq, torch.ones_like(sq))),
                       torch.zeros_like(sq))


def loss_and_grads(color: torch.Tensor, planar: torch.Tensor, target: torch.Tensor, camera,
                   weights: LossWeights):
    """Loss terms and their gradients w.r.t. the shaded colour and the
    G-buffer (regularisers). Mirrors training.py:143-172."""
    color = color.detach().requires_grad_(True)
    gp = planar.detach().requires_grad_(True)
    disp = linear_to_display(color)
    l_img = image_loss(disp, target, weights.dssim)
    l_normal = torch.zeros((), device=color.device, dtype=color.dtype)
    l_smooth = torch.zeros((), device=color.device, dtype=color.dtype)
    if weights.normal > 0.0 or weights.smooth > 0.0:
        alpha = gp[12]
        cover = alpha > REG_COVER_ALPHA
        n_img, n_ok = _normal_image(gp[5:8].permute(1, 2, 0))
        zbar = torch.where(cover, gp[11] / alpha.clamp_min(1e-30), torch.zeros_like(alpha))
        if weights.normal > 0.0:
            n_ref, d_ok = depth_to_normal(zbar, camera, cover)
            valid = n_ok & d_ok & cover
            cnt = max(int(valid.sum()), 1)
            dots = (n_img * n_ref).sum(-1)
            l_normal = torch.where(valid, 1.0 - dots, torch.zeros_like(dots)).sum() / cnt
        if weights.smooth > 0.0:
            l_smooth = smoothness_loss(n_img, target, n_ok & cover)
    loss = l_img + weights.normal * l_normal + weights.smooth * l_smooth
    loss.backward()
    terms = {"loss": float(loss.detach()), "image": float(l_img.detach()),
             "normal": float(l_normal.detach()), "smooth": float(l_smooth.detach()),
             "psnr": psnr(disp.detach(), target)}
    dg = gp.grad if gp.grad is not None else torch.zeros_like(planar)
    return terms, color.grad, dg


