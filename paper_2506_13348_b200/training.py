"""Training step (BASELINE configs[3]) on the B200 render path.

compute_step mirrors texsplat.training.compute_step (training.py:130-184):
forward with tape, deferred shading, display transform, L1 + D-SSIM image
loss, normal-consistency and smoothness regularisers, shading adjoint and
splat adjoint. The hot path (K1-K9) is libtsb; the image-space glue (display
transform, SSIM, regularisers; losses.py:24-277) is small dense image math
and runs as torch ops on the GPU with autograd providing the same adjoints
the reference writes by hand.

DataParallelTrainer: one process per GPU, each rank renders its own view,
gradients are flattened into one float32 buffer and summed with a single
NCCL all-reduce over NVLink (torch.distributed), then averaged and applied
with Adam (training.py:69-100) on the device. SURVEY.md §8(e).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import torch
import torch.nn.functional as F

from .backward import SceneGrads, shade_backward, splat_backward
from .device import DeviceAtlas, DeviceEnvironment, DeviceScene, FrameWorkspace
from .rasterize import PreparedScene, prepare, render_prepared
from .shading import ShadeResult, shade_planar

DISPLAY_GAMMA = 2.2
DISPLAY_TOE = 1e-4
SSIM_C1 = 0.01 ** 2
SSIM_C2 = 0.03 ** 2
REG_COVER_ALPHA = 0.5
PSNR_CAP = 99.0


@dataclass
class LossWeights:
    dssim: float = 0.2
    normal: float = 0.05
    smooth: float = 0.02


# ---------------------------------------------------------------------------
# Image-space glue (losses.py), torch
# ---------------------------------------------------------------------------
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


# ---------------------------------------------------------------------------
# compute_step
# ---------------------------------------------------------------------------
def compute_step(scene, camera, target_display, lut, weights: LossWeights = None,
                 threads: int = 1, *, prep: PreparedScene = None, env=None, tile: int = 16):
    """Full forward + backward for one view (training.py:130-184).

    Returns (metrics dict, SceneGrads, DeviceEnvGrads)."""
    del threads
    weights = weights or LossWeights()
    if prep is None:
        prep = prepare(scene, camera, "perprim")
    env = env if env is not None else scene.environment
    denv = env if isinstance(env, DeviceEnvironment) else DeviceEnvironment(env, lut,
                                                                            prep.scene.device)
    gbuf, tape = render_prepared(prep, camera, tile)
    bg = getattr(scene, "background", None)
    color, _, _ = shade_planar(gbuf.planar, camera, denv, bg, want_split=False)
    target = torch.as_tensor(np.asarray(target_display, np.float32) if not torch.is_tensor(
        target_display) else target_display, device=color.device, dtype=torch.float32)
    terms, dcolor, dg_reg = loss_and_grads(color, gbuf.planar, target, camera, weights)
    sr = ShadeResult(color, None, None, cache=(gbuf.planar, denv, np.asarray(
        bg if bg is not None else np.zeros(3), np.float64)))
    dgbuf, env_grads = shade_backward(sr, camera, None, None, dcolor)
    dgbuf += dg_reg
    grads = splat_backward(None, camera, prep, tape, dgbuf)
    terms["fragments"] = gbuf.fragment_count
    return terms, grads, env_grads


# ---------------------------------------------------------------------------
# Data-parallel training over views
# ---------------------------------------------------------------------------
_COMBINED_TO_INTERLEAVED = [0, 1, 2, 3, 6, 4, 5]  # combined channel c -> 8-channel slot


@dataclass
class TrainState:
    """Device-resident learnable parameters and Adam moments."""

    params: dict
    m: dict = field(default_factory=dict)
    v: dict = field(default_factory=dict)
    t: int = 0


def partition_views(num_views: int, rank: int, world: int) -> list:
    """Views of one rank: round-robin r, r + N, ...."""
    if not 0 <= rank < world:
        raise ValueError("rank out of range")
    return list(range(rank, num_views, world))


def allreduce_mean_(flat: torch.Tensor, group=None) -> torch.Tensor:
    """Sum a flat gradient buffer over the ranks in one collective and divide
    by the world size (in place). No-op without an initialised group."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized():
        dist.all_reduce(flat, op=dist.ReduceOp.SUM, group=group)
        flat /= dist.get_world_size(group)
    return flat


def flatten(tensors) -> torch.Tensor:
    """One float32 buffer from a list of tensors (any float dtype)."""
    return torch.cat([t.reshape(-1).float() for t in tensors])


def unflatten(flat: torch.Tensor, like) -> list:
    if sum(t.numel() for t in like) != flat.numel():
        raise ValueError("flat buffer size does not match the templates")
    out, o = [], 0
    for t in like:
        n = t.numel()
        out.append(flat[o:o + n].view(t.shape))
        o += n
    return out


class DataParallelTrainer:
    """One rank = one GPU = its own views; one NCCL all-reduce per step."""

    def __init__(self, scene, lut, *, lr=None, weights: LossWeights = None, tile: int = 16,
                 device=None, group=None):
        self.dev = device if device is not None else torch.device("cuda",
                                                                  torch.cuda.current_device())
        f64 = dict(dtype=torch.float64, device=self.dev)
        P = scene.num_splats
        T = scene.texture_config.resolution
        self.P, self.T, self.K = P, T, (scene.sh_degree + 1) ** 2
        self.sh_degree = scene.sh_degree
        tex = torch.from_numpy(np.ascontiguousarray(scene.texels, np.float32)).to(self.dev)
        self.params = {
            "positions": torch.as_tensor(scene.positions, **f64).contiguous(),
            "tangent_u": torch.as_tensor(scene.tangent_u, **f64).contiguous(),
            "tangent_v": torch.as_tensor(scene.tangent_v, **f64).contiguous(),
            "scales": torch.as_tensor(scene.scales, **f64).contiguous(),
            "opacities": torch.as_tensor(scene.opacities, **f64).contiguous(),
            "sh": torch.as_tensor(scene.sh, **f64).contiguous(),
            "texels": tex,
        }
        env = scene.environment
        self.env_params = [torch.from_numpy(np.ascontiguousarray(m, np.float32)).to(self.dev)
                           for m in env.spec_mips]
        self.env_params.append(torch.from_numpy(np.ascontiguousarray(env.diffuse, np.float32)
                                                ).to(self.dev))
        self.lut = torch.from_numpy(np.ascontiguousarray(lut.table, np.float32)).to(self.dev)
        self.texels8 = torch.zeros((P, T, T, 8), dtype=torch.float32, device=self.dev)
        self.background = np.asarray(scene.background, np.float64)
        self.weights = weights or LossWeights()
        self.tile = tile
        self.group = group
        self.lr = lr or {"positions": 1.6e-4, "tangent_u": 1e-3, "tangent_v": 1e-3,
                         "scales": 1e-3, "opacities": 5e-2, "sh": 2.5e-3, "texels": 2.5e-3,
                         "env": 1e-2}
        self.adam_m, self.adam_v, self.step_count = {}, {}, 0
        self.workspace = FrameWorkspace(self.dev)
        self._refresh_views()

    def _refresh_views(self):
        p = self.params
        self.texels8[..., _COMBINED_TO_INTERLEAVED] = p["texels"]
        self.dscene = DeviceScene.from_tensors(p["positions"], p["tangent_u"], p["tangent_v"],
                                               p["scales"], p["opacities"], p["sh"],
                                               self.sh_degree, self.T)
        self.datlas = DeviceAtlas.interleaved(self.texels8)
        self.denv = DeviceEnvironment.from_tensors(self.env_params[:-1], self.env_params[-1],
                                                   self.lut)
        self.prep = PreparedScene(self.dscene, self.datlas, "perprim", "verify",
                                  workspace=self.workspace)

    def grads_and_loss(self, camera, target):
        gbuf, tape = render_prepared(self.prep, camera, self.tile)
        color, _, _ = shade_planar(gbuf.planar, camera, self.denv, self.background,
                                   want_split=False)
        terms, dcolor, dg_reg = loss_and_grads(color, gbuf.planar, target, camera, self.weights)
        sr = ShadeResult(color, None, None, cache=(gbuf.planar, self.denv, self.background))
        dgbuf, env_grads = shade_backward(sr, camera, None, None, dcolor)
        dgbuf += dg_reg
        grads = splat_backward(None, camera, self.prep, tape, dgbuf)
        return terms, grads, env_grads

    def _flat_grads(self, grads: SceneGrads, env_grads) -> torch.Tensor:
        parts = [grads.positions, grads.tangent_u, grads.tangent_v, grads.scales,
                 grads.opacities, grads.sh]
        flat = [p.reshape(-1).float() for p in parts]
        flat.append(grads.texels_dense.reshape(-1))
        flat += [m.reshape(-1) for m in env_grads.spec_mips] + [env_grads.diffuse.reshape(-1)]
        return torch.cat(flat)

    def _unflatten(self, flat: torch.Tensor):
        out, o = {}, 0
        for name in ("positions", "tangent_u", "tangent_v", "scales", "opacities", "sh",
                     "texels"):
            n = self.params[name].numel()
            out[name] = flat[o:o + n].view_as(self.params[name])
            o += n
        env = []
        for prm in self.env_params:
            n = prm.numel()
            env.append(flat[o:o + n].view_as(prm))
            o += n
        out["env"] = env
        return out

    def _adam(self, key, param, grad, lr, b1=0.9, b2=0.999, eps=1e-8):
        grad = grad.to(param.dtype)
        if key not in self.adam_m:
            self.adam_m[key] = torch.zeros_like(param)
            self.adam_v[key] = torch.zeros_like(param)
        m, v = self.adam_m[key], self.adam_v[key]
        m.mul_(b1).add_(grad, alpha=1.0 - b1)
        v.mul_(b2).addcmul_(grad, grad, value=1.0 - b2)
        t = self.step_count
        denom = (v / (1.0 - b2 ** t)).sqrt_().add_(eps)
        param.addcdiv_(m, denom, value=-lr / (1.0 - b1 ** t))

    def step(self, camera, target):
        """Forward + backward on this rank's view, all-reduce, Adam update.
        Returns (terms, flat gradient buffer after the all-reduce)."""
        terms, grads, env_grads = self.grads_and_loss(camera, target)
        flat = self._flat_grads(grads, env_grads)
        allreduce_mean_(flat, self.group)
        g = self._unflatten(flat)
        self.step_count += 1
        with torch.no_grad():
            for name in ("positions", "tangent_u", "tangent_v", "scales", "opacities", "sh",
                         "texels"):
                self._adam(name, self.params[name], g[name], self.lr[name])
            p = self.params
            # constraint projections (training.py:270-304)
            p["opacities"].clamp_(0.0, 1.0)
            p["scales"].clamp_(min=1e-6)
            p["texels"].clamp_(0.0, 1.0)
            tu = p["tangent_u"] / torch.linalg.norm(p["tangent_u"], dim=1, keepdim=True)
            tv = p["tangent_v"] - (tu * p["tangent_v"]).sum(1, keepdim=True) * tu
            tv = tv / torch.linalg.norm(tv, dim=1, keepdim=True)
            p["tangent_u"].copy_(tu)
            p["tangent_v"].copy_(tv)
            for i, prm in enumerate(self.env_params):
                self._adam(f"env{i}", prm, g["env"][i], self.lr["env"])
                prm.clamp_(min=0.0)
        self._refresh_views()
        return terms, flat
