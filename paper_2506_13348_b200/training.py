"""Training step (BASELINE configs[3]) on the B200 render path.

compute_step mirrors texsplat.training.compute_step (training.py:130-184):
forward with tape (K1-K5), deferred shading (K6), display transform + L1 +
D-SSIM image loss (K10), shading adjoint (K7), normal-consistency and
smoothness regularisers (K11) and the splat adjoint (K8/K9) — every step
of it a libtsb kernel; the loss terms stay on the device (fp64 sums) until
a caller reads them.

DataParallelTrainer: one process per GPU, each rank renders its own view;
the gradients land directly in one flat float32 buffer (texel and
environment gradients are written in place by the kernels, the float64
geometry gradients are packed with one copy), which a single NCCL
all-reduce over NVLink sums (torch.distributed); then one fused Adam launch
(K12, training.py:69-100 with the step's projections) and the tangent
re-orthonormalisation (K13). The texels live as the (P, T, T, 8)
interleaved verify-mode atlas, so the updated parameters are rendered
directly. SURVEY.md §8(e).
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .backward import DeviceEnvGrads, SceneGrads, shade_backward, splat_backward
from .device import DeviceAtlas, DeviceEnvironment, DeviceScene, FrameWorkspace
from .rasterize import PreparedScene, prepare, render_prepared
from .shading import ShadeResult, shade_planar

DISPLAY_GAMMA = 2.2
DISPLAY_TOE = 1e-4
PSNR_CAP = 99.0
SCALE_FLOOR = 1e-6          # training.py:35


@dataclass
class LossWeights:
    dssim: float = 0.2
    normal: float = 0.05
    smooth: float = 0.02


def linear_to_display(x: torch.Tensor) -> torch.Tensor:
    """Gamma 2.2 with a slope-matched linear toe below 1e-4 (losses.py:24-29);
    used to make display-space targets (not on the step's path, which runs
    the transform inside K10)."""
    p = 1.0 / DISPLAY_GAMMA
    toe_slope = DISPLAY_TOE ** (p - 1.0)
    return torch.where(x >= DISPLAY_TOE, x.clamp_min(DISPLAY_TOE) ** p,
                       toe_slope * x.clamp_min(0.0))


def _psnr_from_mse(mse: float) -> float:
    """losses.py:137-144 on the clipped images' mean squared error."""
    if mse <= 10.0 ** (-PSNR_CAP / 10.0):
        return PSNR_CAP
    return float(10.0 * math.log10(1.0 / mse))


class StepTerms(dict):
    """Loss terms of a step. The device sums (K10/K11) are read back on the
    first access, so a training loop that never looks does not synchronise."""

    def __init__(self, sums: torch.Tensor, n_values: int, weights: LossWeights, extra=None):
        super().__init__()
        self._sums, self._n, self._w, self._extra = sums, n_values, weights, extra or {}
        self._ready = False

    def _fill(self):
        if self._ready:
            return
        t = self._sums.detach().cpu().numpy().astype(np.float64)
        N, w = float(self._n), self._w
        image = (1.0 - w.dssim) * t[0] / N + w.dssim * 0.5 * (1.0 - t[1] / N)
        normal = t[3] / max(t[4], 1.0) if w.normal > 0.0 else 0.0
        smooth = t[5] / max(t[6], 1.0) if w.smooth > 0.0 else 0.0
        super().update({"loss": image + w.normal * normal + w.smooth * smooth,
                        "image": image, "normal": normal, "smooth": smooth,
                        "psnr": _psnr_from_mse(t[2] / N)})
        for k, v in self._extra.items():
            super().__setitem__(k, v() if callable(v) else v)
        self._ready = True

    def __getitem__(self, k):
        self._fill()
        return super().__getitem__(k)

    def __iter__(self):
        self._fill()
        return super().__iter__()

    def __len__(self):
        self._fill()
        return super().__len__()

    def keys(self):
        self._fill()
        return super().keys()

    def items(self):
        self._fill()
        return super().items()

    def get(self, k, default=None):
        self._fill()
        return super().get(k, default)


class _LossBuffers:
    """Per-image-size device buffers of the loss kernels."""

    def __init__(self):
        self._by_size = {}

    def get(self, W, H, dev):
        key = (W, H, dev)
        if key not in self._by_size:
            nb = C.c_uint64()
            _lib.check(_lib.lib().tsb_loss_scratch_size(W, H, C.byref(nb)), "tsb_loss_scratch_size")
            self._by_size[key] = {
                "scratch": torch.empty(int(nb.value), dtype=torch.uint8, device=dev),
                "dcolor": torch.empty((H, W, 3), dtype=torch.float32, device=dev),
                "dgbuf": torch.empty((13, H, W), dtype=torch.float32, device=dev),
                "terms": torch.zeros(8, dtype=torch.float64, device=dev),
            }
        return self._by_size[key]


_BUFFERS = _LossBuffers()


def image_loss_grad(color: torch.Tensor, target: torch.Tensor, weights: LossWeights, bufs,
                    stream=None):
    """K10: dcolor of the display-space image loss; sums into bufs['terms']."""
    H, W = int(color.shape[0]), int(color.shape[1])
    _lib.check(_lib.lib().tsb_loss_image(
        _lib.ptr(color), _lib.ptr(target), W, H, float(weights.dssim), _lib.ptr(bufs["dcolor"]),
        _lib.ptr(bufs["terms"]), _lib.ptr(bufs["scratch"]), int(bufs["scratch"].numel()),
        _lib.stream_handle(stream)), "tsb_loss_image")
    return bufs["dcolor"]


def regularizer_grads(planar: torch.Tensor, target: torch.Tensor, camera, weights: LossWeights,
                      dgbuf: torch.Tensor, terms: torch.Tensor, stream=None):
    """K11: adds the regulariser gradients into the planar dgbuf."""
    cam = _lib.camera_struct(camera)
    _lib.check(_lib.lib().tsb_loss_regularizers(
        _lib.ptr(planar), _lib.ptr(target), C.byref(cam), float(weights.normal),
        float(weights.smooth), _lib.ptr(dgbuf), _lib.ptr(terms), _lib.stream_handle(stream)),
        "tsb_loss_regularizers")


def _target_tensor(target_display, dev) -> torch.Tensor:
    t = target_display if torch.is_tensor(target_display) else torch.from_numpy(
        np.ascontiguousarray(np.asarray(target_display, np.float32)))
    return t.to(device=dev, dtype=torch.float32).contiguous()


# ---------------------------------------------------------------------------
# compute_step
# ---------------------------------------------------------------------------
def compute_step(scene, camera, target_display, lut, weights: LossWeights = None,
                 threads: int = 1, *, prep: PreparedScene = None, env=None, tile: int = 16):
    """Full forward + backward for one view (training.py:130-184).

    Returns (metrics dict, SceneGrads, DeviceEnvGrads); texel gradients in
    the reference's combined (P, T, T, 7) order."""
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
    dev = color.device
    H, W = int(camera.height), int(camera.width)
    target = _target_tensor(target_display, dev)
    bufs = _BUFFERS.get(W, H, dev)
    terms = torch.zeros(8, dtype=torch.float64, device=dev)
    bufs = dict(bufs, terms=terms)
    dcolor = image_loss_grad(color, target, weights, bufs)
    sr = ShadeResult(color, None, None, cache=(gbuf.planar, denv, np.asarray(
        bg if bg is not None else np.zeros(3), np.float64)))
    dgbuf, env_grads = shade_backward(sr, camera, None, None, dcolor)
    regularizer_grads(gbuf.planar, target, camera, weights, dgbuf, terms)
    grads = splat_backward(None, camera, prep, tape, dgbuf)
    metrics = StepTerms(terms, 3 * W * H, weights,
                        extra={"fragments": lambda: gbuf.fragment_count})
    metrics._fill()
    return dict(metrics), grads, env_grads


# ---------------------------------------------------------------------------
# Data-parallel training over views
# ---------------------------------------------------------------------------
_COMBINED_TO_INTERLEAVED = [0, 1, 2, 3, 6, 4, 5]  # combined channel c -> 8-channel slot


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


def world_extent(positions: np.ndarray) -> float:
    """Scene.world_extent (scene.py:146-151): the position learning-rate scale."""
    p = np.asarray(positions, np.float64)
    if p.shape[0] == 0:
        return 1.0
    return float(max(np.linalg.norm(p.max(axis=0) - p.min(axis=0)), 1e-6))


_GEOM = ("positions", "tangent_u", "tangent_v", "scales", "opacities", "sh")


class DataParallelTrainer:
    """One rank = one GPU = its own views; one NCCL all-reduce per step."""

    def __init__(self, scene, lut, *, lr=None, weights: LossWeights = None, tile: int = 16,
                 device=None, group=None, betas=(0.9, 0.999), eps=1e-8):
        self.dev = device if device is not None else torch.device("cuda",
                                                                  torch.cuda.current_device())
        dev = self.dev
        f64 = dict(dtype=torch.float64, device=dev)
        P = scene.num_splats
        T = scene.texture_config.resolution
        self.P, self.T, self.K = P, T, (scene.sh_degree + 1) ** 2
        self.sh_degree = scene.sh_degree
        self.params = {n: torch.as_tensor(np.ascontiguousarray(getattr(scene, n)), **f64)
                       .contiguous() for n in _GEOM}
        tex = torch.from_numpy(np.ascontiguousarray(scene.texels, np.float32)).to(dev)
        self.texels8 = torch.zeros((P, T, T, 8), dtype=torch.float32, device=dev)
        self.texels8[..., _COMBINED_TO_INTERLEAVED] = tex
        env = scene.environment
        self.env_params = [torch.from_numpy(np.ascontiguousarray(m, np.float32)).to(dev)
                           for m in env.spec_mips]
        self.env_params.append(torch.from_numpy(np.ascontiguousarray(env.diffuse, np.float32)
                                                ).to(dev))
        self.lut = torch.from_numpy(np.ascontiguousarray(lut.table, np.float32)).to(dev)
        self.background = np.asarray(scene.background, np.float64)
        self.weights = weights or LossWeights()
        self.tile = tile
        self.group = group
        self.betas, self.eps = betas, eps
        extent = world_extent(scene.positions)
        self.lr = {"positions": 1.6e-4 * extent, "tangent_u": 1e-3, "tangent_v": 1e-3,
                   "scales": 1e-3, "opacities": 5e-2, "sh": 2.5e-3, "texels": 2.5e-3,
                   "env": 1e-2}                   # TrainConfig defaults (training.py:45-52)
        if lr:
            self.lr.update(lr)
        self.step_count = 0

        # device views the kernels render from (parameters updated in place)
        p = self.params
        self.dscene = DeviceScene.from_tensors(p["positions"], p["tangent_u"], p["tangent_v"],
                                               p["scales"], p["opacities"], p["sh"],
                                               self.sh_degree, T)
        self.datlas = DeviceAtlas.interleaved(self.texels8)
        self.denv = DeviceEnvironment.from_tensors(self.env_params[:-1], self.env_params[-1],
                                                   self.lut)
        self.prep = PreparedScene(self.dscene, self.datlas, "perprim", "verify",
                                  workspace=FrameWorkspace(dev))

        # one flat float32 gradient buffer: [geometry | texels (P,T,T,8) | env grids]
        self.n_geom = sum(t.numel() for t in p.values())
        n_tex = self.texels8.numel()
        n_env = sum(t.numel() for t in self.env_params)
        self.flat = torch.zeros(self.n_geom + n_tex + n_env, dtype=torch.float32, device=dev)
        self.geom64 = torch.zeros(self.n_geom, **f64)
        views, o = {}, 0
        for n in _GEOM:
            views[n] = self.geom64[o:o + p[n].numel()].view(p[n].shape)
            o += p[n].numel()
        tex_grad = self.flat[self.n_geom:self.n_geom + n_tex].view(P, T, T, 8)
        self.grads = SceneGrads(views["positions"], views["tangent_u"], views["tangent_v"],
                                views["scales"], views["opacities"], views["sh"], tex_grad,
                                texel_layout=_lib.TEXELS_INTERLEAVED)
        env_views, o = [], self.n_geom + n_tex
        for prm in self.env_params:
            env_views.append(self.flat[o:o + prm.numel()].view(prm.shape))
            o += prm.numel()
        self.env_grads = DeviceEnvGrads(env_views[:-1], env_views[-1])
        nb = C.c_uint64()
        _lib.check(_lib.lib().tsb_backward_scratch_size(P, C.byref(nb)), "tsb_backward_scratch_size")
        self.bwd_scratch = torch.empty(int(nb.value), dtype=torch.uint8, device=dev)

        # Adam groups: (param, grad view of the flat buffer, lr, clamp, floor)
        groups, o = [], 0
        for n in _GEOM:
            k = p[n].numel()
            clamp = {"scales": _lib.CLAMP_FLOOR, "opacities": _lib.CLAMP_UNIT}.get(n, _lib.CLAMP_NONE)
            groups.append((p[n], self.flat[o:o + k], self.lr[n], clamp, SCALE_FLOOR))
            o += k
        groups.append((self.texels8, tex_grad.view(-1), self.lr["texels"], _lib.CLAMP_UNIT, 0.0))
        for prm, gv in zip(self.env_params, env_views):
            groups.append((prm, gv.view(-1), self.lr["env"], _lib.CLAMP_NONE, 0.0))
        if len(groups) > _lib.ADAM_MAX_GROUPS:
            raise ValueError("too many parameter groups for one Adam launch")
        self._moments = []
        arr = (_lib.AdamGroup_t * len(groups))()
        for i, (prm, g, lr_i, clamp, floor) in enumerate(groups):
            m, v = torch.zeros_like(prm), torch.zeros_like(prm)
            self._moments.append((m, v))
            a = arr[i]
            a.param, a.grad, a.m, a.v = _lib.ptr(prm), _lib.ptr(g), _lib.ptr(m), _lib.ptr(v)
            a.count = prm.numel()
            a.lr, a.floor, a.clamp = float(lr_i), float(floor), clamp
            a.dtype = _lib.F64 if prm.dtype == torch.float64 else _lib.F32
        self._adam_groups = arr

    @property
    def texels(self) -> torch.Tensor:
        """Current texels in the reference's combined (P, T, T, 7) order."""
        return self.texels8[..., _COMBINED_TO_INTERLEAVED]

    def grads_and_loss(self, camera, target):
        """Forward + backward of one view into the flat gradient buffer
        (zeroed first). Returns StepTerms."""
        dev = self.dev
        H, W = int(camera.height), int(camera.width)
        bufs = _BUFFERS.get(W, H, dev)
        target = _target_tensor(target, dev)
        self.flat.zero_()
        self.geom64.zero_()
        terms = torch.zeros(8, dtype=torch.float64, device=dev)
        bufs = dict(bufs, terms=terms)
        gbuf, tape = render_prepared(self.prep, camera, self.tile)
        color, _, _ = shade_planar(gbuf.planar, camera, self.denv, self.background,
                                   want_split=False)
        dcolor = image_loss_grad(color, target, self.weights, bufs)
        sr = ShadeResult(color, None, None, cache=(gbuf.planar, self.denv, self.background))
        dgbuf, _ = shade_backward(sr, camera, None, None, dcolor, env_grads=self.env_grads,
                                  dgbuf=bufs["dgbuf"])
        regularizer_grads(gbuf.planar, target, camera, self.weights, dgbuf, terms)
        splat_backward(None, camera, self.prep, tape, dgbuf, grads=self.grads,
                       scratch=self.bwd_scratch)
        self.flat[:self.n_geom].copy_(self.geom64)
        return StepTerms(terms, 3 * W * H, self.weights)

    def step(self, camera, target):
        """Forward + backward on this rank's view, all-reduce, Adam update.
        Returns (terms, flat gradient buffer after the all-reduce)."""
        terms = self.grads_and_loss(camera, target)
        allreduce_mean_(self.flat, self.group)
        self.step_count += 1
        L = _lib.lib()
        st = _lib.stream_handle()
        _lib.check(L.tsb_adam_step(self._adam_groups, len(self._adam_groups), self.step_count,
                                   float(self.betas[0]), float(self.betas[1]), float(self.eps),
                                   st), "tsb_adam_step")
        _lib.check(L.tsb_orthonormalize_tangents(self.P, _lib.ptr(self.params["tangent_u"]),
                                                 _lib.ptr(self.params["tangent_v"]), st),
                   "tsb_orthonormalize_tangents")
        return terms, self.flat
