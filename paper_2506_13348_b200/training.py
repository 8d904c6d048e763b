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
from .scene import scene_texels
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
_ADAM_CLAMP = {"scales": _lib.CLAMP_FLOOR, "opacities": _lib.CLAMP_UNIT, "texels": _lib.CLAMP_UNIT}


class DataParallelTrainer:
    """One rank = one GPU = its own views; the gradient exchange is one
    bucketed all-reduce per step.

    State on the device: float64 splat parameters, texels as the (P, T, T, 8)
    interleaved verify-mode atlas the forward renders from, float32
    environment grids, Adam moments per parameter group with per-group step
    counts (training.py:69-100: the texel moments restart at the stage-2
    broadcast). The gradients land in ONE flat float32 buffer laid out
    [geometry | env grids | texels (P, T, T, 7) combined order]: K8 writes the
    texel gradients straight into it in the 7-channel order (no always-zero
    8th channel on the wire; Adam maps them onto the 8-channel parameters,
    TSB_F32_TEX87). The buffer is all-reduced in buckets — geometry + env
    first, then the texels in splat-range chunks — each bucket's Adam launch
    waiting only on its own all-reduce, so the update of bucket k overlaps
    the transfer of bucket k+1. No host synchronisation per step: the frame
    capacity is validated from the device's running maximum every
    `check_every` steps, the divergence guard is a device flag (`halt`) that
    the guarded Adam / orthonormalisation honour (tsb_guard_finite).
    """

    def __init__(self, scene, lut, *, lr=None, weights: LossWeights = None, tile: int = 16,
                 device=None, group=None, betas=(0.9, 0.999), eps=1e-8,
                 optimize_geometry: bool = True, optimize_environment: bool = True,
                 texel_buckets: int = 4, check_every: int = 32, deterministic: bool = False):
        self.dev = device if device is not None else torch.device("cuda",
                                                                  torch.cuda.current_device())
        dev = self.dev
        f64 = dict(dtype=torch.float64, device=dev)
        self.sh_degree = int(scene.sh_degree)
        self.K = (self.sh_degree + 1) ** 2
        self.T = int(scene.texture_config.resolution)
        self.params = {n: torch.as_tensor(np.ascontiguousarray(getattr(scene, n)), **f64)
                       .contiguous() for n in _GEOM}
        self.P = int(self.params["positions"].shape[0])
        tex = torch.from_numpy(np.ascontiguousarray(scene_texels(scene), np.float32)).to(dev)
        self.texels8 = torch.zeros((self.P, self.T, self.T, 8), dtype=torch.float32, device=dev)
        self.texels8[..., _COMBINED_TO_INTERLEAVED] = tex
        env = scene.environment
        self.env_params = [torch.from_numpy(np.ascontiguousarray(m, np.float32)).to(dev)
                           for m in env.spec_mips]
        self.env_params.append(torch.from_numpy(np.ascontiguousarray(env.diffuse, np.float32)
                                                ).to(dev))
        table = lut.table if hasattr(lut, "table") else lut
        self.lut = torch.as_tensor(np.ascontiguousarray(table, np.float32)).to(dev)
        self.background = np.asarray(scene.background, np.float64)
        self.weights = weights or LossWeights()
        self.tile = tile
        self.group = group
        self.betas, self.eps = betas, eps
        self.optimize_geometry = optimize_geometry
        self.optimize_environment = optimize_environment
        self.texel_buckets = max(1, int(texel_buckets))
        self.check_every = max(1, int(check_every))
        self.deterministic = deterministic
        extent = world_extent(scene.positions)
        self.lr = {"positions": 1.6e-4 * extent, "tangent_u": 1e-3, "tangent_v": 1e-3,
                   "scales": 1e-3, "opacities": 5e-2, "sh": 2.5e-3, "texels": 2.5e-3,
                   "env": 1e-2}                   # TrainConfig defaults (training.py:45-52)
        if lr:
            self.lr.update(lr)
        self.step_count = 0
        self.steps = {}                           # Adam step count per parameter group
        self.moments = {}                         # group name -> (m, v)
        self.halt = torch.zeros(1, dtype=torch.int32, device=dev)
        self.workspace = FrameWorkspace(dev)
        self._frames_since_check = 0
        self._rebuild()

    # -- layout ---------------------------------------------------------------
    def _rebuild(self):
        """(Re)create the device views, the flat gradient buffer, the scratch
        buffers and the Adam groups for the current P and T (after the
        stage-2 broadcast or a prune); moments of unchanged shape are kept."""
        dev, P, T = self.dev, self.P, self.T
        p = self.params
        self.dscene = DeviceScene.from_tensors(p["positions"], p["tangent_u"], p["tangent_v"],
                                               p["scales"], p["opacities"], p["sh"],
                                               self.sh_degree, T)
        self.datlas = DeviceAtlas.interleaved(self.texels8)
        self.denv = DeviceEnvironment.from_tensors(self.env_params[:-1], self.env_params[-1],
                                                   self.lut)
        self.prep = PreparedScene(self.dscene, self.datlas, "perprim", "verify",
                                  workspace=self.workspace)
        n_geom = sum(t.numel() for t in p.values())
        n_env = sum(t.numel() for t in self.env_params)
        # texel gradients: 7 combined channels when they go on the wire (no
        # zero pad channel in the all-reduce); on one GPU the 8-channel
        # interleaved layout of the parameters themselves (32-B aligned texels:
        # fewer L2 sectors per atomic in K8, vectorised Adam)
        self.tex_ch = 7 if _dist_on() else 8
        n_tex = P * T * T * self.tex_ch
        self.n_geom, self.n_env, self.n_tex = n_geom, n_env, n_tex
        self.flat = torch.zeros(n_geom + n_env + n_tex, dtype=torch.float32, device=dev)
        self.geom64 = torch.zeros(n_geom, dtype=torch.float64, device=dev)
        gviews, o = {}, 0
        for n in _GEOM:
            gviews[n] = self.geom64[o:o + p[n].numel()].view(p[n].shape)
            o += p[n].numel()
        tex_grad = self.flat[n_geom + n_env:].view(P, T, T, self.tex_ch)
        self.grads = SceneGrads(gviews["positions"], gviews["tangent_u"], gviews["tangent_v"],
                                gviews["scales"], gviews["opacities"], gviews["sh"], tex_grad,
                                texel_layout=(_lib.TEXELS_COMBINED if self.tex_ch == 7
                                              else _lib.TEXELS_INTERLEAVED))
        env_views, o = [], n_geom
        for prm in self.env_params:
            env_views.append(self.flat[o:o + prm.numel()].view(prm.shape))
            o += prm.numel()
        self.env_grads = DeviceEnvGrads(env_views[:-1], env_views[-1])
        nb = C.c_uint64()
        _lib.check(_lib.lib().tsb_backward_scratch_size(P, C.byref(nb)), "tsb_backward_scratch_size")
        self.bwd_scratch = torch.empty(int(nb.value), dtype=torch.uint8, device=dev)

        # Adam groups -> launches (one per all-reduce bucket)
        def group(name, prm, grad, lr, dtype=None):
            if name not in self.moments or self.moments[name][0].shape != prm.shape:
                self.moments[name] = (torch.zeros_like(prm), torch.zeros_like(prm))
            return (name, prm, grad, lr, _ADAM_CLAMP.get(name.split(":")[0], _lib.CLAMP_NONE),
                    dtype if dtype is not None else
                    (_lib.F64 if prm.dtype == torch.float64 else _lib.F32))

        first, o = [], 0
        for n in _GEOM:
            k = p[n].numel()
            if self.optimize_geometry or n == "sh":
                first.append(group(n, p[n], self.flat[o:o + k], self.lr[n]))
            o += k
        if self.optimize_environment:
            for i, (prm, gv) in enumerate(zip(self.env_params, env_views)):
                name = f"env_spec{i}" if i < len(self.env_params) - 1 else "env_diffuse"
                first.append(group(name, prm, gv.view(-1), self.lr["env"]))
        # texel buckets: splat ranges (a range of the 8-channel parameters maps
        # onto the same range of the 7-channel gradients)
        if "texels" not in self.moments or self.moments["texels"][0].shape != self.texels8.shape:
            self.moments["texels"] = (torch.zeros_like(self.texels8),
                                      torch.zeros_like(self.texels8))
        tm, tv = self.moments["texels"]
        nbk = min(self.texel_buckets, max(P, 1))
        cuts = [P * i // nbk for i in range(nbk + 1)]
        tex_groups, tex_ranges = [], []
        for i in range(nbk):
            a, b = cuts[i], cuts[i + 1]
            if b <= a:
                continue
            tex_groups.append((f"texels:{i}", self.texels8[a:b], tex_grad[a:b],
                               self.lr["texels"], _lib.CLAMP_UNIT,
                               _lib.F32_TEX87 if self.tex_ch == 7 else _lib.F32,
                               tm[a:b], tv[a:b]))
            c = self.tex_ch
            tex_ranges.append((n_geom + n_env + a * T * T * c, n_geom + n_env + b * T * T * c))
        self._buckets = [((0, n_geom + n_env), first)] + [
            (rng, [g]) for rng, g in zip(tex_ranges, tex_groups)]
        self._launches = []
        for rng, groups in self._buckets:
            arr = (_lib.AdamGroup_t * max(1, len(groups)))()
            names = []
            for i, gtuple in enumerate(groups):
                name, prm, g, lr_i, clamp, dtype = gtuple[:6]
                m, v = gtuple[6:8] if len(gtuple) > 6 else self.moments[name]
                a_ = arr[i]
                a_.param, a_.grad, a_.m, a_.v = _lib.ptr(prm), _lib.ptr(g), _lib.ptr(m), _lib.ptr(v)
                a_.count = prm.numel()
                a_.lr, a_.floor, a_.clamp, a_.dtype = float(lr_i), float(SCALE_FLOOR), clamp, dtype
                names.append(name.split(":")[0])
            self._launches.append((rng, arr, len(groups), names))
        if len(first) > _lib.ADAM_MAX_GROUPS:
            raise ValueError("too many parameter groups for one Adam launch")

    # -- one step ------------------------------------------------------------
    @property
    def texels(self) -> torch.Tensor:
        """Current texels in the reference's combined (P, T, T, 7) order."""
        return self.texels8[..., _COMBINED_TO_INTERLEAVED]

    def _check_capacity(self, camera):
        """Device running maximum of the frames' entry counts vs capacity,
        every `check_every` steps (one small host read)."""
        ws = self.workspace
        W, H = int(camera.width), int(camera.height)
        if ws.key != (self.P, W, H, self.tile):
            return True  # first frame of this size: render with a checked frame
        self._frames_since_check += 1
        if self._frames_since_check < self.check_every:
            return False
        self._frames_since_check = 0
        need = ws.max_needed_value()
        if need > ws.capacity:
            raise RuntimeError(f"frame workspace overflow during training ({need} > "
                               f"{ws.capacity} entries); raise the headroom")
        if need > 0.7 * ws.capacity:  # keep >= 30 % headroom as the scene evolves
            ws.ensure(self.P, W, H, self.tile, int(need * 1.6) + 4096)
        return False

    def grads_and_loss(self, camera, target, terms: torch.Tensor = None):
        """Forward + backward of one view into the flat gradient buffer
        (zeroed first). Returns StepTerms (device sums, read lazily)."""
        dev = self.dev
        H, W = int(camera.height), int(camera.width)
        bufs = _BUFFERS.get(W, H, dev)
        target = _target_tensor(target, dev)
        self.flat.zero_()
        self.geom64.zero_()
        if terms is None:
            terms = torch.zeros(8, dtype=torch.float64, device=dev)
        else:
            terms.zero_()
        bufs = dict(bufs, terms=terms)
        checked = self._check_capacity(camera)
        gbuf, tape = render_prepared(self.prep, camera, self.tile, check=checked)
        if checked:  # first frame of this layout: size for the scene's growth (60 % headroom)
            ws = self.workspace
            want = int(int(ws.needed.item()) * 1.6) + 4096
            if ws.capacity < want:
                ws.ensure(self.P, W, H, self.tile, want)
                gbuf, tape = render_prepared(self.prep, camera, self.tile, check=True)
            ws.reset_max()
        color, _, _ = shade_planar(gbuf.planar, camera, self.denv, self.background,
                                   want_split=False)
        dcolor = image_loss_grad(color, target, self.weights, bufs)
        sr = ShadeResult(color, None, None, cache=(gbuf.planar, self.denv, self.background))
        dgbuf, _ = shade_backward(sr, camera, None, None, dcolor, env_grads=self.env_grads,
                                  dgbuf=bufs["dgbuf"])
        regularizer_grads(gbuf.planar, target, camera, self.weights, dgbuf, terms)
        splat_backward(None, camera, self.prep, tape, dgbuf, grads=self.grads,
                       scratch=self.bwd_scratch, deterministic=self.deterministic)
        self.flat[:self.n_geom].copy_(self.geom64)
        self._last_gbuf = gbuf
        return StepTerms(terms, 3 * W * H, self.weights)

    def step(self, camera, target, terms: torch.Tensor = None):
        """Forward + backward on this rank's view, bucketed all-reduce + Adam,
        tangent re-orthonormalisation. Returns (terms, flat gradient buffer)."""
        st = self.grads_and_loss(camera, target, terms)
        L = _lib.lib()
        sh = _lib.stream_handle()
        _lib.check(L.tsb_guard_finite(_lib.ptr(st._sums), 7, _lib.ptr(self.halt), sh),
                   "tsb_guard_finite")
        self.step_count += 1
        stepped = set()
        for names in (n for _, _, _, n in self._launches):
            stepped.update(names)
        for n in stepped:
            self.steps[n] = self.steps.get(n, 0) + 1
        if _dist_on():
            works = self._allreduce_async()
            for (rng, arr, n, names), work in zip(self._launches, works):
                if n == 0:
                    continue
                work.wait()  # (the current stream waits on this bucket only)
                self.flat[rng[0]:rng[1]].div_(_world(self.group))
                t = self.steps[names[0]]
                _lib.check(L.tsb_adam_step_ex(arr, n, t, float(self.betas[0]),
                                              float(self.betas[1]), float(self.eps),
                                              _lib.ptr(self.halt), sh), "tsb_adam_step")
        else:  # one GPU: one Adam launch per distinct step count (normally one)
            for t, (arr, n) in self._single_launches().items():
                _lib.check(L.tsb_adam_step_ex(arr, n, t, float(self.betas[0]),
                                              float(self.betas[1]), float(self.eps),
                                              _lib.ptr(self.halt), sh), "tsb_adam_step")
        if self.optimize_geometry:
            _lib.check(L.tsb_orthonormalize_tangents_ex(
                self.P, _lib.ptr(self.params["tangent_u"]), _lib.ptr(self.params["tangent_v"]),
                _lib.ptr(self.halt), sh), "tsb_orthonormalize_tangents")
        return st, self.flat

    def _single_launches(self):
        """Every bucket's groups merged, keyed by their Adam step count."""
        by_t = {}
        for _, arr, n, names in self._launches:
            for i in range(n):
                by_t.setdefault(self.steps[names[i]], []).append(arr[i])
        out = {}
        for t, gs in by_t.items():
            arr = (_lib.AdamGroup_t * len(gs))(*gs)
            out[t] = (arr, len(gs))
        return out

    def _allreduce_async(self):
        """Start one all-reduce (sum) per bucket; None entries: no group."""
        if not _dist_on():
            return [None] * len(self._launches)
        import torch.distributed as dist
        return [dist.all_reduce(self.flat[a:b], op=dist.ReduceOp.SUM, group=self.group,
                                async_op=True) for (a, b), _, _, _ in self._launches]

    # -- train() schedule ----------------------------------------------------
    def broadcast_textures(self, resolution: int):
        """Stage-2 chart growth (broadcast_textures, training.py:201-221) and
        the Adam reset of the texels (training.py:254-257)."""
        T0, T = self.T, int(resolution)
        if T != T0:
            new = torch.empty((self.P, T, T, 8), dtype=torch.float32, device=self.dev)
            _lib.check(_lib.lib().tsb_broadcast_texels(self.P, T0, T, _lib.ptr(self.texels8),
                                                       _lib.ptr(new), _lib.stream_handle()),
                       "tsb_broadcast_texels")
            self.texels8 = new
            self.T = T
        self.moments.pop("texels", None)
        self.steps.pop("texels", None)
        self._rebuild()

    def prune(self, threshold: float) -> int:
        """Drop splats with opacity <= threshold (_prune, training.py:187-198):
        parameters, texels and their Adam moments compacted on the device (step
        counts kept). Skipped when every or no splat survives, or after a
        divergence. Returns the number of splats (one host read)."""
        P = self.P
        if P == 0 or int(self.halt.item()):
            return P
        L = _lib.lib()
        bufs, dsts = [], {}

        def add(key, t):
            d = torch.empty_like(t)
            dsts[key] = d
            bufs.append((t, d, t.numel() // P * t.element_size()))

        for n in _GEOM:
            add(("p", n), self.params[n])
            if n in self.moments:
                add(("m", n), self.moments[n][0])
                add(("v", n), self.moments[n][1])
        add(("p", "texels"), self.texels8)
        add(("m", "texels"), self.moments["texels"][0])
        add(("v", "texels"), self.moments["texels"][1])
        arr = (_lib.RowBuffer_t * len(bufs))()
        for i, (src, dst, rb) in enumerate(bufs):
            arr[i].src, arr[i].dst, arr[i].row_bytes = _lib.ptr(src), _lib.ptr(dst), int(rb)
        nb = C.c_uint64()
        _lib.check(L.tsb_prune_scratch_size(P, C.byref(nb)), "tsb_prune_scratch_size")
        scratch = torch.empty(int(nb.value), dtype=torch.uint8, device=self.dev)
        kept = torch.zeros(1, dtype=torch.int32, device=self.dev)
        _lib.check(L.tsb_prune_rows(P, _lib.ptr(self.params["opacities"]), float(threshold), arr,
                                    len(bufs), _lib.ptr(kept), _lib.ptr(scratch), int(nb.value),
                                    _lib.stream_handle()), "tsb_prune_rows")
        k = int(kept.item())
        if k == P or k == 0:
            return P
        for n in _GEOM:
            self.params[n] = dsts[("p", n)][:k]
            if n in self.moments:
                self.moments[n] = (dsts[("m", n)][:k], dsts[("v", n)][:k])
        self.texels8 = dsts[("p", "texels")][:k]
        self.moments["texels"] = (dsts[("m", "texels")][:k], dsts[("v", "texels")][:k])
        self.P = k
        self._rebuild()
        return k

    def to_scene(self, template=None) -> "Scene":
        """The current parameters as a host Scene (texels in combined order)."""
        from .scene import Scene, TextureConfig
        from .environment import EnvironmentLight
        env = EnvironmentLight([m.cpu().numpy() for m in self.env_params[:-1]],
                               self.env_params[-1].cpu().numpy())
        p = {n: t.cpu().numpy() for n, t in self.params.items()}
        return Scene(p["positions"], p["tangent_u"], p["tangent_v"], p["scales"],
                     p["opacities"], p["sh"], self.sh_degree,
                     np.ascontiguousarray(self.texels.cpu().numpy()),
                     TextureConfig(self.T), environment=env, background=self.background.copy())


def _ssim_torch(a: torch.Tensor, b: torch.Tensor) -> float:
    """Mean SSIM of two (H, W, C) display images (losses.py:61-99: 11-tap
    sigma-1.5 separable Gaussian, zero padding), float64 on the device — an
    evaluation metric for `fit`'s summary, not part of the training step."""
    import torch.nn.functional as F
    x = torch.arange(-5, 6, dtype=torch.float64, device=a.device)
    w = torch.exp(-0.5 * (x / 1.5) ** 2)
    w = w / w.sum()
    C = a.shape[-1]

    def blur(img):  # (H, W, C) -> (H, W, C)
        t = img.permute(2, 0, 1).unsqueeze(0)
        t = F.conv2d(t, w.view(1, 1, 11, 1).expand(C, 1, 11, 1).contiguous(), padding=(5, 0),
                     groups=C)
        t = F.conv2d(t, w.view(1, 1, 1, 11).expand(C, 1, 1, 11).contiguous(), padding=(0, 5),
                     groups=C)
        return t[0].permute(1, 2, 0)

    mu_a, mu_b = blur(a), blur(b)
    saa = blur(a * a) - mu_a * mu_a
    sbb = blur(b * b) - mu_b * mu_b
    sab = blur(a * b) - mu_a * mu_b
    c1, c2 = 0.01 ** 2, 0.03 ** 2
    m = ((2.0 * mu_a * mu_b + c1) * (2.0 * sab + c2)) / (
        (mu_a * mu_a + mu_b * mu_b + c1) * (saa + sbb + c2))
    return float(m.mean())


def evaluate(scene, cameras, targets_display, lut=None, *, device=None) -> dict:
    """Mean PSNR / SSIM of a scene against display-space targets
    (training.py:325-339): each view rendered and shaded on the GPU
    (per-primitive sampling), display transform, both images clipped to
    [0, 1]."""
    from .environment import BrdfLut
    from .rasterize import render_forward as _rf
    from .shading import shade_gbuffer as _sg
    dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
    lut = lut if lut is not None else BrdfLut.build(device=dev)
    ps, ss = [], []
    for cam, tgt in zip(cameras, targets_display):
        color = _sg(_rf(scene, cam, "perprim"), cam, scene.environment, lut,
                    background=scene.background).color
        disp = linear_to_display(color.to(torch.float64)).clamp(0.0, 1.0)
        t = _target_tensor(tgt, dev).to(torch.float64)
        if t.dim() == 2:
            t = t.unsqueeze(-1).expand(-1, -1, 3)
        t = t.clamp(0.0, 1.0)
        ps.append(_psnr_from_mse(float(((disp - t) ** 2).mean())))
        ss.append(_ssim_torch(disp, t))
    return {"psnr": float(np.mean(ps)), "ssim": float(np.mean(ss))}


def _dist_on() -> bool:
    import torch.distributed as dist
    return dist.is_available() and dist.is_initialized()


def _world(group) -> int:
    import torch.distributed as dist
    return dist.get_world_size(group)


# ---------------------------------------------------------------------------
# train (training.py:38-66, :224-322)
# ---------------------------------------------------------------------------
@dataclass
class TrainConfig:
    """Optimization schedule and learning rates (training.py:38-66)."""

    iterations: int = 400
    stage_split: int = -1            # -1: iterations // 2
    texture_resolution: int = 4
    use_textures: bool = True        # False keeps 1x1 charts throughout
    lr_position: float = 1.6e-4      # scaled by initial scene extent
    lr_frame: float = 1e-3
    lr_scale: float = 1e-3
    lr_opacity: float = 5e-2
    lr_texel: float = 2.5e-3
    lr_sh: float = 2.5e-3
    lr_env: float = 1e-2
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8
    prune_interval: int = 500
    prune_opacity: float = 0.005
    optimize_environment: bool = True
    optimize_geometry: bool = True
    weights: LossWeights = field(default_factory=LossWeights)
    seed: int = 0
    threads: int = 1

    def split_iteration(self) -> int:
        return self.iterations // 2 if self.stage_split < 0 else self.stage_split


HISTORY_KEYS = ("iteration", "stage", "loss", "image", "normal", "smooth", "psnr", "fragments",
                "splats")


def train(scene, cameras, targets_display, config: TrainConfig, lut=None, log_path=None, *,
          device=None, group=None, deterministic: bool = False):
    """Two-stage fit against display-space target images (training.py:224-322)
    on the GPU: per iteration one random view (numpy default_rng(seed), the
    reference's schedule), compute_step's kernels, Adam with the reference's
    projections, the stage-2 chart broadcast with the texel Adam reset,
    opacity pruning every `prune_interval` stage-1 iterations, and the
    non-finite-loss guard. Loss terms accumulate in a device history and are
    read back once at the end (and at pruning steps, which need the kept
    count); a diverged iteration stops all later updates on the device and
    raises RuntimeError like the reference. Under torch.distributed each rank
    draws its views from default_rng(seed + rank) and the gradients are
    averaged (data parallel: a different trajectory from single-view SGD,
    SURVEY.md §8(e)). deterministic=True: bitwise-repeatable runs
    (fixed-point gradient accumulation, tsb_render_backward_ex).
    Returns (fitted Scene, history list of dicts)."""
    import csv

    from .environment import BrdfLut
    from .scene import scene_texels as _texels
    dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
    if lut is None:
        lut = BrdfLut.build(device=dev)
    rank = 0
    if _dist_on():
        import torch.distributed as dist
        rank = dist.get_rank(group)
    rng = np.random.default_rng(config.seed + rank)
    extent = world_extent(scene.positions)
    split = config.split_iteration()
    lr = {"positions": config.lr_position * extent, "tangent_u": config.lr_frame,
          "tangent_v": config.lr_frame, "scales": config.lr_scale,
          "opacities": config.lr_opacity, "sh": config.lr_sh, "texels": config.lr_texel,
          "env": config.lr_env}
    _texels(scene)  # (validates the texture source)
    tr = DataParallelTrainer(scene, lut, lr=lr, weights=config.weights, device=dev, group=group,
                             betas=(config.beta1, config.beta2), eps=config.eps,
                             optimize_geometry=config.optimize_geometry,
                             optimize_environment=config.optimize_environment,
                             deterministic=deterministic)
    targets = [_target_tensor(t, dev) for t in targets_display]
    n_it = int(config.iterations)
    hist = torch.zeros((max(n_it, 1), 9), dtype=torch.float64, device=dev)
    stages, splats, sizes = [], [], []
    for it in range(n_it):
        stage = 1 if it < split else 2
        if it == split and config.use_textures:
            tr.broadcast_textures(config.texture_resolution)
        view = int(rng.integers(0, len(cameras)))
        cam = cameras[view]
        tr.step(cam, targets[view], terms=hist[it, :8])
        hist[it, 8] = tr._last_gbuf.pixels.n_contrib.sum(dtype=torch.int64).double()
        if stage == 1 and it > 0 and it % config.prune_interval == 0:
            tr.prune(config.prune_opacity)
        stages.append(stage)
        splats.append(tr.P)
        sizes.append(3 * int(cam.width) * int(cam.height))
    h = hist.cpu().numpy()
    history = []
    w = config.weights
    for it in range(n_it):
        t = h[it]
        N = float(sizes[it])
        image = (1.0 - w.dssim) * t[0] / N + w.dssim * 0.5 * (1.0 - t[1] / N)
        normal = t[3] / max(t[4], 1.0) if w.normal > 0.0 else 0.0
        smooth = t[5] / max(t[6], 1.0) if w.smooth > 0.0 else 0.0
        loss = image + w.normal * normal + w.smooth * smooth
        if not np.isfinite(loss):
            raise RuntimeError(f"loss diverged at iteration {it}: {loss}")
        history.append({"iteration": it, "stage": stages[it], "loss": loss, "image": image,
                        "normal": normal, "smooth": smooth, "psnr": _psnr_from_mse(t[2] / N),
                        "fragments": int(t[8]), "splats": splats[it]})
    if log_path is not None:
        with open(log_path, "w", newline="") as f:
            wr = csv.writer(f)
            wr.writerow(["iteration", "stage", "loss", "image", "normal", "smooth", "psnr",
                         "splats"])
            for r in history:
                wr.writerow([r["iteration"], r["stage"], r["loss"], r["image"], r["normal"],
                             r["smooth"], r["psnr"], r["splats"]])
    return tr.to_scene(scene), history
