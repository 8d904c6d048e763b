"""Image-based lighting inputs (mirrors texsplat.environment).

Reference: environment.py:28-464. The per-frame samplers run on the GPU
inside k_shade (tsb_math.h tsb_sample_equirect / tsb_sample_specular /
tsb_sample_lut). This module holds the host-side containers and the one-time
precompute (GGX prefilter, cosine irradiance, split-sum LUT). The precompute
runs on the GPU (K15 tsb_env_prefilter, K16 tsb_brdf_lut; pass `device=`);
the vectorised numpy restatement kept here is the host checker those kernels
are tested against (bit-identical to the reference's numpy).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

TWO_PI = 2.0 * np.pi


def equirect_dirs(height: int, width: int) -> np.ndarray:
    """Unit directions at texel centres, (H, W, 3), z-up (environment.py:28-38)."""
    theta = (np.arange(height) + 0.5) / height * np.pi
    phi = (np.arange(width) + 0.5) / width * TWO_PI
    st, ct = np.sin(theta), np.cos(theta)
    return np.stack([st[:, None] * np.cos(phi)[None, :], st[:, None] * np.sin(phi)[None, :],
                     np.broadcast_to(ct[:, None], (height, width))], axis=-1)


def equirect_solid_angles(height: int, width: int) -> np.ndarray:
    theta = (np.arange(height) + 0.5) / height * np.pi
    w = np.sin(theta) * (np.pi / height) * (TWO_PI / width)
    return np.broadcast_to(w[:, None], (height, width)).copy()


def downsample2(grid) -> np.ndarray:
    h, w = grid.shape[:2]
    g = grid[:(h // 2) * 2, :(w // 2) * 2].astype(np.float64)
    return g.reshape(h // 2, 2, w // 2, 2, -1).mean(axis=(1, 3))


def ggx_ndf(cos_h, alpha):
    a2 = alpha * alpha
    d = cos_h * cos_h * (a2 - 1.0) + 1.0
    return a2 / (np.pi * d * d)


def prefilter_specular(base, roughness: float, out_height: int, out_width: int,
                       chunk: int = 512) -> np.ndarray:
    """GGX-weighted prefilter with the n = v = r approximation (environment.py:147-176)."""
    if roughness <= 0.0:
        raise ValueError("prefilter needs roughness > 0; level 0 is the base")
    src = downsample2(base)
    sh_, sw_ = src.shape[:2]
    in_dirs = equirect_dirs(sh_, sw_).reshape(-1, 3)
    in_rad = src.reshape(-1, 3)
    d_omega = equirect_solid_angles(sh_, sw_).reshape(-1)
    out_dirs = equirect_dirs(out_height, out_width).reshape(-1, 3)
    alpha = roughness * roughness
    out = np.empty((out_dirs.shape[0], 3))
    for s in range(0, out_dirs.shape[0], chunk):
        c = np.clip(out_dirs[s:s + chunk] @ in_dirs.T, -1.0, 1.0)
        w = np.where(c > 0.0, ggx_ndf(np.sqrt(0.5 * (1.0 + c)), alpha) * c, 0.0) * d_omega
        out[s:s + chunk] = (w @ in_rad) / np.maximum(w.sum(axis=1, keepdims=True), 1e-30)
    return out.reshape(out_height, out_width, 3)


def diffuse_irradiance(base, out_height: int, out_width: int, chunk: int = 1024) -> np.ndarray:
    """Cosine-weighted irradiance E(N) (environment.py:179-195)."""
    src = downsample2(base)
    sh_, sw_ = src.shape[:2]
    in_dirs = equirect_dirs(sh_, sw_).reshape(-1, 3)
    in_rad = src.reshape(-1, 3) * equirect_solid_angles(sh_, sw_).reshape(-1, 1)
    out_dirs = equirect_dirs(out_height, out_width).reshape(-1, 3)
    out = np.empty((out_dirs.shape[0], 3))
    for s in range(0, out_dirs.shape[0], chunk):
        out[s:s + chunk] = np.maximum(out_dirs[s:s + chunk] @ in_dirs.T, 0.0) @ in_rad
    return out.reshape(out_height, out_width, 3)


@dataclass
class EnvGrads:
    """Gradient accumulators matching EnvironmentLight parameters."""

    spec_mips: list
    diffuse: np.ndarray

    def scaled(self, s: float) -> "EnvGrads":
        return EnvGrads([g * s for g in self.spec_mips], self.diffuse * s)


class EnvironmentLight:
    """Specular mip pyramid (independent grids) + diffuse irradiance, float32."""

    def __init__(self, spec_mips, diffuse):
        self.spec_mips = [np.ascontiguousarray(m, dtype=np.float32) for m in spec_mips]
        self.diffuse = np.ascontiguousarray(diffuse, dtype=np.float32)
        for m in self.spec_mips:
            if m.ndim != 3 or m.shape[2] != 3:
                raise ValueError("mip grids must be (H, W, 3)")
        if self.diffuse.ndim != 3 or self.diffuse.shape[2] != 3:
            raise ValueError("diffuse grid must be (H, W, 3)")

    @property
    def levels(self) -> int:
        return len(self.spec_mips)

    @staticmethod
    def from_base(base, levels: int = 6, diffuse_height: int = 32,
                  device=None) -> "EnvironmentLight":
        """Level l is max(4, h>>l) x max(8, w>>l) at roughness l/(levels-1)
        (environment.py:231-244). With `device` the quadratures run on the
        GPU (K15-K16, tsb_env_prefilter; fp64 sums in another order, so
        float32-rounding-level differences); without, this host restatement
        is bit-identical to the reference."""
        if device is not None:
            return EnvironmentLight._from_base_device(base, levels, diffuse_height, device)
        base = np.asarray(base, dtype=np.float64)
        h, w = base.shape[:2]
        mips = [base.astype(np.float32)]
        for level in range(1, levels):
            mips.append(prefilter_specular(base, level / (levels - 1), max(4, h >> level),
                                           max(8, w >> level)).astype(np.float32))
        dh = min(diffuse_height, h)
        return EnvironmentLight(mips, diffuse_irradiance(base, dh, 2 * dh).astype(np.float32))

    @staticmethod
    def _from_base_device(base, levels, diffuse_height, device):
        import ctypes as C

        import torch

        from . import _lib
        b = torch.as_tensor(np.ascontiguousarray(base, np.float64), device=device)
        h, w = int(b.shape[0]), int(b.shape[1])
        if not 1 <= levels <= _lib.ENV_MAX_LEVELS:
            raise ValueError("levels out of range")
        hs = [h] + [max(4, h >> l) for l in range(1, levels)]
        ws = [w] + [max(8, w >> l) for l in range(1, levels)]
        mips = [torch.empty((hh, ww, 3), dtype=torch.float32, device=device)
                for hh, ww in zip(hs, ws)]
        dh = min(diffuse_height, h)
        diff = torch.empty((dh, 2 * dh, 3), dtype=torch.float32, device=device)
        L = _lib.lib()
        nb = C.c_uint64()
        _lib.check(L.tsb_env_scratch_size(h, w, C.byref(nb)), "tsb_env_scratch_size")
        scratch = torch.empty(int(nb.value), dtype=torch.uint8, device=device)
        ptrs = (C.c_void_p * levels)(*[_lib.ptr(m) for m in mips])
        _lib.check(L.tsb_env_prefilter(_lib.ptr(b), h, w, levels, ptrs,
                                       (C.c_int32 * levels)(*hs), (C.c_int32 * levels)(*ws),
                                       _lib.ptr(diff), dh, 2 * dh, _lib.ptr(scratch),
                                       int(nb.value), _lib.stream_handle()), "tsb_env_prefilter")
        torch.cuda.current_stream().synchronize()
        return EnvironmentLight([m.cpu().numpy() for m in mips], diff.cpu().numpy())

    @staticmethod
    def constant(value, height: int = 64, levels: int = 6) -> "EnvironmentLight":
        value = np.asarray(value, dtype=np.float32) * np.ones(3, np.float32)
        mips = []
        for level in range(levels):
            oh = max(4, height >> level)
            mips.append(np.broadcast_to(value, (oh, 2 * oh, 3)).copy())
        dh = min(32, height)
        diff = np.full((dh, 2 * dh, 3), np.pi, dtype=np.float64) * value
        return EnvironmentLight(mips, diff.astype(np.float32))

    def parameters(self):
        return list(self.spec_mips) + [self.diffuse]

    def copy(self) -> "EnvironmentLight":
        return EnvironmentLight([m.copy() for m in self.spec_mips], self.diffuse.copy())

    def zero_grads(self) -> EnvGrads:
        return EnvGrads([np.zeros(m.shape) for m in self.spec_mips], np.zeros(self.diffuse.shape))


def hammersley(n: int) -> np.ndarray:
    """First n Hammersley points in [0,1)^2 (environment.py:341-355)."""
    i = np.arange(n, dtype=np.uint64)
    bits = i.copy()
    rev = np.zeros_like(bits)
    for b in range(32):
        rev |= ((bits >> np.uint64(b)) & np.uint64(1)) << np.uint64(31 - b)
    return np.stack([i.astype(np.float64) / n, rev.astype(np.float64) * 2.3283064365386963e-10],
                    axis=1)


class BrdfLut:
    """Split-sum (A, B) table over (cos_theta, roughness) (environment.py:362-425).

    table[j, i] = (A, B) at cos = (i+0.5)/res, rough = (j+0.5)/res; GGX
    importance sampling over Hammersley points, Smith-IBL k = r^2/2.
    """

    def __init__(self, table):
        table = np.asarray(table, dtype=np.float64)
        if table.ndim != 3 or table.shape[2] != 2 or table.shape[0] != table.shape[1]:
            raise ValueError("LUT table must be (res, res, 2)")
        self.table = table

    @property
    def resolution(self) -> int:
        return self.table.shape[0]

    @staticmethod
    def build(resolution: int = 64, samples: int = 2048, device=None) -> "BrdfLut":
        """BrdfLut.build (environment.py:381-390). With `device` the table is
        integrated on the GPU (K16, tsb_brdf_lut)."""
        if device is not None:
            import torch

            from . import _lib
            t = torch.empty((resolution, resolution, 2), dtype=torch.float64, device=device)
            _lib.check(_lib.lib().tsb_brdf_lut(resolution, samples, _lib.ptr(t),
                                               _lib.stream_handle()), "tsb_brdf_lut")
            return BrdfLut(t.cpu().numpy())
        return BrdfLut._build_host(resolution, samples)

    @staticmethod
    def _build_host(resolution: int = 64, samples: int = 2048) -> "BrdfLut":
        xi = hammersley(samples)
        phi = TWO_PI * xi[:, 0]
        cphi, sphi = np.cos(phi), np.sin(phi)
        table = np.empty((resolution, resolution, 2))
        cos_v = np.maximum((np.arange(resolution) + 0.5) / resolution, 1e-8)   # (R,)
        sin_v = np.sqrt(np.maximum(0.0, 1.0 - cos_v * cos_v))
        for j in range(resolution):
            r = (j + 0.5) / resolution
            alpha = r * r
            cos_h = np.sqrt((1.0 - xi[:, 1]) / (1.0 + (alpha * alpha - 1.0) * xi[:, 1]))
            sin_h = np.sqrt(np.maximum(0.0, 1.0 - cos_h * cos_h))
            hx, hy, hz = sin_h * cphi, sin_h * sphi, cos_h                     # (S,)
            voh = hx[None, :] * sin_v[:, None] + hz[None, :] * cos_v[:, None]  # (R, S)
            nol = 2.0 * voh * hz[None, :] - cos_v[:, None]
            live = nol > 0.0
            noh = np.maximum(cos_h, 1e-8)[None, :]
            voh_c = np.maximum(voh, 1e-8)
            k = alpha / 2.0
            g1v = cos_v / (cos_v * (1.0 - k) + k)
            nl = np.maximum(nol, 1e-8)
            g1l = nl / (nl * (1.0 - k) + k)
            G = g1v[:, None] * g1l
            gvis = np.where(live, G * voh_c / (noh * cos_v[:, None]), 0.0)
            fc = (1.0 - voh_c) ** 5
            table[j, :, 0] = np.mean((1.0 - fc) * gvis, axis=1)
            table[j, :, 1] = np.mean(fc * gvis, axis=1)
        return BrdfLut(table)
