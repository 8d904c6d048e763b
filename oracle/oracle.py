"""ctypes wrapper of the CPU oracle (oracle/tsb_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference leg, as the checker or the CPU
baseline. The product path (paper_2506_13348_b200) never imports it.

The oracle restates the reference's forward path with the same decision
math as the GPU kernels (shared header tsb_math.h), so structure and the
verify-mode G-buffer are bit-exact with the GPU; it is pinned to the numpy
reference by tests/test_oracle_golden.py.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
BUILD = HERE / "_build"

_lib = None


def _cpu_has_v3() -> bool:
    try:
        flags = Path("/proc/cpuinfo").read_text()
    except OSError:
        return False
    line = next((ln for ln in flags.splitlines() if ln.startswith("flags")), "")
    have = set(line.split())
    return {"avx2", "fma", "bmi2"} <= have


def build():
    subprocess.run(["make", "-C", str(HERE)], check=True, stdout=subprocess.DEVNULL)


def lib():
    global _lib
    if _lib is not None:
        return _lib
    name = "liboracle_v3.so" if _cpu_has_v3() else "liboracle.so"
    path = BUILD / name
    if not path.exists():
        build()
    h = C.CDLL(str(path))
    P = C.c_void_p
    h.oracle_frame_new.restype = P
    h.oracle_frame_new.argtypes = [C.c_int32, C.c_int32, P, P, P, P, P, P, P, C.c_int32, C.c_int32]
    h.oracle_frame_free.argtypes = [P]
    h.oracle_frame_num_entries.restype = C.c_int64
    h.oracle_frame_num_entries.argtypes = [P]
    h.oracle_frame_num_kept.restype = C.c_int32
    h.oracle_frame_num_kept.argtypes = [P]
    h.oracle_frame_num_tiles.restype = C.c_int32
    h.oracle_frame_num_tiles.argtypes = [P]
    h.oracle_frame_export.argtypes = [P, P, P, P, P, P]
    h.oracle_frame_raster.argtypes = [P, C.c_int32, C.c_int32, C.c_int32, C.c_int32, P, P, P, P,
                                      C.c_int32, P, P, P, P, P]
    h.oracle_frame_set_binning.argtypes = [P, C.c_int32]
    h.oracle_frame_entry_stats.argtypes = [P, P, P]
    h.oracle_shade.argtypes = [P, P, C.c_int32, P, P, P, C.c_int32, C.c_int32, P, C.c_int32, P,
                               C.c_int32, P, P, P]
    _lib = h
    return h


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


class _Cam(C.Structure):
    _fields_ = [("w2v", C.c_double * 16), ("fx", C.c_double), ("fy", C.c_double),
                ("cx", C.c_double), ("cy", C.c_double), ("near", C.c_double),
                ("far", C.c_double), ("width", C.c_int32), ("height", C.c_int32)]


def cam_struct(cam) -> _Cam:
    c = _Cam()
    c.w2v[:] = [float(v) for v in np.asarray(cam.world_to_view, np.float64).ravel()]
    c.fx, c.fy, c.cx, c.cy = float(cam.fx), float(cam.fy), float(cam.cx), float(cam.cy)
    c.near, c.far = float(cam.near), float(cam.far)
    c.width, c.height = int(cam.width), int(cam.height)
    return c


def _texels(scene):
    t = getattr(scene, "texels", None)
    if isinstance(t, np.ndarray):
        return t
    return np.stack([s.combined() for s in scene.textures]).astype(np.float32)


def pack(texels, max_dim=4096):
    """Atlas pages + entries in the reference layout (atlas.py:127-167)."""
    P, T = texels.shape[0], texels.shape[1]
    charts_x = max_dim // T
    charts_y = min(max_dim // T, -(-P // charts_x))
    per_page = charts_x * charts_y
    pages = -(-P // per_page)
    k = np.arange(P)
    page, idx = np.divmod(k, per_page)
    cy, cx = np.divmod(idx, charts_x)
    entries = np.stack([cx, cy, page], axis=1).astype(np.int32)
    full = np.zeros((pages * per_page, T, T, 7), np.float32)
    full[:P] = texels
    g = full.reshape(pages, charts_y, charts_x, T, T, 7).transpose(0, 1, 3, 2, 4, 5)
    g = g.reshape(pages, charts_y * T, charts_x * T, 7)
    fa = np.ascontiguousarray(g[..., 0:4])
    fb = np.zeros_like(fa)
    fb[..., 0:2] = g[..., 5:7]
    fb[..., 2] = g[..., 4]
    return fa, fb, entries


def flat_attrs(texels):
    P = texels.shape[0]
    out = np.zeros((P, 5), np.float32)
    for k in range(P):
        b = texels[k]
        out[k, 0:3] = np.ascontiguousarray(b[:, :, 0:3]).reshape(-1, 3).mean(axis=0)
        out[k, 3] = np.ascontiguousarray(b[:, :, 4:5]).mean()
        out[k, 4] = np.ascontiguousarray(b[:, :, 3:4]).mean()
    return out


def render(scene, cam, mode="verify", tile=16, threads=0, atlas=None, binning="box"):
    """Oracle forward. mode 'verify' (fp32 SW bilinear) or 'flat'.
    binning: "rect" = the reference's _tile_lists (rasterize.py:246-258),
    "box" = rect ∩ alpha-cut ellipse box (what the GPU bins with); pixels
    are identical under both when the box is conservative.
    atlas: optional (fam_a, fam_b, entries) from pack(); packed here if None.
    Returns dict with gbuf (13,H,W) f32, n_contrib, last_entry, final_T,
    T_last (H,W), sorted_ids (P,), keys (E,), ranges (tiles,2), rects (P,4),
    view_z (P,), num_kept."""
    L = lib()
    P = int(scene.positions.shape[0])
    K = (int(scene.sh_degree) + 1) ** 2
    arrs = [np.ascontiguousarray(getattr(scene, n), np.float64) for n in
            ("positions", "tangent_u", "tangent_v", "scales", "opacities")]
    sh = np.ascontiguousarray(scene.sh, np.float64).reshape(P, K, 3)
    c = cam_struct(cam)
    f = L.oracle_frame_new(P, int(scene.sh_degree), *[_p(a) for a in arrs], _p(sh), C.byref(c),
                           tile, threads)
    try:
        L.oracle_frame_set_binning(f, 1 if binning == "box" else 0)
        E = L.oracle_frame_num_entries(f)
        NT = L.oracle_frame_num_tiles(f)
        sorted_ids = np.empty(max(P, 1), np.int32)
        keys = np.empty(max(E, 1), np.int64)
        ranges = np.empty((NT, 2), np.int32)
        rects = np.empty((max(P, 1), 4), np.int32)
        view_z = np.empty(max(P, 1), np.float64)
        L.oracle_frame_export(f, _p(sorted_ids), _p(keys), _p(ranges), _p(rects), _p(view_z))
        texels = _texels(scene)
        T = int(texels.shape[1])
        if mode == "flat":
            fa = fb = ent = None
            fl = flat_attrs(texels)
            pw = ph = 0
            m = 2
        else:
            fa, fb, ent = atlas if atlas is not None else pack(texels)
            fl = None
            ph, pw = int(fa.shape[1]), int(fa.shape[2])
            m = 1
        H, W = int(cam.height), int(cam.width)
        gbuf = np.empty((13, H, W), np.float32)
        n = np.empty((H, W), np.int32)
        le = np.empty((H, W), np.int32)
        fT = np.empty((H, W), np.float32)
        Tl = np.empty((H, W), np.float32)
        L.oracle_frame_raster(f, m, T, pw, ph, _p(ent), _p(fa), _p(fb), _p(fl), threads,
                              _p(gbuf), _p(n), _p(le), _p(fT), _p(Tl))
        return {"gbuf": gbuf, "n_contrib": n, "last_entry": le, "final_T": fT, "T_last": Tl,
                "sorted_ids": sorted_ids[:P], "keys": keys[:E], "ranges": ranges,
                "rects": rects[:P], "view_z": view_z[:P],
                "num_kept": L.oracle_frame_num_kept(f)}
    finally:
        L.oracle_frame_free(f)


def shade(gbuf, cam, env, lut_table, background=None, threads=0):
    """Oracle shade_gbuffer (mesh=None); gbuf planar (13,H,W) float32."""
    L = lib()
    H, W = int(cam.height), int(cam.width)
    mips = np.concatenate([np.ascontiguousarray(m, np.float32).ravel() for m in env.spec_mips])
    hw = np.array([[m.shape[0], m.shape[1]] for m in env.spec_mips], np.int32).ravel()
    diff = np.ascontiguousarray(env.diffuse, np.float32)
    lut = np.ascontiguousarray(lut_table, np.float32)
    bg = np.asarray([0, 0, 0] if background is None else background, np.float32)
    color = np.empty((H, W, 3), np.float32)
    dif = np.empty_like(color)
    spe = np.empty_like(color)
    c = cam_struct(cam)
    g = np.ascontiguousarray(gbuf, np.float32)
    L.oracle_shade(_p(g), C.byref(c), len(env.spec_mips), _p(mips), _p(hw), _p(diff),
                   diff.shape[0], diff.shape[1], _p(lut), lut.shape[0], _p(bg), threads,
                   _p(color), _p(dif), _p(spe))
    return color, dif, spe


def cpu_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1
