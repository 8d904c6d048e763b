"""Reference outputs at the cfg3 / cfg5 / cfg4 shapes (round-2 parity pins).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_scale.py [cfg5|cfg3|train|cfg2gb]

The numpy reference is imported read-only, here only; the GPU box reads the
committed .npz files. Scenes at 500k-2M splats come from this package's
vectorised generator (bit-identical to texsplat.synth.make_shell_scene:
tests/test_synth.py; the fixtures also carry sha256 checksums the GPU tests
re-check), converted to reference objects with
MaterialTextureSet.from_combined.

Crop windows: a crop camera (cx - x0, cy - y0, w, h) renders pixels
bit-identical to the full frame. Only the splats whose
reference rect (_cull_rects, rasterize.py:137-169) is non-empty for the crop
camera can reach it, so the reference renders that subset; the subset keeps
the relative id order, hence the same (z, id) draw order
(rasterize.py:178-182). This script asserts that the subset's rects and
depths equal the full-scene rows bit for bit before trusting it.

  cfg5_crop.npz   make_shell_scene(2M, T=16, seed=3), _lobe_environment(rng(0),
                  128, 6), bench_cameras(1, 1920, 1080)[0], two 96x96 crops
                  (centre, silhouette): per-pixel counts, 13-channel G-buffer,
                  colour, draw order (global ids), fragment counts.
  cfg3_crop.npz   make_shell_scene(500k, T=8, seed=3), bench_cameras(256, 1920,
                  1080)[37], 128x128 crop at the silhouette, env (64, 6).
  train_crop.npz  compute_step (training.py:130-184) on the cfg2/cfg4 scene
                  (100k, T=8), init = positions + 0.003, through an 80x80 crop
                  of bench_cameras(1, 800, 800)[0]; target = display(shade(
                  render(truth))) of the same crop. Loss terms, every non-zero
                  SceneGrads row (index + values) and the env gradients.
  cfg2_gbuf.npz   the full-frame cfg2 G-buffer (all 13 channels) on three
                  160x160 windows of the full 800x800 render (centre,
                  silhouette, corner of the shell).
"""

from __future__ import annotations

import hashlib
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(HERE))
sys.path.insert(0, str(HERE.parent.parent))

from make_golden import cam_dict, crop_camera, tape_counts  # noqa: E402
from texsplat.environment import BrdfLut  # noqa: E402
from texsplat.losses import linear_to_display  # noqa: E402
from texsplat.rasterize import _cull_rects, prepare, render_forward  # noqa: E402
from texsplat.scene import Scene as RefScene  # noqa: E402
from texsplat.shading import shade_gbuffer  # noqa: E402
from texsplat.synth import _lobe_environment, bench_cameras  # noqa: E402
from texsplat.textures import MaterialTextureSet, TextureConfig  # noqa: E402
from texsplat.training import compute_step  # noqa: E402

from paper_2506_13348_b200 import synth  # noqa: E402

T0 = time.time()


def log(msg):
    print(f"[{time.time() - T0:7.1f}s] {msg}", flush=True)


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def ref_scene(s, ids=None, env=None):
    """Reference Scene of (a subset of) this package's Scene."""
    sel = slice(None) if ids is None else ids
    tex = s.texels[sel]
    return RefScene(
        positions=s.positions[sel], tangent_u=s.tangent_u[sel], tangent_v=s.tangent_v[sel],
        scales=s.scales[sel], opacities=s.opacities[sel], sh=s.sh[sel], sh_degree=s.sh_degree,
        textures=[MaterialTextureSet.from_combined(t) for t in tex],
        texture_config=TextureConfig(resolution=int(tex.shape[1])),
        environment=env, background=np.zeros(3))


class _Geo:
    """Just the fields _cull_rects reads."""

    def __init__(self, s):
        self.positions, self.tangent_u, self.tangent_v = s.positions, s.tangent_u, s.tangent_v
        self.scales = s.scales

    @property
    def num_splats(self):
        return self.positions.shape[0]


def subset_for(s, cam):
    rects, view_z, keep = _cull_rects(_Geo(s), cam)
    ids = np.nonzero(keep)[0]
    return ids, rects, view_z


def render_crop(s, cam, lut, env, prefix):
    ids, rects, view_z = subset_for(s, cam)
    sub = ref_scene(s, ids, env)
    prep = prepare(sub, cam, "perprim")
    # the subset's rects / depths are the full scene's rows, bit for bit
    r2, z2, k2 = _cull_rects(sub, cam)
    assert np.array_equal(r2, rects[ids]) and np.array_equal(z2, view_z[ids]) and k2.all()
    gbuf, tape = render_forward(sub, cam, "perprim", with_tape=True, prep=prep)
    sr = shade_gbuffer(gbuf, cam, env, lut, background=sub.background)
    d = {
        f"{prefix}gbuf": gbuf.data.astype(np.float32),
        f"{prefix}counts": tape_counts(tape, cam.height, cam.width).astype(np.int16),
        f"{prefix}fragment_count": np.array(gbuf.fragment_count),
        f"{prefix}order": ids[prep.order.indices].astype(np.int32),
        f"{prefix}color": sr.color.astype(np.float32),
    }
    d.update(cam_dict(prefix + "cam_", cam))
    log(f"{prefix}: subset {ids.size} splats, {gbuf.fragment_count} fragments")
    return d


def scene_sha(s):
    return {"sha_positions": sha(s.positions), "sha_tangent_u": sha(s.tangent_u),
            "sha_scales": sha(s.scales), "sha_texels": sha(s.texels)}


def lut():
    return BrdfLut(np.load(HERE / "lut.npz")["table"])


def cfg5():
    s = synth.make_shell_scene(2_000_000, 16, seed=3)
    env = _lobe_environment(np.random.default_rng(0), height=128, levels=6)
    log("cfg5 scene")
    full = bench_cameras(1, 1920, 1080)[0]
    d = scene_sha(s)
    d.update(cam_dict("full_cam_", full))
    windows = {"c_": (912, 492, 96, 96), "s_": (1824, 492, 96, 96)}
    for pre, (x0, y0, w, h) in windows.items():
        d[pre + "crop"] = np.array([x0, y0, w, h])
        d.update(render_crop(s, crop_camera(full, x0, y0, w, h), lut(), env, pre))
    np.savez_compressed(HERE / "cfg5_crop.npz", **d)


def cfg3():
    s = synth.make_shell_scene(500_000, 8, seed=3)
    env = _lobe_environment(np.random.default_rng(0), height=64, levels=6)
    log("cfg3 scene")
    full = bench_cameras(256, 1920, 1080)[37]
    d = scene_sha(s)
    d.update(cam_dict("full_cam_", full))
    x0, y0, w, h = 1792, 476, 128, 128
    d["crop"] = np.array([x0, y0, w, h])
    d.update(render_crop(s, crop_camera(full, x0, y0, w, h), lut(), env, ""))
    np.savez_compressed(HERE / "cfg3_crop.npz", **d)


def train():
    s = synth.make_shell_scene(100_000, 8, seed=3)
    env = _lobe_environment(np.random.default_rng(0), height=64, levels=6)
    full = bench_cameras(1, 800, 800)[0]
    x0, y0, w, h = 650, 90, 80, 80
    cam = crop_camera(full, x0, y0, w, h)
    truth = ref_scene(s, None, env)
    log("train scene")
    L = lut()
    gt = render_forward(truth, cam)
    target = linear_to_display(shade_gbuffer(gt, cam, env, L, background=truth.background).color)
    init = ref_scene(s, None, env)
    init.positions = init.positions + 0.003
    metrics, gr, eg = compute_step(init, cam, target, L)
    log(f"compute_step: {metrics}")
    d = scene_sha(s)
    d.update(cam_dict("full_cam_", full))
    d.update(cam_dict("cam_", cam))
    d["crop"] = np.array([x0, y0, w, h])
    d["target"] = np.asarray(target, dtype=np.float64)
    for k in ("loss", "image", "normal", "smooth", "psnr", "fragments"):
        d[f"m_{k}"] = np.array(metrics[k])
    geo = np.concatenate([gr.positions, gr.tangent_u, gr.tangent_v, gr.scales,
                          gr.opacities[:, None], gr.sh.reshape(len(gr.opacities), -1)], axis=1)
    tex = [t is not None and np.any(t != 0) for t in gr.texels]
    nz = np.nonzero(np.any(geo != 0, axis=1) | np.array(tex))[0]
    d["nz"] = nz.astype(np.int32)
    for name in ("positions", "tangent_u", "tangent_v", "scales", "opacities", "sh"):
        d[f"g_{name}"] = getattr(gr, name)[nz]
    d["g_texels"] = np.stack([gr.texels[i] if gr.texels[i] is not None else np.zeros((8, 8, 7))
                              for i in nz]).astype(np.float64)
    for i, m in enumerate(eg.spec_mips):
        d[f"genv_mip{i}"] = m
    d["genv_diffuse"] = eg.diffuse
    log(f"train: {nz.size} splats with gradients")
    np.savez_compressed(HERE / "train_crop.npz", **d)


def cfg2gb():
    s = synth.make_shell_scene(100_000, 8, seed=3)
    env = _lobe_environment(np.random.default_rng(0), height=64, levels=6)
    full = bench_cameras(1, 800, 800)[0]
    d = scene_sha(s)
    windows = {"c_": (320, 320, 160, 160), "s_": (600, 40, 160, 160), "e_": (40, 600, 160, 160)}
    for pre, (x0, y0, w, h) in windows.items():
        d[pre + "crop"] = np.array([x0, y0, w, h])
        d.update(render_crop(s, crop_camera(full, x0, y0, w, h), lut(), env, pre))
    np.savez_compressed(HERE / "cfg2_gbuf.npz", **d)


if __name__ == "__main__":
    which = sys.argv[1:] or ["cfg2gb", "train", "cfg3", "cfg5"]
    for w in which:
        globals()[w]()
        log(f"{w} done")
