"""Generate the golden fixtures under tests/golden/ from the numpy reference.

Run in the dev container (the reference is importable only there):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

The reference is imported read-only; nothing here is used at run time on the
GPU box, which only reads the committed .npz files. Every fixture stores the
inputs it was rendered from (or, for the 100k-splat scene, checksums that our
own generator must reproduce) plus the reference outputs:

  cfg1.npz      BASELINE configs[0]: make_plane_scene(32, 32, T=4, seed=7),
                camera_ring(1, 128, 128)[0]; G-buffer, per-pixel contributor
                counts (from the tape), draw order, rects, shaded outputs.
  lut.npz       BrdfLut.build() (64 x 64 x 2), shared by every shading test.
  small.npz     make_plane_scene(3, 3, T=4, seed=7) at 48 x 40 (tile/thread
                invariance scene of test_rasterize.py:81-88) and the flat-mode
                scene make_plane_scene(2, 2, T=4, seed=5) at 32 x 32
                (test_rasterize.py:116-123).
  cfg2_crop.npz BASELINE configs[1] scene make_shell_scene(100000, 8, seed=3)
                with _lobe_environment(default_rng(0), 64, 6), rendered
                through a 128 x 128 crop of bench_cameras(1, 800, 800)[0]
                (crop windows are pixel-identical to the full frame).
  backward.npz  splat_backward / shade_backward / compute_step gradients on
                the reference's own FD scenes (test_rasterize.py:173-200,
                test_shading.py:260-315, training.py:130-184).
"""

from __future__ import annotations

import hashlib
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")

from texsplat.environment import BrdfLut  # noqa: E402
from texsplat.rasterize import prepare, render_forward, splat_backward  # noqa: E402
from texsplat.shading import shade_backward, shade_gbuffer  # noqa: E402
from texsplat.splats import Camera  # noqa: E402
from texsplat.synth import (_lobe_environment, bench_cameras, camera_ring,  # noqa: E402
                            make_gradcheck_scene, make_plane_scene,
                            make_shell_scene)

OUT = Path(__file__).resolve().parent


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def cam_dict(prefix, cam):
    return {
        f"{prefix}w2v": cam.world_to_view,
        f"{prefix}intr": np.array([cam.fx, cam.fy, cam.cx, cam.cy, cam.near, cam.far]),
        f"{prefix}size": np.array([cam.width, cam.height], dtype=np.int64),
    }


def scene_dict(prefix, scene, with_texels=True):
    d = {
        f"{prefix}positions": scene.positions,
        f"{prefix}tangent_u": scene.tangent_u,
        f"{prefix}tangent_v": scene.tangent_v,
        f"{prefix}scales": scene.scales,
        f"{prefix}opacities": scene.opacities,
        f"{prefix}sh": scene.sh,
        f"{prefix}sh_degree": np.array(scene.sh_degree),
        f"{prefix}background": scene.background,
    }
    if with_texels:
        d[f"{prefix}texels"] = np.stack([t.combined() for t in scene.textures])
    if scene.environment is not None:
        env = scene.environment
        for i, m in enumerate(env.spec_mips):
            d[f"{prefix}env_mip{i}"] = m
        d[f"{prefix}env_levels"] = np.array(env.levels)
        d[f"{prefix}env_diffuse"] = env.diffuse
    return d


def tape_counts(tape, H, W):
    """Per-pixel composited-fragment counts from the reference tape."""
    counts = np.zeros(H * W, dtype=np.int32)
    for bounds, records in tape:
        tx0, ty0, tx1, ty1 = bounds
        tw = tx1 - tx0
        for k, idx, *_ in records:
            py = ty0 + idx // tw
            px = tx0 + idx % tw
            np.add.at(counts, py * W + px, 1)
    return counts.reshape(H, W)


def render_case(prefix, scene, cam, lut, mode="perprim", atlas=None, shade=True):
    prep = prepare(scene, cam, mode, atlas)
    gbuf, tape = render_forward(scene, cam, mode, atlas, with_tape=True, prep=prep)
    d = {
        f"{prefix}gbuf": gbuf.data.astype(np.float64),
        f"{prefix}fragment_count": np.array(gbuf.fragment_count),
        f"{prefix}counts": tape_counts(tape, cam.height, cam.width),
        f"{prefix}order": prep.order.indices.astype(np.int64),
        f"{prefix}rects": prep.rects.astype(np.int64),
    }
    if shade and scene.environment is not None:
        sr = shade_gbuffer(gbuf, cam, scene.environment, lut, background=scene.background)
        d[f"{prefix}color"] = sr.color
        d[f"{prefix}diffuse"] = sr.diffuse
        d[f"{prefix}specular"] = sr.specular
    return d


def crop_camera(cam: Camera, x0, y0, w, h) -> Camera:
    return Camera(cam.world_to_view.copy(), fx=cam.fx, fy=cam.fy, cx=cam.cx - x0,
                  cy=cam.cy - y0, width=w, height=h, near=cam.near, far=cam.far)


def main():
    t0 = time.time()
    lut = BrdfLut.build()
    np.savez_compressed(OUT / "lut.npz", table=lut.table)
    print(f"lut {time.time() - t0:.1f}s", flush=True)

    # ---- cfg1 -------------------------------------------------------------
    scene = make_plane_scene(nx=32, ny=32, texture_res=4, seed=7)
    cam = camera_ring(1, width=128, height=128)[0]
    d = {}
    d.update(scene_dict("", scene))
    d.update(cam_dict("cam_", cam))
    d.update(render_case("", scene, cam, lut))
    np.savez_compressed(OUT / "cfg1.npz", **d)
    print(f"cfg1 {time.time() - t0:.1f}s frags={d['fragment_count']}", flush=True)

    # ---- small scenes ------------------------------------------------------
    d = {}
    s1 = make_plane_scene(nx=3, ny=3, texture_res=4, seed=7)
    c1 = camera_ring(1, width=48, height=40)[0]
    d.update(scene_dict("inv_", s1))
    d.update(cam_dict("inv_cam_", c1))
    d.update(render_case("inv_", s1, c1, lut))
    s2 = make_plane_scene(nx=2, ny=2, texture_res=4, seed=5)
    c2 = camera_ring(1, width=32, height=32)[0]
    d.update(scene_dict("flat_", s2))
    d.update(cam_dict("flat_cam_", c2))
    d.update(render_case("flat_", s2, c2, lut, mode="flat"))
    d.update(render_case("flatp_", s2, c2, lut, mode="perprim"))
    np.savez_compressed(OUT / "small.npz", **d)
    print(f"small {time.time() - t0:.1f}s", flush=True)

    # ---- backward ----------------------------------------------------------
    d = {}
    sb = make_plane_scene(nx=2, ny=2, texture_res=2, seed=13)
    cb = camera_ring(1, width=16, height=16)[0]
    Wg = np.random.default_rng(0).normal(size=(16, 16, 13))
    prep = prepare(sb, cb)
    gbuf, tape = render_forward(sb, cb, with_tape=True, prep=prep)
    gr = splat_backward(sb, cb, prep, tape, Wg)
    d.update(scene_dict("bw_", sb))
    d.update(cam_dict("bw_cam_", cb))
    d["bw_dbuf"] = Wg
    d["bw_gbuf"] = gbuf.data
    for name in ("positions", "tangent_u", "tangent_v", "scales", "opacities", "sh"):
        d[f"bw_g_{name}"] = getattr(gr, name)
    d["bw_g_texels"] = np.stack([t if t is not None else np.zeros((2, 2, 7))
                                 for t in gr.texels])
    # gradcheck scene: full G-buffer + shading adjoints on a random dcolor
    sg = make_gradcheck_scene(seed=11)
    cg = camera_ring(1, width=32, height=32)[0]
    prep = prepare(sg, cg)
    gbuf, tape = render_forward(sg, cg, with_tape=True, prep=prep)
    sr = shade_gbuffer(gbuf, cg, sg.environment, lut, background=sg.background)
    dcolor = np.random.default_rng(1).normal(size=(32, 32, 3))
    dgbuf, eg = shade_backward(sr, cg, sg.environment, lut, dcolor)
    gr = splat_backward(sg, cg, prep, tape, dgbuf)
    d.update(scene_dict("gc_", sg))
    d.update(cam_dict("gc_cam_", cg))
    d["gc_gbuf"] = gbuf.data
    d["gc_color"] = sr.color
    d["gc_dcolor"] = dcolor
    d["gc_dgbuf"] = dgbuf
    for i, m in enumerate(eg.spec_mips):
        d[f"gc_genv_mip{i}"] = m
    d["gc_genv_diffuse"] = eg.diffuse
    for name in ("positions", "tangent_u", "tangent_v", "scales", "opacities", "sh"):
        d[f"gc_g_{name}"] = getattr(gr, name)
    d["gc_g_texels"] = np.stack([t if t is not None else np.zeros((4, 4, 7))
                                 for t in gr.texels])
    np.savez_compressed(OUT / "backward.npz", **d)
    print(f"backward {time.time() - t0:.1f}s", flush=True)

    # ---- compute_step (training.py:130-184) --------------------------------
    from texsplat.losses import linear_to_display
    from texsplat.training import compute_step
    truth = make_gradcheck_scene(seed=11)
    ct = camera_ring(1, width=32, height=32)[0]
    gt = render_forward(truth, ct)
    target = linear_to_display(shade_gbuffer(gt, ct, truth.environment, lut,
                                             background=truth.background).color)
    init = truth.copy()
    init.positions = init.positions + 0.003
    metrics, gr, eg = compute_step(init, ct, target, lut)
    d = {}
    d.update(scene_dict("st_", init))
    d.update(cam_dict("st_cam_", ct))
    d["st_target"] = target
    for k in ("loss", "image", "normal", "smooth", "psnr", "fragments"):
        d[f"st_m_{k}"] = np.array(metrics[k])
    for name in ("positions", "tangent_u", "tangent_v", "scales", "opacities", "sh"):
        d[f"st_g_{name}"] = getattr(gr, name)
    d["st_g_texels"] = np.stack([t if t is not None else np.zeros((4, 4, 7)) for t in gr.texels])
    for i, m in enumerate(eg.spec_mips):
        d[f"st_genv_mip{i}"] = m
    d["st_genv_diffuse"] = eg.diffuse
    np.savez_compressed(OUT / "train.npz", **d)
    print(f"train {time.time() - t0:.1f}s", flush=True)

    # ---- cfg2 crop ---------------------------------------------------------
    shell = make_shell_scene(100_000, 8, seed=3)
    shell.environment = _lobe_environment(np.random.default_rng(0), height=64, levels=6)
    print(f"shell built {time.time() - t0:.1f}s", flush=True)
    full = bench_cameras(1, 800, 800)[0]
    x0, y0, w, h = 336, 336, 128, 128
    cc = crop_camera(full, x0, y0, w, h)
    d = {
        "sha_positions": sha(shell.positions), "sha_tangent_u": sha(shell.tangent_u),
        "sha_tangent_v": sha(shell.tangent_v), "sha_scales": sha(shell.scales),
        "sha_texels": sha(np.stack([t.combined() for t in shell.textures])),
        "crop": np.array([x0, y0, w, h]),
    }
    d.update(scene_dict("", shell, with_texels=False))
    for k in ("positions", "tangent_u", "tangent_v", "scales", "opacities", "sh"):
        d.pop(k)
    d.update(cam_dict("full_cam_", full))
    d.update(cam_dict("cam_", cc))
    rc = render_case("", shell, cc, lut)
    rc.pop("rects")
    d.update(rc)
    np.savez_compressed(OUT / "cfg2_crop.npz", **d)
    print(f"cfg2 crop {time.time() - t0:.1f}s frags={d['fragment_count']}", flush=True)


if __name__ == "__main__":
    main()
