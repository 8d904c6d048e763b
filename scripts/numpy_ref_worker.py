"""Times the numpy reference renderer (texsplat, installed in baseline/_ref)
on crop windows of one view; prints one JSON line. Used by bench.py's CPU
baseline (single-process and one-process-per-core figures).

    python scripts/numpy_ref_worker.py [--train] SPLATS T W H ENV_H VIEW x0,y0,w,h [...]

Per crop: the reference's prepare (rasterize.py:172-243, all splats, atlas
mode incl. the page concat) and render_forward of the crop window
(rasterize.py:395-438), then shade_gbuffer (shading.py:126-183), each timed;
a crop camera renders pixels identical to the full frame.
--train: the reference's compute_step (training.py:130-184) of the cfg4 step
(init = positions + 0.003, target = the unperturbed scene's display render
of the same window), timed whole, and its prepare on its own.
"""
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT / "baseline" / "_ref"))
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402


def main():
    argv = sys.argv[1:]
    train = argv and argv[0] == "--train"
    if train:
        argv = argv[1:]
    P, T, W, H, env_h, view = (int(v) for v in argv[:6])
    crops = [tuple(int(c) for c in s.split(",")) for s in argv[6:]]
    from texsplat.environment import BrdfLut
    from texsplat.environment import EnvironmentLight as RefEnv
    from texsplat.rasterize import prepare, render_forward
    from texsplat.scene import Scene as RefScene
    from texsplat.shading import shade_gbuffer
    from texsplat.splats import Camera
    from texsplat.textures import MaterialTextureSet, TextureConfig

    from paper_2506_13348_b200 import pack_atlases, synth
    s = synth.make_shell_scene(P, T, seed=3, with_environment=True, env_height=env_h)
    scene = RefScene(positions=s.positions, tangent_u=s.tangent_u, tangent_v=s.tangent_v,
                     scales=s.scales, opacities=s.opacities, sh=s.sh, sh_degree=s.sh_degree,
                     textures=[MaterialTextureSet.from_combined(t) for t in s.texels],
                     texture_config=TextureConfig(resolution=T),
                     environment=RefEnv(list(s.environment.spec_mips), s.environment.diffuse),
                     background=np.zeros(3))
    atlas = pack_atlases(s)  # bit-identical pages (tests/test_formats.py)
    lut = BrdfLut(np.load(ROOT / "tests" / "golden" / "lut.npz")["table"])
    cam = synth.bench_cameras(256, W, H)[view]
    out = []
    if train:
        from texsplat.losses import linear_to_display
        from texsplat.training import compute_step
        init = RefScene(positions=scene.positions + 0.003, tangent_u=scene.tangent_u,
                        tangent_v=scene.tangent_v, scales=scene.scales,
                        opacities=scene.opacities, sh=scene.sh, sh_degree=scene.sh_degree,
                        textures=scene.textures, texture_config=scene.texture_config,
                        environment=scene.environment, background=scene.background)
        for x0, y0, w, h in crops:
            cc = Camera(np.asarray(cam.world_to_view), fx=cam.fx, fy=cam.fy, cx=cam.cx - x0,
                        cy=cam.cy - y0, width=w, height=h, near=cam.near, far=cam.far)
            tgt = linear_to_display(shade_gbuffer(render_forward(scene, cc), cc,
                                                  scene.environment, lut,
                                                  background=scene.background).color)
            t0 = time.perf_counter()
            prepare(init, cc, "perprim")
            t1 = time.perf_counter()
            m, _, _ = compute_step(init, cc, tgt, lut)
            t2 = time.perf_counter()
            out.append({"crop": [x0, y0, w, h], "prepare_s": t1 - t0, "step_s": t2 - t1,
                        "fragments": int(m["fragments"])})
        print(json.dumps(out), flush=True)
        return
    for x0, y0, w, h in crops:
        cc = Camera(np.asarray(cam.world_to_view), fx=cam.fx, fy=cam.fy, cx=cam.cx - x0,
                    cy=cam.cy - y0, width=w, height=h, near=cam.near, far=cam.far)
        t0 = time.perf_counter()
        prep = prepare(scene, cc, "atlas", atlas)
        t1 = time.perf_counter()
        g = render_forward(scene, cc, "atlas", atlas, prep=prep)
        t2 = time.perf_counter()
        shade_gbuffer(g, cc, scene.environment, lut, background=scene.background)
        t3 = time.perf_counter()
        out.append({"crop": [x0, y0, w, h], "prepare_s": t1 - t0, "render_s": t2 - t1,
                    "shade_s": t3 - t2, "fragments": int(g.fragment_count)})
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
