"""Reference train() history for the GPU train loop's parity test.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_train.py

A 4 x 3 plane scene at T=1 (stage 1) fitted for 24 iterations: the stage-2
broadcast to T=4 with the texel Adam reset at iteration 12, opacity pruning
every 5 stage-1 iterations (three extra splats far outside every view, at
opacity 0.001, are pruned at iteration 5), the reference's Adam and
projections (training.py:224-322). Stores the inputs (scene arrays, cameras,
display targets), the config, the per-iteration history and the fitted
parameters, plus a stage-1-only run (12 iterations) whose fitted parameters
are compared tightly.
"""
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(HERE))

from make_golden import cam_dict, scene_dict  # noqa: E402
from texsplat.environment import BrdfLut  # noqa: E402
from texsplat.scene import Scene  # noqa: E402
from texsplat.synth import camera_ring, make_plane_scene, render_targets  # noqa: E402
from texsplat.training import TrainConfig, _texel_tensor, train  # noqa: E402


def build_inputs():
    """(lut, init scene, cameras, display targets) of the train-loop fixture."""
    lut = BrdfLut(np.load(HERE / "lut.npz")["table"])
    gt = make_plane_scene(nx=4, ny=3, texture_res=1, seed=2, sh_degree=1)
    cams = camera_ring(3, radius=3.0, width=40, height=40)
    targets = render_targets(gt, cams, lut)
    init = gt.copy()
    init.positions = init.positions + 0.01
    n_extra = 3
    far = np.array([[60.0, 60.0, 60.0]]) + np.arange(n_extra)[:, None]
    init = Scene(positions=np.concatenate([init.positions, far]),
                 tangent_u=np.concatenate([init.tangent_u, init.tangent_u[:n_extra]]),
                 tangent_v=np.concatenate([init.tangent_v, init.tangent_v[:n_extra]]),
                 scales=np.concatenate([init.scales, init.scales[:n_extra]]),
                 opacities=np.concatenate([init.opacities, np.full(n_extra, 0.001)]),
                 sh=np.concatenate([init.sh, init.sh[:n_extra]]), sh_degree=init.sh_degree,
                 textures=list(init.textures) + list(init.textures[:n_extra]),
                 texture_config=init.texture_config, environment=init.environment,
                 background=init.background)
    return lut, init, cams, targets


def main():
    lut, init, cams, targets = build_inputs()
    config = TrainConfig(iterations=24, stage_split=12, texture_resolution=4, prune_interval=5,
                         prune_opacity=0.005, seed=4)
    fitted, hist = train(init, cams, targets, config, lut)
    d = {}
    d.update(scene_dict("init_", init))
    for i, c in enumerate(cams):
        d.update(cam_dict(f"cam{i}_", c))
        d[f"target{i}"] = np.asarray(targets[i], np.float64)
    d["n_cams"] = np.array(len(cams))
    for k in ("loss", "image", "normal", "smooth", "psnr", "fragments", "splats", "stage"):
        d[f"h_{k}"] = np.array([h[k] for h in hist])
    for k in ("positions", "tangent_u", "tangent_v", "scales", "opacities", "sh"):
        d[f"fit_{k}"] = getattr(fitted, k)
    d["fit_texels"] = _texel_tensor(fitted)
    d["fit_env_diffuse"] = fitted.environment.diffuse
    # stage 1 only (the parameters can be compared tightly before the
    # stage-2 texels make the fp32 / fp64 trajectories drift)
    cfg1 = TrainConfig(iterations=12, stage_split=12, texture_resolution=4, prune_interval=5,
                       prune_opacity=0.005, seed=4)
    fit1, hist1 = train(init, cams, targets, cfg1, lut)
    for k in ("loss", "splats"):
        d[f"s1_h_{k}"] = np.array([h[k] for h in hist1])
    for k in ("positions", "tangent_u", "tangent_v", "scales", "opacities", "sh"):
        d[f"s1_fit_{k}"] = getattr(fit1, k)
    d["s1_fit_texels"] = _texel_tensor(fit1)
    d["s1_fit_env_diffuse"] = fit1.environment.diffuse
    np.savez_compressed(HERE / "train_loop.npz", **d)
    print("losses", [round(h["loss"], 6) for h in hist])
    print("splats", [h["splats"] for h in hist])


if __name__ == "__main__":
    main()
