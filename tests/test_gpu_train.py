"""Training-step kernels (K10-K13, csrc/tsb_train.cu) against a plain
PyTorch fp32 reference of the same ops (tests/torch_loss_ref.py, autograd
adjoints) and against the reference's numpy Adam / Gram-Schmidt.

Tolerances: loss terms 1e-5 relative; gradients max abs error <= 2e-3 of the
array's max magnitude (fp32 blur sums in a different order than conv2d)."""
import ctypes as C

import numpy as np
import pytest
import torch

from paper_2506_13348_b200 import _lib, render_forward, shade_gbuffer, synth
from paper_2506_13348_b200.training import (LossWeights, _BUFFERS, image_loss_grad,
                                            linear_to_display, regularizer_grads)

import golden_io as gio
import torch_loss_ref as ref

pytestmark = pytest.mark.gpu


def _close(name, got, want, rel=2e-3):
    got = got.detach().double().cpu().numpy()
    want = want.detach().double().cpu().numpy()
    scale = max(np.abs(want).max(), 1e-12)
    err = np.abs(got - want).max()
    assert err <= rel * scale, (name, err, scale)


def _frame(seed=11, size=48):
    truth = synth.make_gradcheck_scene(seed)
    cam = synth.camera_ring(1, width=size, height=size)[0]
    lut = gio.lut()
    gb = render_forward(truth, cam, "perprim")
    res = shade_gbuffer(gb, cam, truth.environment, lut, background=truth.background)
    other = truth.copy()
    other.texels = np.clip(other.texels * 0.7 + 0.2, 0.0, 1.0).astype(np.float32)
    tgt = linear_to_display(shade_gbuffer(render_forward(other, cam, "perprim"), cam,
                                          other.environment, lut,
                                          background=other.background).color)
    return cam, gb.planar.contiguous(), res.color.contiguous(), tgt.contiguous()


@pytest.mark.parametrize("weights", [LossWeights(), LossWeights(0.5, 0.0, 0.0),
                                     LossWeights(0.2, 0.3, 0.0), LossWeights(0.2, 0.0, 0.4)])
def test_loss_kernels_match_torch(weights):
    cam, planar, color, tgt = _frame()
    H, W = planar.shape[1:]
    bufs = dict(_BUFFERS.get(W, H, color.device))
    terms = torch.zeros(8, dtype=torch.float64, device=color.device)
    bufs["terms"] = terms
    dcolor = image_loss_grad(color, tgt, weights, bufs).clone()
    dg = torch.zeros_like(planar)
    regularizer_grads(planar, tgt, cam, weights, dg, terms)
    t = terms.cpu().numpy()
    N = 3 * W * H
    rterms, rdcolor, rdg = ref.loss_and_grads(color, planar, tgt, cam, weights)
    image = (1 - weights.dssim) * t[0] / N + weights.dssim * 0.5 * (1 - t[1] / N)
    assert abs(image - rterms["image"]) <= 1e-5 * max(1.0, abs(rterms["image"]))
    if weights.normal > 0:
        assert abs(t[3] / max(t[4], 1) - rterms["normal"]) <= 1e-5
    if weights.smooth > 0:
        assert abs(t[5] / max(t[6], 1) - rterms["smooth"]) <= 1e-5
    _close("dcolor", dcolor, rdcolor)
    for c in (5, 6, 7, 11, 12):
        if rdg[c].abs().max() > 0:
            _close(f"dgbuf[{c}]", dg[c], rdg[c])
    for c in (0, 1, 2, 3, 4, 8, 9, 10):
        assert float(dg[c].abs().max()) == 0.0


def _np_adam(p, g, m, v, t, lr, b1=0.9, b2=0.999, eps=1e-8):
    m = b1 * m + (1 - b1) * g
    v = b2 * v + (1 - b2) * g * g
    mh, vh = m / (1 - b1 ** t), v / (1 - b2 ** t)
    return p - lr * mh / (np.sqrt(vh) + eps), m, v


def test_adam_matches_reference_numpy():
    rng = np.random.default_rng(0)
    dev = torch.device("cuda")
    specs = [("f64", np.float64, 1000, _lib.CLAMP_NONE, 0.0, 1e-2),
             ("f64floor", np.float64, 333, _lib.CLAMP_FLOOR, 0.4, 5e-2),
             ("f32unit", np.float32, 4097, _lib.CLAMP_UNIT, 0.0, 5e-2)]
    params, grads, moms, host = [], [], [], []
    arr = (_lib.AdamGroup_t * len(specs))()
    for i, (_, dt, n, clamp, floor, lr) in enumerate(specs):
        p0 = rng.uniform(0.0, 1.0, n).astype(dt)
        prm = torch.from_numpy(p0.copy()).to(dev)
        g = torch.zeros(n, dtype=torch.float32, device=dev)
        m, v = torch.zeros_like(prm), torch.zeros_like(prm)
        params.append(prm); grads.append(g); moms.append((m, v))
        host.append([p0.astype(np.float64), np.zeros(n), np.zeros(n)])
        a = arr[i]
        a.param, a.grad, a.m, a.v = _lib.ptr(prm), _lib.ptr(g), _lib.ptr(m), _lib.ptr(v)
        a.count, a.lr, a.floor, a.clamp = n, lr, floor, clamp
        a.dtype = _lib.F64 if dt == np.float64 else _lib.F32
    L = _lib.lib()
    for step in range(1, 4):
        for i, (_, dt, n, clamp, floor, lr) in enumerate(specs):
            gh = rng.normal(0.0, 1.0, n).astype(np.float32)
            grads[i].copy_(torch.from_numpy(gh))
            p, m, v = _np_adam(host[i][0], gh.astype(np.float64), host[i][1], host[i][2], step, lr)
            if clamp == _lib.CLAMP_UNIT:
                p = np.clip(p, 0.0, 1.0)
            elif clamp == _lib.CLAMP_FLOOR:
                p = np.maximum(p, floor)
            host[i] = [p, m, v]
        _lib.check(L.tsb_adam_step(arr, len(specs), step, 0.9, 0.999, 1e-8, None), "adam")
        torch.cuda.synchronize()
        for i, (name, dt, *_r) in enumerate(specs):
            got = params[i].cpu().numpy().astype(np.float64)
            tol = 1e-12 if dt == np.float64 else 2e-6
            assert np.abs(got - host[i][0]).max() <= tol, (name, step)


def test_orthonormalize_tangents_matches_reference():
    rng = np.random.default_rng(1)
    P = 1000
    tu = rng.normal(size=(P, 3))
    tv = rng.normal(size=(P, 3))
    u = tu / np.linalg.norm(tu, axis=-1, keepdims=True)
    v = tv - np.sum(u * tv, axis=-1, keepdims=True) * u
    v = v / np.linalg.norm(v, axis=-1, keepdims=True)
    du, dv = torch.from_numpy(tu).cuda(), torch.from_numpy(tv).cuda()
    _lib.check(_lib.lib().tsb_orthonormalize_tangents(P, _lib.ptr(du), _lib.ptr(dv), None), "o")
    assert np.abs(du.cpu().numpy() - u).max() < 1e-14
    assert np.abs(dv.cpu().numpy() - v).max() < 1e-14


def test_trainer_step_gradient_equals_compute_step():
    """The trainer's flat buffer (texel gradients in the atlas's 8-channel
    order on one GPU, 7 combined channels under torch.distributed) holds
    exactly compute_step's gradients for the same parameters."""
    from paper_2506_13348_b200.training import DataParallelTrainer, compute_step
    truth = synth.make_gradcheck_scene(11)
    cam = synth.camera_ring(1, width=32, height=32)[0]
    lut = gio.lut()
    tgt = linear_to_display(shade_gbuffer(render_forward(truth, cam, "perprim"), cam,
                                          truth.environment, lut,
                                          background=truth.background).color)
    init = truth.copy()
    init.texels = np.clip(init.texels + 0.1, 0.0, 1.0).astype(np.float32)
    tr = DataParallelTrainer(init, lut)
    terms = tr.grads_and_loss(cam, tgt)
    m, grads, eg = compute_step(init, cam, tgt.cpu().numpy(), lut)
    assert abs(terms["loss"] - m["loss"]) <= 1e-6 * max(1.0, abs(m["loss"]))
    for name in ("positions", "tangent_u", "tangent_v", "scales", "opacities", "sh"):
        _close(name, getattr(tr.grads, name), getattr(grads, name), rel=1e-3)
    got = tr.grads.texels_dense
    if tr.grads.texel_layout == _lib.TEXELS_INTERLEAVED:  # one GPU: the atlas's own order
        got = got[..., [0, 1, 2, 3, 6, 4, 5]]
    _close("texels", got, grads.texels_dense, rel=1e-3)
    for a, b in zip(tr.env_grads.spec_mips, eg.spec_mips):
        _close("env", a, b, rel=1e-3)


def _train_golden():
    from paper_2506_13348_b200.training import TrainConfig
    g = gio.load("train_loop")
    scene = gio.scene(g, "init_")
    cams = [gio.camera(g, f"cam{i}_") for i in range(int(g["n_cams"]))]
    targets = [g[f"target{i}"] for i in range(len(cams))]
    cfg = TrainConfig(iterations=24, stage_split=12, texture_resolution=4, prune_interval=5,
                      prune_opacity=0.005, seed=4)
    return g, scene, cams, targets, cfg


def test_train_loop_matches_reference_history():
    """GPU train() vs the reference's train() (training.py:224-322) on the
    same scene, views, targets and config: the same view schedule (numpy
    default_rng(seed)), the stage-2 broadcast 1x1 -> 4x4 with the texel Adam
    reset at iteration 12, the prune at iteration 5 (15 -> 12 splats, Adam
    moments compacted), per-step losses within the fp32-vs-fp64 drift."""
    from paper_2506_13348_b200.training import train
    g, scene, cams, targets, cfg = _train_golden()
    fitted, hist = train(scene, cams, targets, cfg, gio.lut())
    assert [h["stage"] for h in hist] == list(g["h_stage"])
    assert [h["splats"] for h in hist] == list(g["h_splats"])
    frag = np.array([h["fragments"] for h in hist])
    assert np.array_equal(frag[:5], g["h_fragments"][:5])  # before parameters drift
    assert np.abs(frag - g["h_fragments"]).max() <= 1e-3 * g["h_fragments"].max()
    ref = g["h_loss"]
    got = np.array([h["loss"] for h in hist])
    rel = np.abs(got - ref) / np.abs(ref)
    print("train loop loss relative error per step:", rel.max(), rel)
    # Stage 1 agrees to <= 2.5e-4 (observed over repeated runs). In stage 2
    # (16 texels per splat, Adam reset) Adam's per-component normalisation
    # turns the fp32 noise of near-zero texel gradients into full-size steps;
    # on this 40x40, 12-splat problem one coverage decision can then flip a
    # few steps later. Observed over repeated runs (scripts/train_drift.py):
    # max 0.3 % or 7.7 % at one step depending on the run, run-to-run spread
    # of the GPU itself of the same size.
    stage2 = np.array([h["stage"] for h in hist]) == 2
    assert rel[~stage2].max() <= 1e-3, rel
    assert rel[stage2].max() <= 0.12, rel
    assert np.median(rel[stage2]) <= 1e-2, rel
    assert fitted.num_splats == 12 and fitted.texture_config.resolution == 4
    assert fitted.texels.shape == (12, 4, 4, 7)


def test_train_stage1_parameters_match_reference():
    """Stage 1 only (12 iterations, prunes at 5 and 10): every fitted
    parameter array, the texels and the environment vs the reference's."""
    from paper_2506_13348_b200.training import train
    g, scene, cams, targets, cfg = _train_golden()
    cfg.iterations, cfg.stage_split = 12, 12
    fitted, hist = train(scene, cams, targets, cfg, gio.lut())
    assert [h["splats"] for h in hist] == list(g["s1_h_splats"])
    rel = np.abs(np.array([h["loss"] for h in hist]) - g["s1_h_loss"]) / g["s1_h_loss"]
    assert rel.max() <= 1e-3, rel  # observed <= 2.5e-4 over repeated runs
    # Adam moves every component by ~lr per step whatever the gradient's size,
    # so a near-zero fp32 gradient of the other sign costs (part of) a step:
    # the bar is one step of each group's learning rate (observed: positions
    # 1.7e-4 of 4.2e-4, env 5.2e-3 of 1e-2, opacities 3.2e-4 of 5e-2,
    # texels 4.4e-5 of 2.5e-3)
    errs = {}
    for name in ("positions", "tangent_u", "tangent_v", "scales", "opacities", "sh"):
        errs[name] = float(np.abs(getattr(fitted, name) - g[f"s1_fit_{name}"]).max())
    errs["texels"] = float(np.abs(fitted.texels - g["s1_fit_texels"]).max())
    errs["env"] = float(np.abs(fitted.environment.diffuse - g["s1_fit_env_diffuse"]).max())
    print("stage-1 parameter errors:", errs)
    from paper_2506_13348_b200.training import world_extent
    step = {"positions": cfg.lr_position * world_extent(scene.positions),
            "tangent_u": cfg.lr_frame, "tangent_v": cfg.lr_frame, "scales": cfg.lr_scale,
            "opacities": cfg.lr_opacity, "sh": cfg.lr_sh, "texels": cfg.lr_texel,
            "env": cfg.lr_env}
    for name, e in errs.items():  # within one Adam step of the reference, per component
        assert e <= step[name], (name, e, step[name])


def test_train_loop_divergence_guard():
    """A non-finite loss stops every later update on the device and raises
    like the reference (training.py:263-265)."""
    from paper_2506_13348_b200.training import train
    g, scene, cams, targets, cfg = _train_golden()
    bad = [t.copy() for t in targets]
    for b in bad:
        b[0, 0, 0] = np.nan
    cfg.iterations = 6
    with pytest.raises(RuntimeError, match="diverged"):
        train(scene, cams, bad, cfg, gio.lut())


def test_stage_transition_is_bitwise():
    """Reference acceptance c06 (pkg/tests/test_acceptance.py:317): growing
    the trained 1x1 charts to the stage-2 resolution (tsb_broadcast_texels)
    changes no bit of the rendered images — the first stage-2 render equals
    the last stage-1 render (fp32 verify-mode sampling of a constant chart is
    exact)."""
    from paper_2506_13348_b200.training import (DataParallelTrainer, TrainConfig, train)
    lut = gio.lut()
    gt = synth.make_plane_scene(nx=3, ny=3, texture_res=1, seed=2, sh_degree=1)
    cams = synth.camera_ring(2, radius=3.0, width=32, height=32)
    targets = [linear_to_display(shade_gbuffer(render_forward(gt, c, "perprim"), c,
                                               gt.environment, lut,
                                               background=gt.background).color).cpu().numpy()
               for c in cams]
    init = gt.copy()
    init.positions = init.positions + 0.01
    cfg = TrainConfig(iterations=6, stage_split=6, texture_resolution=4, seed=3,
                      prune_interval=100)
    stage1, _ = train(init, cams, targets, cfg, lut)
    assert stage1.texture_config.resolution == 1
    tr = DataParallelTrainer(stage1, lut)
    tr.broadcast_textures(4)
    stage2 = tr.to_scene()
    assert stage2.texture_config.resolution == 4
    for cam in cams:
        r1 = shade_gbuffer(render_forward(stage1, cam, "perprim"), cam, stage1.environment, lut,
                           background=stage1.background).color
        r2 = shade_gbuffer(render_forward(stage2, cam, "perprim"), cam, stage2.environment, lut,
                           background=stage2.background).color
        assert torch.equal(r1, r2)


def test_evaluate_matches_reference():
    """evaluate() (the GPU render + display transform + clipped PSNR / SSIM of
    training.py:325-339) vs the reference's on the train-loop fixture's
    initial scene (tests/golden/make_golden_eval.py)."""
    from paper_2506_13348_b200.training import evaluate
    _, scene, cams, targets, _ = _train_golden()
    ev = gio.load("evaluate")
    r = evaluate(scene, cams, targets, gio.lut())
    # fp32 render vs fp64 at ~50 dB: the PSNR moves by thousandths of a dB
    assert abs(r["psnr"] - float(ev["psnr"])) <= 0.05, (r, float(ev["psnr"]))
    assert abs(r["ssim"] - float(ev["ssim"])) <= 1e-5, (r, float(ev["ssim"]))


def test_fit_cli_end_to_end(tmp_path, capsys):
    """`cli fit` (cli.py:127-156): manifest + 8-bit PNG targets -> GPU train()
    -> checkpoint, CSV log and a JSON summary; the checkpoint reloads."""
    import json

    from paper_2506_13348_b200 import cli, formats
    _, scene, cams, targets, _ = _train_golden()
    names = []
    for i, t in enumerate(targets):
        name = f"view_{i}.png"
        cli.write_png(tmp_path / name, np.round(np.clip(t, 0.0, 1.0) * 255.0).astype(np.uint8))
        names.append(name)
    formats.save_manifest(tmp_path / "manifest.json", cams, names)
    formats.save_scene(scene, tmp_path / "init")
    (tmp_path / "cfg.json").write_text(json.dumps({"iterations": 6, "stage_split": 3,
                                                    "prune_interval": 100}))
    rc = cli.main(["fit", "--manifest", str(tmp_path / "manifest.json"), "--scene",
                   str(tmp_path / "init"), "--out", str(tmp_path / "out"), "--config",
                   str(tmp_path / "cfg.json"), "--texture-res", "2"])
    assert rc == 0
    summary = json.loads(capsys.readouterr().out)
    assert summary["command"] == "fit" and summary["iterations"] == 6
    assert np.isfinite(summary["psnr"]) and 0.0 < summary["ssim"] <= 1.0
    log = (tmp_path / "out" / "train_log.csv").read_text().splitlines()
    assert len(log) == 1 + 6
    fitted = formats.load_scene(tmp_path / "out" / "scene")
    assert fitted.texture_config.resolution == 2 and fitted.num_splats == summary["splats"]


def test_train_loop_at_scale():
    """train() on a 20k-splat shell (1x1 charts growing to 8x8 at the stage
    split, three 256x256 views, pruning on): every logged loss finite, the
    fit improves, the broadcast and the prune run at scale."""
    from paper_2506_13348_b200.scene import TextureConfig
    from paper_2506_13348_b200.training import TrainConfig, train
    lut = gio.lut()
    truth = synth.make_shell_scene(20000, 8, seed=5, with_environment=True)
    cams = synth.bench_cameras(3, 256, 256)
    targets = [linear_to_display(shade_gbuffer(render_forward(truth, c, "perprim"), c,
                                               truth.environment, lut,
                                               background=truth.background).color).cpu().numpy()
               for c in cams]
    init = truth.copy()
    init.positions = init.positions + 0.002
    init.texels = np.ascontiguousarray(truth.texels.mean(axis=(1, 2), keepdims=True))
    init.texture_config = TextureConfig(1, truth.texture_config.support)
    init.opacities[::50] = 0.001  # a few to prune
    cfg = TrainConfig(iterations=30, stage_split=15, texture_resolution=8, prune_interval=10,
                      prune_opacity=0.005, seed=1)
    fitted, hist = train(init, cams, targets, cfg, lut)
    loss = np.array([h["loss"] for h in hist])
    assert np.isfinite(loss).all(), loss
    assert [h["stage"] for h in hist] == [1] * 15 + [2] * 15
    assert loss[14] < loss[0]
    assert fitted.texture_config.resolution == 8 and fitted.texels.shape[1:3] == (8, 8)
    assert fitted.num_splats < init.num_splats  # the near-transparent splats were pruned
