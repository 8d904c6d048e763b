"""GPU parity of the backward pass against the numpy reference.

Fixtures (tests/golden/make_golden.py) hold the reference's fp64
splat_backward / shade_backward / compute_step gradients. Tolerance: per
gradient array, max |ours - ref| <= GRAD_RTOL * max |ref| (+ a tiny absolute
floor). The GPU computes in fp32 with float atomics (order-dependent low
bits), the reference in fp64.
"""
import numpy as np
import pytest
import torch

import golden_io as gio
from paper_2506_13348_b200 import render_forward, synth
from paper_2506_13348_b200.backward import shade_backward, splat_backward
from paper_2506_13348_b200.environment import EnvironmentLight
from paper_2506_13348_b200.shading import ShadeResult, device_environment
from paper_2506_13348_b200.training import DataParallelTrainer, compute_step

pytestmark = pytest.mark.gpu
GRAD_RTOL = 2e-3


def _close(name, ours, ref, rtol=GRAD_RTOL, atol=1e-9):
    ours = np.asarray(ours, np.float64)
    ref = np.asarray(ref, np.float64)
    assert ours.shape == ref.shape, (name, ours.shape, ref.shape)
    err = float(np.abs(ours - ref).max()) if ref.size else 0.0
    scale = float(np.abs(ref).max()) if ref.size else 0.0
    assert err <= rtol * scale + atol, f"{name}: max err {err:.3e} vs scale {scale:.3e}"
    return err / max(scale, 1e-30)


def _grads_vs(g, pre, grads):
    errs = {}
    for name in ("positions", "tangent_u", "tangent_v", "scales", "opacities", "sh"):
        errs[name] = _close(name, getattr(grads, name).cpu().numpy(), g[f"{pre}g_{name}"])
    errs["texels"] = _close("texels", grads.texels_dense.cpu().numpy(), g[f"{pre}g_texels"])
    return errs


def test_splat_backward_random_dbuf_matches_reference():
    g = gio.load("backward")
    scene, cam = gio.scene(g, "bw_"), gio.camera(g, "bw_cam_")
    gbuf, tape = render_forward(scene, cam, "perprim", with_tape=True)
    assert np.abs(gbuf.numpy() - g["bw_gbuf"]).max() <= 1e-3
    grads = splat_backward(scene, cam, None, tape, g["bw_dbuf"])
    _grads_vs(g, "bw_", grads)


def test_shade_backward_matches_reference(lut_table):
    g = gio.load("backward")
    scene, cam = gio.scene(g, "gc_"), gio.camera(g, "gc_cam_")
    planar = torch.from_numpy(g["gc_gbuf"].astype(np.float32)).permute(2, 0, 1).contiguous().cuda()
    denv = device_environment(scene.environment, gio.lut())
    sr = ShadeResult(None, None, None, cache=(planar, denv, scene.background))
    dgbuf, eg = shade_backward(sr, cam, None, None, g["gc_dcolor"])
    ours = dgbuf.permute(1, 2, 0).cpu().numpy()
    ref = g["gc_dgbuf"]
    for c in range(13):
        _close(f"dgbuf[{c}]", ours[..., c], ref[..., c], rtol=2e-3, atol=1e-6)
    for i, m in enumerate(eg.spec_mips):
        _close(f"env mip {i}", m.cpu().numpy(), g[f"gc_genv_mip{i}"])
    _close("env diffuse", eg.diffuse.cpu().numpy(), g["gc_genv_diffuse"])


def test_splat_backward_from_shading_matches_reference():
    g = gio.load("backward")
    scene, cam = gio.scene(g, "gc_"), gio.camera(g, "gc_cam_")
    gbuf, tape = render_forward(scene, cam, "perprim", with_tape=True)
    grads = splat_backward(scene, cam, None, tape, g["gc_dgbuf"])
    _grads_vs(g, "gc_", grads)


def test_backward_requires_perprim():
    g = gio.load("backward")
    scene, cam = gio.scene(g, "bw_"), gio.camera(g, "bw_cam_")
    _, tape = render_forward(scene, cam, "flat", with_tape=True)
    with pytest.raises(ValueError):
        splat_backward(scene, cam, None, tape, np.zeros((16, 16, 13)))


def test_compute_step_matches_reference():
    g = gio.load("train")
    scene, cam = gio.scene(g, "st_"), gio.camera(g, "st_cam_")
    metrics, grads, eg = compute_step(scene, cam, g["st_target"], gio.lut())
    for k in ("loss", "image", "normal", "smooth"):
        ref = float(g[f"st_m_{k}"])
        assert abs(metrics[k] - ref) <= 1e-4 * max(1.0, abs(ref)), (k, metrics[k], ref)
    assert metrics["fragments"] == int(g["st_m_fragments"])
    _grads_vs(g, "st_", grads)
    for i, m in enumerate(eg.spec_mips):
        _close(f"env mip {i}", m.cpu().numpy(), g[f"st_genv_mip{i}"])
    _close("env diffuse", eg.diffuse.cpu().numpy(), g["st_genv_diffuse"])


def test_alpha_one_backward_is_finite():
    """alpha == 1 is allowed by the reference; the adjoint must stay finite."""
    from paper_2506_13348_b200 import MaterialTextureSet, Scene, TextureConfig
    from paper_2506_13348_b200.splats import Camera
    P = 2
    tex = np.stack([MaterialTextureSet.constant((0.5, 0.4, 0.3), 0.5, 0.1, resolution=2).combined()
                    for _ in range(P)])
    s = Scene(np.array([[0.0, 0.0, 0.0], [0.0, 0.0, 1.0]]), np.tile([1.0, 0.0, 0.0], (P, 1)),
              np.tile([0.0, 1.0, 0.0], (P, 1)), np.full((P, 2), 0.8), np.ones(P),
              np.zeros((P, 1, 3)), 0, tex, TextureConfig(2))
    cam = Camera.look_at((0.0, 0.0, -2.0), (0.0, 0.0, 1.0), width=33, height=33)
    gb, tape = render_forward(s, cam, "perprim", with_tape=True)
    assert float(gb.alpha.max()) == 1.0
    grads = splat_backward(s, cam, None, tape, np.ones((33, 33, 13)))
    for t in grads.flat():
        assert torch.isfinite(t).all()


def test_data_parallel_trainer_reduces_loss():
    truth = synth.make_gradcheck_scene(11)
    cam = synth.camera_ring(1, width=32, height=32)[0]
    from paper_2506_13348_b200.training import linear_to_display
    from paper_2506_13348_b200 import shade_gbuffer
    lut = gio.lut()
    tgt = linear_to_display(shade_gbuffer(render_forward(truth, cam, "perprim"), cam,
                                          truth.environment, lut,
                                          background=truth.background).color)
    init = truth.copy()
    init.texels = np.clip(init.texels + 0.1, 0.0, 1.0).astype(np.float32)
    lr = {"positions": 1e-5, "tangent_u": 1e-4, "tangent_v": 1e-4, "scales": 1e-5,
          "opacities": 1e-3, "sh": 1e-3, "texels": 5e-3, "env": 1e-3}
    tr = DataParallelTrainer(init, lut, lr=lr)
    losses = [tr.step(cam, tgt)[0]["loss"] for _ in range(20)]
    assert all(np.isfinite(losses))
    assert max(losses[-5:]) < 0.8 * losses[0], losses


def test_deterministic_backward_is_bitwise_repeatable():
    """tsb_render_backward_ex(deterministic=1): int64 fixed-point sums, so two
    runs agree bit for bit (the float-atomic default need not), and both
    modes agree with each other and with the reference's gradients."""
    g = gio.load("backward")
    scene, cam = gio.scene(g, "gc_"), gio.camera(g, "gc_cam_")
    gbuf, tape = render_forward(scene, cam, "perprim", with_tape=True)
    a = splat_backward(scene, cam, None, tape, g["gc_dgbuf"], deterministic=True)
    b = splat_backward(scene, cam, None, tape, g["gc_dgbuf"], deterministic=True)
    for x, y in zip(a.flat(), b.flat()):
        assert torch.equal(x, y)
    _grads_vs(g, "gc_", a)
    f = splat_backward(scene, cam, None, tape, g["gc_dgbuf"])
    for x, y in zip(a.flat(), f.flat()):
        scale = float(y.abs().max()) if y.numel() else 0.0
        assert float((x - y).abs().max()) <= 1e-4 * scale + 1e-9


def test_deterministic_backward_at_cfg4_scale():
    """The same on an 80x80 window of the 100k-splat cfg4 scene (real list
    lengths, many warps adding into the same splats and texels)."""
    gc_ = gio.load("train_crop")
    scene = gio.cfg2_scene()
    cam = gio.camera(gc_)
    dbuf = np.random.default_rng(7).normal(size=(cam.height, cam.width, 13))
    gbuf, tape = render_forward(scene, cam, "perprim", with_tape=True)
    runs = [splat_backward(scene, cam, None, tape, dbuf, deterministic=True) for _ in range(3)]
    for r in runs[1:]:
        for x, y in zip(runs[0].flat(), r.flat()):
            assert torch.equal(x, y)
    f = splat_backward(scene, cam, None, tape, dbuf)
    for x, y in zip(runs[0].flat(), f.flat()):
        scale = float(y.abs().max()) if y.numel() else 0.0
        assert float((x - y).abs().max()) <= 1e-4 * scale + 1e-9
