"""GPU parity at the BASELINE shapes (round-2 pins, tests/golden/make_golden_scale.py).

  * cfg2 full frame: all 13 G-buffer channels on three 160x160 windows vs the
    numpy reference;
  * cfg3 shape: 500k splats, T=8, a 2-page layered atlas, 1920x1080 view 37,
    a silhouette crop — GPU vs the CPU oracle bit-exact (verify mode), HW mode
    same counts + PSNR >= 50 dB, both vs the reference within the bar;
  * cfg5 shape: 2M splats, T=16, a 31-page layered atlas (16.6 GB per copy),
    1920x1080, two crops — the same checks;
  * cfg4 scale backward: compute_step through an 80x80 crop of the cfg2
    scene (1,250 splats with gradients, real list lengths and contention)
    vs the reference's fp64 gradients.

Crop cameras render pixels bit-identical to the full frame.
"""
import gc
import hashlib

import numpy as np
import pytest
import torch

import golden_io as gio
from oracle import oracle
from paper_2506_13348_b200 import pack_atlases, render_forward, shade_gbuffer, synth
from paper_2506_13348_b200.device import DeviceAtlas
from paper_2506_13348_b200.environment import BrdfLut
from paper_2506_13348_b200.rasterize import frame_structure, prepare, render_prepared
from paper_2506_13348_b200.training import compute_step

pytestmark = pytest.mark.gpu
TOL = 1e-3
# fp32 gradients with float atomics vs the reference's fp64, at cfg4 scale
# (~120k fragments through 1,250 splats): max |ours - ref| per array
# relative to the array's max |ref|
GRAD_RTOL_SCALE = 5e-3


def _gate_flips_only(ours, ref):
    """Contributor counts equal the reference's except T > 1e-4 gate flips
    (fp32 vs fp64 transmittance): each differs by one fragment, and at most
    one pixel in 2000 flips (observed: 15 / 640,000 on the full cfg2 frame)."""
    d = np.asarray(ours, np.int64) - np.asarray(ref, np.int64)
    assert np.abs(d).max() <= 1
    assert int((d != 0).sum()) <= max(2, d.size // 2000), int((d != 0).sum())


def _np(t):
    return t.detach().cpu().numpy()


def psnr(a, b, peak=1.0):
    mse = float(np.mean((np.asarray(a, np.float64) - np.asarray(b, np.float64)) ** 2))
    return float("inf") if mse == 0 else 10.0 * np.log10(peak * peak / mse)


def _sha_ok(g, scene):
    for k in ("positions", "tangent_u", "scales", "texels"):
        h = hashlib.sha256(np.ascontiguousarray(getattr(scene, k)).tobytes()).hexdigest()
        assert h == str(g["sha_" + k]), k


class _Shape:
    """A large scene + its atlas: device copies (linear + layered texture) and
    the oracle's page arrays, built with one host copy of the pages."""

    def __init__(self, n, T, env_height):
        self.scene = synth.make_shell_scene(n, T, seed=3, with_environment=True,
                                            env_height=env_height, env_levels=6)
        aset = pack_atlases(self.scene)
        self.pages = len(aset.family_a)
        self.scene.texels = self.scene.texels[:0]  # the oracle reads only T from it
        gc.collect()
        self.datlas = DeviceAtlas(aset, linear=True, hw=True)
        entries = aset.indirection.entries
        fa = np.stack([p.texels for p in aset.family_a])
        aset.family_a.clear()
        gc.collect()
        fb = np.stack([p.texels for p in aset.family_b])
        aset.family_b.clear()
        gc.collect()
        self.oracle_atlas = (fa, fb, entries)
        self.lut = gio.lut()

    def check_crop(self, g, pre):
        cam = gio.camera(g, pre + "cam_")
        ref = oracle.render(self.scene, cam, atlas=self.oracle_atlas)
        out = {}
        for smp in ("verify", "hw"):
            prep = prepare(self.scene, cam, "atlas", self.datlas, sampler=smp)
            gb, tape = render_prepared(prep, cam, 16)
            out[smp] = gb
            assert np.array_equal(_np(gb.pixels.n_contrib), ref["n_contrib"]), smp
            st = frame_structure(tape)
            K = ref["num_kept"]
            assert np.array_equal(st["sorted_ids"][:K], ref["sorted_ids"][:K]), smp
            assert np.array_equal(st["keys"], ref["keys"]), smp
            assert np.array_equal(st["ranges"], ref["ranges"]), smp
        gv, gh = out["verify"], out["hw"]
        # verify mode: bit-exact vs the oracle
        assert np.array_equal(_np(gv.planar), ref["gbuf"])
        assert np.array_equal(_np(gv.pixels.final_T), ref["final_T"])
        # vs the numpy reference (order, counts up to T-gate flips, every channel)
        K = ref["num_kept"]
        assert np.array_equal(ref["sorted_ids"][:K], g[pre + "order"])
        _gate_flips_only(_np(gv.pixels.n_contrib), g[pre + "counts"])
        gref = g[pre + "gbuf"].transpose(2, 0, 1)
        for c in range(13):
            assert np.abs(_np(gv.planar)[c] - gref[c]).max() <= TOL, c
        env = self.scene.environment
        sv = shade_gbuffer(gv, cam, env, self.lut, background=self.scene.background)
        assert np.abs(_np(sv.color) - g[pre + "color"]).max() <= TOL
        # HW mode: same counts (above), PSNR >= 50 dB vs the oracle and the reference
        assert psnr(_np(gh.planar)[:12], ref["gbuf"][:12]) >= 50.0
        sh = shade_gbuffer(gh, cam, env, self.lut, background=self.scene.background)
        assert psnr(_np(sh.color), g[pre + "color"]) >= 50.0
        return ref


def test_cfg2_full_frame_gbuffer_windows():
    """Every G-buffer channel of the full 800x800 cfg2 frame (three windows
    of the full render) vs the reference, verify and HW modes."""
    g = gio.load("cfg2_gbuf")
    scene = gio.cfg2_scene()
    _sha_ok(g, scene)
    full = gio.camera(gio.load("cfg2_crop"), "full_cam_")
    lut = gio.lut()
    gv = render_forward(scene, full, "perprim")
    gh = render_forward(scene, full, "atlas", pack_atlases(scene))
    assert torch.equal(gv.pixels.n_contrib, gh.pixels.n_contrib)
    for pre in ("c_", "s_", "e_"):
        x0, y0, w, h = (int(v) for v in g[pre + "crop"])
        win = (slice(None), slice(y0, y0 + h), slice(x0, x0 + w))
        ref = g[pre + "gbuf"].transpose(2, 0, 1)
        ours = _np(gv.planar)[win]
        for c in range(13):
            assert np.abs(ours[c] - ref[c]).max() <= TOL, (pre, c)
        _gate_flips_only(_np(gv.pixels.n_contrib)[win[1:]], g[pre + "counts"])
        assert psnr(_np(gh.planar)[win][:12], ref[:12]) >= 50.0
        cam = gio.camera(g, pre + "cam_")
        sr = shade_gbuffer(render_forward(scene, cam, "perprim"), cam, scene.environment, lut,
                           background=scene.background)
        assert np.abs(_np(sr.color) - g[pre + "color"]).max() <= TOL


def test_cfg3_shape_two_pages():
    g = gio.load("cfg3_crop")
    sh = _Shape(500_000, 8, 64)
    assert sh.pages == 2
    sh.check_crop(g, "")


def test_cfg5_shape_thirty_one_pages():
    """2M splats, T=16: 31 layered pages per family, two crops (centre and
    the right silhouette) of the 1920x1080 view."""
    g = gio.load("cfg5_crop")
    sh = _Shape(2_000_000, 16, 128)
    assert sh.pages == 31
    for pre in ("c_", "s_"):
        sh.check_crop(g, pre)
    del sh
    gc.collect()
    torch.cuda.empty_cache()


def test_compute_step_cfg4_scale_crop():
    """compute_step at cfg4 scale: 100k splats, T=8, 80x80 window of the
    800x800 view (the reference's fp64 gradients of 1,250 splats; every
    other row must be zero)."""
    g = gio.load("train_crop")
    scene = gio.cfg2_scene()
    _sha_ok(g, scene)
    init = scene.copy()
    init.positions = init.positions + 0.003
    cam = gio.camera(g)
    metrics, grads, eg = compute_step(init, cam, g["target"], gio.lut())
    for k in ("loss", "image", "normal", "smooth"):
        ref = float(g[f"m_{k}"])
        assert abs(metrics[k] - ref) <= 1e-4 * max(1.0, abs(ref)), (k, metrics[k], ref)
    assert metrics["fragments"] == int(g["m_fragments"])
    nz = g["nz"]
    mask = np.zeros(scene.num_splats, bool)
    mask[nz] = True
    errs = {}
    for name in ("positions", "tangent_u", "tangent_v", "scales", "opacities", "sh"):
        ours = getattr(grads, name).cpu().numpy()
        ref = g[f"g_{name}"]
        err = np.abs(ours[nz].reshape(ref.shape) - ref).max()
        errs[name] = err / max(np.abs(ref).max(), 1e-30) if np.abs(ref).max() > 0 else err
        assert not np.any(ours[~mask]), name
    print("cfg4-scale relative gradient errors:", errs)
    for name, e in errs.items():
        assert e <= GRAD_RTOL_SCALE, (name, e)
    tex = grads.texels_dense.cpu().numpy()
    err = np.abs(tex[nz] - g["g_texels"]).max()
    assert err <= 2e-3 * np.abs(g["g_texels"]).max(), err
    assert not np.any(tex[~mask])
    for i, m in enumerate(eg.spec_mips):
        ref = g[f"genv_mip{i}"]
        assert np.abs(m.cpu().numpy() - ref).max() <= 2e-3 * np.abs(ref).max() + 1e-9, i
    ref = g["genv_diffuse"]
    assert np.abs(eg.diffuse.cpu().numpy() - ref).max() <= 2e-3 * np.abs(ref).max() + 1e-9
