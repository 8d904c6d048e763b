"""Pin the CPU oracle to the numpy reference (golden fixtures, no GPU).

The fixtures were produced by tests/golden/make_golden*.py from the
reference itself. The reference computes in float64; the oracle (and the
GPU) in float32 with an fp64 guard band on the alpha cut, so:
  * draw order, rects, per-pixel contributor counts: exact;
  * G-buffer / colour: max abs <= 1e-3 (north_star bar), observed ~1e-6.
"""
import numpy as np
import pytest

import golden_io as gio
from oracle import oracle

TOL = 1e-3


def _check_forward(g, pre, scene, cam, mode="verify"):
    r = oracle.render(scene, cam, mode=mode, tile=16)
    ref = g[pre + "gbuf"].transpose(2, 0, 1)
    assert np.abs(r["gbuf"] - ref).max() <= TOL
    assert np.array_equal(r["n_contrib"], g[pre + "counts"])
    assert int(r["n_contrib"].sum()) == int(g[pre + "fragment_count"])
    K = r["num_kept"]
    assert np.array_equal(r["sorted_ids"][:K], g[pre + "order"])
    if pre + "rects" in g:
        assert np.array_equal(r["rects"], g[pre + "rects"])
    return r


def test_cfg1_forward_and_shade():
    g = gio.load("cfg1")
    scene, cam = gio.scene(g), gio.camera(g)
    r = _check_forward(g, "", scene, cam)
    assert np.abs(r["gbuf"] - g["gbuf"].transpose(2, 0, 1)).max() < 1e-5
    color, dif, spe = oracle.shade(r["gbuf"], cam, scene.environment, gio.load("lut")["table"],
                                   scene.background)
    assert np.abs(color - g["color"]).max() <= TOL
    assert np.abs(dif - g["diffuse"]).max() <= TOL
    assert np.abs(spe - g["specular"]).max() <= TOL


@pytest.mark.parametrize("tile", [8, 16, 32, 64])
def test_oracle_tile_invariance(tile):
    g = gio.load("small")
    scene, cam = gio.scene(g, "inv_"), gio.camera(g, "inv_cam_")
    r = oracle.render(scene, cam, tile=tile)
    base = oracle.render(scene, cam, tile=16)
    assert np.array_equal(r["gbuf"], base["gbuf"])
    assert np.array_equal(r["n_contrib"], g["inv_counts"])
    assert np.abs(r["gbuf"] - g["inv_gbuf"].transpose(2, 0, 1)).max() <= TOL


def test_flat_mode():
    g = gio.load("small")
    scene, cam = gio.scene(g, "flat_"), gio.camera(g, "flat_cam_")
    _check_forward(g, "flat_", scene, cam, mode="flat")
    _check_forward(g, "flatp_", scene, cam, mode="verify")


def test_threads_do_not_change_output():
    g = gio.load("cfg1")
    scene, cam = gio.scene(g), gio.camera(g)
    a = oracle.render(scene, cam, threads=1)
    b = oracle.render(scene, cam, threads=4)
    for k in ("gbuf", "n_contrib", "final_T", "keys", "ranges"):
        assert np.array_equal(a[k], b[k])


def test_cfg2_crop():
    g = gio.load("cfg2_crop")
    scene, cam = gio.cfg2_scene(), gio.camera(g)
    r = _check_forward(g, "", scene, cam)
    color, _, _ = oracle.shade(r["gbuf"], cam, scene.environment, gio.load("lut")["table"],
                               scene.background)
    assert np.abs(color - g["color"]).max() <= TOL


def test_cfg2_full_frame():
    """Full 800x800 cfg2 frame: contributor counts vs the reference.

    fp32 intersection math can flip the T > 1e-4 gate on a handful of
    pixels (effect <= 1e-4 on the G-buffer); everything else is exact."""
    path = gio.GOLDEN / "cfg2_full.npz"
    if not path.exists():
        pytest.skip("cfg2_full.npz not generated")
    g = np.load(path)
    scene = gio.cfg2_scene()
    cam = gio.camera(gio.load("cfg2_crop"), "full_cam_")
    r = oracle.render(scene, cam)
    K = r["num_kept"]
    assert np.array_equal(r["sorted_ids"][:K], g["order"])
    diff = r["n_contrib"] != g["counts"]
    assert diff.sum() <= 15, diff.sum()  # observed: 15 gate flips
    assert np.abs(r["gbuf"][12] - g["alpha"]).max() <= TOL
    color, _, _ = oracle.shade(r["gbuf"], cam, scene.environment, gio.load("lut")["table"],
                               scene.background)
    assert np.abs(color - g["color"]).max() <= TOL


@pytest.mark.parametrize("case", ["cfg1", "small_inv", "cfg2_crop"])
def test_box_binning_is_conservative(case):
    """Binning by rect ∩ alpha-cut ellipse box (the GPU's) renders exactly
    what the reference's rect binning (_tile_lists) renders."""
    if case == "cfg1":
        g = gio.load("cfg1")
        scene, cam = gio.scene(g), gio.camera(g)
    elif case == "small_inv":
        g = gio.load("small")
        scene, cam = gio.scene(g, "inv_"), gio.camera(g, "inv_cam_")
    else:
        g = gio.load("cfg2_crop")
        scene, cam = gio.cfg2_scene(), gio.camera(g)
    a = oracle.render(scene, cam, binning="rect")
    b = oracle.render(scene, cam, binning="box")
    assert len(b["keys"]) <= len(a["keys"])
    for k in ("gbuf", "n_contrib", "final_T", "T_last"):
        assert np.array_equal(a[k], b[k]), k


def _gate_flips_only(ours, ref):
    """Contributor counts equal the reference's except T > 1e-4 gate flips
    (fp32 vs fp64 transmittance): each differs by one fragment, and at most
    one pixel in 2000 flips (observed: 15 / 640,000 on the full cfg2 frame)."""
    d = np.asarray(ours, np.int64) - np.asarray(ref, np.int64)
    assert np.abs(d).max() <= 1
    assert int((d != 0).sum()) <= max(2, d.size // 2000), int((d != 0).sum())


def _crop_case(g, pre, scene, lut_table, env):
    """Oracle vs a reference crop window (tests/golden/make_golden_scale.py):
    counts exact except T-gate flips, all 13 G-buffer channels and the
    colour within the north_star bar."""
    cam = gio.camera(g, pre + "cam_")
    r = oracle.render(scene, cam)
    K = r["num_kept"]
    assert np.array_equal(r["sorted_ids"][:K], g[pre + "order"])
    _gate_flips_only(r["n_contrib"], g[pre + "counts"])
    ref = g[pre + "gbuf"].transpose(2, 0, 1)
    for c in range(13):
        assert np.abs(r["gbuf"][c] - ref[c]).max() <= TOL, c
    color, _, _ = oracle.shade(r["gbuf"], cam, env, lut_table, scene.background)
    assert np.abs(color - g[pre + "color"]).max() <= TOL
    return r


def _check_sha(g, scene):
    import hashlib
    for k in ("positions", "tangent_u", "scales", "texels"):
        h = hashlib.sha256(np.ascontiguousarray(getattr(scene, k)).tobytes()).hexdigest()
        assert h == str(g["sha_" + k]), k


def test_cfg2_full_frame_gbuffer_windows(lut_table):
    """All 13 G-buffer channels of the full cfg2 frame on three 160x160
    windows (centre, two silhouette windows)."""
    g = gio.load("cfg2_gbuf")
    scene = gio.cfg2_scene()
    _check_sha(g, scene)
    for pre in ("c_", "s_", "e_"):
        _crop_case(g, pre, scene, lut_table, scene.environment)


def test_cfg3_crop_two_page_shape(lut_table):
    """cfg3 geometry: 500k splats, T=8 (a 2-page atlas), 1920x1080 view 37
    of the 256-view orbit, 128x128 silhouette crop."""
    from paper_2506_13348_b200 import synth
    g = gio.load("cfg3_crop")
    scene = synth.make_shell_scene(500_000, 8, seed=3, with_environment=True)
    _check_sha(g, scene)
    _crop_case(g, "", scene, lut_table, scene.environment)
