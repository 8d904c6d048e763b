"""GPU parity tests for the forward path (libtsb via the C ABI).

Bars:
  * vs the CPU oracle (shared decision math): draw order, (tile<<32|rank)
    sort keys, tile ranges, rects, per-pixel contributor counts, final T and
    the fp32 verify-mode / flat-mode G-buffer are BIT-EXACT;
  * vs the numpy reference (golden fixtures): G-buffer / colour max abs <= 1e-3;
  * hardware texture mode: PSNR >= 50 dB vs the oracle's verify G-buffer/colour.
"""
import numpy as np
import pytest
import torch

import golden_io as gio
from oracle import oracle
from paper_2506_13348_b200 import (MaterialTextureSet, Renderer, Scene, TextureConfig, pack_atlases,
                                   render_forward, shade_gbuffer, synth)
from paper_2506_13348_b200.rasterize import frame_structure, prepare, render_prepared
from paper_2506_13348_b200.splats import Camera

pytestmark = pytest.mark.gpu
TOL = 1e-3


def _np(t):
    return t.detach().cpu().numpy()


def _assert_structure_equal(tape, ref):
    st = frame_structure(tape)
    assert np.array_equal(st["sorted_ids"], ref["sorted_ids"])
    assert np.array_equal(st["rects"], ref["rects"])
    assert np.array_equal(st["keys"], ref["keys"])
    assert np.array_equal(st["ranges"], ref["ranges"])


def _assert_pixels_equal(gbuf, ref):
    px = gbuf.pixels
    assert np.array_equal(_np(px.n_contrib), ref["n_contrib"])
    assert np.array_equal(_np(px.last_entry), ref["last_entry"])
    assert np.array_equal(_np(px.final_T), ref["final_T"])
    assert np.array_equal(_np(px.T_last), ref["T_last"])


def psnr(a, b, peak=1.0):
    mse = float(np.mean((np.asarray(a, np.float64) - np.asarray(b, np.float64)) ** 2))
    return float("inf") if mse == 0 else 10.0 * np.log10(peak * peak / mse)


def test_cfg1_bit_exact_vs_oracle_and_golden(lut_table):
    g = gio.load("cfg1")
    scene, cam = gio.scene(g), gio.camera(g)
    gbuf, tape = render_forward(scene, cam, "perprim", with_tape=True)
    ref = oracle.render(scene, cam, tile=16)
    _assert_structure_equal(tape, ref)
    _assert_pixels_equal(gbuf, ref)
    assert np.array_equal(_np(gbuf.planar), ref["gbuf"])
    # vs the numpy reference
    assert np.abs(gbuf.numpy() - g["gbuf"]).max() <= TOL
    assert np.array_equal(_np(gbuf.pixels.n_contrib), g["counts"])
    assert gbuf.fragment_count == int(g["fragment_count"])
    sr = shade_gbuffer(gbuf, cam, scene.environment, gio.lut(), background=scene.background)
    assert np.abs(_np(sr.color) - g["color"]).max() <= TOL
    assert np.abs(_np(sr.diffuse) - g["diffuse"]).max() <= TOL
    assert np.abs(_np(sr.specular) - g["specular"]).max() <= TOL
    c_or, _, _ = oracle.shade(ref["gbuf"], cam, scene.environment, lut_table, scene.background)
    assert np.abs(_np(sr.color) - c_or).max() <= 1e-5


@pytest.mark.parametrize("tile", [8, 16, 32])
def test_tile_size_never_changes_output(tile):
    g = gio.load("small")
    scene, cam = gio.scene(g, "inv_"), gio.camera(g, "inv_cam_")
    gb = render_forward(scene, cam, "perprim", tile=tile)
    base = oracle.render(scene, cam, tile=16)
    assert np.array_equal(_np(gb.planar), base["gbuf"])
    assert np.array_equal(_np(gb.pixels.n_contrib), g["inv_counts"])
    gbt, tape = render_forward(scene, cam, "perprim", tile=tile, with_tape=True)
    _assert_structure_equal(tape, oracle.render(scene, cam, tile=tile))


def test_flat_mode_bit_exact_and_same_alpha():
    g = gio.load("small")
    scene, cam = gio.scene(g, "flat_"), gio.camera(g, "flat_cam_")
    flat = render_forward(scene, cam, "flat")
    per = render_forward(scene, cam, "perprim")
    assert np.array_equal(_np(flat.planar), oracle.render(scene, cam, mode="flat")["gbuf"])
    assert np.abs(flat.numpy() - g["flat_gbuf"]).max() <= TOL
    assert torch.equal(flat.alpha, per.alpha)
    assert not torch.equal(flat.albedo, per.albedo)


def test_atlas_verify_matches_perprim_bitwise_multipage():
    scene = synth.make_plane_scene(3, 3, 4, 7)
    cam = synth.camera_ring(1, width=48, height=48)[0]
    a = pack_atlases(scene, max_dim=8)  # 3 pages
    ref = render_forward(scene, cam, "perprim")
    alt = render_forward(scene, cam, "atlas", a, sampler="verify")
    assert torch.equal(ref.planar, alt.planar)
    hw = render_forward(scene, cam, "atlas", a, sampler="hw")
    assert psnr(_np(hw.planar), _np(ref.planar)) >= 50.0
    assert torch.equal(hw.pixels.n_contrib, ref.pixels.n_contrib)


def test_hw_texture_mode_psnr(lut_table):
    g = gio.load("cfg1")
    scene, cam = gio.scene(g), gio.camera(g)
    hw = render_forward(scene, cam, "atlas", pack_atlases(scene))
    ref = oracle.render(scene, cam)
    assert np.array_equal(_np(hw.pixels.n_contrib), ref["n_contrib"])
    assert psnr(_np(hw.planar)[:12], ref["gbuf"][:12]) >= 50.0
    sr = shade_gbuffer(hw, cam, scene.environment, gio.lut(), background=scene.background)
    c_or, _, _ = oracle.shade(ref["gbuf"], cam, scene.environment, lut_table, scene.background)
    assert psnr(_np(sr.color), c_or) >= 50.0
    hw16 = render_forward(scene, cam, "atlas", pack_atlases(scene), texel_format="rgba16f")
    assert psnr(_np(hw16.planar)[:12], ref["gbuf"][:12]) >= 50.0


def _facing_scene(zs, opacities, albedos, res=2):
    P = len(zs)
    tex = np.stack([MaterialTextureSet.constant(albedos[k], 0.5, 0.0, resolution=res).combined()
                    for k in range(P)])
    return Scene(np.array([[0.0, 0.0, z] for z in zs]), np.tile([1.0, 0.0, 0.0], (P, 1)),
                 np.tile([0.0, 1.0, 0.0], (P, 1)), np.full((P, 2), 0.8),
                 np.asarray(opacities, np.float64), np.zeros((P, 1, 3)), 0, tex,
                 TextureConfig(res))


def _center_camera():
    return Camera.look_at((0.0, 0.0, -2.0), (0.0, 0.0, 1.0), width=33, height=33, fov_x_deg=60.0)


def test_hand_values_single_and_two_splats():
    # rasterize tests :39-67 with fp32 tolerances
    gb = render_forward(_facing_scene([0.0], [0.7], [(0.8, 0.2, 0.1)]), _center_camera())
    assert abs(float(gb.alpha[16, 16]) - 0.7) < 1e-6
    exp = 0.7 * np.float32([0.8, 0.2, 0.1]).astype(np.float64)
    assert np.allclose(_np(gb.albedo[16, 16]), exp, atol=1e-6)
    gb = render_forward(_facing_scene([0.0, 1.0], [0.7, 0.5],
                                      [(0.8, 0.2, 0.1), (0.1, 0.9, 0.3)]), _center_camera())
    a = 0.7 + 0.5 * 0.3
    assert abs(float(gb.alpha[16, 16]) - a) < 1e-6
    cf, cb = np.float32([0.8, 0.2, 0.1]), np.float32([0.1, 0.9, 0.3])
    assert np.allclose(_np(gb.albedo[16, 16]), cf * 0.7 + cb * 0.5 * 0.3, atol=1e-6)
    assert abs(float(gb.depth[16, 16]) - (2.0 * 0.7 + 3.0 * 0.15)) < 1e-5
    assert np.allclose(_np(gb.normal[16, 16]), [0.0, 0.0, a], atol=1e-6)


def test_draw_order_is_depth_not_input_order():
    a = _facing_scene([0.0, 1.0], [0.7, 0.5], [(0.8, 0.2, 0.1), (0.1, 0.9, 0.3)])
    b = _facing_scene([1.0, 0.0], [0.5, 0.7], [(0.1, 0.9, 0.3), (0.8, 0.2, 0.1)])
    cam = _center_camera()
    assert torch.equal(render_forward(a, cam).planar, render_forward(b, cam).planar)


def test_culling_and_empty_frames():
    cam = _center_camera()
    gb = render_forward(_facing_scene([-5.0], [0.9], [(0.5, 0.5, 0.5)]), cam)
    assert gb.fragment_count == 0 and float(gb.planar.abs().max()) == 0.0
    s = _facing_scene([0.0], [0.9], [(0.5, 0.5, 0.5)])
    s.positions[0, 0] = 50.0
    assert render_forward(s, cam).fragment_count == 0


def test_saturation_alpha_one():
    s = _facing_scene([0.0, 1.0], [1.0, 1.0], [(1.0, 0.0, 0.0), (0.0, 1.0, 0.0)])
    gb = render_forward(s, _center_camera())
    assert float(gb.albedo[16, 16, 1]) == 0.0
    assert abs(float(gb.alpha[16, 16]) - 1.0) < 1e-6
    ref = oracle.render(s, _center_camera())
    assert np.array_equal(_np(gb.planar), ref["gbuf"])


def test_view_dependent_indirect_channel():
    s = _facing_scene([0.0], [1.0], [(0.5, 0.5, 0.5)])
    s.sh = np.zeros((1, 4, 3))
    s.sh[0, 0] = 0.5
    s.sh[0, 3] = 0.4
    s.sh_degree = 1
    cl = Camera.look_at((-1.5, 0.0, -2.0), (0.0, 0.0, 0.0), width=33, height=33)
    cr = Camera.look_at((1.5, 0.0, -2.0), (0.0, 0.0, 0.0), width=33, height=33)
    gl, gr = render_forward(s, cl), render_forward(s, cr)
    il = _np(gl.indirect[16, 16] / gl.alpha[16, 16])
    ir = _np(gr.indirect[16, 16] / gr.alpha[16, 16])
    assert not np.allclose(il, ir)
    d = s.positions[0] - cl.center
    d /= np.linalg.norm(d)
    C1 = 0.4886025119029199
    expect = np.maximum(0.0, 0.28209479177387814 * 0.5 + (-C1 * d[0]) * 0.4)
    assert np.allclose(il, expect, atol=1e-6)


def test_capacity_overflow_rerenders():
    g = gio.load("cfg1")
    scene, cam = gio.scene(g), gio.camera(g)
    prep = prepare(scene, cam, "perprim")
    prep.workspace.ensure(scene.num_splats, 128, 128, 16, 16)  # far too small
    gb, tape = render_prepared(prep, cam, 16)
    assert tape.capacity >= int(prep.workspace.needed.item())
    assert gb.fragment_count == int(g["fragment_count"])


def test_renderer_matches_one_shot_and_is_deterministic():
    g = gio.load("cfg1")
    scene, cam = gio.scene(g), gio.camera(g)
    r = Renderer(scene, pack_atlases(scene), scene.environment, gio.lut(), sampler="verify")
    c1, gb1 = r.render(cam)
    c1 = c1.clone()
    c2, _ = r.render(cam)
    assert torch.equal(c1, c2)
    sr = shade_gbuffer(render_forward(scene, cam, "perprim"), cam, scene.environment, gio.lut(),
                       background=scene.background)
    assert torch.equal(c1, sr.color)


def test_cfg2_crop_vs_golden():
    g = gio.load("cfg2_crop")
    scene, cam = gio.cfg2_scene(), gio.camera(g)
    gb = render_forward(scene, cam, "perprim")
    assert np.abs(gb.numpy() - g["gbuf"]).max() <= TOL
    assert np.array_equal(_np(gb.pixels.n_contrib), g["counts"])
    sr = shade_gbuffer(gb, cam, scene.environment, gio.lut(), background=scene.background)
    assert np.abs(_np(sr.color) - g["color"]).max() <= TOL


def test_cfg2_full_frame_bit_exact_vs_oracle(lut_table):
    """BASELINE configs[1] at full size: every structural output bit-exact."""
    scene = gio.cfg2_scene()
    cam = synth.bench_cameras(1, 800, 800)[0]
    atlas = pack_atlases(scene)
    gb, tape = render_forward(scene, cam, "atlas", atlas, sampler="verify", with_tape=True)
    ref = oracle.render(scene, cam, tile=16)
    _assert_structure_equal(tape, ref)
    _assert_pixels_equal(gb, ref)
    assert np.array_equal(_np(gb.planar), ref["gbuf"])
    # the reference's rect binning renders the same pixels (box is conservative)
    ref_rect = oracle.render(scene, cam, tile=16, binning="rect")
    assert np.array_equal(_np(gb.planar), ref_rect["gbuf"])
    assert np.array_equal(_np(gb.pixels.n_contrib), ref_rect["n_contrib"])
    full = np.load(gio.GOLDEN / "cfg2_full.npz")
    assert np.abs(_np(gb.alpha) - full["alpha"]).max() <= TOL
    sr = shade_gbuffer(gb, cam, scene.environment, gio.lut(), background=scene.background)
    assert np.abs(_np(sr.color) - full["color"]).max() <= TOL
    hw = render_forward(scene, cam, "atlas", atlas)
    assert torch.equal(hw.pixels.n_contrib, gb.pixels.n_contrib)
    c_or, _, _ = oracle.shade(ref["gbuf"], cam, scene.environment, lut_table, scene.background)
    srh = shade_gbuffer(hw, cam, scene.environment, gio.lut(), background=scene.background)
    assert psnr(_np(srh.color), c_or) >= 50.0


def test_empty_scene_and_odd_sizes():
    """P = 0, and image sizes that are not tile multiples (rasterize.py
    clips the last tiles to the image)."""
    s = _facing_scene([0.0], [0.9], [(0.5, 0.5, 0.5)])
    empty = Scene(np.zeros((0, 3)), np.zeros((0, 3)), np.zeros((0, 3)), np.zeros((0, 2)),
                  np.zeros(0), np.zeros((0, 1, 3)), 0, np.zeros((0, 2, 2, 7), np.float32),
                  TextureConfig(2))
    cam = Camera.look_at((0.0, 0.0, -2.0), (0.0, 0.0, 1.0), width=37, height=23)
    gb = render_forward(empty, cam, "flat")
    assert gb.fragment_count == 0 and float(gb.planar.abs().max()) == 0.0
    for tile in (8, 16, 32):
        gb = render_forward(s, cam, "perprim", tile=tile)
        ref = oracle.render(s, cam, tile=tile)
        assert np.array_equal(_np(gb.planar), ref["gbuf"])


def test_splat_crossing_near_plane_gets_fullscreen_rect():
    """Centre in front, a rect corner behind the near plane: full-screen rect
    (rasterize.py:151-168); results still match the oracle bit for bit."""
    s = _facing_scene([0.0], [0.9], [(0.5, 0.5, 0.5)])
    s.tangent_v[0] = [0.0, 0.0, 1.0]          # splat plane contains the view axis
    s.tangent_u[0] = [1.0, 0.0, 0.0]
    s.scales[0] = [0.8, 1.0]
    cam = Camera.look_at((0.0, 0.3, -1.0), (0.0, 0.0, 1.0), width=40, height=40, near=0.05)
    gb, tape = render_forward(s, cam, "perprim", with_tape=True)
    ref = oracle.render(s, cam)
    _assert_structure_equal(tape, ref)
    assert np.array_equal(_np(gb.planar), ref["gbuf"])
    assert ref["rects"][0].tolist() == [0, 40, 0, 40]


def test_bad_inputs_raise_reference_exceptions():
    from paper_2506_13348_b200 import prepare as prep
    s = synth.make_plane_scene(2, 2, 4, 5)
    cam = synth.camera_ring(1, width=16, height=16)[0]
    with pytest.raises(ValueError):
        prep(s, cam, "atlas", None)                      # rasterize.py:220-221
    with pytest.raises(ValueError):
        prep(s, cam, "atlas", pack_atlases(synth.make_plane_scene(2, 2, 2, 5)))  # :223-224
    with pytest.raises(ValueError):
        render_forward(s, cam, "perprim", tile=12)
    a = pack_atlases(s)
    a.indirection.entries[0, 0] = 10_000                 # chart out of range
    with pytest.raises(ValueError):
        render_forward(s, cam, "atlas", a)


def test_hw_rgba16f_and_multipage_hw_match_counts():
    scene = synth.make_plane_scene(6, 6, 4, 3)
    cam = synth.camera_ring(1, width=64, height=64)[0]
    ref = oracle.render(scene, cam)
    for fmt in ("rgba32f", "rgba16f"):
        gb = render_forward(scene, cam, "atlas", pack_atlases(scene, max_dim=16),
                            texel_format=fmt)                 # 3 pages, layered texture
        assert np.array_equal(_np(gb.pixels.n_contrib), ref["n_contrib"])
        assert psnr(_np(gb.planar)[:12], ref["gbuf"][:12]) >= 50.0


def test_frame_graph_matches_launches_and_rejects_other_sizes():
    """tsb_frame_graph_*: replaying the captured frame for new cameras gives
    bit-identical colour and G-buffers to the per-launch path."""
    from paper_2506_13348_b200 import Renderer, pack_atlases
    from paper_2506_13348_b200.environment import BrdfLut
    scene = synth.make_shell_scene(3000, 4, seed=3, with_environment=True, env_height=16,
                                   env_levels=3)
    cams = synth.bench_cameras(5, 96, 80)
    r = Renderer(scene, pack_atlases(scene), scene.environment, BrdfLut.build())
    for c in cams:
        r.render(c)
    r.reserve(cams[0], int(r.entries_needed() * 2) + 4096)
    ref = [(c_, g_.planar.clone()) for c_, g_ in (
        (lambda o: (o[0].clone(), o[1]))(r.render(c, check=True)) for c in cams)]
    for (col_ref, gb_ref), c in zip(ref, cams):
        col, gb = r.render(c, check=False)
        assert torch.equal(col, col_ref)
        assert torch.equal(gb.planar, gb_ref)
    other = synth.bench_cameras(1, 64, 64)[0]
    import ctypes as C
    from paper_2506_13348_b200 import _lib
    h, _ = r._graph(cams[0], 96, 80)
    with pytest.raises(ValueError):
        _lib.check(_lib.lib().tsb_frame_graph_launch(h, C.byref(_lib.camera_struct(other)), None,
                                                     None), "graph")
    r.close()


def test_full_hd_tile8_many_tiles_bit_exact():
    """1920x1080 at 8-px tiles (32,400 tiles: the one-CTA tile schedule loops,
    several hundred blocks per raster launch) and a camera close enough that
    splats cross the near plane and fill blocks whole (z-safe / surely-live
    block tests on both sides): structure and verify-mode pixels bit-exact."""
    scene = synth.make_shell_scene(6000, 4, seed=11)
    cam = synth.bench_cameras(8, 1920, 1080)[3]
    gbuf, tape = render_forward(scene, cam, "perprim", tile=8, with_tape=True)
    ref = oracle.render(scene, cam, tile=8)
    _assert_structure_equal(tape, ref)
    _assert_pixels_equal(gbuf, ref)
    assert np.array_equal(_np(gbuf.planar), ref["gbuf"])
    # inside-out close-up: the eye 0.12 from the shell, splats near the eye
    # reach behind the near plane (full-screen rects, not z-safe blocks)
    near = Camera.look_at((0.0, 0.0, 1.12), (0.0, 0.0, 0.0), fov_x_deg=100.0, width=320,
                          height=240, near=0.05)
    gbuf, tape = render_forward(scene, near, "perprim", tile=16, with_tape=True)
    ref = oracle.render(scene, near, tile=16)
    _assert_structure_equal(tape, ref)
    _assert_pixels_equal(gbuf, ref)
    assert np.array_equal(_np(gbuf.planar), ref["gbuf"])


@pytest.mark.parametrize("use_graph", [True, False])
def test_stream_views_yields_each_frame_in_order(use_graph):
    """Renderer.stream_views (the e2e path: read-back of frame i overlapped
    with frame i+1, started from an event inside the frame graph) returns
    every view's colour image, in order, identical to a plain render."""
    from paper_2506_13348_b200.environment import BrdfLut
    scene = synth.make_shell_scene(3000, 4, seed=5, with_environment=True)
    cams = synth.bench_cameras(7, 160, 120)
    r = Renderer(scene, pack_atlases(scene), scene.environment, BrdfLut.build(32, 128))
    need = 0
    for c in cams:
        r.render(c)
        need = max(need, r.entries_needed())
    r.reserve(cams[0], need + 1024)
    r.use_graph = use_graph
    expect = [_np(r.render(c)[0]).copy() for c in cams]
    for n in (1, 2, 5, 7):
        got = [(i, img.numpy().copy()) for i, img in r.stream_views(cams[:n])]
        assert [i for i, _ in got] == list(range(n))
        for i, img in got:
            assert np.array_equal(img, expect[i]), (n, i)


def test_render_normal_and_depth_maps():
    """reference test_rasterize.py:150-161 (fp32 tolerances)."""
    from paper_2506_13348_b200.rasterize import render_depth_map, render_normal_map
    scene = _facing_scene([0.0], [0.9], [(0.3, 0.3, 0.3)])
    scene.scales[:] = 0.05  # tiny footprint so the corners stay uncovered
    cam = _center_camera()
    gb = render_forward(scene, cam)
    assert float(gb.alpha[0, 0]) == 0.0
    n = _np(render_normal_map(scene, cam))
    assert np.allclose(n[16, 16], [0.5, 0.5, 1.0], atol=1e-6)
    assert np.allclose(n[0, 0], 0.5)  # uncovered -> mid-gray
    d = _np(render_depth_map(scene, cam))
    assert abs(float(d[16, 16]) - 2.0) < 1e-5
    assert float(d[0, 0]) == 0.0


def test_record_slot_permutation_never_changes_results():
    """Per-splat records stored by Morton slot (DeviceScene from a host scene)
    vs by id (record_slot = NULL): identical structure, pixels and G-buffer."""
    scene = synth.make_shell_scene(4000, 4, seed=9)
    cam = synth.bench_cameras(4, 200, 160)[1]
    out = []
    for morton in (True, False):
        prep = prepare(scene, cam, "perprim", sampler="verify")
        assert prep.scene.record_slot is not None
        if not morton:
            prep.scene.record_slot = None
        gb, tape = render_prepared(prep, cam, 16)
        out.append((gb, frame_structure(tape)))
    (g1, s1), (g2, s2) = out
    for k in ("sorted_ids", "keys", "ranges", "rects"):
        assert np.array_equal(s1[k], s2[k]), k
    assert np.array_equal(_np(g1.planar), _np(g2.planar))
    assert np.array_equal(_np(g1.pixels.n_contrib), _np(g2.pixels.n_contrib))
