"""GPU binning (tsb_binning.cu) edge cases vs the CPU oracle, bit-exact.

The draw order is np.lexsort((ids, z)) (rasterize.py:178-182) and the tile
lists keep it (rasterize.py:246-258). The GPU sorts a 32-bit depth key with
one-sweep radix passes and re-orders runs of equal keys by the full fp64
depth; these scenes stress exactly that:
  * a frontal plane: 100k splats at ONE depth (a single run of equal full
    keys, ties broken by id) — must stay fast (no O(run^2) path);
  * far content: depths 1000..1001 with near = 0.01 (the old 24-bit key
    clamped every depth beyond near * 2^16 to one key);
  * a long run of distinct depths inside one 2^-20 key bucket in reverse id
    order (k_sort_long_runs re-sorts it);
  * sizes / tiles that exercise the one-sweep tails (P not a multiple of
    4096, entries not a multiple of 4096, tile 8 / 32).
"""
import time

import numpy as np
import pytest
import torch

from oracle import oracle
from paper_2506_13348_b200 import MaterialTextureSet, Scene, TextureConfig, render_forward, synth
from paper_2506_13348_b200.rasterize import frame_structure
from paper_2506_13348_b200.splats import Camera

pytestmark = pytest.mark.gpu


def _np(t):
    return t.detach().cpu().numpy()


def _plane_scene(n_side, z_of, scale=0.01, seed=0):
    """n_side^2 facing splats on a grid in [-1, 1]^2 at depths z_of(ids)."""
    P = n_side * n_side
    g = (np.arange(n_side) + 0.5) / n_side * 2.0 - 1.0
    xx, yy = np.meshgrid(g, g)
    pos = np.stack([xx.ravel(), yy.ravel(), z_of(np.arange(P))], 1)
    rng = np.random.default_rng(seed)
    base = MaterialTextureSet.constant((0.5, 0.5, 0.5), 0.5, 0.0, resolution=2).combined()
    tex = np.repeat(base[None], P, 0)
    tex[:, :, :, 0:3] = rng.uniform(0.1, 0.9, (P, 1, 1, 3)).astype(np.float32)
    return Scene(pos, np.tile([1.0, 0.0, 0.0], (P, 1)), np.tile([0.0, 1.0, 0.0], (P, 1)),
                 np.full((P, 2), scale * 2.0 / n_side * 30), np.full(P, 0.6),
                 np.zeros((P, 1, 3)), 0, tex, TextureConfig(2))


def _check(scene, cam, tile=16):
    gb, tape = render_forward(scene, cam, "perprim", tile=tile, with_tape=True)
    ref = oracle.render(scene, cam, tile=tile)
    st = frame_structure(tape)
    K = ref["num_kept"]
    assert np.array_equal(st["sorted_ids"][:K], ref["sorted_ids"][:K])
    assert np.array_equal(st["keys"], ref["keys"])
    assert np.array_equal(st["ranges"], ref["ranges"])
    assert np.array_equal(_np(gb.pixels.n_contrib), ref["n_contrib"])
    assert np.array_equal(_np(gb.planar), ref["gbuf"])
    return gb, ref


def _timed_frame(scene, cam):
    render_forward(scene, cam, "perprim")
    torch.cuda.synchronize()
    t = time.perf_counter()
    render_forward(scene, cam, "perprim")
    torch.cuda.synchronize()
    return time.perf_counter() - t


def test_frontal_plane_one_depth():
    scene = _plane_scene(316, lambda i: np.full(i.shape, 3.0))  # 99,856 splats, z = 3 exactly
    cam = Camera.look_at((0.0, 0.0, 0.0), (0.0, 0.0, 1.0), width=256, height=256, fov_x_deg=50.0)
    gb, ref = _check(scene, cam)
    assert ref["num_kept"] == scene.num_splats
    assert np.array_equal(ref["sorted_ids"], np.arange(scene.num_splats))  # ties: by id
    assert _timed_frame(scene, cam) < 0.5  # (the host path dominates; no O(run^2) sort)


def test_far_content_beyond_old_key_clamp():
    rng = np.random.default_rng(5)
    scene = _plane_scene(200, lambda i: 1000.0 + rng.random(i.shape), scale=0.8)
    cam = Camera.look_at((0.0, 0.0, 0.0), (0.0, 0.0, 1.0), width=160, height=120,
                         fov_x_deg=0.2, near=0.01, far=5000.0)
    _check(scene, cam)


def test_long_run_of_distinct_depths_in_one_key_bucket():
    # 2^-20 relative key resolution at z = 2: depths 2 + i * 1e-13 share one
    # 32-bit key but differ in the fp64 pattern; decreasing in id => the whole
    # run must be reversed by the full-key re-sort
    P = 120 * 120
    scene = _plane_scene(120, lambda i: 2.0 + (P - i) * 1e-13, scale=0.3)
    cam = Camera.look_at((0.0, 0.0, 0.0), (0.0, 0.0, 1.0), width=96, height=96, fov_x_deg=40.0)
    gb, ref = _check(scene, cam)
    K = ref["num_kept"]
    assert K > 1000 and np.all(np.diff(ref["sorted_ids"][:K]) < 0)


@pytest.mark.parametrize("tile", [8, 16, 32])
def test_onesweep_tails_and_tiles(tile):
    scene = synth.make_shell_scene(9_001, 2, seed=4)
    cam = synth.bench_cameras(3, 203, 147)[1]
    _check(scene, cam, tile)
