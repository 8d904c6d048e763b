"""Input generators reproduce the reference's scenes bit-for-bit."""
import hashlib

import numpy as np

import golden_io as gio
from paper_2506_13348_b200 import synth
from paper_2506_13348_b200.environment import BrdfLut


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def test_plane_scene_matches_reference():
    g = gio.load("cfg1")
    s = synth.make_plane_scene(32, 32, 4, 7)
    for k in ("positions", "tangent_u", "tangent_v", "scales", "opacities", "sh", "texels"):
        assert np.array_equal(getattr(s, k), g[k]), k
    for i in range(int(g["env_levels"])):
        assert np.array_equal(s.environment.spec_mips[i], g[f"env_mip{i}"])
    assert np.array_equal(s.environment.diffuse, g["env_diffuse"])
    cam = synth.camera_ring(1, width=128, height=128)[0]
    assert np.array_equal(cam.world_to_view, g["cam_w2v"])


def test_shell_scene_matches_reference():
    g = gio.load("cfg2_crop")
    s = gio.cfg2_scene()
    for k in ("positions", "tangent_u", "tangent_v", "scales"):
        assert _sha(getattr(s, k)) == str(g["sha_" + k]), k
    assert _sha(s.texels) == str(g["sha_texels"])
    for i in range(6):
        assert np.array_equal(s.environment.spec_mips[i], g[f"env_mip{i}"])
    full = synth.bench_cameras(1, 800, 800)[0]
    assert np.array_equal(full.world_to_view, g["full_cam_w2v"])


def test_brdf_lut_matches_reference():
    ref = gio.load("lut")["table"]
    assert np.abs(BrdfLut.build().table - ref).max() < 1e-12
