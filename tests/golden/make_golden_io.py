"""Generate the on-disk-format fixtures with the REFERENCE writers (run here,
where /root/reference exists): a small checkpoint, its atlas pages and a
manifest, plus the arrays they hold (io_expected.npz). The tests read them
with paper_2506_13348_b200.formats and re-write them byte for byte.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_io.py
"""
import shutil
from pathlib import Path

import numpy as np
from texsplat.atlas import pack_atlases, save_atlases
from texsplat.scene import save_manifest, save_scene
from texsplat.synth import camera_ring, make_plane_scene

HERE = Path(__file__).resolve().parent
for d in ("io_ckpt", "io_atlas"):
    shutil.rmtree(HERE / d, ignore_errors=True)
scene = make_plane_scene(nx=4, ny=4, texture_res=2, seed=7)
save_scene(scene, HERE / "io_ckpt")
save_atlases(pack_atlases(scene.textures, max_dim=8), HERE / "io_atlas")
cams = camera_ring(2, width=16, height=12)
save_manifest(HERE / "io_manifest.json", cams, ["a.png", "b.png"])
np.savez_compressed(
    HERE / "io_expected.npz", positions=scene.positions, tangent_u=scene.tangent_u,
    tangent_v=scene.tangent_v, scales=scene.scales, opacities=scene.opacities, sh=scene.sh,
    texels=np.stack([t.combined() for t in scene.textures]),
    spec0=scene.environment.spec_mips[0], diffuse=scene.environment.diffuse,
    background=scene.background, cam0=cams[0].world_to_view, cam1=cams[1].world_to_view)
print("ok", scene.num_splats)

# reference `render --decompose` of the checkpoint (default camera), both
# texture modes: the 8-bit images the CLI test compares against
from texsplat.cli import main as ref_main  # noqa: E402

for mode, extra in (("perprim", []), ("atlas", ["--atlas"])):
    out = HERE / f"io_render_{mode}"
    shutil.rmtree(out, ignore_errors=True)
    ref_main(["render", "--scene", str(HERE / "io_ckpt"), "--decompose", "--out", str(out)]
             + extra)
