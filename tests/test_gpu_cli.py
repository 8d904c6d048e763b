"""`render --decompose` on the B200 path against the reference CLI's own
8-bit images (tests/golden/make_golden_io.py ran the reference's cmd_render on
the same checkpoint and camera). fp32 vs fp64 moves a value across a
quantisation step now and then: per-pixel difference <= 1 LSB in the
fp32-verify (perprim) mode; texture-unit sampling (--atlas) uses 8-bit
filter weights, so there the bar is PSNR >= 40 dB per image."""
import json
from pathlib import Path

import numpy as np
import pytest
from PIL import Image

from paper_2506_13348_b200 import cli

pytestmark = pytest.mark.gpu
G = Path(__file__).resolve().parent / "golden"
NAMES = ["albedo", "normal", "roughness", "metallic", "diffuse", "specular", "final"]


@pytest.mark.parametrize("atlas", [False, True])
def test_render_decompose_matches_reference(tmp_path, capsys, atlas):
    args = ["render", "--scene", str(G / "io_ckpt"), "--decompose", "--out", str(tmp_path)]
    assert cli.main(args + (["--atlas"] if atlas else [])) == 0
    summary = json.loads(capsys.readouterr().out)
    assert summary["command"] == "render" and summary["views"] == 1
    assert len(summary["files"]) == 7
    ref_dir = G / ("io_render_atlas" if atlas else "io_render_perprim")
    for n in NAMES:
        got = np.asarray(Image.open(tmp_path / f"view_000_{n}.png")).astype(np.int32)
        ref = np.asarray(Image.open(ref_dir / f"view_000_{n}.png")).astype(np.int32)
        assert got.shape == ref.shape, n
        d = np.abs(got - ref)
        if not atlas:
            assert d.max() <= 1, (n, d.max())
            assert (d > 0).mean() <= 0.01, (n, (d > 0).mean())
        else:
            mse = (d.astype(np.float64) ** 2).mean()
            assert mse == 0 or 10 * np.log10(255.0 ** 2 / mse) >= 40.0, (n, mse)


def test_bench_atlas_summary(capsys, tmp_path):
    cfg = tmp_path / "b.json"
    cfg.write_text(json.dumps({"splats": 2000, "views": 1, "width": 64, "rounds": 2}))
    assert cli.main(["bench-atlas", "--texture-res", "4", "--config", str(cfg)]) == 0
    s = json.loads(capsys.readouterr().out)
    for k in ("baseline", "software", "atlas"):
        assert s[k]["fps"] > 0 and s[k]["fragments_per_frame"] > 0
    assert s["baseline"]["fragments_per_frame"] == s["atlas"]["fragments_per_frame"]


def test_cli_errors_exit_2(tmp_path):
    assert cli.main(["render", "--scene", str(tmp_path / "missing")]) == 2
