"""On-disk formats (paper_2506_13348_b200.formats) against files written by
the REFERENCE writers (tests/golden/make_golden_io.py): readers recover the
reference's arrays exactly, writers reproduce its files byte for byte, and
the reference's error types are raised."""
import filecmp
import json
from pathlib import Path

import numpy as np
import pytest

from paper_2506_13348_b200 import formats

G = Path(__file__).resolve().parent / "golden"


@pytest.fixture(scope="module")
def expected():
    return np.load(G / "io_expected.npz")


def test_load_scene_matches_reference_arrays(expected):
    s = formats.load_scene(G / "io_ckpt")
    for name in ("positions", "tangent_u", "tangent_v", "scales", "opacities", "sh", "texels",
                 "background"):
        assert np.array_equal(getattr(s, name), expected[name]), name
    assert np.array_equal(s.environment.spec_mips[0], expected["spec0"])
    assert np.array_equal(s.environment.diffuse, expected["diffuse"])


def test_save_scene_is_byte_identical(tmp_path):
    s = formats.load_scene(G / "io_ckpt" / "scene.json")
    formats.save_scene(s, tmp_path / "out")
    names = sorted(p.name for p in (G / "io_ckpt").iterdir())
    assert sorted(p.name for p in (tmp_path / "out").iterdir()) == names
    for n in names:
        assert filecmp.cmp(G / "io_ckpt" / n, tmp_path / "out" / n, shallow=False), n


def test_atlas_round_trip_is_byte_identical(tmp_path):
    a = formats.load_atlases(G / "io_atlas" / "atlas.json")
    formats.save_atlases(a, tmp_path)
    for p in (G / "io_atlas").iterdir():
        assert filecmp.cmp(p, tmp_path / p.name, shallow=False), p.name


def test_manifest_round_trip(tmp_path, expected):
    cams, imgs = formats.load_manifest(G / "io_manifest.json")
    assert [p.name for p in imgs] == ["a.png", "b.png"]
    assert np.array_equal(cams[0].world_to_view, expected["cam0"])
    formats.save_manifest(tmp_path / "m.json", cams, ["a.png", "b.png"])
    assert json.loads((tmp_path / "m.json").read_text()) == json.loads(
        (G / "io_manifest.json").read_text())


def test_reference_error_types(tmp_path):
    with pytest.raises(formats.MissingReferenceError):
        formats.load_scene(tmp_path / "nothing")
    d = tmp_path / "bad"
    d.mkdir()
    (d / "scene.json").write_text(json.dumps({"version": 99}))
    with pytest.raises(formats.VersionError):
        formats.load_scene(d)
    (d / "scene.json").write_text("{not json")
    with pytest.raises(formats.SchemaError):
        formats.load_scene(d)
    blob = d / "x.bin"
    blob.write_bytes(b"XXXX" + b"\0" * 12)
    with pytest.raises(formats.SchemaError):
        formats.read_splats_blob(blob)
    assert issubclass(formats.SchemaError, ValueError)
    assert issubclass(formats.MissingReferenceError, FileNotFoundError)
