"""Host-side logic: atlas packing, ABI surface, error mapping (no GPU)."""
import ctypes
import re

import numpy as np
import pytest

from conftest import ROOT
from paper_2506_13348_b200 import _lib, atlas, synth
from paper_2506_13348_b200.scene import MaterialTextureSet


def test_library_exports_every_declared_symbol():
    h = ctypes.CDLL(str(_lib.LIB_PATH))
    declared = _lib.exported_symbols()
    assert "tsb_render_forward" in declared and "tsb_shade_forward" in declared
    for name in declared:
        assert hasattr(h, name), name


def test_header_is_plain_c():
    hdr = (ROOT / "include" / "tsb.h").read_text()
    assert 'extern "C"' in hdr
    assert "torch" not in hdr and "at::" not in hdr


def test_chart_grid_values():
    assert atlas.chart_grid(10, 4, 16) == (4, 3, 1)
    assert atlas.chart_grid(100, 4, 16) == (4, 4, 7)
    assert atlas.chart_grid(100_000, 8, 4096) == (512, 196, 1)
    with pytest.raises(ValueError):
        atlas.chart_grid(1, 32, 16)
    with pytest.raises(ValueError):
        atlas.chart_grid(0, 4, 16)


def test_pack_places_every_chart_once():
    s = synth.make_plane_scene(3, 3, 4, 7)
    a = atlas.pack_atlases(s, max_dim=8)
    assert a.indirection.pages == 3
    for k in range(9):
        cx, cy, pg = a.indirection.lookup(k)
        blk = s.texels[k]
        pa = a.family_a[pg].texels[cy * 4:(cy + 1) * 4, cx * 4:(cx + 1) * 4]
        pb = a.family_b[pg].texels[cy * 4:(cy + 1) * 4, cx * 4:(cx + 1) * 4]
        assert np.array_equal(pa[..., 0:3], blk[..., 0:3])
        assert np.array_equal(pa[..., 3], blk[..., 3])
        assert np.array_equal(pb[..., 0:2], blk[..., 5:7])
        assert np.array_equal(pb[..., 2], blk[..., 4])
        assert np.all(pb[..., 3] == 0)
    with pytest.raises(LookupError):
        a.indirection.lookup(9)


def test_pack_from_material_sets_equals_array_path():
    s = synth.make_plane_scene(2, 2, 4, 5)
    a1 = atlas.pack_atlases(s.texels)
    a2 = atlas.pack_atlases([MaterialTextureSet.from_combined(b) for b in s.texels])
    assert np.array_equal(a1.family_a[0].texels, a2.family_a[0].texels)
    assert np.array_equal(a1.indirection.entries, a2.indirection.entries)


def test_pack_matches_oracle_layout():
    from oracle import oracle
    s = synth.make_plane_scene(5, 5, 4, 3)
    a = atlas.pack_atlases(s, max_dim=16)
    fa, fb, ent = oracle.pack(s.texels, max_dim=16)
    assert np.array_equal(np.stack([p.texels for p in a.family_a]), fa)
    assert np.array_equal(np.stack([p.texels for p in a.family_b]), fb)
    assert np.array_equal(a.indirection.entries, ent)


def test_error_mapping():
    class FakeLib:
        def tsb_last_error(self):
            return b"boom"
    old = _lib._lib
    _lib._lib = FakeLib()
    try:
        with pytest.raises(ValueError):
            _lib.check(_lib.TSB_ERR_VALUE, "x")
        with pytest.raises(LookupError):
            _lib.check(_lib.TSB_ERR_LOOKUP, "x")
        with pytest.raises(_lib.TsbError):
            _lib.check(_lib.TSB_ERR_CUDA, "x")
        _lib.check(_lib.TSB_OK, "x")
    finally:
        _lib._lib = old


def test_ctypes_struct_layouts_match_header():
    assert ctypes.sizeof(_lib.Camera_t) == 16 * 8 + 6 * 8 + 8
    assert ctypes.sizeof(_lib.Scene_t) == 8 + 7 * 8
    assert ctypes.sizeof(_lib.Atlas_t) == 16 + 5 * 8 + 8
    assert ctypes.sizeof(_lib.PixelState_t) == 5 * 8


def test_product_path_never_imports_oracle():
    pkg = ROOT / "paper_2506_13348_b200"
    for f in pkg.rglob("*.py"):
        txt = f.read_text()
        assert not re.search(r"^\s*(from|import)\s+oracle", txt, re.M), f


def test_prepare_rejects_bad_mode():
    from paper_2506_13348_b200 import prepare
    s = synth.make_plane_scene(2, 2, 4, 5)
    with pytest.raises(ValueError):
        prepare(s, None, "bogus")
