"""The drop-in boundary under the reference's calling patterns (GPU).

  * resident device copies: texsplat's per-view loop (cli.py:63-68) calls
    render_forward / shade_gbuffer with the same host objects every view;
    nothing is re-uploaded, and an in-place update of the host arrays is
    picked up (resident.py);
  * capacity: frames replayed without a host check (CUDA graph) are
    validated through the device-side running maximum of the entry counts;
    stream_views re-renders from the first unverified frame after growing;
  * tapes: a tape whose workspace was reused by a later frame is refused.
"""
import numpy as np
import pytest
import torch

import golden_io as gio
from paper_2506_13348_b200 import (Renderer, pack_atlases, render_forward, resident,
                                   shade_gbuffer, synth)
from paper_2506_13348_b200.backward import splat_backward
from paper_2506_13348_b200.environment import BrdfLut
from paper_2506_13348_b200.rasterize import prepare, render_prepared

pytestmark = pytest.mark.gpu


def _scene():
    return synth.make_shell_scene(6000, 4, seed=3, with_environment=True, env_height=16,
                                  env_levels=3)


def test_cmd_render_loop_uploads_once_and_sees_in_place_updates():
    scene = _scene()
    atlas = pack_atlases(scene)
    lut = gio.lut()
    cams = synth.bench_cameras(3, 96, 80)
    outs = []
    for cam in cams:  # cli.py:63-68
        gbuf = render_forward(scene, cam, "atlas", atlas)
        sr = shade_gbuffer(gbuf, cam, scene.environment, lut, background=scene.background)
        outs.append(sr.color.clone())
    keys = [k for k in resident._cache if k[1] in (id(scene), id(atlas), id(scene.environment))]
    kinds = sorted(k[0] for k in keys)
    assert kinds == ["atlas", "env", "scene"], kinds  # one device copy of each
    first_scene = resident._cache[next(k for k in keys if k[0] == "scene")][2]
    # same objects again: same device copies, identical pixels
    gbuf = render_forward(scene, cams[0], "atlas", atlas)
    again = shade_gbuffer(gbuf, cams[0], scene.environment, lut, background=scene.background)
    assert torch.equal(again.color, outs[0])
    assert resident._cache[next(k for k in keys if k[0] == "scene")][2] is first_scene
    # an in-place update of the host arrays (e.g. an optimizer step) re-uploads
    scene.positions += 0.01
    gbuf = render_forward(scene, cams[0], "atlas", atlas)
    moved = shade_gbuffer(gbuf, cams[0], scene.environment, lut, background=scene.background)
    assert not torch.equal(moved.color, outs[0])
    fresh = synth.make_shell_scene(6000, 4, seed=3, with_environment=True, env_height=16,
                                   env_levels=3)
    fresh.positions += 0.01
    ref = render_forward(fresh, cams[0], "atlas", pack_atlases(fresh))
    assert torch.equal(gbuf.planar, ref.planar)


def test_graph_replays_report_overflow():
    scene = _scene()
    r = Renderer(scene, pack_atlases(scene), scene.environment, gio.lut())
    cams = synth.bench_cameras(6, 96, 80)
    r.render(cams[0], check=True)
    need = r.entries_needed()
    r.reserve(cams[0], need // 2)          # too small for every view
    r.prep.workspace.reset_max()
    for c in cams:
        r.render(c, check=False)           # CUDA graph, no host sync
    with pytest.raises(RuntimeError, match="overflow"):
        r.check_capacity()
    r.reserve(cams[0], 4 * need)
    for c in cams:
        r.render(c, check=False)
    r.check_capacity()                     # fits: no error


def test_stream_views_recovers_from_overflow():
    scene = _scene()
    r = Renderer(scene, pack_atlases(scene), scene.environment, gio.lut())
    cams = synth.bench_cameras(8, 96, 80)
    ref = []
    for c in cams:
        col, _ = r.render(c, check=True)
        ref.append(col.cpu().clone())
    need = max(_need(r, c) for c in cams)
    r.reserve(cams[0], need // 3)
    got = {}
    for i, img in r.stream_views(cams, pipeline=1):  # one view at a time
        got[i] = img.clone()
    assert sorted(got) == list(range(len(cams)))
    for i in range(len(cams)):
        assert torch.equal(got[i], ref[i]), i
    assert r.prep.workspace.capacity >= need


def _need(r, cam):
    r.render(cam, check=True)
    return r.entries_needed()


def test_stale_tape_is_refused():
    g = gio.load("backward")
    scene, cam = gio.scene(g, "bw_"), gio.camera(g, "bw_cam_")
    prep = prepare(scene, cam, "perprim")
    _, tape1 = render_prepared(prep, cam, 16)
    render_prepared(prep, cam, 16)  # a second frame into the same workspace
    with pytest.raises(RuntimeError, match="stale tape"):
        splat_backward(scene, cam, prep, tape1, g["bw_dbuf"])
    # separate render_forward(with_tape=True) calls keep independent tapes
    _, ta = render_forward(scene, cam, "perprim", with_tape=True)
    _, tb = render_forward(scene, cam, "perprim", with_tape=True)
    ga = splat_backward(scene, cam, None, ta, g["bw_dbuf"])
    gb = splat_backward(scene, cam, None, tb, g["bw_dbuf"])
    assert torch.allclose(ga.positions, gb.positions)


def test_pipelined_stream_views_match_and_recover():
    """Two frames in flight (independent workspaces on their own streams):
    the same images as one-at-a-time checked renders, also after an
    overflow restart."""
    scene = _scene()
    r = Renderer(scene, pack_atlases(scene), scene.environment, gio.lut())
    cams = synth.bench_cameras(9, 96, 80)
    ref = []
    for c in cams:
        col, _ = r.render(c, check=True)
        ref.append(col.cpu().clone())
    need = max(_need(r, c) for c in cams)
    for cap in (4 * need, need // 3):
        r.reserve(cams[0], cap)
        got = {i: img.clone() for i, img in r.stream_views(cams, pipeline=2)}
        assert sorted(got) == list(range(len(cams)))
        for i in range(len(cams)):
            assert torch.equal(got[i], ref[i]), (cap, i)


def test_integration_md_ctypes_stub_renders_like_the_package():
    """The ctypes binding INTEGRATION.md shows a texsplat maintainer (section
    2) runs as written against libtsb.so and gives the package's G-buffer."""
    import re
    from pathlib import Path
    root = Path(__file__).resolve().parent.parent
    code = re.search(r"## 2\..*?```python\n(.*?)```", (root / "INTEGRATION.md").read_text(),
                     re.S).group(1)
    code = code.replace('C.CDLL("libtsb.so")',
                        f'C.CDLL("{root / "paper_2506_13348_b200" / "libtsb.so"}")')
    ns = {}
    exec(compile(code, "INTEGRATION.md", "exec"), ns)
    scene = _scene()
    atlas = pack_atlases(scene)
    cam = synth.bench_cameras(1, 96, 80)[0]
    got = ns["render_forward_gpu"](scene, cam, atlas)
    ref = render_forward(scene, cam, "atlas", atlas).data
    assert torch.equal(got.contiguous(), ref.contiguous())


def test_concurrent_renders_on_two_streams():
    """Different cameras rendered at once from two host threads, each on its
    own stream, through the one-shot API: each result equals
    the serial render of its camera (no shared per-frame state)."""
    import threading
    scene = _scene()
    atlas = pack_atlases(scene)
    lut = gio.lut()
    cams = synth.bench_cameras(2, 96, 80)
    ref = [shade_gbuffer(render_forward(scene, c, "atlas", atlas), c, scene.environment, lut,
                         background=scene.background).color.clone() for c in cams]
    torch.cuda.synchronize()
    out = [None, None]
    dev = torch.cuda.current_device()

    def work(i):
        torch.cuda.set_device(dev)
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            for _ in range(20):
                g = render_forward(scene, cams[i], "atlas", atlas)
                out[i] = shade_gbuffer(g, cams[i], scene.environment, lut,
                                       background=scene.background).color.clone()
            s.synchronize()

    th = [threading.Thread(target=work, args=(i,)) for i in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for i in range(2):
        assert torch.equal(out[i], ref[i]), i
