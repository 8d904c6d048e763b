"""A reference checkpoint loaded straight to the device renders exactly like
the same scene loaded on the host."""
from pathlib import Path

import pytest
import torch

from paper_2506_13348_b200 import formats, render_forward, synth
from paper_2506_13348_b200.rasterize import render_prepared

pytestmark = pytest.mark.gpu
G = Path(__file__).resolve().parent / "golden"


def test_device_checkpoint_renders_like_host():
    host = formats.load_scene(G / "io_ckpt")
    ds, tex, env, bg, meta = formats.load_scene_device(G / "io_ckpt", "cuda")
    assert ds.num_splats == host.num_splats == meta["num_splats"]
    prep = formats.prepare_device(ds, tex)
    cam = synth.camera_ring(1, width=48, height=40)[0]
    gb_dev, _ = render_prepared(prep, cam, 16)
    gb_host = render_forward(host, cam, "perprim")
    assert torch.equal(gb_dev.planar, gb_host.planar)
    assert torch.equal(gb_dev.pixels.n_contrib, gb_host.pixels.n_contrib)
