"""Data-parallel training step across 2 ranks (gloo) on ONE GPU.

Each rank runs DataParallelTrainer.step on its own view; the flat gradient
buffer after the bucketed all-reduce must equal the mean of the two
single-rank gradients (computed by each rank for both views without a
group), and the post-Adam parameters must be bitwise identical on both
ranks. The ranks share the device only for this
correctness check; nothing here is timed.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_dir):
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parent.parent
    sys.path.insert(0, str(root))
    sys.path.insert(0, str(root / "tests"))
    import torch.distributed as dist

    import golden_io as gio
    from paper_2506_13348_b200 import render_forward, shade_gbuffer, synth
    from paper_2506_13348_b200.training import DataParallelTrainer, linear_to_display

    torch.cuda.set_device(0)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    truth = synth.make_gradcheck_scene(11)
    cams = synth.camera_ring(2, width=32, height=32)
    lut = gio.lut()
    tgts = [linear_to_display(shade_gbuffer(render_forward(truth, c, "perprim"), c,
                                            truth.environment, lut,
                                            background=truth.background).color) for c in cams]
    init = truth.copy()
    init.texels = np.clip(init.texels + 0.1, 0.0, 1.0).astype(np.float32)
    init.positions = init.positions + 0.002

    # single-rank gradients of both views (no group: no all-reduce)
    solo = DataParallelTrainer(init, lut, texel_buckets=3)
    solo.group = None
    singles = []
    for c, t in zip(cams, tgts):
        solo.grads_and_loss(c, t)
        singles.append(solo.flat.clone())
    mean = (singles[0] + singles[1]) / 2

    tr = DataParallelTrainer(init, lut, texel_buckets=3)
    _, flat = tr.step(cams[rank], tgts[rank])
    torch.cuda.synchronize()
    np.save(os.path.join(out_dir, f"flat{rank}.npy"), flat.cpu().numpy())
    np.save(os.path.join(out_dir, f"mean{rank}.npy"), mean.cpu().numpy())
    for n, p in tr.params.items():
        np.save(os.path.join(out_dir, f"{n}{rank}.npy"), p.cpu().numpy())
    np.save(os.path.join(out_dir, f"texels{rank}.npy"), tr.texels8.cpu().numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_two_ranks_mean_gradient_and_identical_parameters(tmp_path):
    world, port = 2, _free_port()
    mp.start_processes(_worker, args=(world, port, str(tmp_path)), nprocs=world, join=True,
                       start_method="spawn")
    f0, f1 = np.load(tmp_path / "flat0.npy"), np.load(tmp_path / "flat1.npy")
    assert np.array_equal(f0, f1)  # every rank holds the same reduced buffer
    m = np.load(tmp_path / "mean0.npy")
    scale = np.abs(m).max()
    assert np.abs(f0 - m).max() <= 1e-5 * scale
    for n in ("positions", "tangent_u", "tangent_v", "scales", "opacities", "sh", "texels"):
        assert np.array_equal(np.load(tmp_path / f"{n}0.npy"), np.load(tmp_path / f"{n}1.npy")), n
