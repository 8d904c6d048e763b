"""Run-to-run and GPU-vs-reference drift of train() on the train_loop golden
(diagnostic for the tolerance in tests/test_gpu_train.py)."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "tests"))
import golden_io as gio  # noqa: E402
from paper_2506_13348_b200.training import TrainConfig, train  # noqa: E402

g = gio.load("train_loop")
scene = gio.scene(g, "init_")
cams = [gio.camera(g, f"cam{i}_") for i in range(int(g["n_cams"]))]
targets = [g[f"target{i}"] for i in range(len(cams))]
cfg = TrainConfig(iterations=24, stage_split=12, texture_resolution=4, prune_interval=5,
                  prune_opacity=0.005, seed=4)
ref = g["h_loss"]
for det in (False, True):
    runs = [np.array([h["loss"] for h in train(scene, cams, targets, cfg, gio.lut(),
                                               deterministic=det)[1]]) for _ in range(3)]
    for r in runs:
        print("det" if det else "atomics", "vs ref max rel", float(np.max(np.abs(r - ref) / ref)),
              "stage1", float(np.max(np.abs(r - ref)[:12] / ref[:12])))
    print("  run-to-run max rel", float(np.max(np.abs(runs[0] - runs[1]) / ref)),
          float(np.max(np.abs(runs[0] - runs[2]) / ref)))
