"""A few cfg4 training steps for ncu (no timing)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

from paper_2506_13348_b200 import render_forward, shade_gbuffer, synth  # noqa: E402
from paper_2506_13348_b200.environment import BrdfLut  # noqa: E402
from paper_2506_13348_b200.training import DataParallelTrainer, linear_to_display  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
scene = synth.make_shell_scene(100_000, 8, seed=3, with_environment=True)
cam = synth.bench_cameras(256, 800, 800)[0]
lut = BrdfLut.build()
tgt = linear_to_display(shade_gbuffer(render_forward(scene, cam, "perprim"), cam,
                                      scene.environment, lut, background=scene.background).color)
init = scene.copy()
init.positions = init.positions + 0.003
tr = DataParallelTrainer(init, lut)
for _ in range(steps):
    terms, _ = tr.step(cam, tgt)
torch.cuda.synchronize()
print("ok", terms["loss"])
