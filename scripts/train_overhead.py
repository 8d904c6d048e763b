"""Host-side cost of one DataParallelTrainer.step (cfg4) vs its device time:
is the training step launch-bound? (diagnostic, prints one line)"""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_2506_13348_b200 import render_forward, shade_gbuffer, synth
from paper_2506_13348_b200.environment import BrdfLut
from paper_2506_13348_b200.training import DataParallelTrainer, linear_to_display

scene = synth.make_shell_scene(100_000, 8, seed=3, with_environment=True)
lut = BrdfLut.build()
views = synth.bench_cameras(8, 800, 800)
tg = [linear_to_display(shade_gbuffer(render_forward(scene, c, "perprim"), c, scene.environment,
                                      lut, background=scene.background).color) for c in views]
init = scene.copy(); init.positions = init.positions + 0.003
tr = DataParallelTrainer(init, lut)
for i in range(5):
    tr.step(views[i % 8], tg[i % 8])
torch.cuda.synchronize()
N = 40
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
cpu = 0.0
e0.record()
t0 = time.perf_counter()
for i in range(N):
    a = time.perf_counter()
    tr.step(views[i % 8], tg[i % 8])
    cpu += time.perf_counter() - a
e1.record()
torch.cuda.synchronize()
wall = time.perf_counter() - t0
print(f"device {e0.elapsed_time(e1) / N:.3f} ms/step, host enqueue {1e3 * cpu / N:.3f} ms/step, "
      f"wall {1e3 * wall / N:.3f} ms/step")

if len(sys.argv) > 1 and sys.argv[1] == "--profile":
    import cProfile, pstats
    pr = cProfile.Profile()
    pr.enable()
    for i in range(N):
        tr.step(views[i % 8], tg[i % 8])
    torch.cuda.synchronize()
    pr.disable()
    pstats.Stats(pr).sort_stats("tottime").print_stats(30)
