"""Renderer.stream_views throughput with and without the frame graph."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2506_13348_b200 import Renderer, pack_atlases, synth  # noqa: E402
from paper_2506_13348_b200.environment import BrdfLut  # noqa: E402

scene = synth.make_shell_scene(100_000, 8, seed=3, with_environment=True)
cams = synth.bench_cameras(64, 800, 800)
r = Renderer(scene, pack_atlases(scene), scene.environment, BrdfLut.build())
for c in cams[:4]:
    r.render(c)
r.reserve(cams[0], int(r.entries_needed() * 1.3) + 4096)
for use in (False, True, False, True):
    r.use_graph = use
    for _ in r.stream_views(cams[:4]):
        pass
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    n = 0
    for _, img in r.stream_views(cams * 2):
        n += 1
    t1 = time.perf_counter()
    print(f"graph={use}: {n / (t1 - t0):.1f} fps")
