"""Frame graph vs the per-launch path: identical colour images, host cost."""
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
ref = [r.render(c, check=True)[0].clone() for c in cams[:6]]
got = [r.render(c, check=False)[0].clone() for c in cams[:6]]
torch.cuda.synchronize()
print("max diff graph vs launches", max(float((a - b).abs().max()) for a, b in zip(ref, got)))
for use in (False, True):
    r.use_graph = use
    torch.cuda.synchronize()
    x = torch.empty(1 << 28, device="cuda")
    x.fill_(1.0)
    N = 200
    t0 = time.perf_counter()
    for i in range(N):
        r.render(cams[i % 64], check=False)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"graph={use}: host per frame {1e3 * (t1 - t0) / N:.3f} ms; wall {1e3 * (t2 - t0) / N:.3f} ms")
