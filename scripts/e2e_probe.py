"""Where the e2e frame time goes: graph replays alone (host-timed), with the
colour readback (stream_views), and device-timed graph replays."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2506_13348_b200 import Renderer, pack_atlases, synth  # noqa: E402
from paper_2506_13348_b200.environment import BrdfLut  # noqa: E402

scene = synth.make_shell_scene(100_000, 8, seed=3, with_environment=True)
cams = synth.bench_cameras(256, 800, 800)
r = Renderer(scene, pack_atlases(scene), scene.environment, BrdfLut.build())
need = 0
for c in cams[::16]:
    r.render(c)
    need = max(need, r.entries_needed())
r.reserve(cams[0], int(need * 1.15) + 4096)
N = 100
views = [cams[i % len(cams)] for i in range(N)]
for rep in range(2):
    for c in views[:5]:
        r.render(c, check=False)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    for c in views:
        r.render(c, check=False)
    e1.record()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"graph replays: host launch {1e3 * (t1 - t0) / N:.3f} ms/frame, wall "
          f"{1e3 * (t2 - t0) / N:.3f}, device {e0.elapsed_time(e1) / N:.3f} ms/frame")
    for _ in r.stream_views(views[:4]):
        pass
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in r.stream_views(views):
        pass
    t1 = time.perf_counter()
    print(f"stream_views: {1e3 * (t1 - t0) / N:.3f} ms/frame ({N / (t1 - t0):.0f} fps)")
for depth in (2, 3, 4):
    for _ in r.stream_views(views[:6], depth=depth):
        pass
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in r.stream_views(views, depth=depth):
        pass
    t1 = time.perf_counter()
    print(f"stream_views depth {depth}: {1e3 * (t1 - t0) / N:.3f} ms/frame ({N / (t1 - t0):.0f} fps)")
src = torch.empty((800, 800, 3), device="cuda")
dst = torch.empty((800, 800, 3), pin_memory=True)
for _ in range(3):
    dst.copy_(src, non_blocking=True)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(20):
    dst.copy_(src, non_blocking=True)
torch.cuda.synchronize()
t1 = time.perf_counter()
print(f"D2H 7.68 MB pinned: {1e3 * (t1 - t0) / 20:.3f} ms ({7.68e6 * 20 / (t1 - t0) / 1e9:.1f} GB/s)")
copy = torch.cuda.Stream()
comp = torch.cuda.current_stream()
dcol = [torch.empty((800, 800, 3), device="cuda") for _ in range(4)]
hcol = [torch.empty((800, 800, 3), pin_memory=True) for _ in range(4)]
ev = [torch.cuda.Event() for _ in range(4)]
for variant in ("dep-copies", "indep-copies", "no-copies-events"):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i, c in enumerate(views):
        b = i % 4
        r.render(c, check=False, stream=comp, color=dcol[b])
        if variant == "dep-copies":
            ev[b].record(comp)
            copy.wait_event(ev[b])
            with torch.cuda.stream(copy):
                hcol[b].copy_(dcol[b], non_blocking=True)
        elif variant == "indep-copies":
            with torch.cuda.stream(copy):
                hcol[b].copy_(dcol[(b + 2) % 4], non_blocking=True)
        else:
            ev[b].record(comp)
            copy.wait_event(ev[b])
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    print(f"{variant}: {1e3 * (t1 - t0) / N:.3f} ms/frame")
