"""Work counters of k_raster_fwd for one cfg2 frame (instrumented build:
make -C paper_2506_13348_b200/csrc EXTRA=-DTSB_STATS OUT=../libtsb_stats.so BUILD=build_stats,
run with TSB_LIB=paper_2506_13348_b200/libtsb_stats.so)."""
import ctypes as C
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2506_13348_b200 import Renderer, pack_atlases, synth, _lib  # noqa: E402
from paper_2506_13348_b200.environment import BrdfLut  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
P, T, W, H = {"cfg2": (100_000, 8, 800, 800), "cfg5": (2_000_000, 16, 1920, 1080)}[cfg]
scene = synth.make_shell_scene(P, T, seed=3, with_environment=True)
cam = synth.bench_cameras(256, W, H)[0]
r = Renderer(scene, pack_atlases(scene), scene.environment, BrdfLut.build(), texture_mode="atlas",
             sampler="hw")
lib = _lib.lib()
buf = (C.c_ulonglong * 16)()
r.render(cam, check=True)
torch.cuda.synchronize()
lib.tsb_debug_stats(buf, 1)
r.render(cam)
torch.cuda.synchronize()
lib.tsb_debug_stats(buf, 1)
s = list(buf)
names = {0: "units", 1: "steps", 2: "candidates", 3: "full_candidates", 5: "pair_iterations",
         6: "composited_pairs", 8: "undone_lanes_at_decide", 9: "live_pairs_decided",
         10: "undone_lane_x_candidate_tests"}
out = {v: s[k] for k, v in names.items()}
out["pair_lane_util"] = s[6] / max(1, s[5] * 32 * 2)
out["full_frac"] = s[3] / max(1, s[2])
out["cand_per_step"] = s[2] / max(1, s[1])
out["live_per_test"] = s[9] / max(1, s[10])
print(json.dumps(out, indent=1))
