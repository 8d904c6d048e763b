"""Full-frame cfg2 reference outputs (BASELINE configs[1]) for the oracle pin.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_full.py

Renders make_shell_scene(100000, 8, seed=3) + _lobe_environment(rng(0), 64, 6)
through bench_cameras(1, 800, 800)[0] with the numpy reference (~1 min) and
stores per-pixel contributor counts, alpha and the shaded colour.
"""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(Path(__file__).resolve().parent))

from make_golden import tape_counts  # noqa: E402
from texsplat.environment import BrdfLut, EnvironmentLight  # noqa: E402
from texsplat.rasterize import prepare, render_forward  # noqa: E402
from texsplat.shading import shade_gbuffer  # noqa: E402
from texsplat.synth import _lobe_environment, bench_cameras, make_shell_scene  # noqa: E402

OUT = Path(__file__).resolve().parent


def main():
    t0 = time.time()
    lut = BrdfLut(np.load(OUT / "lut.npz")["table"])
    shell = make_shell_scene(100_000, 8, seed=3)
    shell.environment = _lobe_environment(np.random.default_rng(0), height=64, levels=6)
    cam = bench_cameras(1, 800, 800)[0]
    prep = prepare(shell, cam, "perprim")
    gbuf, tape = render_forward(shell, cam, "perprim", with_tape=True, prep=prep)
    print(f"render {time.time() - t0:.1f}s", flush=True)
    sr = shade_gbuffer(gbuf, cam, shell.environment, lut, background=shell.background)
    np.savez_compressed(OUT / "cfg2_full.npz",
                        counts=tape_counts(tape, 800, 800).astype(np.int16),
                        fragment_count=np.array(gbuf.fragment_count),
                        alpha=gbuf.alpha.astype(np.float32),
                        color=sr.color.astype(np.float32),
                        order=prep.order.indices.astype(np.int32))
    print(f"done {time.time() - t0:.1f}s", flush=True)


if __name__ == "__main__":
    main()
