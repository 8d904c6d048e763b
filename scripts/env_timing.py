"""GPU vs host environment precompute time (cfg5 env: 128x256 base, 6 levels;
BRDF LUT 64x64x2048)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2506_13348_b200.environment import BrdfLut, EnvironmentLight  # noqa: E402

base = np.random.default_rng(0).uniform(0.0, 2.0, (128, 256, 3))
EnvironmentLight.from_base(base[:16, :32], 3, device="cuda")
BrdfLut.build(8, 64, device="cuda")
for name, fn in (("env gpu", lambda: EnvironmentLight.from_base(base, 6, device="cuda")),
                 ("env host", lambda: EnvironmentLight.from_base(base, 6)),
                 ("lut gpu", lambda: BrdfLut.build(device="cuda")),
                 ("lut host", lambda: BrdfLut.build())):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    fn()
    torch.cuda.synchronize()
    print(f"{name}: {1e3 * (time.perf_counter() - t0):.1f} ms")
