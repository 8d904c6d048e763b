"""Environment precompute on the GPU (K15-K16, csrc/tsb_env.cu) against the
host restatement, which is bit-identical to the reference's numpy
(tests/test_host.py pins that). Tolerance: relative 1e-5 of each grid's
max (fp64 sums in another order, rounded to float32); LUT 1e-9 absolute."""
import numpy as np
import pytest

from paper_2506_13348_b200.environment import BrdfLut, EnvironmentLight

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("height,levels", [(16, 4), (64, 6)])
def test_env_prefilter_matches_host(height, levels):
    rng = np.random.default_rng(0)
    base = rng.uniform(0.0, 2.0, (height, 2 * height, 3))
    host = EnvironmentLight.from_base(base, levels)
    dev = EnvironmentLight.from_base(base, levels, device="cuda")
    assert len(dev.spec_mips) == len(host.spec_mips)
    for a, b in zip(dev.spec_mips + [dev.diffuse], host.spec_mips + [host.diffuse]):
        assert a.shape == b.shape and a.dtype == np.float32
        assert np.abs(a.astype(np.float64) - b).max() <= 1e-5 * max(np.abs(b).max(), 1e-12)


def test_brdf_lut_matches_host():
    host = BrdfLut.build(32, 512)
    dev = BrdfLut.build(32, 512, device="cuda")
    assert np.abs(dev.table - host.table).max() <= 1e-9
