"""Reference evaluate() (training.py:325-339) on the train-loop fixture's
initial scene, for the GPU evaluate() used by `cli fit`.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_eval.py
"""
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(HERE))

from make_golden_train import build_inputs  # noqa: E402
from texsplat.training import evaluate  # noqa: E402


def main():
    lut, init, cams, targets = build_inputs()
    r = evaluate(init, cams, targets, lut)
    np.savez_compressed(HERE / "evaluate.npz", psnr=np.array(r["psnr"]), ssim=np.array(r["ssim"]))
    print(r)


if __name__ == "__main__":
    main()
