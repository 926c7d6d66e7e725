"""Accuracy of the two coarse formulations against the FP64 oracle (oracle.port_mgift):
max |X_gpu - X_oracle| / max |X_oracle| over the whole range-pulse cube, for full-band white
noise (the worst case for the interpolation window) at the BASELINE shapes.  One JSON line per
(shape, coarse vector): K1 (transform) and K1g (gather) side by side."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as O  # noqa: E402
from paper_2403_06788_b200 import mgift, scene  # noqa: E402
from paper_2403_06788_b200.model import RadarParams  # noqa: E402

for M, K in ((256, 512), (512, 1024), (1024, 2048), (2048, 4096)):
    p = RadarParams.create(3e9, 20e6 if K != 2048 else 25e6, 20e6, 1000.0, M, K)
    x = scene.to_complex64_roundtrip(scene.add_noise(np.zeros((M, K), complex), 1.0, M + K))
    for c, v in (([87.0, 2.0], 0), ([-300.0, 10.0], 0), ([150.0, -5.0, 0.3], 0), ([4.0, 7.5], 1)):
        ref = O.port_mgift(x, p, c, v)
        row = {"M": M, "K": K, "ctilde": c, "variant": "kt" if v else "grft"}
        for mode in ("transform", "gather"):
            os.environ["LTCI_COARSE"] = mode
            got = mgift(x, p, c, v)
            row[mode] = float(np.abs(got - ref).max() / np.abs(ref).max())
            row[mode + "_rms"] = float(np.sqrt(np.mean(np.abs(got - ref) ** 2)) / np.sqrt(np.mean(np.abs(ref) ** 2)))
        print(json.dumps(row), flush=True)
