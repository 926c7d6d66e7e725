"""Randomised sweep of the interpolating coarse gather against the FP64 oracle: shapes, shifts of
every size and sign (including exact half-cell and whole-cell shifts), orders 1-3 and the keystone
variant.  Prints the worst case; exits 1 when any case exceeds 2e-5."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["LTCI_COARSE"] = "gather"
import oracle as O  # noqa: E402
from paper_2403_06788_b200 import mgift, scene  # noqa: E402
from paper_2403_06788_b200.model import RadarParams  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 200
rng = np.random.default_rng(2024)
worst = (0.0, None)
for it in range(n):
    K = int(2 ** rng.integers(6, 12))
    M = int(2 ** rng.integers(5, 9))
    p = RadarParams.create(3e9, 25e6, 20e6, 1000.0, M, K)
    x = scene.to_complex64_roundtrip(scene.add_noise(np.zeros((M, K), complex), 1.0, 1000 + it))
    v = int(rng.integers(0, 4) == 0)
    kind = int(rng.integers(0, 5))
    dR, T = p.delta_R(), p.T()
    if v:
        c = [float(rng.integers(-8, 9)), float(rng.uniform(-30, 30))]
    elif kind == 0:   # whole- and half-cell shifts at the last pulse
        c = [float(rng.integers(-40, 41)) * 0.5 * dR / T]
    elif kind == 1:   # zero
        c = [0.0]
    elif kind == 2:   # large
        c = [float(rng.uniform(-5e4, 5e4)), float(rng.uniform(-500, 500))]
    elif kind == 3:
        c = [float(rng.uniform(-300, 300)), float(rng.uniform(-20, 20)), float(rng.uniform(-1, 1))]
    else:
        c = [float(rng.uniform(-300, 300)), float(rng.uniform(-20, 20))]
    ref = O.port_mgift(x, p, c, v)
    err = float(np.abs(mgift(x, p, c, v) - ref).max() / np.abs(ref).max())
    if err > worst[0]:
        worst = (err, (K, M, v, c))
print("cases", n, "worst", worst)
sys.exit(1 if worst[0] > 2e-5 else 0)
