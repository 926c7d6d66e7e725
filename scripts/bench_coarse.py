"""Coarse-stage (K1) A/B timing: device time of the coarse and fine stages of
one engine pass per BASELINE config, with whatever library LTCI_LIB_PATH
selects (A/B builds from scripts/build_ab.sh) and LTCI_COARSE_GENERIC.
Prints one JSON line per config: coarse ms and the HBM fraction it implies."""
import argparse, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2403_06788_b200 import configs, scene
from paper_2403_06788_b200.detectors import Engine, detection_threshold
from paper_2403_06788_b200.model import DetectorOptions

ap = argparse.ArgumentParser()
ap.add_argument("--configs", default="1,3")
ap.add_argument("--runs", type=int, default=5)
ap.add_argument("--tag", default=os.environ.get("LTCI_LIB_PATH", "default"))
a = ap.parse_args()
hbm = 6551.7
for ci in map(int, a.configs.split(",")):
    w = configs.config(ci)
    p, s = w.params, w.space
    e = Engine(p, s, w.variant, w.amb, DetectorOptions(retain_threshold=detection_threshold(p, w.sigma2, 1e-6)))
    x = torch.from_numpy(scene.to_complex64_roundtrip(w.cube()).astype(np.complex64)).cuda()
    e.run_device(x.data_ptr())
    torch.cuda.synchronize()
    e.set_timing(True)
    cms, fms = [], []
    for _ in range(a.runs):
        e.run_device(x.data_ptr())
        st = e.stats()
        cms.append(st["coarse_ms"])
        fms.append(st["fine_ms"])
    coarse = int(np.prod([g.count for g in s.coarse])) if w.variant == 0 else w.amb.count() * s.coarse[1].count
    byts = 8.0 * coarse * s.roi.count() * p.M + 8.0 * p.K * p.M
    cm = float(np.median(cms))
    print(json.dumps({"config": ci, "tag": a.tag, "generic": os.environ.get("LTCI_COARSE_GENERIC", "0"),
                      "coarse_ms": cm, "fine_ms": float(np.median(fms)), "coarse_gbs": byts / cm / 1e6,
                      "coarse_frac": byts / cm / 1e6 / hbm}), flush=True)
    e.close()
