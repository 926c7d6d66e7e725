"""Where the end-to-end time of one engine call goes (bench.py's e2e path):
run_host (H2D + f64->c64 + kernels enqueued), device completion, result()."""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2403_06788_b200 import configs, scene
from paper_2403_06788_b200.detectors import Engine, detection_threshold
from paper_2403_06788_b200.model import DetectorOptions

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 0
w = configs.config(cfg)
p, s = w.params, w.space
gamma = detection_threshold(p, w.sigma2, min(1e-6, 1e5 / float(w.hypotheses())))
eng = Engine(p, s, w.variant, w.amb, DetectorOptions(retain_threshold=gamma))
cube = scene.to_complex64_roundtrip(w.cube(cpi=0))
host = torch.from_numpy(cube.view(np.float64).reshape(-1)).pin_memory()
st = torch.cuda.current_stream()
sp = st.cuda_stream
rows = []
for i in range(30):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    eng.run_host_ptr(host.data_ptr(), sp)
    t1 = time.perf_counter()
    st.synchronize()
    t2 = time.perf_counter()
    m = eng.result(sp)
    t3 = time.perf_counter()
    if i >= 5:
        rows.append(((t1 - t0) * 1e3, (t2 - t1) * 1e3, (t3 - t2) * 1e3, len(m.cand_index)))
a = np.array(rows)
print(f"config {cfg}: enqueue {np.median(a[:,0]):.3f} ms, device wait {np.median(a[:,1]):.3f} ms, "
      f"result {np.median(a[:,2]):.3f} ms, total {np.median(a[:,:3].sum(1)):.3f} ms, candidates {int(a[0,3])}")
