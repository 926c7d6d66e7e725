"""Engine hazards found in round-1 review, each pinned by a GPU test:

* the candidate-overflow re-run (``assemble`` grows the buffer and runs the
  cascade again) must use the echo of the run being assembled, even when the
  caller overwrote its own device buffer before ``result()`` (CPI streams
  double-buffer their inputs);
* back-to-back ``run_file`` calls reuse the two pinned staging blocks: a call
  must not refill a block whose DMA from an earlier call is still queued;
* one-shot ``ds_grft`` calls from many host threads (the reference's callers
  fan detector calls out over threads, proj/src/bench.cpp:94-110) leave a
  bounded number of idle engines behind.
"""
from __future__ import annotations

import ctypes as C
import threading

import numpy as np
import pytest

from paper_2403_06788_b200 import _lib, scene
from paper_2403_06788_b200.configs import config
from paper_2403_06788_b200.cube_io import CubeFile, write_cube_file
from paper_2403_06788_b200.detectors import Engine, detection_threshold, ds_grft
from paper_2403_06788_b200.model import DetectorOptions

from helpers import cube, load, radar, space

pytestmark = pytest.mark.gpu


def _dev_cube(torch, x):
    """complex64 column-major cube (k + K m) on the device as a float32 tensor."""
    a = np.ascontiguousarray(x.astype(np.complex64)).view(np.float32)
    return torch.from_numpy(a.copy()).cuda()


def test_overflow_rerun_uses_the_runs_cube(monkeypatch):
    import torch
    g = load("small_grft.npz")
    p, s = radar(g), space(g, radar(g))
    x = scene.to_complex64_roundtrip(cube(g))
    y = scene.to_complex64_roundtrip(scene.add_noise(np.zeros_like(x), 4.0, 99))  # a different CPI
    opt = DetectorOptions(retain_threshold=float(g["retain"]) * 0.25)  # many retained cells
    ref_eng = Engine(p, s, opt=opt)
    ref_eng.run_host(x)
    ref = ref_eng.result()
    ref_eng.close()
    assert ref.cand_index.size > 16
    monkeypatch.setenv("LTCI_CAND_CAP", "8")  # the first run overflows and assemble() re-runs
    e = Engine(p, s, opt=opt)
    d = _dev_cube(torch, x)
    e.run_device(d.data_ptr())
    torch.cuda.synchronize()
    d.copy_(_dev_cube(torch, y))  # the caller reuses its buffer for the next CPI
    torch.cuda.synchronize()
    m = e.result()
    e.close()
    assert np.array_equal(m.cand_index, ref.cand_index)
    assert np.array_equal(m.cand_value, ref.cand_value)
    assert np.array_equal(m.peak_index, ref.peak_index) and m.argmax == ref.argmax


def test_chained_run_file_calls_use_their_own_files(tmp_path):
    """Three run_file calls queued back to back (no result() in between); each
    run's per-row peaks, copied on the stream right behind it, equal the host
    path's for that file."""
    import torch
    w = config(4)
    p, s = w.params, w.space
    gamma = detection_threshold(p, w.sigma2, 1e-6)
    opt = DetectorOptions(retain_threshold=gamma)
    cubes = [scene.to_complex64_roundtrip(w.cube(cpi)) for cpi in range(3)]
    paths = []
    for i, x in enumerate(cubes):
        paths.append(tmp_path / f"cpi{i}.bin")
        write_cube_file(paths[-1], CubeFile.from_cube(x, p, w.sigma2))
    e = Engine(p, s, opt=opt)
    lib = _lib.load()
    ptr, n = e.peaks_device()
    st = torch.cuda.Stream()
    got = torch.empty((3, n, 4), dtype=torch.int32, device="cuda")
    torch.cuda.synchronize()
    for i, path in enumerate(paths):
        e.run_file(path, st.cuda_stream)
        # a one-map "merge" is a device copy of the slots on the same stream
        _lib.raise_for(lib.ltci_cuda_merge_peaks(C.c_void_p(ptr), 1, n, C.c_void_p(got[i].data_ptr()),
                                                 C.c_void_p(st.cuda_stream)), lib)
    st.synchronize()
    for i, x in enumerate(cubes):
        e.run_host(x)
        e.result()
        torch.cuda.synchronize()
        want = torch.empty((n, 4), dtype=torch.int32, device="cuda")
        _lib.raise_for(lib.ltci_cuda_merge_peaks(C.c_void_p(ptr), 1, n, C.c_void_p(want.data_ptr()), None), lib)
        torch.cuda.synchronize()
        assert torch.equal(got[i], want), f"run_file call {i} saw another call's cube"
    e.close()


def test_one_shot_pool_is_bounded_across_threads():
    g = load("small_grft.npz")
    p, s = radar(g), space(g, radar(g))
    x = scene.to_complex64_roundtrip(cube(g))
    opt = DetectorOptions(retain_threshold=float(g["retain"]))
    want = ds_grft(x, p, s, opt)
    out, errs = [None] * 12, []

    def work(i):
        try:
            out[i] = ds_grft(x, p, s, opt)
        except Exception as ex:  # pragma: no cover - reported below
            errs.append(ex)

    ts = [threading.Thread(target=work, args=(i,)) for i in range(len(out))]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errs, errs
    for m in out:
        assert m.argmax == want.argmax and np.array_equal(m.cand_index, want.cand_index)
        assert np.array_equal(m.peak_value, want.peak_value)
    lib = _lib.load()
    ne, nf = C.c_int64(), C.c_int64()
    _lib.raise_for(lib.ltci_cuda_pool_idle(0, C.byref(ne), C.byref(nf)), lib)
    assert 1 <= ne.value <= 2, ne.value
