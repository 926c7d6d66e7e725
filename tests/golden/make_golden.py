"""Generate the golden vectors in tests/golden/ from the REFERENCE itself.

Run in the build container (needs oracle/_ref/libltci_ref.so, i.e. the
reference compiled read-only from /root/reference by oracle/Makefile):

    python tests/golden/make_golden.py

Every input is seeded and rounded to complex64 before the reference sees it
(the GPU computes from that rounding).  Outputs are
what the reference's own functions return:
  transforms.npz   mgift (RM and KtRm), gft (sub-ROI), keystone on small cubes
  small_grft.npz   ds_grft, small space built by the reference's build_dual_scale,
                   keep_dense=true (full complex map) + candidates
  small_kt.npz     ds_kt_mfp, same cube, build_ambiguity
  c0.npz           BASELINE config 0 (512x256, hand-built space): ds_grft with
                   retain = detection_threshold(sigma2=1/K, Pfa=1e-6) --
                   candidates, argmax, counters -- and the per-range-cell peak
                   map from ref_peak_map (reference mgift+gft in run_dual_scale's loop)
  p1_p3.npz        order-1 and order-3 ds_grft (dense) on a tiny instance
  fd.npz           fd_grft at orders 1, 2 and 3 on
                   build_single_scale spaces, keep_dense + candidates; the order-2
                   case with a sub-ROI
  td_kt.npz        td_grft on a range-pulse cube (orders 1 and 2, ROI subset, the
                   ZeroOutside and Wrap trajectory policies) and kt_mfp (three
                   folding numbers), keep_dense + candidates
  range_fft.npz    range_fft (the configs[3] front end K0) of seeded range-pulse
                   cubes: a noise cube, and range_ifft of a synthesized
                   DS-KT-MFP scene (K_valid < K guard band) with its round trip

    python tests/golden/make_golden.py [fd|td_kt|range]     (only that file)
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle as O  # noqa: E402
from paper_2403_06788_b200 import configs, scene  # noqa: E402
from paper_2403_06788_b200.model import DetectorOptions  # noqa: E402


def c64(x):
    return np.ascontiguousarray(x).astype(np.complex64).astype(np.complex128)


def space_arrays(prefix, s):
    out = {}
    out[prefix + "coarse"] = np.array([[g.start, g.step, g.count] for g in s.coarse])
    out[prefix + "fine"] = np.array([[g.start, g.step, g.count] for g in s.fine])
    out[prefix + "steps"] = np.array([s.steps.rm, s.steps.dfm, s.steps.alpha])
    out[prefix + "kappa"] = np.array(s.kappa)
    out[prefix + "roi"] = np.array([s.roi.first, s.roi.last])
    return out


def radar_arrays(prefix, p):
    return {prefix + "radar": np.array([p.fc, p.fs, p.Br, p.delta_f, p.PRF, p.M, p.K, p.K_valid])}


def map_arrays(prefix, m):
    return {prefix + "cand_index": m.cand_index, prefix + "cand_value": m.cand_value,
            prefix + "argmax": np.array(m.argmax, np.uint64), prefix + "argmax_value": np.array(m.argmax_value),
            prefix + "counters": np.array(m.counters, np.uint64),
            prefix + "axes": np.array([[a.role, a.order, a.size] for a in m.axes]),
            prefix + "doppler_first": np.array(m.doppler_first),
            **({prefix + "dense": m.dense} if m.dense_stored else {})}


def single_arrays(prefix, s):
    return {prefix + "c": np.array([[g.start, g.step, g.count] for g in s.c]),
            prefix + "steps": np.array([s.steps.rm, s.steps.dfm, s.steps.alpha]),
            prefix + "roi": np.array([s.roi.first, s.roi.last])}


def make_fd():
    p = O.ref_radar(8 * 100e6, 100e6, 50e6, 2000.0, 32, 64)
    tgt = [(0.4 + 0.1j, [21 * p.delta_R(), 13.3, 240.0]), (0.3, [40 * p.delta_R(), -22.0, -400.0])]
    cube = c64(O.ref_synthesize(p, tgt, 1.0 / p.K, 91))
    spaces = {"s2_": O.ref_single_scale(p, 2, [(-30.0, 30.0), (-1100.0, 1100.0)], [0.5, 0.5], 3, p.K - 5),
              "s1_": O.ref_single_scale(p, 1, [(-30.0, 30.0)], [1.0], 0, p.K - 1),
              "s3_": O.ref_single_scale(p, 3, [(-20.0, 20.0), (-450.0, 450.0), (-30000.0, 30000.0)],
                                        [0.4, 0.3, 0.3], 0, p.K - 1)}
    # retention at the 80th percentile of the order-2 dense map
    probe = O.ref_fd(cube, p, spaces["s2_"], DetectorOptions(keep_dense=True))
    retain = float(np.quantile(np.abs(probe.dense), 0.8))
    opt = DetectorOptions(retain_threshold=retain, keep_dense=True)
    out = {"cube": cube.astype(np.complex64), "retain": np.array(retain), **radar_arrays("", p)}
    for key, sp in spaces.items():
        out.update(single_arrays(key, sp), **map_arrays("m" + key[1:], O.ref_fd(cube, p, sp, opt)))
    np.savez_compressed(os.path.join(HERE, "fd.npz"), **out)


def make_td_kt():
    """td_grft (range-pulse cube, the three trajectory policies) and kt_mfp from the reference."""
    p = O.ref_radar(8 * 100e6, 100e6, 50e6, 2000.0, 32, 64)
    tgt = [(0.4 + 0.1j, [21 * p.delta_R(), 13.3, 240.0]), (0.3, [40 * p.delta_R(), -22.0, -400.0])]
    freq = c64(O.ref_synthesize(p, tgt, 1.0 / p.K, 92))
    rng_cube = c64(O.ref_range_ifft(freq, p))
    out = {"freq": freq.astype(np.complex64), "range": rng_cube.astype(np.complex64), **radar_arrays("", p)}
    # td_grft: order 2 with an ROI subset (trajectories leave the cube at both ends) and order 1
    s2 = O.ref_single_scale(p, 2, [(-30.0, 30.0), (-1100.0, 1100.0)], [0.5, 0.5], 2, p.K - 3)
    s1 = O.ref_single_scale(p, 1, [(-30.0, 30.0)], [1.0], 0, p.K - 1)
    probe = O.ref_td(rng_cube, p, s2, DetectorOptions(keep_dense=True))
    retain = float(np.quantile(np.abs(probe.dense), 0.8))
    out["td_retain"] = np.array(retain)
    out.update(single_arrays("s2_", s2), **single_arrays("s1_", s1))
    for pol, name in ((0, "zero"), (1, "wrap")):
        opt = DetectorOptions(retain_threshold=retain, keep_dense=True, trajectory=pol)
        out.update(map_arrays(f"td2_{name}_", O.ref_td(rng_cube, p, s2, opt)))
    out.update(map_arrays("td1_zero_", O.ref_td(rng_cube, p, s1, DetectorOptions(retain_threshold=retain,
                                                                                   keep_dense=True))))
    # kt_mfp: three folding numbers, acceleration grid of the order-2 space
    amb = O.ref_ambiguity(p, -1.4 * p.Va(), 1.4 * p.Va())
    sk = O.ref_single_scale(p, 2, [(-30.0, 30.0), (-1100.0, 1100.0)], [0.5, 0.5], 4, p.K - 9)
    probe = O.ref_kt(freq, p, amb, sk, DetectorOptions(keep_dense=True))
    kret = float(np.quantile(np.abs(probe.dense), 0.9))
    out["kt_retain"] = np.array(kret)
    out["amb"] = np.array([amb.q_min, amb.q_max])
    out.update(single_arrays("sk_", sk),
               **map_arrays("kt_", O.ref_kt(freq, p, amb, sk, DetectorOptions(retain_threshold=kret, keep_dense=True))))
    np.savez_compressed(os.path.join(HERE, "td_kt.npz"), **out)


def make_range():
    # noise cube straight in the range domain, and a C3-like scene (fs > Br) taken
    # to the range domain by the reference's range_ifft
    p = O.ref_radar(3e9, 25e6, 20e6, 1000.0, 16, 128)
    noise = c64(scene.add_noise(np.zeros((p.M, p.K), complex), 1.0, 303))
    tgt = [(0.5 + 0.2j, [40 * p.delta_R(), 31.0, 2.5]), (0.3 - 0.1j, [90.4 * p.delta_R(), -55.0, -4.0])]
    freq = c64(O.ref_synthesize(p, tgt, 1.0 / p.K, 404))
    rng_scene = c64(O.ref_range_ifft(freq, p))
    np.savez_compressed(os.path.join(HERE, "range_fft.npz"), noise=noise.astype(np.complex64),
                        noise_fft=O.ref_range_fft(noise, p), scene_range=rng_scene.astype(np.complex64),
                        scene_fft=O.ref_range_fft(rng_scene, p), **radar_arrays("", p))


def main():
    assert O.have_ref(), "build the reference first: make -C oracle"
    if sys.argv[1:] == ["fd"]:
        make_fd()
        print("fd.npz written to", HERE)
        return
    if sys.argv[1:] == ["td_kt"]:
        make_td_kt()
        print("td_kt.npz written to", HERE)
        return
    if sys.argv[1:] == ["range"]:
        make_range()
        print("range_fft.npz written to", HERE)
        return
    # ---- transforms
    p = O.ref_radar(4 * 100e6, 100e6, 50e6, 2000.0, 32, 64)
    cube = c64(scene.add_noise(np.zeros((p.M, p.K), complex), 1.0, 101))
    mg = O.ref_mgift(cube, p, [11.7, -4.1])
    mgk = O.ref_mgift(cube, p, [2.0, 3.3], 1)
    rows = c64(O.ref_mgift(cube, p, [0.0, 0.0]))
    gf = O.ref_gft(rows, p, [1.2], 1, p.K - 2)
    ks = O.ref_keystone(cube, p, 8)
    ks4 = O.ref_keystone(cube, p, 4)
    np.savez_compressed(os.path.join(HERE, "transforms.npz"), cube=cube.astype(np.complex64), rows=rows,
                        mgift=mg, mgift_kt=mgk, gft=gf, keystone=ks, keystone4=ks4, **radar_arrays("", p))

    # ---- small ds_grft / ds_kt_mfp with dense maps
    p = O.ref_radar(8 * 100e6, 100e6, 50e6, 2000.0, 32, 64)
    s = O.ref_dual_scale(p, 2, [(-40.0, 40.0), (-15.0, 15.0)], [0.5, 0.5], 0, p.K - 1)
    tgt = [(0.35 + 0.1j, [30 * p.delta_R(), float(s.coarse[0].value(1)) + 1.3, float(s.coarse[1].value(0)) + 0.4])]
    cube = c64(O.ref_synthesize(p, tgt, 1.0 / p.K, 77))
    opt = DetectorOptions(retain_threshold=3.0, keep_dense=True)
    m = O.ref_ds(cube, p, s, opt)
    pi, pv = O.ref_peak_map(cube, p, s)
    np.savez_compressed(os.path.join(HERE, "small_grft.npz"), cube=cube.astype(np.complex64), peak_index=pi,
                        peak_value=pv, retain=np.array(3.0), **radar_arrays("", p), **space_arrays("", s),
                        **map_arrays("", m))
    amb = O.ref_ambiguity(p, -1.6 * p.Va(), 1.6 * p.Va())
    m = O.ref_ds(cube, p, s, opt, 1, amb)
    pi, pv = O.ref_peak_map(cube, p, s, 1, amb)
    np.savez_compressed(os.path.join(HERE, "small_kt.npz"), cube=cube.astype(np.complex64), peak_index=pi,
                        peak_value=pv, retain=np.array(3.0), amb=np.array([amb.q_min, amb.q_max]),
                        **radar_arrays("", p), **space_arrays("", s), **map_arrays("", m))

    # ---- order 1 and order 3
    p = O.ref_radar(4 * 100e6, 100e6, 50e6, 2000.0, 16, 32)
    s1 = O.ref_dual_scale(p, 1, [(-40.0, 40.0)], [1.0], 0, p.K - 1)
    s3 = O.ref_dual_scale(p, 3, [(-40.0, 40.0), (-15.0, 15.0), (-30.0, 30.0)], [0.4, 0.3, 0.3], 2, p.K - 3)
    cube = c64(O.ref_synthesize(p, [(0.5, [9 * p.delta_R(), 12.0, 2.0, 1.0])], 1.0 / p.K, 5))
    opt = DetectorOptions(retain_threshold=1.0, keep_dense=True)
    m1 = O.ref_ds(cube, p, s1, opt)
    m3 = O.ref_ds(cube, p, s3, opt)
    np.savez_compressed(os.path.join(HERE, "p1_p3.npz"), cube=cube.astype(np.complex64), **radar_arrays("", p),
                        **space_arrays("s1_", s1), **space_arrays("s3_", s3), **map_arrays("m1_", m1),
                        **map_arrays("m3_", m3))

    # ---- BASELINE config 0
    w = configs.config(0)
    cube = c64(w.cube())
    gamma = O.ref_threshold(w.params, w.sigma2, 1e-6)
    m = O.ref_ds(cube, w.params, w.space, DetectorOptions(retain_threshold=gamma, threads=0))
    pi, pv = O.ref_peak_map(cube, w.params, w.space)
    np.savez_compressed(os.path.join(HERE, "c0.npz"), cube=cube.astype(np.complex64), gamma=np.array(gamma),
                        peak_index=pi, peak_value=pv, **map_arrays("", m))
    make_fd()
    make_td_kt()
    make_range()
    print("golden vectors written to", HERE)


if __name__ == "__main__":
    main()
