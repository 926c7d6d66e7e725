"""Cube file container: the library's C++ reader/writer
(csrc/cube_io.cpp) against the reference's own read_cube_file/write_cube_file
(oracle/_ref), after proj/tests/test_cli_io.cpp:21-70; and the GPU wire path
(Engine.run_file) against the host-buffer path on the same cube."""
from __future__ import annotations

import os

import numpy as np
import pytest

import oracle as O
from paper_2403_06788_b200 import _lib
from paper_2403_06788_b200.cube_io import (CubeFile, RANGE_PULSE, cube_file_info, read_cube_file,
                                           write_cube_file)
from paper_2403_06788_b200.model import RadarParams

from helpers import cube, load, radar, space

needs_ref = pytest.mark.skipif(not O.have_ref(), reason="reference not built (oracle/_ref)")


def _small(M=32, K=16):
    # fixtures::small analogue (proj/tests/fixtures.hpp): any valid radar works
    return RadarParams.create(1.0e10, 4.0e6, 4.0e6 * 0.8, 1000.0, M, K)


def _random_cube(p, seed):
    rng = np.random.default_rng(seed)
    return (rng.standard_normal((p.M, p.K)) + 1j * rng.standard_normal((p.M, p.K)))


def test_round_trip_bit_exact_and_documented_size(tmp_path):
    p = _small()
    x = _random_cube(p, 3)
    path = tmp_path / "cube.bin"
    write_cube_file(path, CubeFile.from_cube(x, p, 0.25))
    assert os.path.getsize(path) == 61 + p.K * p.M * 16
    assert not os.path.exists(str(path) + ".tmp")
    back = read_cube_file(path)
    assert back.domain == 0 and back.sigma2 == 0.25
    assert (back.params.K, back.params.M, back.params.K_valid, back.params.fc) == (p.K, p.M, p.K_valid, p.fc)
    assert np.array_equal(back.data, x)
    d, q, s2 = cube_file_info(path)
    assert d == 0 and q.K == p.K and s2 == 0.25


@needs_ref
def test_files_are_byte_identical_to_the_reference_and_cross_readable(tmp_path):
    p = _small(64, 32)
    x = _random_cube(p, 5)
    ours, theirs = tmp_path / "ours.bin", tmp_path / "ref.bin"
    write_cube_file(ours, CubeFile.from_cube(x, p, 1.5))
    O.ref_write_cube_file(theirs, p, x, 1.5)
    assert ours.read_bytes() == theirs.read_bytes()
    d, q, s2, y = O.ref_read_cube_file(ours)
    assert (d, s2, q.K, q.M, q.K_valid, q.fc, q.fs, q.Br, q.PRF) == (0, 1.5, p.K, p.M, p.K_valid, p.fc, p.fs, p.Br,
                                                                    p.PRF)
    assert np.array_equal(y, x)
    back = read_cube_file(theirs)
    assert np.array_equal(back.data, x) and back.params.delta_f == q.delta_f


def _corruptions(tmp_path, p):
    base = tmp_path / "good.bin"
    write_cube_file(base, CubeFile.from_cube(np.zeros((p.M, p.K)), p, 0.0))
    raw = base.read_bytes()
    cases = {}

    def put(name, data):
        f = tmp_path / name
        f.write_bytes(data)
        cases[name] = f

    put("truncated_payload.bin", raw[:-8])
    put("trailing.bin", raw + b"\0")
    put("short_header.bin", raw[:40])
    put("bad_magic.bin", b"X" + raw[1:])
    put("bad_version.bin", raw[:4] + (2).to_bytes(4, "little") + raw[8:])
    put("bad_domain.bin", raw[:8] + b"\x05" + raw[9:])
    put("bad_params.bin", raw[:9] + (12).to_bytes(4, "little") + raw[13:])  # K = 12: not a power of two
    cases["missing.bin"] = tmp_path / "missing.bin"
    return cases


def test_reader_rejects_corrupted_containers(tmp_path):
    p = _small(16, 4)
    for name, path in _corruptions(tmp_path, p).items():
        with pytest.raises(_lib.IoError):
            read_cube_file(path)


@needs_ref
def test_reader_errors_match_the_reference(tmp_path):
    p = _small(16, 4)
    for name, path in _corruptions(tmp_path, p).items():
        with pytest.raises(_lib.IoError) as ours:
            read_cube_file(path)
        with pytest.raises(O.OracleError) as theirs:
            O.ref_read_cube_file(path)
        assert theirs.value.code == 6, name  # LTCI_IO_ERROR <- ltci::IoError
        assert str(ours.value) == str(theirs.value).split("] ", 1)[1], name


def test_writer_failure_leaves_nothing(tmp_path):
    p = _small(16, 4)
    target = tmp_path / "no_such_dir" / "cube.bin"
    with pytest.raises(_lib.IoError, match="for writing"):
        write_cube_file(target, CubeFile.from_cube(np.zeros((p.M, p.K)), p))
    assert not target.parent.exists()


def test_range_domain_flag_carries_through(tmp_path):
    p = _small(16, 4)
    x = _random_cube(p, 4)
    path = tmp_path / "rp.bin"
    write_cube_file(path, CubeFile.from_cube(x, p, 1.0, RANGE_PULSE))
    back = read_cube_file(path)
    assert back.domain == 1
    with pytest.raises(_lib.ConditionViolated):
        back.to_freq_cube()
    assert np.array_equal(back.to_range_cube(), x)


@pytest.mark.gpu
@pytest.mark.parametrize("variant", [0, 1])
def test_engine_run_file_equals_run_host(tmp_path, variant):
    """File -> pinned staging -> device gives the identical map to the host path."""
    from paper_2403_06788_b200 import AmbiguitySpace, DetectorOptions
    from paper_2403_06788_b200.detectors import Engine

    g = load("small_kt.npz" if variant else "small_grft.npz")
    p = radar(g)
    s = space(g, p)
    amb = AmbiguitySpace(int(g["amb"][0]), int(g["amb"][1])) if variant else None
    x = cube(g)
    path = tmp_path / "cpi.bin"
    write_cube_file(path, CubeFile.from_cube(x, p, 1.0))
    opt = DetectorOptions(retain_threshold=float(g["retain"]), keep_dense=True)
    eng = Engine(p, s, variant, amb, opt)
    eng.run_host(x)
    a = eng.result()
    eng.run_file(path)
    b = eng.result()
    assert np.array_equal(a.dense, b.dense)
    assert np.array_equal(a.cand_index, b.cand_index) and np.array_equal(a.cand_value, b.cand_value)
    assert a.argmax == b.argmax

    # the reference's errors on the wire path
    rp = tmp_path / "rp.bin"
    write_cube_file(rp, CubeFile.from_cube(x, p, 1.0, RANGE_PULSE))
    with pytest.raises(_lib.ConditionViolated):
        eng.run_file(rp)
    other = RadarParams.create(p.fc * 2, p.fs, p.Br, p.PRF, p.M, p.K, p.K_valid)
    op = tmp_path / "other.bin"
    write_cube_file(op, CubeFile.from_cube(x, other, 1.0))
    with pytest.raises(ValueError, match="different radar"):
        eng.run_file(op)
    with pytest.raises(_lib.IoError):
        eng.run_file(tmp_path / "missing.bin")
    eng.close()


@pytest.mark.gpu
def test_engine_run_file_multi_block(tmp_path):
    """A cube larger than one 32 MiB staging block (C1 size, 2 blocks)."""
    from paper_2403_06788_b200 import DetectorOptions
    from paper_2403_06788_b200.configs import config
    from paper_2403_06788_b200.detectors import Engine

    w = config(1)
    x = w.cube(noise=True)
    path = tmp_path / "c1.bin"
    write_cube_file(path, CubeFile.from_cube(x, w.params, 1.0))
    gamma = float(np.sqrt(-w.params.M * w.params.K * w.sigma2 * np.log(1e-6)))
    eng = Engine(w.params, w.space, 0, None, DetectorOptions(retain_threshold=gamma))
    eng.run_host(x)
    a = eng.result()
    eng.run_file(path)
    b = eng.result()
    assert np.array_equal(a.cand_index, b.cand_index) and np.array_equal(a.cand_value, b.cand_value)
    assert np.array_equal(a.peak_index, b.peak_index)
    eng.close()
