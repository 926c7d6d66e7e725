"""CPU: the multi-rank path (range-cell shards + gathered peak map) with the
gloo backend at world size 2 (and 3), checked against the single-rank map of
the oracle on the same seeded cube."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import oracle as O
from paper_2403_06788_b200 import parallel
from paper_2403_06788_b200.configs import baseline_space, doppler_window
from paper_2403_06788_b200.model import DetectorOptions, RadarParams
from paper_2403_06788_b200 import scene


def _small():
    p = RadarParams.create(3e9, 20e6, 20e6, 1000.0, 64, 128)
    s = baseline_space(p, [(-150.0, 150.0), (-20.0, 20.0)])
    x = scene.to_complex64_roundtrip(
        scene.add_noise(scene.synthesize_cube(p, [(0.2, [40 * p.delta_R(), 61.0, 3.0])]), 1.0 / p.K, 7))
    full = O.port_ds(x, p, s, DetectorOptions(retain_threshold=2.0))
    return p, s, full


def test_shard_rows_cover_exactly():
    for R in (1, 7, 128, 2048):
        for world in (1, 2, 3, 8):
            sl = [parallel.shard_rows(R, world, r) for r in range(world)]
            assert sl[0][0] == 0 and sl[-1][1] == R
            assert all(a[1] == b[0] for a, b in zip(sl[:-1], sl[1:]))
            assert max(h - l for l, h in sl) - min(h - l for l, h in sl) <= 1


def test_host_merge_reproduces_full_map():
    p, s, full = _small()
    D = doppler_window(p, s)[1]
    for world in (2, 3, 5):
        parts = parallel.split_map_by_rows(full, s.roi.count(), D, world)
        m = parallel.merge_rank_maps(parts, full.counters)
        assert np.array_equal(m.peak_index, full.peak_index)
        assert np.array_equal(m.peak_value, full.peak_value)
        assert np.array_equal(m.cand_index, full.cand_index)
        assert np.array_equal(m.cand_value, full.cand_value)
        assert m.argmax == full.argmax and m.argmax_value == full.argmax_value


def _small_dense():
    p = RadarParams.create(3e9, 20e6, 20e6, 1000.0, 64, 128)
    s = baseline_space(p, [(-150.0, 150.0), (-20.0, 20.0)])
    x = scene.to_complex64_roundtrip(
        scene.add_noise(scene.synthesize_cube(p, [(0.2, [40 * p.delta_R(), 61.0, 3.0])]), 1.0 / p.K, 7))
    full = O.port_ds(x, p, s, DetectorOptions(retain_threshold=2.0, keep_dense=True))
    C = int(np.prod([g.count for g in s.coarse]))
    return p, s, full, C


def test_shard_coarse_cover_exactly():
    for C in (8, 83, 332, 3960):
        for world in (1, 2, 3, 8):
            sl = [parallel.shard_coarse(C, world, r) for r in range(world)]
            assert sl[0][0] == 0 and sl[-1][1] == C
            assert all(a[1] == b[0] for a, b in zip(sl[:-1], sl[1:]))
    with pytest.raises(ValueError):
        parallel.shard_coarse(3, 4, 0)


def test_host_coarse_merge_reproduces_full_map():
    """Coarse-cell partition: per-row max across ranks + concatenated candidates
    reproduce the single-rank map (the oracle's, FP64)."""
    p, s, full, C = _small_dense()
    assert np.array_equal(full.peak_index, parallel.split_map_by_coarse(full, C, 1)[0].peak_index)
    for world in (2, 3, 4):  # C = 4 coarse cells here
        parts = parallel.split_map_by_coarse(full, C, world)
        m = parallel.merge_coarse_maps(parts, full.counters)
        assert np.array_equal(m.peak_index, full.peak_index)
        assert np.array_equal(m.peak_value, full.peak_value)
        assert np.array_equal(m.cand_index, full.cand_index)
        assert np.array_equal(m.cand_value, full.cand_value)
        assert m.argmax == full.argmax and m.argmax_value == full.argmax_value


def _free_port():
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        p, s, full = _small()
        D = doppler_window(p, s)[1]
        local = parallel.split_map_by_rows(full, s.roi.count(), D, world)[rank]
        merged = parallel.gather_map(local)
        if rank == 0:
            ok = (np.array_equal(merged.peak_index, full.peak_index)
                  and np.array_equal(merged.peak_value, full.peak_value)
                  and np.array_equal(merged.cand_index, full.cand_index)
                  and np.array_equal(merged.cand_value, full.cand_value)
                  and merged.argmax == full.argmax)
            q.put(ok)
    finally:
        dist.destroy_process_group()


def _worker_coarse(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        p, s, full, C = _small_dense()
        local = parallel.split_map_by_coarse(full, C, world)[rank]
        merged = parallel.gather_coarse_map(local)
        if rank == 0:
            ok = (np.array_equal(merged.peak_index, full.peak_index)
                  and np.array_equal(merged.peak_value, full.peak_value)
                  and np.array_equal(merged.cand_index, full.cand_index)
                  and np.array_equal(merged.cand_value, full.cand_value)
                  and merged.argmax == full.argmax)
            q.put(ok)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_coarse_gather_matches_single_rank(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_coarse, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    for pr in procs:
        pr.join(timeout=180)
        assert pr.exitcode == 0
    assert q.get(timeout=10) is True


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_gather_matches_single_rank(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    for pr in procs:
        pr.join(timeout=180)
        assert pr.exitcode == 0
    assert q.get(timeout=10) is True


# ---- bench.py's own collectives (parallel.RankComm / PeakGather), both branches

def _worker_bench_comm(rank, world, port, staged, shard, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        p, s, full, C = _small_dense()
        R = s.roi.count()
        comm = parallel.RankComm(world, host_staged=staged)
        # max-over-ranks timing, as bench.py reduces its event times
        t = torch.tensor([10.0 + rank], dtype=torch.float64)
        comm.all_reduce_max(t)
        ok = float(t.item()) == 10.0 + world - 1

        def merge(gathered, merged):
            merged.copy_(torch.from_numpy(parallel.merge_peak_records(gathered.numpy())))

        g = parallel.PeakGather(comm, shard, R, torch.zeros(1), merge=merge)
        if shard == "coarse":
            local = parallel.split_map_by_coarse(full, C, world)[rank]
        else:
            D = doppler_window(p, s)[1]
            local = parallel.split_map_by_rows(full, R, D, world)[rank]
        g(torch.from_numpy(parallel.encode_peak_records(local.peak_index, local.peak_value)))
        got = g.full_map().numpy().view(np.uint32)
        want = parallel.encode_peak_records(full.peak_index, full.peak_value).view(np.uint32)
        ok = ok and np.array_equal(got, want)
        q.put((rank, bool(ok)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("staged", [False, True])
@pytest.mark.parametrize("shard", ["coarse", "rows"])
def test_gloo_bench_collectives(staged, shard):
    """bench.py's N>1 helpers on both transports (direct and host-staged):
    max-over-ranks reduction and the peak exchange reproduce the single-rank map."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_bench_comm, args=(r, world, port, staged, shard, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    for pr in procs:
        pr.join(timeout=180)
        assert pr.exitcode == 0
    res = sorted(q.get(timeout=10) for _ in range(world))
    assert res == [(r, True) for r in range(world)]


def test_merge_peak_records_tie_break():
    """Host mirror of merge_peaks_kernel: magnitude first, lowest index on ties,
    empty slots lose."""
    E = np.uint64(0xFFFFFFFFFFFFFFFF)
    a = parallel.encode_peak_records(np.array([5, 9, E, 3], np.uint64), np.array([1 + 0j, 2j, 0, 3], np.complex128))
    b = parallel.encode_peak_records(np.array([4, 8, 7, E], np.uint64), np.array([1j, 2 + 0j, 1e-3, 0], np.complex128))
    m = parallel.merge_peak_records(np.stack([a, b])).view(np.uint32)
    idx = m[:, 2].astype(np.uint64) | (m[:, 3].astype(np.uint64) << np.uint64(32))
    assert idx.tolist() == [4, 8, 7, 3]
