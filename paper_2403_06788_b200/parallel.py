"""Multi-GPU sharding: range cells or coarse cells.

Every (coarse cell, ROI row) output of the cascade is independent, so ranks
own contiguous slices of ROI rows (``shard_rows``): each replicates the echo,
runs the coarse stage storing only its rows and the fine stage on them, and
reduces into its own per-cell peak records.  The only exchange is gathering:

* per-cell peak map: fixed-size 16-byte records {f32 re, f32 im, u64 flat
  index} per row -> ``all_gather`` (rows are disjoint, no arithmetic);
* candidates: counts, then a padded ``all_gather`` of records, merged and
  re-sorted by flat index (r is not the slowest axis of the flat index);
* global argmax: max over the gathered peaks with the reference's total order
  (magnitude desc, flat index asc; proj/src/detectors.cpp:34-50).

The collectives run through ``torch.distributed`` (NCCL between GPUs; gloo in
the CPU tests).  ``merge_rank_maps`` is the deterministic host-side merge used
by both; results are bit-identical for any rank count.

Coarse-cell sharding (``shard_coarse``, SURVEY.md §8(e) "Alternative") is the
partition that scales: each rank searches a contiguous slice of coarse cells
over every ROI row, so no work is replicated (range sharding repeats the
K-point coarse transforms on every rank: 2.9 ms against 28 ms of fine work per
rank at C1 on 8 GPUs, a 4.8x ceiling).  The exchange becomes a per-row max:
every rank holds a peak for every row, combined with the kernels' own
magnitude and lowest-index tie-break (``ltci_cuda_merge_peaks`` on the device;
``merge_coarse_maps`` on the host), and candidates concatenate.
"""
from __future__ import annotations

from typing import List, Optional, Sequence, Tuple

import numpy as np

from .model import DetectionMap


def shard_rows(R: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous [lo, hi) slice of R ROI rows for ``rank`` (sizes differ by <= 1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("shard_rows: bad world/rank")
    return rank * R // world, (rank + 1) * R // world


def shard_coarse(C: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous [lo, hi) slice of C coarse cells for ``rank`` (sizes differ by <= 1)."""
    if world < 1 or not 0 <= rank < world or C < world:
        raise ValueError("shard_coarse: need 1 <= world <= coarse cells and a valid rank")
    return rank * C // world, (rank + 1) * C // world


def _mag2_f32(v: np.ndarray) -> np.ndarray:
    # magnitude order used everywhere on the device: fmaf(re, re, im*im) in fp32
    re = v.real.astype(np.float32)
    im = v.imag.astype(np.float32)
    return (re * re + im * im).astype(np.float32)


def argmax_total_order(index: np.ndarray, value: np.ndarray) -> int:
    """Position of the strongest cell, ties to the lowest flat index."""
    if index.size == 0:
        return -1
    m = np.abs(value)
    best = np.max(m)
    cand = np.nonzero(m == best)[0]
    return int(cand[np.argmin(index[cand])])


def merge_rank_maps(maps: Sequence[DetectionMap], full_counters: Optional[tuple] = None) -> DetectionMap:
    """Merge per-rank maps (rank order = row order) into the single-GPU map."""
    if not maps:
        raise ValueError("merge_rank_maps: no maps")
    base = maps[0]
    out = DetectionMap(kind=base.kind, params=base.params, axes=list(base.axes),
                       counters=full_counters if full_counters is not None else base.counters,
                       retain_threshold=base.retain_threshold, dual=base.dual, amb=base.amb,
                       doppler_first=base.doppler_first)
    out.peak_index = np.concatenate([m.peak_index for m in maps])
    out.peak_value = np.concatenate([m.peak_value for m in maps])
    ci = np.concatenate([m.cand_index for m in maps]) if maps else np.zeros(0, np.uint64)
    cv = np.concatenate([m.cand_value for m in maps]) if maps else np.zeros(0, np.complex128)
    order = np.argsort(ci, kind="stable")
    out.cand_index, out.cand_value = ci[order], cv[order]
    k = argmax_total_order(out.peak_index, out.peak_value)
    if k >= 0:
        out.argmax = int(out.peak_index[k])
        out.argmax_value = complex(out.peak_value[k])
    return out


def merge_coarse_maps(maps: Sequence[DetectionMap], full_counters: Optional[tuple] = None) -> DetectionMap:
    """Merge per-rank maps of a coarse-cell partition (every map covers every
    row): per-row best (magnitude desc, flat index asc), candidates concatenated
    and sorted.  Host-side: magnitudes of the recentred FP64 values; the bench
    path merges the raw FP32 slots on the device (``ltci_cuda_merge_peaks``)."""
    if not maps:
        raise ValueError("merge_coarse_maps: no maps")
    base = maps[0]
    R = base.peak_index.size
    if any(m.peak_index.size != R for m in maps):
        raise ValueError("merge_coarse_maps: every map must cover the same rows")
    out = DetectionMap(kind=base.kind, params=base.params, axes=list(base.axes),
                       counters=full_counters if full_counters is not None else base.counters,
                       retain_threshold=base.retain_threshold, dual=base.dual, amb=base.amb,
                       doppler_first=base.doppler_first)
    idx = np.stack([m.peak_index for m in maps])          # (ranks, R)
    val = np.stack([m.peak_value for m in maps])
    mag = np.where(idx == np.uint64(0xFFFFFFFFFFFFFFFF), -1.0, np.abs(val))
    best = np.zeros(R, np.int64)
    for k in range(1, len(maps)):
        better = (mag[k] > mag[best, np.arange(R)]) | ((mag[k] == mag[best, np.arange(R)]) &
                                                        (idx[k] < idx[best, np.arange(R)]))
        best = np.where(better, k, best)
    out.peak_index = idx[best, np.arange(R)].copy()
    out.peak_value = val[best, np.arange(R)].copy()
    ci = np.concatenate([m.cand_index for m in maps])
    cv = np.concatenate([m.cand_value for m in maps])
    order = np.argsort(ci, kind="stable")
    out.cand_index, out.cand_value = ci[order], cv[order]
    k = argmax_total_order(out.peak_index, out.peak_value)
    if k >= 0:
        out.argmax = int(out.peak_index[k])
        out.argmax_value = complex(out.peak_value[k])
    return out


def gather_coarse_map(local: DetectionMap, group=None, device=None) -> Optional[DetectionMap]:
    """Coarse-cell partition: all-gather every rank's per-row peaks and
    candidates; rank 0 returns the merged map (``merge_coarse_maps``)."""
    maps = _gather_maps(local, group, device)
    return merge_coarse_maps(maps, local.counters) if maps is not None else None


def gather_map(local: DetectionMap, group=None, device=None) -> Optional[DetectionMap]:
    """Range-cell partition: all-gather every rank's peaks and candidates;
    rank 0 returns the merged map, other ranks None.  NCCL or gloo."""
    maps = _gather_maps(local, group, device)
    return merge_rank_maps(maps, local.counters) if maps is not None else None


def _gather_maps(local: DetectionMap, group=None, device=None) -> Optional[List[DetectionMap]]:
    """All-gather every rank's peaks and candidates; rank 0 gets the list of
    rank maps, other ranks None.  Works with NCCL (device tensors) and gloo."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    dev = device if device is not None else torch.device("cpu")

    def pack(idx: np.ndarray, val: np.ndarray, n: int) -> "torch.Tensor":
        rec = np.zeros((n, 4), np.float64)  # idx (as int64 bits), re, im, valid
        rec[: idx.size, 0] = idx.astype(np.int64).view(np.float64)
        rec[: idx.size, 1] = val.real
        rec[: idx.size, 2] = val.imag
        rec[: idx.size, 3] = 1.0
        return torch.from_numpy(rec).to(dev)

    def unpack(t: "torch.Tensor"):
        a = t.cpu().numpy()
        keep = a[:, 3] == 1.0
        return a[keep, 0].copy().view(np.int64).astype(np.uint64), a[keep, 1] + 1j * a[keep, 2]

    # sizes first (peaks: rows per rank; candidates: counts)
    sizes = torch.tensor([local.peak_index.size, local.cand_index.size], dtype=torch.int64, device=dev)
    all_sizes = [torch.zeros_like(sizes) for _ in range(world)]
    dist.all_gather(all_sizes, sizes, group=group)
    all_sizes = [s.cpu().numpy() for s in all_sizes]
    pmax = max(int(s[0]) for s in all_sizes)
    cmax = max(int(s[1]) for s in all_sizes)
    peaks = pack(local.peak_index, local.peak_value, pmax)
    cands = pack(local.cand_index, local.cand_value, max(cmax, 1))
    pg = [torch.zeros_like(peaks) for _ in range(world)]
    cg = [torch.zeros_like(cands) for _ in range(world)]
    dist.all_gather(pg, peaks, group=group)
    dist.all_gather(cg, cands, group=group)
    if rank != 0:
        return None
    maps = []
    for r in range(world):
        m = DetectionMap(kind=local.kind, params=local.params, axes=list(local.axes), counters=local.counters,
                         retain_threshold=local.retain_threshold, dual=local.dual, amb=local.amb,
                         doppler_first=local.doppler_first)
        m.peak_index, m.peak_value = unpack(pg[r])
        m.cand_index, m.cand_value = unpack(cg[r])
        maps.append(m)
    return maps


def split_map_by_rows(full: DetectionMap, R: int, D: int, world: int) -> List[DetectionMap]:
    """Test helper: the per-rank maps a row-sharded run produces, cut from a full map."""
    out = []
    r_of = (full.cand_index // np.uint64(D)) % np.uint64(R)
    for rank in range(world):
        lo, hi = shard_rows(R, world, rank)
        m = DetectionMap(kind=full.kind, params=full.params, axes=list(full.axes), counters=full.counters,
                         retain_threshold=full.retain_threshold, dual=full.dual, amb=full.amb,
                         doppler_first=full.doppler_first)
        m.peak_index = full.peak_index[lo:hi].copy()
        m.peak_value = full.peak_value[lo:hi].copy()
        sel = (r_of >= lo) & (r_of < hi)
        m.cand_index = full.cand_index[sel].copy()
        m.cand_value = full.cand_value[sel].copy()
        k = argmax_total_order(m.peak_index, m.peak_value)
        m.argmax, m.argmax_value = int(m.peak_index[k]), complex(m.peak_value[k])
        out.append(m)
    return out


def split_map_by_coarse(full: DetectionMap, C: int, world: int) -> List[DetectionMap]:
    """Test helper: the per-rank maps a coarse-sharded run produces, cut from a
    full map that kept its dense statistic (per-row best over the rank's coarse
    cells, ties to the lowest flat index; candidates of those cells)."""
    if not full.dense_stored:
        raise ValueError("split_map_by_coarse: needs a dense map")
    H = full.dense.size
    per_c = H // C                      # flat = c * per_c + rest, rest = (f*R + r)*D + jj
    R = full.peak_index.size
    D = full.axes[-1].size
    flat = np.arange(H, dtype=np.uint64)
    row = ((flat // np.uint64(D)) % np.uint64(R)).astype(np.int64)
    mag = np.abs(full.dense)
    out = []
    for rank in range(world):
        lo, hi = shard_coarse(C, world, rank)
        sel = slice(lo * per_c, hi * per_c)
        m = DetectionMap(kind=full.kind, params=full.params, axes=list(full.axes), counters=full.counters,
                         retain_threshold=full.retain_threshold, dual=full.dual, amb=full.amb,
                         doppler_first=full.doppler_first)
        # per-row best: sort by (row, -mag, flat) and take the first of each row
        r_s, m_s, f_s = row[sel], mag[sel], flat[sel]
        order = np.lexsort((f_s, -m_s, r_s))
        first = np.ones(order.size, bool)
        first[1:] = r_s[order][1:] != r_s[order][:-1]
        pick = order[first]
        m.peak_index = f_s[pick].copy()
        m.peak_value = full.dense[sel][pick].copy()
        cs = (full.cand_index >= np.uint64(lo * per_c)) & (full.cand_index < np.uint64(hi * per_c))
        m.cand_index, m.cand_value = full.cand_index[cs].copy(), full.cand_value[cs].copy()
        out.append(m)
    return out


# ---------------------------------------------------------------------------
# Collectives of the N-rank bench path (bench.py).  One object, two transports:
# device tensors over NCCL (the real path: one GPU per rank), or, when every
# rank shares one GPU for a functional check (LTCI_BENCH_SHARED_GPU=1), host
# copies over gloo.  Both branches run under gloo in tests/test_multi.py.

class RankComm:
    """``all_gather_into`` / ``all_reduce_max`` for the bench's peak records
    and timings.  ``host_staged=False``: the tensors go to the collective as
    they are (NCCL with device tensors, or gloo with host tensors);
    ``host_staged=True``: device tensors are staged through host memory
    (gloo cannot take them)."""

    def __init__(self, world: int, host_staged: bool = False, group=None):
        self.world = world
        self.host_staged = host_staged
        self.group = group

    def all_gather_into(self, out, inp) -> None:
        """``out`` (world x inp.numel(), rank-major) <- every rank's ``inp``."""
        import torch
        import torch.distributed as dist
        if not self.host_staged:
            # rank-major concatenation along dim 0 (gloo checks the shape, NCCL only numel)
            dist.all_gather_into_tensor(out.view(-1, *inp.shape[1:]), inp, group=self.group)
            return
        parts = [torch.empty_like(inp, device="cpu") for _ in range(self.world)]
        dist.all_gather(parts, inp.cpu(), group=self.group)
        out.copy_(torch.cat(parts).view_as(out))

    def all_reduce_max(self, t) -> None:
        """Element-wise max over ranks, in place (the max-over-ranks timing)."""
        import torch.distributed as dist
        if not self.host_staged:
            dist.all_reduce(t, op=dist.ReduceOp.MAX, group=self.group)
            return
        h = t.cpu()
        dist.all_reduce(h, op=dist.ReduceOp.MAX, group=self.group)
        t.copy_(h)


def _mag2f_np(re: np.ndarray, im: np.ndarray) -> np.ndarray:
    """fmaf(re, re, im*im) in FP32, as ``mag2f`` (csrc/common.cuh) evaluates it:
    re*re is exact in FP64, so one FP32 rounding of the FP64 sum matches the
    fused form except at double-rounding boundaries."""
    im2 = (im.astype(np.float32) * im.astype(np.float32)).astype(np.float32)
    return (re.astype(np.float64) * re.astype(np.float64) + im2.astype(np.float64)).astype(np.float32)


def merge_peak_records(gathered: np.ndarray) -> np.ndarray:
    """Host mirror of ``merge_peaks_kernel`` (csrc/engine.cu): per row, the
    best 16-byte slot {f32 re, f32 im, u64 flat index} over the ranks of a
    coarse-cell partition -- magnitude first, lowest flat index on ties, empty
    slots (index 2^64-1) lose -- the reference's total order
    (proj/src/detectors.cpp:23-31, 34-50).  ``gathered``: (ranks, R, 4) int32."""
    g = np.ascontiguousarray(gathered).view(np.uint32).reshape(gathered.shape[0], -1, 4)
    re = g[..., 0].view(np.float32)
    im = g[..., 1].view(np.float32)
    idx = g[..., 2].astype(np.uint64) | (g[..., 3].astype(np.uint64) << np.uint64(32))
    empty = idx == np.uint64(0xFFFFFFFFFFFFFFFF)
    mag = np.where(empty, np.float32(-1.0), _mag2f_np(re, im))
    R = g.shape[1]
    rows = np.arange(R)
    best = np.zeros(R, np.int64)
    for k in range(1, g.shape[0]):
        bm, bi = mag[best, rows], idx[best, rows]
        better = ~empty[k] & ((mag[k] > bm) | ((mag[k] == bm) & (idx[k] < bi)))
        best = np.where(better, k, best)
    return g[best, rows].view(np.int32).copy()


def encode_peak_records(index: np.ndarray, value: np.ndarray) -> np.ndarray:
    """(R, 4) int32 slots {re, im, idx lo, idx hi} as the engine stores them."""
    out = np.zeros((index.size, 4), np.uint32)
    out[:, 0] = value.real.astype(np.float32).view(np.uint32)
    out[:, 1] = value.imag.astype(np.float32).view(np.uint32)
    out[:, 2] = (index.astype(np.uint64) & np.uint64(0xFFFFFFFF)).astype(np.uint32)
    out[:, 3] = (index.astype(np.uint64) >> np.uint64(32)).astype(np.uint32)
    return out.view(np.int32)


class PeakGather:
    """The per-row peak exchange of one sharded CPI (bench.py's N-rank step).

    * ``shard="coarse"``: every rank holds a slot for every row R; all-gather the
      (R, 4) records into (world, R, 4) and reduce per row with ``merge``
      (``ltci_cuda_merge_peaks`` on the device; ``merge_peak_records`` on the
      host) into ``merged``.
    * ``shard="rows"``: rank k holds rows ``shard_rows(R, world, k)``; slices
      differ by at most one row, so each is padded to R // world + 1 records,
      all-gathered, and ``full_map`` cuts the padding back out.
    """

    def __init__(self, comm: RankComm, shard: str, R: int, like, merge=None):
        import torch
        if shard not in ("coarse", "rows"):
            raise ValueError("PeakGather: shard must be 'coarse' or 'rows'")
        self.comm, self.shard, self.R, self.merge = comm, shard, R, merge
        w = comm.world
        kw = dict(dtype=torch.int32, device=like.device)
        if shard == "coarse":
            self.gathered = torch.empty((w, R, 4), **kw)
            self.merged = torch.empty((R, 4), **kw)
        else:
            self.stride = R // w + 1
            self.gathered = torch.empty((w * self.stride, 4), **kw)
            self.pad = torch.zeros((self.stride, 4), **kw)

    def __call__(self, local) -> None:
        """``local``: this rank's (rows, 4) int32 peak slots."""
        if self.shard == "coarse":
            self.comm.all_gather_into(self.gathered, local)
            self.merge(self.gathered, self.merged)
        else:
            self.pad[: local.shape[0]].copy_(local)
            self.comm.all_gather_into(self.gathered, self.pad)

    def full_map(self):
        """(R, 4) slots of the whole job after the last call."""
        import torch
        if self.shard == "coarse":
            return self.merged
        w = self.comm.world
        return torch.cat([self.gathered[k * self.stride: k * self.stride + (hi - lo)]
                          for k, (lo, hi) in enumerate(shard_rows(self.R, w, k) for k in range(w))])
