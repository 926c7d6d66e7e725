"""bench.py's N-rank helpers (parallel.RankComm / PeakGather) over REAL NCCL
on the one GPU the build has: a world of one rank executes the NCCL branch --
`dist.all_reduce(op=MAX)`, `all_gather_into_tensor` on device tensors, then
the device peak merge (`ltci_cuda_merge_peaks`) -- the lines that had only
ever run over gloo (round 1's NCCL branch recursed into itself).  With more
ranks the same calls move more records; the gloo world-size-2/3 tests cover
the indexing across ranks."""
from __future__ import annotations

import os
import socket
import subprocess
import sys
import textwrap

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = textwrap.dedent("""
    import ctypes, sys
    import numpy as np
    import torch
    import torch.distributed as dist
    sys.path.insert(0, %r)
    from paper_2403_06788_b200 import _lib, parallel
    from paper_2403_06788_b200.parallel import PeakGather, RankComm

    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", device_id=dev)
    assert dist.get_backend() == "nccl" and dist.get_world_size() == 1
    comm = RankComm(1, host_staged=False)

    t = torch.tensor([3.25, -1.0], device=dev)
    comm.all_reduce_max(t)                       # NCCL all_reduce(MAX)
    assert t.tolist() == [3.25, -1.0]

    rng = np.random.default_rng(3)
    R = 37
    idx = rng.integers(0, 2**40, R).astype(np.uint64)
    val = (rng.standard_normal(R) + 1j * rng.standard_normal(R)).astype(np.complex64)
    rec = torch.from_numpy(parallel.encode_peak_records(idx, val).view(np.int32).reshape(R, 4).copy()).to(dev)

    g = PeakGather(comm, "rows", R, rec)         # padded NCCL all_gather_into_tensor
    g(rec)
    assert torch.equal(g.full_map(), rec)

    lib = _lib.load()
    stream = torch.cuda.current_stream().cuda_stream

    def merge_on_device(gathered, merged):
        _lib.raise_for(lib.ltci_cuda_merge_peaks(ctypes.c_void_p(gathered.data_ptr()), 1, R,
                                                 ctypes.c_void_p(merged.data_ptr()), ctypes.c_void_p(stream)), lib)

    g = PeakGather(comm, "coarse", R, rec, merge=merge_on_device)
    g(rec)
    torch.cuda.synchronize()
    assert torch.equal(g.full_map(), rec)
    want = parallel.merge_peak_records(rec.cpu().numpy().reshape(1, R, 4))
    assert np.array_equal(g.full_map().cpu().numpy().view(np.uint32), np.asarray(want).view(np.uint32).reshape(R, 4))
    dist.destroy_process_group()
    print("nccl-ok")
""") % ROOT


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_bench_collectives_over_nccl_one_rank():
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()), RANK="0", LOCAL_RANK="0",
               WORLD_SIZE="1")
    r = subprocess.run([sys.executable, "-c", SCRIPT], env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "nccl-ok" in r.stdout, r.stdout[-2000:] + r.stderr[-4000:]
