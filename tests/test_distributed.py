"""N>1 host logic on CPU with gloo (world_size 2): nnz-balanced row sharding,
row-disjoint partial SpMMs reassembled by all-gather, and the max-over-ranks
timing reduction used by bench.py (the product's sharded GCN path:
tests/test_distributed_product.py)."""

import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2405_16883_b200 import dist as sdist
from paper_2405_16883_b200 import synthetic


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _csr_matmul(rp, ci, v, X):
    """Local row-shard product on the host (float64 torch CSR): the CUDA kernels need a GPU;
    this test covers the sharding, exchange and reduction logic."""
    A = torch.sparse_csr_tensor(torch.as_tensor(rp).long(), torch.as_tensor(ci).long(),
                                torch.as_tensor(v).double(), size=(len(rp) - 1, X.shape[0]))
    return A @ torch.as_tensor(X).double()


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        A, X, _, _ = synthetic.cfg2(n=3000, feat=16)
        shards = sdist.nnz_balanced_row_shards(A.rowptr, world)
        r0, r1 = shards[rank]
        rp, ci, v = sdist.shard_csr(A.rowptr, A.colidx, A.vals, r0, r1)
        local = _csr_matmul(rp, ci, v, X)
        full = sdist.allgather_rows(local, shards)
        want = _csr_matmul(A.rowptr, A.colidx, A.vals, X)
        ok = bool(torch.equal(full, want))
        t = sdist.max_over_ranks(float(rank + 1))
        q.put((rank, ok, t, shards))
    finally:
        dist.destroy_process_group()


def test_row_shards_balance():
    A, _, _, _ = synthetic.cfg2(n=20000, feat=8)
    for world in (2, 3, 8):
        sh = sdist.nnz_balanced_row_shards(A.rowptr, world)
        assert sh[0][0] == 0 and sh[-1][1] == A.shape[0]
        assert all(a[1] == b[0] for a, b in zip(sh, sh[1:]))
        work = [A.rowptr[r1] - A.rowptr[r0] + (r1 - r0) for r0, r1 in sh]
        heavy = int(np.diff(A.rowptr).max())
        assert max(work) - min(work) <= heavy + 2 * (A.nnz + A.shape[0]) // (world * 1000) + 2


def test_gloo_world2_sharded_spmm_and_max_reduction():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, ok, t, shards in res:
        assert ok, f"rank {rank}: reassembled sharded SpMM differs from the full oracle"
        assert t == float(world)
