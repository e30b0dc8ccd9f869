"""Sweep SpMM variants / merge granularity on configs[1] (GCN graph), L2 flushed per launch."""
import statistics
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2405_16883_b200 as st  # noqa: E402
from paper_2405_16883_b200 import ops, synthetic  # noqa: E402

A, X, _, _ = synthetic.cfg2()
At = st.csr_from_arrays(A.rowptr, A.colidx, A.vals, A.shape, name="A")
R, C, V = At.storage.levels[1].pos, At.storage.levels[1].crd, At.storage.values
Z = torch.from_numpy(X).cuda()
out = torch.empty_like(Z)
flush = torch.empty(128 * 1024 * 1024, device="cuda")
byts = 4 * (A.shape[0] + 1) + 8 * A.nnz + 2 * 4 * A.shape[0] * 128


PERSIST = [a for a in sys.argv if a.startswith("persist=")]
NOFLUSH = "noflush" in sys.argv
sys.argv = [a for a in sys.argv if a != "noflush"]


def timeit(fn, reps=30):
    ts = []
    for _ in range(reps):
        if not NOFLUSH:
            if PERSIST:
                ops.l2_reset_persisting()
            flush.zero_()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    return statistics.median(ts)


sys.argv = [a for a in sys.argv if not a.startswith("persist=")]
if PERSIST:
    got = ops.l2_set_persisting(int(float(PERSIST[0].split("=")[1]) * 2**20))
    print("persisting L2 carve-out:", got / 2**20, "MiB")
for ipg in [int(x) for x in (sys.argv[1:] or ["0", "256", "512"])]:
    part = ops.merge_partition(R, A.nnz, ipg, k=128)
    ipg = part.items_per_group
    ws = ops.spmm_workspace(A.shape[0], A.nnz, 128, "merge", ipg, 1, "cuda")
    ms = timeit(lambda: ops.spmm_csr(R, C, V, Z, out=out, variant="merge", partition=part, workspace=ws))
    print(f"merge ipg={ipg:4d}: {ms*1e3:8.1f} us  {byts/ms/1e6:8.1f} GB/s")
ms = timeit(lambda: ops.spmm_csr(R, C, V, Z, out=out, variant="row"))
print(f"row           : {ms*1e3:8.1f} us  {byts/ms/1e6:8.1f} GB/s")
