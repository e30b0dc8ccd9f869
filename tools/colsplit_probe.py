"""cfg2 layer: one K=128 merge SpMM vs. the same product as K/S-column slices run one after
another (S = 2, 4), so each launch's working set of B is n x (128/S) floats (51 MB at S = 2)
instead of the 102 MB table that does not stay in L2 next to the streaming output.
L2 flushed (512 MB write) before every rep; median of REPS reps by CUDA events."""
import os
import statistics
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2405_16883_b200 import ops, synthetic  # noqa: E402

A, X, _, _ = synthetic.cfg2()
R = torch.from_numpy(A.rowptr).int().cuda()
Ci = torch.from_numpy(A.colidx).int().cuda()
V = torch.from_numpy(A.vals).cuda()
Xd = torch.from_numpy(X).cuda()
m, k = A.shape[0], Xd.shape[1]
flush = torch.empty(128 * 1024 * 1024, device="cuda")
REPS = int(os.environ.get("REPS", "30"))
ref = ops.spmm_csr(R, Ci, V, Xd, variant="merge")


def timed(fn):
    ts = []
    for _ in range(REPS):
        flush.zero_()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e) * 1e3)
    return statistics.median(ts), min(ts)


out = torch.empty((m, k), device="cuda")
for S in (1, 2, 4):
    w = k // S
    part = ops.merge_partition(R, Ci.numel(), k=w, colidx=Ci, vals=V)
    ws = part.workspace(w, 1, Xd.device)

    def run():
        for s in range(S):
            ops.spmm_csr(R, Ci, V, Xd[:, s * w:(s + 1) * w], out=out[:, s * w:(s + 1) * w], variant="merge",
                         partition=part, workspace=ws)

    run()
    torch.cuda.synchronize()
    diff = (out - ref).abs().max().item()
    med, mn = timed(run)
    print(f"S={S} ({w} columns per launch, ipg {part.items_per_group}): median {med:.1f} us (min {mn:.1f}), "
          f"max |diff vs K=128| {diff:.3g}")
