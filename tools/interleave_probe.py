"""cfg2: does interleaving the entries of long rows (a fixed permutation inside each row
longer than one group) balance the merge kernel's groups? Times the merge kernel on the
original and the interleaved CSR (same values, same per-row sums up to order), and, with the
STC_DBG_TIMING build, prints the per-group finish spread.
  python tools/interleave_probe.py"""
import ctypes
import statistics
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2405_16883_b200 import ops, synthetic  # noqa: E402

FL = torch.empty(128 * 1024 * 1024, device="cuda")


def interleave(rowptr, colidx, vals, span):
    ci, va = colidx.copy(), vals.copy()
    lens = np.diff(rowptr)
    for r in np.flatnonzero(lens > span):
        a, b = rowptr[r], rowptr[r + 1]
        g = -(-(b - a) // span)                   # groups the row spans
        order = np.concatenate([np.arange(j, b - a, g) for j in range(g)])
        ci[a:b], va[a:b] = colidx[a:b][order], vals[a:b][order]
    return ci, va


def run(A, ci, va, Z, label):
    R = torch.from_numpy(A.rowptr).int().cuda()
    C = torch.from_numpy(ci).int().cuda()
    V = torch.from_numpy(va).cuda()
    out = torch.empty_like(Z)
    part = ops.merge_partition(R, A.nnz, k=128)
    ws = ops.spmm_workspace(A.shape[0], A.nnz, 128, "merge", part.items_per_group, 1, "cuda")
    f = lambda: ops.spmm_csr(R, C, V, Z, out=out, relu=True, variant="merge", partition=part, workspace=ws)  # noqa
    for _ in range(3):
        f()
    ts = []
    for _ in range(30):
        FL.zero_()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        f()
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e) * 1000)
    line = f"{label}: {statistics.median(ts):.1f} us (ipg {part.items_per_group})"
    lib = ops.lib()
    if hasattr(lib, "stc_debug_timing"):
        FL.zero_()
        torch.cuda.synchronize()
        f()
        torch.cuda.synchronize()
        buf = np.zeros((1 << 16, 4), dtype=np.uint64)
        lib.stc_debug_timing(ctypes.c_void_p(buf.ctypes.data), ctypes.c_size_t(buf.nbytes))
        d = buf[:part.n_groups]
        end = (d[:, 1].astype(np.int64) - d[:, 0].astype(np.int64).min()) / 1e3
        rows = d[:, 2].astype(np.int64)
        line += " | finish p10/p50/p90/max %.1f/%.1f/%.1f/%.1f" % tuple(np.percentile(end, [10, 50, 90, 100]))
        z = rows == 0
        if z.any():
            line += " | 0-row groups p10/p90 %.1f/%.1f" % tuple(np.percentile(end[z], [10, 90]))
        h = rows >= 100
        if h.any():
            line += " | >=100-row groups mean %.1f" % end[h].mean()
    print(line, flush=True)
    return out


A, X, W1, _ = synthetic.cfg2()
Z = torch.from_numpy(X).cuda() @ torch.from_numpy(W1).cuda()
o1 = run(A, A.colidx, A.vals, Z, "original")
ci, va = interleave(A.rowptr, A.colidx, A.vals, 505)
o2 = run(A, ci, va, Z, "interleaved rows > 505")
print("max |diff| between orders:", float((o1 - o2).abs().max()))
