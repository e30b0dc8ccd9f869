"""Per-group finish times of the cfg5 MTTKRP merge kernel (diagnostic STC_DBG_TIMING build,
see tools/merge_balance_probe.py for the build line)."""
import ctypes
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2405_16883_b200 import ops, synthetic  # noqa: E402

(i, j, k), vals, B, C = synthetic.cfg5()
It, Jt, Kt = (torch.from_numpy(x).int().cuda() for x in (i, j, k))
Vt = torch.from_numpy(vals).cuda()
seg = ops.coo_segments(It)
Bt, Ct = torch.from_numpy(B).cuda(), torch.from_numpy(C).cuda()
part = ops.merge_partition(seg.ptr, len(vals), k=32, kind="mttkrp")
FL = torch.empty(128 * 1024 * 1024, device="cuda")
for _ in range(3):
    ops.mttkrp_coo3(seg, Jt, Kt, Vt, Bt, Ct, partition=part)
FL.zero_()
torch.cuda.synchronize()
ops.mttkrp_coo3(seg, Jt, Kt, Vt, Bt, Ct, partition=part)
torch.cuda.synchronize()
G = part.n_groups
buf = np.zeros((1 << 16, 4), dtype=np.uint64)
assert ops.lib().stc_debug_timing(ctypes.c_void_p(buf.ctypes.data), ctypes.c_size_t(buf.nbytes)) == 0
d = buf[:min(G, 1 << 16)]
t0, t1 = d[:, 0].astype(np.int64), d[:, 1].astype(np.int64)
end = (t1 - t0.min()) / 1e3
rows = d[:, 2].astype(np.int64)
nnz = (d[:, 3] >> np.uint64(32)).astype(np.int64)
print(f"groups {G} ipg {part.items_per_group}; span {end.max():.1f} us")
print("finish p1/p10/p50/p90/p99/max: %.1f %.1f %.1f %.1f %.1f %.1f" % tuple(np.percentile(end, [1, 10, 50, 90, 99, 100])))
print("corr(end, rows) %.2f  corr(end, nnz) %.2f" % (np.corrcoef(end, rows)[0, 1], np.corrcoef(end, nnz)[0, 1]))
z = rows == 0
print("0-row groups: %d, finish p10/p90 %.1f/%.1f; >0-row groups p10/p90 %.1f/%.1f" % (
    z.sum(), *np.percentile(end[z], [10, 90]), *np.percentile(end[~z], [10, 90])))
# fiber starts per group: entries whose (i, j) differs from the previous entry's gather B[j]
st = part.starts.cpu().numpy().reshape(-1, 2).astype(np.int64)
fs = np.ones(len(j), bool)
fs[1:] = (i[1:] != i[:-1]) | (j[1:] != j[:-1])
cfs = np.concatenate([[0], np.cumsum(fs)])
fib = cfs[st[1:G + 1, 1]] - cfs[st[:G, 1]]
print("corr(end, fibers) %.2f  (fibers per group p10/p50/p90 %d/%d/%d)" % (
    np.corrcoef(end, fib[:len(end)])[0, 1], *np.percentile(fib, [10, 50, 90])))
gathers = nnz + fib[:len(end)]
print("corr(end, entries + fibers) %.2f" % np.corrcoef(end, gathers)[0, 1])
# least squares: finish = a + b * fibers + c * rows; what an equal-cost partition would give
X = np.stack([np.ones(len(end)), fib[:len(end)].astype(float), rows.astype(float)], 1)
coef, *_ = np.linalg.lstsq(X, end, rcond=None)
pred = X @ coef
print("fit a=%.1f us, per fiber %.4f us, per row %.4f us; residual sd %.2f us" % (
    coef[0], coef[1], coef[2], np.std(end - pred)))
print("equal-cost groups would finish near %.1f us (+ residual p99 %.1f)" % (
    pred.mean(), np.percentile(end - pred, 99)))
