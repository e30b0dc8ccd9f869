"""Per-group finish times of the cfg2 merge kernel. Needs the diagnostic build of
libstc.so (globaltimer stamps per group, `#ifdef STC_DBG_TIMING` in segreduce.cuh):
  cd paper_2405_16883_b200 && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
      -Xcompiler -fPIC --expt-relaxed-constexpr -DSTC_DBG_TIMING -I ../include -c csrc/spmm.cu \
      -o build/spmm_dbg.o && nvcc -gencode arch=compute_100a,code=sm_100a -shared -o libstc.so \
      build/abi_common.o build/spmm_dbg.o build/spmm_wide.o build/attention.o build/spgemm.o
  python tools/merge_balance_probe.py
Prints the spread of finish times and how it correlates with each group's row / entry counts.
Round 1 (kRowCost = 1): finish p10/p50/p90/max 71.7/79.5/90.9/95.7 us, corr(duration, rows) 0.84."""
import ctypes
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2405_16883_b200 import ops, synthetic  # noqa: E402

A, X, W1, _ = synthetic.cfg2()
R, C, V = (torch.from_numpy(A.rowptr).int().cuda(), torch.from_numpy(A.colidx).int().cuda(),
           torch.from_numpy(A.vals).cuda())
Z = torch.from_numpy(X).cuda() @ torch.from_numpy(W1).cuda()
out = torch.empty_like(Z)
part = ops.merge_partition(R, A.nnz, k=128, colidx=C, vals=V)  # the shipped plan: long rows interleaved
ws = ops.spmm_workspace(A.shape[0], A.nnz, 128, "merge", part.items_per_group, 1, "cuda")
FL = torch.empty(128 * 1024 * 1024, device="cuda")
for _ in range(5):
    ops.spmm_csr(R, C, V, Z, out=out, relu=True, variant="merge", partition=part, workspace=ws)
FL.zero_()
torch.cuda.synchronize()
ops.spmm_csr(R, C, V, Z, out=out, relu=True, variant="merge", partition=part, workspace=ws)
torch.cuda.synchronize()
G = part.n_groups
buf = np.zeros((1 << 16, 4), dtype=np.uint64)
lib = ops.lib()
rc = lib.stc_debug_timing(ctypes.c_void_p(buf.ctypes.data), ctypes.c_size_t(buf.nbytes))
assert rc == 0, rc
d = buf[:G]
t0, t1 = d[:, 0].astype(np.int64), d[:, 1].astype(np.int64)
base = t0.min()
start, end = (t0 - base) / 1e3, (t1 - base) / 1e3
rows = (d[:, 2] & np.uint64(0xffffffff)).astype(np.int64)
smid = (d[:, 2] >> np.uint64(32)).astype(np.int64)
nnz = (d[:, 3] >> np.uint64(32)).astype(np.int64)
dur = end - start
print(f"groups {G} ipg {part.items_per_group}; kernel span {end.max():.1f} us")
print("start  us: p50 %.1f p99 %.1f max %.1f" % tuple(np.percentile(start, [50, 99, 100])))
print("finish us: p1 %.1f p10 %.1f p50 %.1f p90 %.1f p99 %.1f max %.1f" % tuple(np.percentile(end, [1, 10, 50, 90, 99, 100])))
print("duration: p10 %.1f p50 %.1f p90 %.1f max %.1f" % tuple(np.percentile(dur, [10, 50, 90, 100])))
print("corr(duration, rows) %.3f  corr(duration, nnz) %.3f" % (np.corrcoef(dur, rows)[0, 1], np.corrcoef(dur, nnz)[0, 1]))
for lo, hi in [(0, 50), (50, 100), (100, 200), (200, 400), (400, 1000)]:
    m = (rows >= lo) & (rows < hi)
    if m.any():
        print(f"  rows in [{lo},{hi}): {m.sum():5d} groups, mean duration {dur[m].mean():.1f} us, mean nnz {nnz[m].mean():.0f}")
cta = (d[:, 3] & np.uint64(0xffffff)).astype(np.int64) >> 8
cta_end = np.zeros(cta.max() + 1)
np.maximum.at(cta_end, cta, end)
print("CTA finish: p10 %.1f p50 %.1f p90 %.1f max %.1f" % tuple(np.percentile(cta_end, [10, 50, 90, 100])))
slow = np.argsort(-end)[:12]
print("slowest groups (g, cta, rows, nnz, start us, end us):")
for gi in slow:
    print(f"  {gi:5d} {cta[gi]:4d} {rows[gi]:4d} {nnz[gi]:4d} {start[gi]:6.1f} {end[gi]:6.1f}")
fast = np.argsort(end)[:5]
print("fastest groups:")
for gi in fast:
    print(f"  {gi:5d} {cta[gi]:4d} {rows[gi]:4d} {nnz[gi]:4d} {start[gi]:6.1f} {end[gi]:6.1f}")

# ---- what explains the spread: cold gathers per group, or the SM a group ran on? ----
st = part.starts.cpu().numpy().reshape(-1, 2)
ci = (part.colidx if part.colidx is not None else C).cpu().numpy()
p0, p1 = st[:G, 1], st[1:G + 1, 1]
for thr in (2000, 20000, 60000):
    cold_pref = np.concatenate([[0], np.cumsum(ci >= thr)])
    cold = cold_pref[p1] - cold_pref[p0]
    X_ = np.stack([np.ones(G), rows, cold], 1)
    coef, *_ = np.linalg.lstsq(X_, end, rcond=None)
    res = end - X_ @ coef
    print(f"cold = col >= {thr}: corr(finish, cold) {np.corrcoef(end, cold)[0, 1]:.3f}; finish ~ {coef[0]:.1f} + "
          f"{coef[1]:.4f} rows + {coef[2]:.4f} cold; residual sd {res.std():.2f} us (finish sd {end.std():.2f})")
sm_mean = np.zeros(smid.max() + 1)
sm_cnt = np.zeros(smid.max() + 1)
np.add.at(sm_mean, smid, end)
np.add.at(sm_cnt, smid, 1)
sm_mean = sm_mean[sm_cnt > 0] / sm_cnt[sm_cnt > 0]
print(f"per-SM mean finish: min {sm_mean.min():.1f} p50 {np.median(sm_mean):.1f} max {sm_mean.max():.1f} us; "
      f"sd between SMs {sm_mean.std():.2f}, sd within SMs {np.sqrt(max(end.var() - sm_mean.var(), 0)):.2f}")
