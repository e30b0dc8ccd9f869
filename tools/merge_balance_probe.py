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
part = ops.merge_partition(R, A.nnz, k=128)
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
rows = d[:, 2].astype(np.int64)
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
