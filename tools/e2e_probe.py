"""Where does bench.py's e2e step time go? (pipelined upload / compute / download)
  python tools/e2e_probe.py"""
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402

work = bench.GCN(base=0, device=torch.device("cuda", 0))
for steps in (20, 40):
    ms, h2d, d2h = work.e2e(steps=steps, warmup=3)
    print(f"e2e as shipped, {steps} steps: {ms:.3f} ms/step", flush=True)

ops = work.ops
orig = ops.spmm_csr
plan = dict(variant=work.variant, partition=work.partition, workspace=None, stats=work.stats)
ws = [ops.spmm_workspace(work.n, work.nnz, work.k, "merge", work.ipg, 1, "cuda") for _ in range(2)]
cnt = [0]


def cached(rp, ci, v, B, **kw):
    for key in ("variant", "partition", "stats"):
        kw.pop(key, None)
    cnt[0] += 1
    return orig(rp, ci, v, B, variant=work.variant, partition=work.partition, workspace=ws[cnt[0] % 2],
                stats=work.stats, **kw)


ops.spmm_csr = cached
ms, _, _ = work.e2e(steps=20, warmup=3)
print(f"e2e with cached plan: {ms:.3f} ms/step", flush=True)
ops.spmm_csr = lambda rp, ci, v, B, out=None, relu=False, **kw: out  # noqa: E731
ms, _, _ = work.e2e(steps=20, warmup=3)
print(f"e2e copies only (no SpMM; GEMMs kept): {ms:.3f} ms/step", flush=True)
