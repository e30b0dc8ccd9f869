"""cfg4: is the CSR remainder faster as two gather passes (SDDMM, then PV as a batched
SpMM) than in the fused per-row online-softmax kernel? Times each piece with L2 flushed.
  python tools/cfg4_rem_probe.py"""
import statistics
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2405_16883_b200 import ops, synthetic  # noqa: E402

FL = torch.empty(128 * 1024 * 1024, device="cuda")


def t(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        FL.zero_()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e) * 1000)
    return statistics.median(ts)


M, Q, K, V = synthetic.cfg4()
R, C, MV = (torch.from_numpy(M.rowptr).int().cuda(), torch.from_numpy(M.colidx).int().cuda(),
            torch.from_numpy(M.vals).cuda())
Qt, Kt, Vt = (torch.from_numpy(x).cuda() for x in (Q, K, V))
plan = ops.attention_tile_plan(R, C, MV, M.shape[1])
ws = torch.empty(int(ops.lib().stc_attention_tiled_workspace_bytes(M.shape[0], 16)) // 4, device="cuda")
print("tiled total", round(t(lambda: ops.sparse_attention_tiled(plan, Qt, Kt, Vt, scale=0.125, workspace=ws)), 1), "us")
rr, rc, rv = plan.rem_rowptr, plan.rem_colidx, plan.rem_vals
print("remainder nnz/head", rc.numel(), "dense share", round(plan.dense_share, 3))
print("fused per-row kernel on the remainder only",
      round(t(lambda: ops.sparse_attention(rr, rc, Qt, Kt, Vt, maskvals=rv, scale=0.125)), 1), "us")
S = torch.empty((16, rc.numel()), device="cuda")
print("SDDMM on the remainder", round(t(lambda: ops.sddmm_csr(rr, rc, Qt, Kt, maskvals=rv, scale=0.125, out=S)), 1), "us")
P = torch.rand_like(S)
O = torch.empty_like(Qt)
for variant in ("row", "merge"):
    print(f"PV batched SpMM ({variant}) on the remainder",
          round(t(lambda: ops.spmm_csr_batched(rr, rc, P, Vt, out=O, variant=variant)), 1), "us")
