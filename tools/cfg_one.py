"""Run one configuration's hot kernel a few times (for ncu captures): python tools/cfg_one.py 5"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2405_16883_b200 import ops, synthetic  # noqa: E402


def cfg5():
    (i, j, k), vals, B, C = synthetic.cfg5()
    It, Jt, Kt = (torch.from_numpy(x).int().cuda() for x in (i, j, k))
    Vt = torch.from_numpy(vals).cuda()
    seg = ops.coo_segments(It)
    Bt, Ct = torch.from_numpy(B).cuda(), torch.from_numpy(C).cuda()
    part = ops.merge_partition(seg.ptr, len(vals), k=32, kind="mttkrp", jcrd=Jt, kcrd=Kt, vals=Vt,
                               factors=(Bt.shape[0], Bt.stride(0), Ct.shape[0], Ct.stride(0)))
    return lambda: ops.mttkrp_coo3(seg, Jt, Kt, Vt, Bt, Ct, partition=part)


def cfg3():
    W, XT = synthetic.cfg3()
    R, C, V = (torch.from_numpy(W.rowptr).int().cuda(), torch.from_numpy(W.colidx).int().cuda(),
               torch.from_numpy(W.vals).cuda())
    Xt = torch.from_numpy(XT).cuda()
    out = torch.empty((W.shape[0], 4096), device="cuda")
    return lambda: ops.spmm_csr(R, C, V, Xt, out=out, variant="coltile")


def cfg4():
    M, Q, K, V = synthetic.cfg4()
    R, C, MV = (torch.from_numpy(M.rowptr).int().cuda(), torch.from_numpy(M.colidx).int().cuda(),
                torch.from_numpy(M.vals).cuda())
    Qt, Kt, Vt = (torch.from_numpy(x).cuda() for x in (Q, K, V))
    plan = ops.attention_tile_plan(R, C, MV, M.shape[1])
    ws = torch.empty(int(ops.lib().stc_attention_tiled_workspace_bytes(M.shape[0], 16)) // 4, device="cuda")
    return lambda: ops.sparse_attention_tiled(plan, Qt, Kt, Vt, scale=0.125, workspace=ws)


def cfg2():
    A, X, W1, _ = synthetic.cfg2()
    R, C, V = (torch.from_numpy(A.rowptr).int().cuda(), torch.from_numpy(A.colidx).int().cuda(),
               torch.from_numpy(A.vals).cuda())
    Z = torch.from_numpy(X).cuda() @ torch.from_numpy(W1).cuda()
    out = torch.empty_like(Z)
    part = ops.merge_partition(R, A.nnz, k=128, colidx=C, vals=V)
    ws = ops.spmm_workspace(A.shape[0], A.nnz, 128, "merge", part.items_per_group, 1, "cuda")
    return lambda: ops.spmm_csr(R, C, V, Z, out=out, relu=True, variant="merge", partition=part, workspace=ws)


if __name__ == "__main__":
    fn = {"2": cfg2, "3": cfg3, "4": cfg4, "5": cfg5}[sys.argv[1]]()
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
