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
    part = ops.merge_partition(seg.ptr, len(vals), k=32, kind="mttkrp")
    return lambda: ops.mttkrp_coo3(seg, Jt, Kt, Vt, Bt, Ct, partition=part)


def cfg3():
    W, XT = synthetic.cfg3()
    R, C, V = (torch.from_numpy(W.rowptr).int().cuda(), torch.from_numpy(W.colidx).int().cuda(),
               torch.from_numpy(W.vals).cuda())
    Xt = torch.from_numpy(XT).cuda()
    out = torch.empty((W.shape[0], 4096), device="cuda")
    return lambda: ops.spmm_csr(R, C, V, Xt, out=out, variant="coltile")


fn = {"3": cfg3, "5": cfg5}[sys.argv[1]]()
for _ in range(3):
    fn()
torch.cuda.synchronize()
