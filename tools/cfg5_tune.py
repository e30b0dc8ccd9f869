"""cfg5 MTTKRP: GPU time against items-per-group (L2 flushed before every rep)."""
import statistics
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2405_16883_b200 import ops, synthetic  # noqa: E402

(i, j, k), vals, B, C = synthetic.cfg5()
It, Jt, Kt = (torch.from_numpy(x).int().cuda() for x in (i, j, k))
Vt = torch.from_numpy(vals).cuda()
seg = ops.coo_segments(It)
Bt, Ct = torch.from_numpy(B).cuda(), torch.from_numpy(C).cuda()
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


for ipg in [None, 32, 48, 64, 96, 128, 232, 400]:
    part = ops.merge_partition(seg.ptr, len(vals), ipg, k=32, kind="mttkrp")
    ws = ops.spmm_workspace(seg.n_seg, len(vals), 32, "merge", part.items_per_group, 1, "cuda")
    us = t(lambda: ops.mttkrp_coo3(seg, Jt, Kt, Vt, Bt, Ct, partition=part, workspace=ws))
    print(f"ipg {part.items_per_group:5d}  {us:8.1f} us")
