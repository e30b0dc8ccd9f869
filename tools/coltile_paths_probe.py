"""COLTILE operand staging: the tiled TMA copy (tensor map) against the per-row bulk copies forced with
STC_COLTILE_ROW_COPIES=1, across operand widths -- also shows that the tensor-map path is the one in use for
narrow operands (k < 128: the 128-column box reaches past the operand and is zero-filled).
  python tools/coltile_paths_probe.py
One B200, 4096 x 4096 at 5 % density: k = 4 / 64 / 132 / 512: 157.6 / 156.6 / 157.6 / 158.8 us tiled,
323.0 / 322.8 / 322.8 / 255.1 us by rows."""
import os, sys, statistics, numpy as np, torch
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), '..'))
from paper_2405_16883_b200 import ops
rng = np.random.default_rng(0)
m, n = 4096, 4096
for k in (4, 64, 132, 512):
    dens = 0.05
    mask = rng.random((m, n)) < dens
    rp = np.concatenate([[0], np.cumsum(mask.sum(1))]).astype(np.int32)
    ci = np.nonzero(mask)[1].astype(np.int32)
    v = rng.standard_normal(ci.size).astype(np.float32)
    R, C, V = (torch.from_numpy(x).cuda() for x in (rp, ci, v))
    B = torch.randn(n, k, device='cuda')
    plan = ops.coltile_plan(R, C, n, V)
    res = {}
    for mode in ("0", "1"):
        os.environ["STC_COLTILE_ROW_COPIES"] = mode
        ts = []
        for _ in range(20):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record(); ops.spmm_csr(R, C, V, B, variant="coltile", partition=plan); e.record()
            torch.cuda.synchronize(); ts.append(s.elapsed_time(e) * 1e3)
        res[mode] = statistics.median(ts)
    print(f"k={k}: tiled-copy path {res['0']:.1f} us, row-copy path {res['1']:.1f} us")
