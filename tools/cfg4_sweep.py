import sys, statistics, torch
sys.path.insert(0, '.')
from paper_2405_16883_b200 import ops, synthetic
M, Q, K, V = synthetic.cfg4()
R, C, MV = (torch.from_numpy(M.rowptr).int().cuda(), torch.from_numpy(M.colidx).int().cuda(), torch.from_numpy(M.vals).cuda())
Qt, Kt, Vt = (torch.from_numpy(x).cuda() for x in (Q, K, V))
flush = torch.empty(128*1024*1024, device="cuda")
ws = torch.empty(int(ops.lib().stc_attention_tiled_workspace_bytes(M.shape[0], 16)) // 4, device="cuda")
def t(fn, reps=20):
    fn(); torch.cuda.synchronize(); ts=[]
    for _ in range(reps):
        flush.zero_(); s=torch.cuda.Event(enable_timing=True); e=torch.cuda.Event(enable_timing=True)
        s.record(); fn(); e.record(); torch.cuda.synchronize(); ts.append(s.elapsed_time(e)*1e3)
    return statistics.median(ts)
for fill in (1/4, 1/8, 1/16, 1/32, 1/64):
    for mx in (8, 12, 16):
        plan = ops.attention_tile_plan(R, C, MV, M.shape[1], min_fill=fill, max_tiles=mx)
        us = t(lambda: ops.sparse_attention_tiled(plan, Qt, Kt, Vt, scale=0.125, workspace=ws))
        print(f"fill {fill:.4f} max {mx}: dense share {plan.dense_share:.3f} tiles/block {(plan.tile_cols>=0).sum(1).float().mean().item():.2f} -> {us:.1f} us", flush=True)
