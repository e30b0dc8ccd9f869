import torch, time
n = 120_849_444 // 4
h = torch.empty(n, dtype=torch.float32).pin_memory()
d = torch.empty(n, dtype=torch.float32, device="cuda")
o = torch.empty(102_400_000 // 4, dtype=torch.float32, device="cuda")
ho = torch.empty(o.numel(), dtype=torch.float32).pin_memory()
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(fn, reps=20):
    for _ in range(3): fn()
    torch.cuda.synchronize(); a = time.perf_counter()
    for _ in range(reps): fn()
    torch.cuda.synchronize(); return (time.perf_counter() - a) / reps * 1e3
h2d = t(lambda: d.copy_(h, non_blocking=True))
d2h = t(lambda: ho.copy_(o, non_blocking=True))
def both():
    with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2): ho.copy_(o, non_blocking=True)
bo = t(both)
print(f"H2D 120.8 MB: {h2d:.3f} ms ({120.85/h2d:.1f} GB/s); D2H 102.4 MB: {d2h:.3f} ms ({102.4/d2h:.1f} GB/s); both concurrently: {bo:.3f} ms")

# the e2e step's transfers alone, pipelined like bench.py (uploads two steps ahead, 6 copies per step)
sizes = [800_004, 8_759_184, 8_759_184, 102_400_000, 65_536, 65_536]
hs = [torch.empty(b // 4, dtype=torch.float32).pin_memory() for b in sizes]
NB = 3
ds = [[torch.empty_like(h, device="cuda") for h in hs] for _ in range(NB)]
outs = [torch.empty(102_400_000 // 4, device="cuda") for _ in range(NB)]
hos = [torch.empty(102_400_000 // 4).pin_memory() for _ in range(NB)]
s_up, s_dn = torch.cuda.Stream(), torch.cuda.Stream()
ev_up = [torch.cuda.Event() for _ in range(NB)]
ev_dn = [torch.cuda.Event() for _ in range(NB)]
def pipe(n):
    for i in range(n):
        b = i % NB
        with torch.cuda.stream(s_up):
            if i >= NB:
                s_up.wait_event(ev_dn[b])
            for d, h in zip(ds[b], hs):
                d.copy_(h, non_blocking=True)
            ev_up[b].record(s_up)
        with torch.cuda.stream(s_dn):
            s_dn.wait_event(ev_up[b])
            hos[b].copy_(outs[b], non_blocking=True)
            ev_dn[b].record(s_dn)
    torch.cuda.current_stream().wait_stream(s_up); torch.cuda.current_stream().wait_stream(s_dn)
for n in (20, 50):
    pipe(3); torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(s_up); pipe(n); e.record(); torch.cuda.synchronize()
    print(f"transfers only, {n} pipelined steps: {s.elapsed_time(e) / n:.3f} ms/step")
