import torch, time
n = 120_849_444 // 4
h = torch.empty(n, dtype=torch.float32).pin_memory()
d = torch.empty(n, dtype=torch.float32, device="cuda")
ho = torch.empty(102_400_000 // 4, dtype=torch.float32).pin_memory()
do = torch.empty(102_400_000 // 4, dtype=torch.float32, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(fn, reps=10):
    fn(); torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps
def up():
    d.copy_(h, non_blocking=True)
def down():
    ho.copy_(do, non_blocking=True)
def both():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur); s2.wait_stream(cur)
    with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2): ho.copy_(do, non_blocking=True)
    cur.wait_stream(s1); cur.wait_stream(s2)
for name, fn, nb in [("h2d", up, n*4), ("d2h", down, 102_400_000), ("both", both, n*4)]:
    ms = t(fn)
    print(name, f"{ms:.3f} ms", f"{nb/ms/1e6:.1f} GB/s")
# chunked h2d
def up_chunks(k=8):
    c = n // k
    for i in range(k):
        d[i*c:(i+1)*c].copy_(h[i*c:(i+1)*c], non_blocking=True)
print("h2d 8 chunks", f"{t(up_chunks):.3f} ms")
