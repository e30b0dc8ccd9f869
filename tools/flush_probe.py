"""How the L2 flush before a timed launch is done changes what the launch pays for: a 512 MB write leaves
the L2 full of dirty lines that the kernel's own misses must first write back; a read pass after the write
leaves clean lines. cfg2 SpMM layer, median of 30:  python tools/flush_probe.py"""
import importlib.util
import statistics
import sys
from pathlib import Path

import torch

sys.argv = sys.argv[:1] + ["2"]
spec = importlib.util.spec_from_file_location("cfg_one", Path(__file__).with_name("cfg_one.py"))
cfg_one = importlib.util.module_from_spec(spec)
spec.loader.exec_module(cfg_one)
fn = cfg_one.cfg2()
buf = torch.empty(128 * 1024 * 1024, device="cuda")
buf2 = torch.empty(128 * 1024 * 1024, device="cuda")


def timed(flush):
    ts = []
    for _ in range(30):
        flush()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e) * 1e3)
    return statistics.median(ts), min(ts)


modes = {
    "no flush (warm L2)": lambda: None,
    "512 MB write (dirty L2)": lambda: buf.zero_(),
    "512 MB write then 512 MB read of it (clean L2)": lambda: (buf.zero_(), buf.sum()),
    "512 MB write then device-to-device copy of another 512 MB": lambda: (buf.zero_(), buf2.copy_(buf)),
    "512 MB read only": lambda: buf.sum(),
}
for name, f in modes.items():
    med, mn = timed(f)
    print(f"{name:60s} median {med:6.1f} us  min {mn:6.1f} us")
