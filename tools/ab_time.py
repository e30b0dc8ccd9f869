"""Median device time of one configuration's hot op (L2 flushed before every rep), for A/B runs
over library builds: STC_LIBRARY=ab/x.so python tools/ab_time.py 5   (see tools/ab.sh)."""
import importlib.util
import os
import statistics
import sys
from pathlib import Path

import torch

cfg = sys.argv[1]
sys.argv = sys.argv[:1] + [cfg]
spec = importlib.util.spec_from_file_location("cfg_one", Path(__file__).with_name("cfg_one.py"))
cfg_one = importlib.util.module_from_spec(spec)
spec.loader.exec_module(cfg_one)
fn = {"2": cfg_one.cfg2, "3": cfg_one.cfg3, "4": cfg_one.cfg4, "5": cfg_one.cfg5}[cfg]()
flush = torch.empty(128 * 1024 * 1024, device="cuda")
ts = []
for _ in range(int(os.environ.get("REPS", "30"))):
    flush.zero_()
    flush.sum()  # clean L2 (bench.py flush_l2)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    fn()
    e.record()
    torch.cuda.synchronize()
    ts.append(s.elapsed_time(e) * 1e3)
print(f"{os.path.basename(os.environ.get('STC_LIBRARY', 'libstc.so'))} cfg{cfg}: median {statistics.median(ts):.1f} us "
      f"(min {min(ts):.1f})")
