"""Long differential fuzz on the GPU (same generators as tests/test_gpu_fuzz.py, many
more seeds): every hot-path case must run on a dedicated kernel in the inferred format
and match the float64 dense evaluation; every random expression of the reference's
strategy must run (kernel or device walker) and match.
  python tools/fuzz_long.py [n_hot] [n_random] [extent_cap]"""
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import paper_2405_16883_b200 as st  # noqa: E402
from helpers import abs_bound, random_expression  # noqa: E402
from oracle.restate import parity_gate  # noqa: E402
from test_gpu_fuzz import _hot_path_case  # noqa: E402

n_hot = int(sys.argv[1]) if len(sys.argv) > 1 else 4000
n_rand = int(sys.argv[2]) if len(sys.argv) > 2 else 2000
cap = int(sys.argv[3]) if len(sys.argv) > 3 else 40   # extent cap of the hot-path cases
fails = []
t0 = time.time()
for seed in range(n_hot):
    rng = np.random.default_rng(100_000 + seed)
    src, tensors = _hot_path_case(rng, cap)
    try:
        e = st.parse(src, tensors)
        out, _, report = st.run_with_report(e)
        assert not any(v.startswith("generic") for v in report["variants"]), report["variants"]
        assert out.format == st.infer_format(e), (out.format, st.infer_format(e))
        want = st.eval_dense(e)
        ok, worst = parity_gate(np.asarray(st.to_dense(out), dtype=np.float64), want, abs_bound(e, tensors), 1e-5)
        assert ok, worst
    except Exception as err:  # noqa: BLE001
        fails.append(("hot", seed, src, repr(err)[:200]))
print(f"hot-path: {n_hot} cases, {len(fails)} failures ({time.time() - t0:.0f} s)", flush=True)
nf = len(fails)
t0 = time.time()
for seed in range(n_rand):
    rng = np.random.default_rng(200_000 + seed)
    e = random_expression(rng, extent_cap=12, device="cuda")
    tensors = {a.tensor.name: a.tensor for a in e.accesses}
    try:
        out, _, _ = st.run_with_report(e)
        want = st.eval_dense(e)
        ok, worst = parity_gate(np.asarray(st.to_dense(out), dtype=np.float64).reshape(want.shape), want,
                                abs_bound(e, tensors), 1e-5)
        assert ok, worst
    except Exception as err:  # noqa: BLE001
        fails.append(("random", seed, st.render(e), repr(err)[:200]))
print(f"random: {n_rand} expressions, {len(fails) - nf} failures ({time.time() - t0:.0f} s)", flush=True)
for f in fails[:30]:
    print(f)
