import sys, collections
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import numpy as np
import paper_2405_16883_b200 as st
from helpers import random_expression
msgs = collections.Counter(); ex = {}
ran = 0
for seed in range(240):
    rng = np.random.default_rng(1000 + seed)
    e = random_expression(rng, extent_cap=9, device="cuda")
    try:
        st.run_with_report(e); ran += 1
    except st.UnsupportedExpressionError as err:
        key = str(err)[:90]
        msgs[key] += 1; ex.setdefault(key, st.render(e) if hasattr(st, 'render') else str(e))
print('ran', ran)
for k, n in msgs.most_common(15):
    print(n, k, '|', ex[k][:100])
