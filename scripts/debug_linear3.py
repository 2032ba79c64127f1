import sys
import numpy as np
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import oracle
from conftest import GOLDEN
from paper_2512_08365_b200 import PowerSignal
from paper_2512_08365_b200 import energy as E
g = dict(np.load(GOLDEN / "integrate_linear.npz"))
s = 6
sl = slice(g["sig_off"][s], g["sig_off"][s + 1]); iv = slice(g["iv_off"][s], g["iv_off"][s + 1])
ts, w, lo, hi = g["ts"][sl], g["watts"][sl], g["lo"][iv], g["hi"][iv]
print("ts", ts, "w", w)
got = E.integrate_many(PowerSignal.from_columns(ts, w, kind="linear"), lo, hi).cpu().numpy()
dev = oracle.integrate_linear(ts, w, lo, hi, oracle.MODE_DEVICE)
o = np.argsort(lo, kind="stable")
for i in o:
    print(i, lo[i], hi[i], got[i], dev[i], "BAD" if got[i] != dev[i] else "")
