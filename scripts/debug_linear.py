"""Print the first mismatches of the linear integrate against the oracle (debug aid)."""
import sys
import numpy as np
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import oracle
from conftest import GOLDEN
from paper_2512_08365_b200 import PowerSignal
from paper_2512_08365_b200 import energy as E
g = dict(np.load(GOLDEN / "integrate_linear.npz"))
for s in range(len(g["sig_off"]) - 1):
    sl = slice(g["sig_off"][s], g["sig_off"][s + 1]); iv = slice(g["iv_off"][s], g["iv_off"][s + 1])
    ts, w, lo, hi = g["ts"][sl], g["watts"][sl], g["lo"][iv], g["hi"][iv]
    got = E.integrate_many(PowerSignal.from_columns(ts, w, kind="linear"), lo, hi).cpu().numpy()
    dev = oracle.integrate_linear(ts, w, lo, hi, oracle.MODE_DEVICE)
    bad = np.nonzero(got != dev)[0]
    print(f"signal {s}: S={len(ts)} n={len(lo)} mismatches={len(bad)}")
    for i in bad[:6]:
        a = np.searchsorted(ts, lo[i], side="right") - 1
        b = np.searchsorted(ts, hi[i], side="left") - 1
        print(f"  i={i} lo={lo[i]} hi={hi[i]} a={a} b={b} ts[a..a+1]={ts[max(a,0):a+2]} got={got[i]!r} dev={dev[i]!r} rel={(got[i]-dev[i])/dev[i] if dev[i] else 0}")
