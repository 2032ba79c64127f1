import sys, ctypes
import numpy as np, torch
sys.path.insert(0, ".")
import oracle
from paper_2512_08365_b200 import PowerSignal, _native
from paper_2512_08365_b200 import energy as E
ts = np.array([2300, 2334, 2336], dtype=np.int64); w = np.array([100.0, 300.0, 500.0])
for lo, hi in [(2335, 2335), (2334, 2334), (2300, 2300), (2336, 2336), (2301, 2301), (2335, 2336), (2300, 2336)]:
    L = np.array([lo]); H = np.array([hi])
    got = E.integrate_many(PowerSignal.from_columns(ts, w, kind="linear"), L, H).cpu().numpy()
    st = _native.Status(); ws = _native.Workspace.get(0)
    _native.lib().dw_status(ws.data_ptr(), _native.stream_handle(), ctypes.byref(st))
    dev = oracle.integrate_linear(ts, w, L, H, oracle.MODE_DEVICE)
    print(lo, hi, got, dev, "long", st.long_intervals)
