"""CPU-side checks of the native boundary: the C-ABI library loads, exports
every symbol include/dwb200.h declares, and the package fails loudly (never
falls back) when no GPU is present."""
import ctypes
import re
from pathlib import Path

import pytest
import torch

from conftest import ROOT

import paper_2512_08365_b200 as dw
from paper_2512_08365_b200 import _native, build


def _declared():
    text = (ROOT / "include" / "dwb200.h").read_text()
    return sorted(set(re.findall(r"^\s*(?:[\w\s\*]+?)\b(dw_\w+)\s*\(", text, re.M)))


def test_header_declares_exactly_the_exported_list():
    assert _declared() == sorted(_native.EXPORTED)


def test_library_builds_and_exports_every_symbol():
    build.build()
    L = ctypes.CDLL(str(_native.LIB_PATH))
    for name in _native.EXPORTED:
        assert hasattr(L, name), name
    assert _native.version().startswith("dwb200")
    assert _native.error_string(_native.DW_E_SPAN) == "interval outside signal span"


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU behaviour")
def test_no_cpu_fallback_without_gpu():
    import numpy as np
    cols = dw.TraceColumns.from_arrays(np.array([0, 10]), np.array([1.0, 2.0]),
                                       np.array([0]), np.array([5]))
    with pytest.raises(_native.NativeUnavailable):
        dw.build_ledger(cols)


def test_unfold_descriptor_layout_matches_header():
    """tensor_equiv.UNFOLD_DTYPE mirrors dw_unfold_t (include/dwb200.h)."""
    from paper_2512_08365_b200.tensor_equiv import UNFOLD_DTYPE
    assert UNFOLD_DTYPE.itemsize == 64
    assert [UNFOLD_DTYPE.fields[n][1] for n in ("value_off", "out_off", "scratch_off", "order", "mask", "dims")] \
        == [0, 8, 16, 24, 28, 32]
    hdr = (Path(__file__).resolve().parent.parent / "include" / "dwb200.h").read_text()
    body = hdr[hdr.index("typedef struct {\n    int64_t value_off;"):hdr.index("} dw_unfold_t;")]
    fields = re.findall(r"^\s*(int64_t|int32_t)\s+(\w+)(\[8\])?;", body, flags=re.M)
    assert [(t, n) for t, n, _ in fields] == [("int64_t", "value_off"), ("int64_t", "out_off"),
                                             ("int64_t", "scratch_off"), ("int32_t", "order"),
                                             ("int32_t", "mask"), ("int32_t", "dims")]


def test_new_entry_points_reject_bad_arguments_before_touching_the_device():
    """Argument validation of the 8(f) entry points runs on the host: bad sizes
    and widths return DW_E_ARG (no CUDA call is made, so this runs without a
    GPU)."""
    L = ctypes.CDLL(str(_native.LIB_PATH))
    E_ARG = _native.DW_E_ARG
    i64 = ctypes.c_int64
    assert L.dw_tensor_norms(None, None, i64(-1), None, None) == E_ARG
    assert L.dw_tensor_prefilter(2, i64(1), i64(1), 1, None, None, None, None, ctypes.c_double(1e-3), None, None,
                                 None, None, None) == E_ARG
    assert L.dw_unfold_spectra(None, None, i64(-1), i64(0), None, None, None, None) == E_ARG
    assert L.dw_unfold_spectra(None, None, i64(0), i64(1 << 40), None, None, None, None) == E_ARG
    assert L.dw_spectra_embed(None, None, None, None, None, i64(-1), None, None, ctypes.c_double(1e-3), None,
                              None) == E_ARG
    assert L.dw_unpack_deltas_w(None, 3, i64(0), i64(5), i64(0), None, None, 4, None, None, ctypes.c_size_t(0),
                                None) == E_ARG
    assert L.dw_unpack_dict(None, None, 1, i64(4), None, None) == E_ARG
    assert L.dw_unpack_decimal(None, i64(-1), 6, None, None) == E_ARG
    assert L.dw_unpack_decimal(None, i64(0), 30, None, None) == E_ARG
