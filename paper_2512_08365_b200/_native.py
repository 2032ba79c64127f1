"""ctypes binding of libdwb200.so (include/dwb200.h).

There is no CPU fallback: importing the compute entry points on a machine
without the built library or without a CUDA device raises ``NativeUnavailable``
the first time a kernel is needed.
"""

from __future__ import annotations

import ctypes
import threading
from pathlib import Path

import torch

_PKG = Path(__file__).resolve().parent
import os as _os

# DWB200_LIB selects a diagnostic build (e.g. _lib/libdwb200_prof.so); the
# default is the product library
LIB_PATH = Path(_os.environ.get("DWB200_LIB") or (_PKG / "_lib" / "libdwb200.so"))

DW_OK = 0
DW_E_REVERSED = -1
DW_E_SPAN = -2
DW_E_EMPTY = -3
DW_E_ORDER = -4
DW_E_ARG = -5
DW_E_CUDA = -6
DW_E_WORKSPACE = -7
DW_E_UNSORTED = -8

DW_SIGNAL_STEP = 0
DW_SIGNAL_LINEAR = 1
DW_MAX_SETS = 4
DW_STATUS_BYTES = 256  # include/dwb200.h
DW_DIRECT_MAX = 256

# every symbol include/dwb200.h declares (tests check the .so exports them all)
EXPORTED = (
    "dw_attribute_workspace_size", "dw_attribute", "dw_ledger", "dw_status", "dw_status_copy", "dw_status_decode",
    "dw_attribute_split_workspace_size", "dw_attribute_split", "dw_attribute_window", "dw_fx_sum_exact", "dw_replay",
    "dw_unpack_workspace_size", "dw_unpack_deltas", "dw_unpack_deltas_w", "dw_unpack_decimal",
    "dw_unpack_decimal_rep_workspace_size", "dw_unpack_decimal_rep", "dw_unpack_decimal_rep_bits",
    "dw_unpack_dict", "dw_unpack_grid", "dw_unpack_bits", "dw_unpack_bits_w", "dw_unpack_bits_dur", "dw_unpack_dict_bits",
    "dw_join_prepare", "dw_join_findings",
    "dw_set_attribute_sms", "dw_ig_nl_count", "dw_ig_nl_write", "dw_ig_classify", "dw_ig_parse_power",
    "dw_ig_parse_op", "dw_ig_parse_kernel", "dw_ig_hash", "dw_ig_id_words", "dw_ig_kernel_lists",
    "dw_fx_sum_workspace_size", "dw_fx_sum", "dw_step_value_at", "dw_detect_pairs",
    "dw_rank_workspace_size", "dw_rank", "dw_rank_segmented_workspace_size", "dw_rank_segmented", "dw_topk_rows",
    "dw_join_workspace_size", "dw_join_diff",
    "dw_exchange_count", "dw_exchange_scatter", "dw_exchange_signal", "dw_exchange_wait",
    "dw_ipc_handle", "dw_ipc_open", "dw_ipc_close",
    "dw_tensor_norms", "dw_tensor_prefilter", "dw_unfold_smem_doubles", "dw_unfold_spectra", "dw_spectra_embed",
    "dw_lcs_matched", "dw_version", "dw_error_string", "dw_launch_count", "dw_kernel_timing", "dw_kernel_time_ms",
    "dw_kernel_timed_count",
)


class NativeUnavailable(RuntimeError):
    """libdwb200.so or a CUDA device is missing: the GPU path cannot run."""


class NativeError(RuntimeError):
    def __init__(self, code: int, where: str):
        self.code = code
        super().__init__(f"{where}: dwb200 error {code} ({error_string(code)})")


c_i64 = ctypes.c_int64
c_i32 = ctypes.c_int32
c_vp = ctypes.c_void_p


class Signal(ctypes.Structure):
    _fields_ = [("d_ts", c_vp), ("d_watts", c_vp), ("n", c_i64), ("span_hi", c_i64),
                ("kind", c_i32), ("validate_order", c_i32), ("sum_mode", c_i32), ("pad", c_i32)]


SUM_REFERENCE, SUM_EXACT = 0, 1  # dw_signal_t.sum_mode


class IntervalSet(ctypes.Structure):
    _fields_ = [("d_start", c_vp), ("d_end", c_vp), ("n", c_i64), ("d_joules", c_vp),
                ("sorted", c_i32), ("pad", c_i32)]


class Window(ctypes.Structure):
    _fields_ = [("g_off", c_i64), ("n_samples_global", c_i64), ("piece_lo", c_i64), ("piece_hi", c_i64),
                ("ts_first", c_i64), ("ts_last", c_i64), ("w_first", ctypes.c_double),
                ("w_last", ctypes.c_double)]


class Status(ctypes.Structure):
    _fields_ = [("code", c_i32), ("bad_set", c_i32), ("bad_index", c_i64 * DW_MAX_SETS),
                ("order_index", c_i64), ("unsorted_index", c_i64 * DW_MAX_SETS),
                ("long_intervals", c_i64), ("totals", ctypes.c_double * 4)]


class Findings(ctypes.Structure):
    _fields_ = [("d_energy_a", c_vp), ("d_energy_b", c_vp), ("d_ratio", c_vp),
                ("d_latency_a", c_vp), ("d_latency_b", c_vp), ("d_verdict", c_vp),
                ("d_side", c_vp), ("d_informational", c_vp), ("d_wasted", c_vp),
                ("d_key_hi", c_vp), ("d_key_lo", c_vp), ("d_tie_rank", c_vp), ("n_a", c_i64),
                ("d_delta_e", c_vp), ("d_delta_t", c_vp), ("d_epw_ratio", c_vp)]


class RankSegment(ctypes.Structure):
    _fields_ = [("d_key_hi", c_vp), ("d_key_lo", c_vp), ("d_tie_rank", c_vp), ("n_a", c_i64), ("P", c_i64)]


class JoinSide(ctypes.Structure):
    _fields_ = [("d_sig", c_vp), ("d_start", c_vp), ("d_end", c_vp), ("d_joules", c_vp),
                ("d_work", c_vp), ("d_rank", c_vp), ("n", c_i64)]


_lib = None
_lock = threading.Lock()


def lib():
    """Load libdwb200.so (loudly failing when absent)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not LIB_PATH.exists():
            raise NativeUnavailable(
                f"{LIB_PATH} is not built; run `python -m paper_2512_08365_b200.build` "
                "(there is no CPU fallback)")
        L = ctypes.CDLL(str(LIB_PATH))
        L.dw_attribute_workspace_size.restype = ctypes.c_size_t
        L.dw_attribute_workspace_size.argtypes = [c_i64, ctypes.POINTER(c_i64), c_i32]
        L.dw_attribute.argtypes = [ctypes.POINTER(Signal), ctypes.POINTER(IntervalSet), c_i32,
                                   c_vp, ctypes.c_size_t, c_vp]
        L.dw_ledger.argtypes = [ctypes.POINTER(Signal), ctypes.POINTER(IntervalSet),
                                ctypes.POINTER(IntervalSet), c_vp, ctypes.c_size_t, c_vp]
        L.dw_status.argtypes = [c_vp, c_vp, ctypes.POINTER(Status)]
        L.dw_status_copy.argtypes = [c_vp, c_vp, c_vp]
        L.dw_status_decode.argtypes = [c_vp, ctypes.POINTER(Status)]
        L.dw_attribute_window.argtypes = [ctypes.POINTER(Signal), ctypes.POINTER(IntervalSet), c_i32,
                                          ctypes.POINTER(Window), c_vp, c_vp, c_i64, c_vp, c_vp, c_vp,
                                          ctypes.c_size_t, c_vp]
        L.dw_fx_sum_exact.argtypes = [c_vp, c_i64, c_vp, c_vp, ctypes.c_size_t, c_vp]
        L.dw_set_attribute_sms.argtypes = [ctypes.c_int]
        L.dw_ig_nl_count.argtypes = [c_vp, c_i64, c_vp, c_vp, c_vp]
        L.dw_ig_nl_write.argtypes = [c_vp, c_i64, c_vp, c_vp, c_vp]
        L.dw_ig_classify.argtypes = [c_vp, c_i64, c_vp, c_i64, c_vp, c_vp, c_vp]
        L.dw_ig_parse_power.argtypes = [c_vp, c_vp, c_vp, c_i64, c_vp, c_vp, c_vp, c_vp]
        L.dw_ig_parse_op.argtypes = [c_vp, c_vp, c_vp, c_i64] + [c_vp] * 12
        L.dw_ig_parse_kernel.argtypes = [c_vp, c_vp, c_vp, c_i64] + [c_vp] * 9
        L.dw_ig_hash.argtypes = [c_vp, c_vp, c_vp, c_i64, c_vp, c_vp, c_vp]
        L.dw_ig_id_words.argtypes = [c_vp, c_vp, c_vp, c_i64, c_i32, c_vp, c_vp]
        L.dw_ig_kernel_lists.argtypes = [c_vp, c_i64, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_i64] + [c_vp] * 11
        L.dw_unpack_workspace_size.restype = ctypes.c_size_t
        L.dw_unpack_workspace_size.argtypes = [c_i64]
        L.dw_unpack_deltas.argtypes = [c_vp, c_i64, c_i64, c_vp, c_vp, c_vp, c_vp, ctypes.c_size_t, c_vp]
        L.dw_unpack_deltas_w.argtypes = [c_vp, c_i32, c_i64, c_i64, c_i64, c_vp, c_vp, c_i32, c_vp, c_vp,
                                         ctypes.c_size_t, c_vp]
        L.dw_unpack_dict.argtypes = [c_vp, c_vp, c_i32, c_i64, c_vp, c_vp]
        L.dw_unpack_bits.argtypes = [c_vp, c_i32, c_i64, c_i64, c_i64, c_vp, c_vp, ctypes.c_size_t, c_vp]
        L.dw_unpack_bits_dur.argtypes = [c_vp, c_vp, c_i32, c_i64, c_i64, c_vp, c_vp]
        L.dw_unpack_grid.argtypes = [c_vp, c_i32, c_i64, c_i64, c_i64, ctypes.c_uint64, c_vp, c_vp]
        L.dw_unpack_bits_w.argtypes = [c_vp, c_i32, c_i64, c_i64, c_i64, c_vp, c_vp, c_i32, c_i64, c_vp, c_vp,
                                       ctypes.c_size_t, c_vp]
        L.dw_unpack_dict_bits.argtypes = [c_vp, c_vp, c_i32, c_i64, c_vp, c_vp]
        L.dw_unpack_decimal.argtypes = [c_vp, c_i64, c_i32, c_vp, c_vp]
        L.dw_unpack_decimal_rep_workspace_size.restype = ctypes.c_size_t
        L.dw_unpack_decimal_rep_workspace_size.argtypes = [c_i64]
        L.dw_unpack_decimal_rep.argtypes = [c_vp, c_vp, c_i64, c_i32, c_vp, c_vp, ctypes.c_size_t, c_vp]
        L.dw_unpack_decimal_rep_bits.argtypes = [c_vp, c_i32, ctypes.c_uint32, c_vp, c_i64, c_i32, c_vp, c_vp,
                                                 ctypes.c_size_t, c_vp]
        L.dw_replay.argtypes = [ctypes.POINTER(Signal), c_vp, c_vp, c_i64, c_i64, c_i64, c_vp, c_i64, c_vp, c_vp,
                                c_vp, c_vp]
        L.dw_tensor_norms.argtypes = [c_vp, c_vp, c_i64, c_vp, c_vp]
        L.dw_exchange_count.argtypes = [c_vp, c_i64, c_i32, c_vp, c_vp]
        L.dw_exchange_scatter.argtypes = [c_vp, c_i32, c_vp, c_i64, c_i32, c_vp, c_vp, c_vp, c_vp]
        L.dw_exchange_signal.argtypes = [c_vp, c_i32, c_i32, ctypes.c_uint64, c_vp]
        L.dw_exchange_wait.argtypes = [c_vp, c_i32, ctypes.c_uint64, c_vp, c_vp]
        L.dw_ipc_handle.argtypes = [c_vp, c_vp, c_vp]
        L.dw_ipc_open.argtypes = [c_vp, ctypes.POINTER(c_vp)]
        L.dw_ipc_close.argtypes = [c_vp]
        L.dw_tensor_prefilter.argtypes = [ctypes.c_int, c_i64, c_i64, c_i32, c_vp, c_vp, c_vp, c_vp,
                                          ctypes.c_double, c_vp, c_vp, c_vp, c_vp, c_vp]
        L.dw_unfold_smem_doubles.restype = c_i64
        L.dw_unfold_smem_doubles.argtypes = []
        L.dw_unfold_spectra.argtypes = [c_vp, c_vp, c_i64, c_i64, c_vp, c_vp, c_vp, c_vp]
        L.dw_spectra_embed.argtypes = [c_vp, c_vp, c_vp, c_vp, c_vp, c_i64, c_vp, c_vp, ctypes.c_double, c_vp,
                                       c_vp]
        L.dw_attribute_split_workspace_size.restype = ctypes.c_size_t
        L.dw_attribute_split_workspace_size.argtypes = [c_i64, c_i64]
        L.dw_attribute_split.argtypes = [ctypes.POINTER(Signal), ctypes.POINTER(IntervalSet), c_vp,
                                         ctypes.c_size_t, c_vp]
        L.dw_fx_sum_workspace_size.restype = ctypes.c_size_t
        L.dw_fx_sum_workspace_size.argtypes = [c_i64]
        L.dw_fx_sum.argtypes = [c_vp, c_i64, c_vp, c_vp, ctypes.c_size_t, c_vp]
        L.dw_step_value_at.argtypes = [ctypes.POINTER(Signal), c_vp, c_i64, c_vp, c_vp]
        L.dw_lcs_matched.argtypes = [c_vp, c_vp, c_vp, c_vp, c_i64, c_vp, c_vp, c_vp, c_vp, c_vp]
        L.dw_version.restype = ctypes.c_char_p
        L.dw_error_string.restype = ctypes.c_char_p
        L.dw_error_string.argtypes = [ctypes.c_int]
        L.dw_launch_count.restype = c_i64
        L.dw_launch_count.argtypes = [ctypes.c_int]
        L.dw_kernel_timing.argtypes = [ctypes.c_int]
        L.dw_kernel_time_ms.restype = ctypes.c_double
        L.dw_kernel_time_ms.argtypes = [ctypes.c_int]
        L.dw_kernel_timed_count.restype = c_i64
        L.dw_kernel_timed_count.argtypes = [ctypes.c_int]
        if hasattr(L, "dw_detect_pairs"):
            L.dw_detect_pairs.argtypes = [c_i64] + [c_vp] * 12 + [ctypes.c_double,
                                                                  ctypes.POINTER(Findings), c_vp]
            L.dw_rank_workspace_size.restype = ctypes.c_size_t
            L.dw_rank_workspace_size.argtypes = [c_i64, c_i64]
            L.dw_rank.argtypes = [c_i64, ctypes.POINTER(Findings), c_i64, c_vp, c_vp, c_vp,
                                  ctypes.c_size_t, c_vp]
            L.dw_topk_rows.argtypes = [c_vp, c_i64, c_i64] + [c_vp] * 9 + [c_vp]
            L.dw_rank_segmented_workspace_size.restype = ctypes.c_size_t
            L.dw_rank_segmented_workspace_size.argtypes = [c_i32, c_i64]
            L.dw_rank_segmented.argtypes = [ctypes.POINTER(RankSegment), c_i32, c_i64, c_vp, c_vp, c_vp,
                                            ctypes.c_size_t, c_vp]
            L.dw_join_workspace_size.restype = ctypes.c_size_t
            L.dw_join_workspace_size.argtypes = [c_i64, c_i64, c_i64]
            L.dw_join_diff.argtypes = [ctypes.POINTER(JoinSide), ctypes.POINTER(JoinSide), c_i64,
                                       ctypes.c_double, ctypes.POINTER(Findings), c_vp, c_vp,
                                       c_vp, c_vp, c_vp, c_vp, ctypes.c_size_t, c_vp]
            L.dw_join_prepare.argtypes = [ctypes.POINTER(JoinSide), ctypes.POINTER(JoinSide), c_i64, c_vp, c_vp,
                                          ctypes.POINTER(c_i64), c_vp, ctypes.c_size_t, c_vp]
            L.dw_join_findings.argtypes = [ctypes.POINTER(JoinSide), ctypes.POINTER(JoinSide), c_i64,
                                           ctypes.c_double, ctypes.POINTER(Findings), c_vp, c_vp, c_i64, c_vp,
                                           c_vp, c_vp, c_vp, ctypes.c_size_t, c_vp]
        _lib = L
        return L


def error_string(code: int) -> str:
    try:
        return lib().dw_error_string(int(code)).decode()
    except NativeUnavailable:
        return str(code)


def version() -> str:
    return lib().dw_version().decode()


def launch_count(reset: bool = False) -> int:
    return int(lib().dw_launch_count(1 if reset else 0))


_DEVICES: dict = {}


def device() -> torch.device:
    """The CUDA device the GPU path runs on (current torch device)."""
    idx = torch.cuda.current_device() if _DEVICES else None
    d = _DEVICES.get(idx)
    if d is None:  # first call (or a new device): check once, then cache
        if not torch.cuda.is_available():
            raise NativeUnavailable("no CUDA device: the dwb200 GPU path cannot run "
                                    "(there is no CPU fallback)")
        lib()
        idx = torch.cuda.current_device()
        d = _DEVICES.setdefault(idx, torch.device("cuda", idx))
    return d


def stream_handle(stream=None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def ptr(t) -> int | None:
    if t is None:
        return None
    return t.data_ptr() if t.numel() else None


def check(rc: int, where: str) -> None:
    if rc != DW_OK:
        raise NativeError(rc, where)


class Workspace:
    """Grow-only device scratch, one per (device, stream); caller-owned by the
    library's contract (the library itself never allocates)."""

    _pool: dict = {}

    @classmethod
    def get(cls, nbytes: int, stream=None) -> torch.Tensor:
        dev = device()
        key = (dev.index, stream_handle(stream))
        buf = cls._pool.get(key)
        if buf is None or buf.numel() < nbytes:
            cls._pool[key] = None
            buf = torch.empty(max(int(nbytes * 1.25), 1 << 20), dtype=torch.uint8, device=dev)
            cls._pool[key] = buf
        return buf

    @classmethod
    def clear(cls) -> None:
        cls._pool.clear()


def num_sms() -> int:
    """Streaming multiprocessors of the current device."""
    return int(torch.cuda.get_device_properties(device()).multi_processor_count)
