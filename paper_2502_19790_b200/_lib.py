"""ctypes binding of the C-ABI in ``include/mixtera_b200.h`` (libmxb200.so).

The product path has no CPU fallback: if the shared library is missing, or no
CUDA device is visible when a kernel is needed, ``lib()`` raises
``DeviceError``. Status codes map to the reference's exception types.
"""

from __future__ import annotations

import ctypes as C
import threading
from pathlib import Path

from .errors import (
    DataReadError,
    DeviceError,
    FeedbackError,
    IndexBuildError,
    MixtureError,
    QueryError,
)

LIB_PATH = Path(__file__).resolve().parent / "libmxb200.so"

MX_OK = 0
MX_EXHAUSTED = 1
_ERRORS = {
    -1: DeviceError,
    -2: ValueError,
    -3: QueryError,
    -4: IndexBuildError,
    -5: MixtureError,
    -6: FeedbackError,
    -7: DataReadError,
    -8: NotImplementedError,
}

MAX_PROPS = 16

i32, i64, u32, u64, dbl, vp = C.c_int32, C.c_int64, C.c_uint32, C.c_uint64, C.c_double, C.c_void_p
P = C.POINTER


class CatalogDesc(C.Structure):
    _fields_ = [
        ("n_props", i32),
        ("columns", P(vp)),
        ("lut", P(u32)),
        ("lut_offsets", P(i32)),
        ("n_samples", i64),
        ("n_files", i32),
        ("file_offsets", vp),
        ("file_ds", P(i32)),
        ("file_ids", P(i64)),
        ("key_bits", u32),
        ("rank_mask", u32),
        ("field_shift", P(u32)),
        ("field_width", P(u32)),
        ("key_strings", P(C.c_uint8)),
        ("key_string_offsets", P(i64)),
        ("key_string_base", P(i32)),
        ("n_columns", i32),
        ("n_key_pieces", i32),
        ("column_bytes", i32),
    ]


class MixtureDesc(C.Structure):
    _fields_ = [
        ("n_mkeys", i32),
        ("allow", P(u32)),
        ("allow_words", i32),
        ("allow_base", P(i32)),
        ("weights", P(dbl)),
        ("chunk_size", i64),
        ("strict", i32),
    ]


class ShardDesc(C.Structure):
    _fields_ = [
        ("world", i32),
        ("rank", i32),
        ("file_lo", i64),
        ("file_hi", i64),
        ("n_files", i32),
        ("file_ds", P(i32)),
        ("file_ids", P(i64)),
        ("tables", vp),
        ("counts", P(i64)),
        ("cap", i64),
        ("global_keys", P(u32)),
        ("n_global_keys", i64),
    ]


class RowsDesc(C.Structure):
    _fields_ = [
        ("n_rows", i64),
        ("key", P(u32)),
        ("file", P(u32)),
        ("start", P(u32)),
        ("end", P(u32)),
        ("n_files", i32),
        ("file_ds", P(i32)),
        ("file_ids", P(i64)),
        ("n_keys", i32),
        ("key_bits", u32),
        ("key_strings", P(C.c_uint8)),
        ("key_string_offsets", P(i64)),
    ]


class JsonDesc(C.Structure):
    _fields_ = [
        ("n_keys", i64),
        ("key_json", P(C.c_uint8)),
        ("key_json_off", P(i64)),
        ("key_rank", P(u32)),
        ("file_rank", P(u32)),
        ("mixture_json", P(C.c_uint8)),
        ("mixture_len", i32),
    ]


_SIGS = {
    "mx_last_error": (C.c_char_p, []),
    "mx_abi_version": (C.c_int, []),
    "mx_launch_count": (i64, []),
    "mx_profile_enable": (C.c_int, [C.c_int]),
    "mx_profile_reset": (C.c_int, []),
    "mx_profile_read": (C.c_int, [C.c_char_p, P(dbl), P(i64)]),
    "mx_index_build": (C.c_int, [P(CatalogDesc), vp, P(vp)]),
    "mx_index_build_rows": (C.c_int, [P(RowsDesc), vp, P(vp)]),
    "mx_index_free": (C.c_int, [vp]),
    "mx_index_sizes": (C.c_int, [vp, P(i64), P(i64), P(i64), P(i64)]),
    "mx_index_export_keys": (C.c_int, [vp, vp, vp]),
    "mx_index_export_intervals": (C.c_int, [vp, vp, vp, vp, vp, vp]),
    "mx_gen_create": (C.c_int, [vp, vp, i32, vp, i32, u64, vp, P(vp)]),
    "mx_gen_free": (C.c_int, [vp]),
    "mx_gen_plan": (C.c_int, [vp, P(MixtureDesc), i64, P(i64)]),
    "mx_gen_plan_arbitrary": (C.c_int, [vp, i64, i64, P(i64)]),
    "mx_gen_result_sizes": (C.c_int, [vp, P(i64), P(i64)]),
    "mx_gen_result_copy": (C.c_int, [vp, vp, vp, vp, vp, vp, vp, vp, vp]),
    "mx_gen_result_device": (C.c_int, [vp, P(vp), P(vp), P(vp), P(vp), P(vp), P(vp)]),
    "mx_gen_report": (C.c_int, [vp, vp]),
    "mx_gen_result_export": (C.c_int, [vp, vp, vp, vp, vp, vp, vp]),
    "mx_gen_result_json": (C.c_int, [vp, P(JsonDesc), P(i64), vp]),
    "mx_gen_result_json_copy": (C.c_int, [vp, vp, vp]),
    "mx_gen_mark": (C.c_int, [vp]),
    "mx_gen_reset_to_mark": (C.c_int, [vp]),
    "mx_gen_next_chunk_id": (C.c_int, [vp, P(i64)]),
    "mx_gen_set_next_chunk_id": (C.c_int, [vp, i64]),
    "mx_gen_get_cursors": (C.c_int, [vp, vp, vp]),
    "mx_gen_set_cursors": (C.c_int, [vp, vp, vp]),
    "mx_gen_component_order": (C.c_int, [vp, vp]),
    "mx_gen_cursor_ranges": (C.c_int, [vp, u32, P(i64), vp, vp, vp, vp, i64]),
    "mx_index_block_table": (C.c_int, [vp, i64, vp, vp]),
    "mx_index_packed_keys": (C.c_int, [vp, vp]),
    "mx_index_build_sharded": (C.c_int, [vp, P(ShardDesc), vp, P(vp)]),
    "mx_gen_cursor_to_consumed": (C.c_int, [vp, vp, vp, vp]),
    "mx_gen_set_consumed": (C.c_int, [vp, vp]),
    "mx_index_build_owner": (C.c_int, [vp, vp, i64, i32, vp, vp, i32, vp, P(vp)]),
    "mx_gen_block_offsets": (C.c_int, [vp, vp, vp]),
    "mx_gen_set_local": (C.c_int, [vp, vp, vp, vp, i64]),
    "mx_gen_set_handoff": (C.c_int, [vp, i32]),
    "mx_gen_handoff": (C.c_int, [vp, P(i64), P(i64), P(vp), P(vp)]),
    "mx_gen_finish_owned": (C.c_int, [vp, i32, i64, i64, i64, vp, vp, i64, vp]),
    "mx_chunks_merge": (C.c_int, [i32, i64, i64, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp]),
    "mx_domain_loss": (C.c_int, [vp, vp, i64, i32, vp, vp, vp]),
    "mx_fit_power_law": (C.c_int, [i32, vp, vp, vp, vp, vp, vp]),
    "mx_ado_pi": (C.c_int, [i32, vp, vp, vp, dbl, dbl, dbl, vp, vp, vp, vp]),
    "mx_ado_credit": (C.c_int, [i32, dbl, vp, vp, vp]),
    "mx_jsonl_records": (C.c_int, [vp, i64, vp, vp, vp, i64, P(i64), P(i64), vp]),
    "mx_jsonl_extract": (C.c_int, [vp, vp, vp, i64, vp, vp, i32, vp, vp, vp, vp, vp, vp, vp, vp]),
    "mx_jsonl_tokenize": (C.c_int, [vp, vp, vp, i64, vp, i32, i32, u32, vp, vp, vp, vp, vp]),
    "mx_pack_tokens": (C.c_int, [i64, i32, i32, vp, vp, vp, vp, vp, vp, vp, vp, vp, i32, vp, vp, vp]),
}

EXPORTED = tuple(_SIGS)

_lock = threading.Lock()
_handle = None


def load_library(path: Path | str = LIB_PATH) -> C.CDLL:
    """Load the .so and declare every symbol (no GPU needed)."""
    if not Path(path).exists():
        raise DeviceError(
            f"CUDA extension {path} is missing; build it with "
            "`python -m paper_2502_19790_b200.build` (there is no CPU fallback)"
        )
    h = C.CDLL(str(path))
    for name, (res, args) in _SIGS.items():
        fn = getattr(h, name)
        fn.restype = res
        fn.argtypes = args
    return h


def lib() -> C.CDLL:
    """The loaded library, after checking a CUDA device is visible."""
    global _handle
    with _lock:
        if _handle is None:
            import torch

            if not torch.cuda.is_available():
                raise DeviceError("no CUDA device visible: the Mixtera B200 path needs a GPU (no CPU fallback)")
            torch.cuda.init()
            _handle = load_library()
        return _handle


def check(rc: int) -> int:
    if rc >= 0:
        return rc
    msg = _handle.mx_last_error().decode("utf-8", "replace") if _handle else "error"
    raise _ERRORS.get(rc, DeviceError)(msg)


def profile_read(phase: str) -> tuple[float, int]:
    ms, n = dbl(), i64()
    check(lib().mx_profile_read(phase.encode(), C.byref(ms), C.byref(n)))
    return ms.value, n.value


def stream_ptr(stream=None) -> int:
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


def ptr(arr) -> int:
    """Address of a numpy array / torch tensor buffer (0 for None)."""
    if arr is None:
        return 0
    if hasattr(arr, "data_ptr"):
        return int(arr.data_ptr())
    return int(arr.ctypes.data)
