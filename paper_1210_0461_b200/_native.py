"""ctypes binding of libcrop_b200.so (include/crop_b200.h).

The product path has no CPU fallback: if the library is missing or no CUDA
device is visible, every call raises `DeviceError` loudly.
"""

import ctypes
import os

from .errors import ConfigError, CropError, DeviceError, InputError, ResourceCapError

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "_lib", "libcrop_b200.so")
ABI_VERSION = 1

_lib = None

P = ctypes.c_void_p
i64, u64, u32, i32 = ctypes.c_int64, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_int


class Interval(ctypes.Structure):
    """crop_interval: the owned bucket range plus device hash tables."""

    _fields_ = [("kappa", u32), ("start", u32), ("stop", u32), ("h_row", P), ("h_col", P)]


class OuterShape(ctypes.Structure):
    """crop_outer_shape: what crop_outer_create_ex needs to plan without a sync."""

    _fields_ = [("all_terms", u64), ("max_row", u32), ("max_col", u32), ("nnz_a", i64), ("nnz_b", i64)]


_SIGS = {
    "crop_abi_version": (i32, []),
    "crop_last_error": (ctypes.c_char_p, []),
    "crop_launch_counter": (u64, []),
    "crop_hash_tables": (i32, [u32, u64, u64, u64, u64, u32, P, P, P]),
    "crop_sign_hash": (i32, [P, P, u64, u64, u64, P, P]),
    "crop_selfjoin_bucket_loads": (i32, [P, P, i64, P, P, u32, i32, P, P]),
    "crop_outer_bucket_loads": (i32, [P, P, P, P, i64, P, P, u32, i32, P, P]),
    "crop_pairs_create": (i32, [P, P, i64, u32, i32, ctypes.POINTER(Interval), P,
                                ctypes.POINTER(P)]),
    "crop_pairs_create_sharded": (i32, [P, P, i64, u32, i32, ctypes.POINTER(Interval), u32, u32, P,
                                        ctypes.POINTER(P)]),
    "crop_pairs_create_ex": (i32, [P, P, i64, u32, i32, ctypes.POINTER(Interval), u32, u32, u32, P,
                                   ctypes.POINTER(P)]),
    "crop_pairs_own": (i32, [P, ctypes.POINTER(i32)]),
    "crop_pairs_info": (i32, [P, ctypes.POINTER(u64), ctypes.POINTER(u64), ctypes.POINTER(u64),
                              ctypes.POINTER(u64)]),
    "crop_pairs_own_terms": (i32, [P, ctypes.POINTER(u64)]),
    "crop_pairs_run": (i32, [P, P, P, P, P, P]),
    "crop_pairs_set_timing": (i32, [P, i32]),
    "crop_pairs_phase_ms": (i32, [P, ctypes.POINTER(ctypes.c_float)]),
    "crop_pairs_overflowed": (i32, [P, ctypes.POINTER(i32)]),
    "crop_pairs_mode": (i32, [P, ctypes.POINTER(i32)]),
    "crop_pairs_set_capacity": (i32, [P, u64]),
    "crop_fimi_parse": (i32, [ctypes.c_char_p, i32, ctypes.POINTER(P), ctypes.POINTER(i64),
                              ctypes.POINTER(i64), ctypes.POINTER(u32), ctypes.POINTER(i64),
                              ctypes.POINTER(i64)]),
    "crop_fimi_copy": (i32, [P, P, P]),
    "crop_fimi_free": (None, [P]),
    "crop_triple_parse": (i32, [ctypes.c_char_p, i32, ctypes.POINTER(P), P, ctypes.POINTER(i64),
                                ctypes.POINTER(i64), ctypes.POINTER(i64)]),
    "crop_triple_copy": (i32, [P, P, P, P]),
    "crop_triple_free": (None, [P]),
    "crop_pairs_set_topk": (i32, [P, P, P, P, u64]),
    "crop_topk_fused": (i32, [P, P, P, P, u64, u32, P, P, P, P, P, P]),
    "crop_bucket_topk": (i32, [P, P, P, P, u64, P, P, u32, u32, P, P, P, P]),
    "crop_pairs_destroy": (None, [P]),
    "crop_entry_bucket_stats": (i32, [P, P, P, P, u64, i32, u32, P, P, u32, P, P, P, P, P]),
    "crop_entry_buckets": (i32, [P, P, u64, P, P, u32, P, P]),
    "crop_entry_bucket_stats_f64": (i32, [P, P, P, P, u64, i32, u32, P, P, u32, P, P, P, P]),
    "crop_product_worker_loads": (i32, [P, P, P, P, i64, P, P, u32, u32, i32, P, P]),
    "crop_topk": (i32, [P, P, P, P, u64, u32, P, P, P]),
    "crop_outer_create": (i32, [P, P, P, P, P, P, i64, i32, ctypes.POINTER(Interval), P,
                                ctypes.POINTER(P)]),
    "crop_outer_create_ex": (i32, [P, P, P, P, P, P, i64, i32, ctypes.POINTER(Interval),
                                   ctypes.POINTER(OuterShape), P, ctypes.POINTER(P)]),
    "crop_outer_info": (i32, [P, ctypes.POINTER(u64), ctypes.POINTER(u64)]),
    "crop_outer_own_terms": (i32, [P, P, P]),
    "crop_outer_run": (i32, [P, P, P, P, P, P, P]),
    "crop_outer_destroy": (None, [P]),
    "crop_ss_index": (i32, [P, P, u64, P, u64, P, u64, P]),
    "crop_ss_keep": (i32, [P, P, u64, P, P, P, P, P, P, P, P, P, P]),
    "crop_ss_probe": (i32, [P, P, P, P, u64, P, u64, P, u64, u64, P, P, u32, u32, P, P, P, P, P, P, P, P, P]),
    "crop_ss_append": (i32, [P, P, P, P, u64, P, P, P, P, P, u32, P, P, P, P, P, P, P, P]),
    "crop_gen_lengths": (i32, [i64, u64, P, u32, u32, P, P]),
    "crop_gen_items": (i32, [i64, u64, u32, P, P, P, P, P]),
}

EXPORTED = tuple(_SIGS)

PAIRS_SAFE_UNITS = 1  # include/crop_b200.h CROP_PAIRS_SAFE_UNITS
PAIRS_NO_OWN = 2


def load(path: str = LIB_PATH):
    """Load (once) and type the native library; raises DeviceError if absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise DeviceError(
            f"native library {path} is missing: build it with "
            "`python -m paper_1210_0461_b200.build` (there is no CPU fallback)")
    lib = ctypes.CDLL(path)
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.crop_abi_version() != ABI_VERSION:
        raise DeviceError(f"ABI mismatch: library {lib.crop_abi_version()} != {ABI_VERSION}")
    _lib = lib
    return lib


_STATUS = {2: InputError, 3: ConfigError, 4: ResourceCapError, 5: DeviceError}


def check(status: int) -> None:
    if status == 0:
        return
    msg = load().crop_last_error().decode(errors="replace")
    raise _STATUS.get(status, CropError)(msg)


def call(name: str, *args) -> None:
    check(getattr(load(), name)(*args))


def require_cuda():
    """The CUDA device every product call runs on (fails loudly without one)."""
    import torch

    if not torch.cuda.is_available():
        raise DeviceError("no CUDA device visible: the CRoP B200 path has no CPU fallback")
    load()
    return torch.device("cuda", torch.cuda.current_device())


def stream_ptr(stream=None) -> int:
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


def ptr(t) -> int | None:
    return None if t is None else int(t.data_ptr())
