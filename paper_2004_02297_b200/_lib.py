"""ctypes binding of the in-tree C-ABI library `libadt.so` (include/adt.h).

There is no CPU fallback: if the library is missing, or no CUDA device is
present when a compute entry point is called, the call raises. Status codes
map to the reference's exception types (ValueError for a bad round_to,
codec.py:52-57) or RuntimeError for CUDA failures.
"""

from __future__ import annotations

import ctypes
import os
import threading

PKG = os.path.dirname(os.path.abspath(__file__))
# ADT_LIB may point at an in-tree build variant (scripts/build_variants.sh) for A/B runs.
LIB_PATH = os.environ.get("ADT_LIB") or os.path.join(PKG, "libadt.so")

ADT_OK = 0
ADT_ERR_ROUND_TO = -1
ADT_ERR_ALIGN = -2
ADT_ERR_ARG = -3
ADT_ERR_NO_DEVICE = -4
ADT_ERR_CUDA_BASE = -1000
TILE_WEIGHTS = 4096
ABI_VERSION = 11
H2D_DIRECT_FULL = 1      # adt_host_to_device_ex flags (include/adt.h)
H2D_SKIP_DIRECT_NORMS = 2
H2D_ZERO_COPY = 4
MAX_SOURCES = 16
PARTIALS_PER_TILE = 8

EXPORTS = ("adt_abi_version", "adt_strerror", "adt_partials_count", "adt_pack", "adt_norm_finalize",
           "adt_unpack", "adt_unpack_multi", "adt_unpack_multi_ex", "adt_copy_multi", "adt_peer_barrier", "adt_ipc_handle_bytes", "adt_ipc_get_handle",
           "adt_ipc_open", "adt_ipc_close", "adt_sumsq", "adt_sgd_pack", "adt_reduce_sgd_pack", "adt_pack_dyn", "adt_unpack_dyn", "adt_sgd_pack_dyn", "adt_reduce_sgd_pack_dyn",
           "adt_awp_observe", "adt_awp_fixup", "adt_unpack_multi_dyn", "adt_awp_combine", "adt_awp_fixup_pieces",
           "adt_awp_fixup_gather", "adt_device_sm_count", "adt_pack_host", "adt_host_to_device", "adt_host_threads",
           "adt_host_simd", "adt_sumsq_f64_partials", "adt_sumsq_f64", "adt_roundtrip", "adt_roundtrip_max_tiles",
           "adt_host_to_device_ring", "adt_host_to_device_ex")


class Segment(ctypes.Structure):
    """adt_segment (include/adt.h)."""

    _fields_ = [
        ("weights", ctypes.c_void_p),
        ("count", ctypes.c_uint64),
        ("offset", ctypes.c_uint64),
        ("round_to", ctypes.c_int32),
        ("reserved", ctypes.c_int32),
    ]


class SgdSegment(ctypes.Structure):
    """adt_sgd_segment (include/adt.h)."""

    _fields_ = [
        ("weights", ctypes.c_void_p),
        ("velocity", ctypes.c_void_p),
        ("grad", ctypes.c_void_p),
        ("count", ctypes.c_uint64),
        ("offset", ctypes.c_uint64),
        ("round_to", ctypes.c_int32),
        ("reserved", ctypes.c_int32),
    ]


class GradSegment(ctypes.Structure):
    """adt_grad_segment (include/adt.h)."""

    _fields_ = [
        ("weights", ctypes.c_void_p),
        ("velocity", ctypes.c_void_p),
        ("count", ctypes.c_uint64),
        ("offset", ctypes.c_uint64),
        ("grad_offset", ctypes.c_uint64),
        ("round_to", ctypes.c_int32),
        ("reserved", ctypes.c_int32),
    ]


class AwpConfig(ctypes.Structure):
    """adt_awp_config (include/adt.h)."""

    _fields_ = [("threshold", ctypes.c_double), ("interval", ctypes.c_int32), ("step_bits", ctypes.c_int32),
                ("max_bits", ctypes.c_int32), ("consecutive", ctypes.c_int32)]


class AwpGroup(ctypes.Structure):
    """adt_awp_group: one LayerPrecisionState (32 bytes, device memory)."""

    _fields_ = [("prev_norm", ctypes.c_double), ("last_delta", ctypes.c_double), ("bits", ctypes.c_int32),
                ("counter", ctypes.c_int32), ("has_prev", ctypes.c_int32), ("has_delta", ctypes.c_int32)]


class AwpRow(ctypes.Structure):
    """adt_awp_row: one trace row (40 bytes, device memory)."""

    _fields_ = [("norm", ctypes.c_double), ("delta", ctypes.c_double), ("batch", ctypes.c_int32),
                ("layer", ctypes.c_int32), ("counter", ctypes.c_int32), ("bits", ctypes.c_int32),
                ("has_delta", ctypes.c_int32), ("pad", ctypes.c_int32)]


class AwpDevice(ctypes.Structure):
    """adt_awp_device: device pointers of the on-GPU controller."""

    _fields_ = [("groups", ctypes.c_void_p), ("members", ctypes.c_void_p), ("member_start", ctypes.c_void_p),
                ("widths_in", ctypes.c_void_p), ("widths_out", ctypes.c_void_p), ("escalated", ctypes.c_void_p),
                ("ring", ctypes.c_void_p),
                ("counter", ctypes.c_void_p), ("nlayers", ctypes.c_int32), ("ngroups", ctypes.c_int32),
                ("ring_steps", ctypes.c_int32), ("reserved", ctypes.c_int32)]


class AdtError(RuntimeError):
    """A CUDA or argument failure reported by libadt."""

    def __init__(self, status: int, text: str):
        super().__init__(f"libadt status {status}: {text}")
        self.status = status


_lock = threading.Lock()
_lib = None


def load() -> ctypes.CDLL:
    """Load libadt.so once; raise loudly if it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build the sm_100a library first "
                "(python -m paper_2004_02297_b200._build, or __graft_entry__.build()). "
                "There is no CPU fallback.")
        lib = ctypes.CDLL(LIB_PATH)
        P = ctypes.POINTER
        seg_p = P(Segment)
        vp = ctypes.c_void_p
        lib.adt_abi_version.restype = ctypes.c_int
        lib.adt_abi_version.argtypes = []
        lib.adt_strerror.restype = ctypes.c_char_p
        lib.adt_strerror.argtypes = [ctypes.c_int]
        lib.adt_partials_count.restype = ctypes.c_int
        lib.adt_partials_count.argtypes = [seg_p, ctypes.c_int, P(ctypes.c_uint64)]
        lib.adt_norm_finalize.restype = ctypes.c_int
        lib.adt_norm_finalize.argtypes = [seg_p, ctypes.c_int, vp, vp, vp]
        lib.adt_pack.restype = ctypes.c_int
        lib.adt_pack.argtypes = [seg_p, ctypes.c_int, vp, vp, vp, vp]
        lib.adt_unpack.restype = ctypes.c_int
        lib.adt_unpack.argtypes = [seg_p, ctypes.c_int, vp, vp]
        lib.adt_unpack_multi_ex.restype = ctypes.c_int
        lib.adt_unpack_multi_ex.argtypes = [seg_p, ctypes.c_int, P(ctypes.c_void_p), ctypes.c_int, vp, ctypes.c_int, vp,
                                            vp]
        lib.adt_unpack_multi.restype = ctypes.c_int
        lib.adt_unpack_multi.argtypes = [seg_p, ctypes.c_int, P(ctypes.c_void_p), ctypes.c_int, vp]
        lib.adt_copy_multi.restype = ctypes.c_int
        lib.adt_copy_multi.argtypes = [vp, P(ctypes.c_void_p), ctypes.c_int, ctypes.c_uint64, ctypes.c_uint64, vp, vp]
        lib.adt_peer_barrier.restype = ctypes.c_int
        lib.adt_peer_barrier.argtypes = [P(ctypes.c_void_p), ctypes.c_int, ctypes.c_int, vp, ctypes.c_uint64, vp]
        lib.adt_ipc_handle_bytes.restype = ctypes.c_int
        lib.adt_ipc_handle_bytes.argtypes = []
        lib.adt_ipc_get_handle.restype = ctypes.c_int
        lib.adt_ipc_get_handle.argtypes = [vp, vp, P(ctypes.c_uint64)]
        lib.adt_ipc_open.restype = ctypes.c_int
        lib.adt_ipc_open.argtypes = [vp, P(ctypes.c_void_p)]
        lib.adt_ipc_close.restype = ctypes.c_int
        lib.adt_ipc_close.argtypes = [vp]
        lib.adt_sgd_pack.restype = ctypes.c_int
        lib.adt_sgd_pack.argtypes = [P(SgdSegment), ctypes.c_int, ctypes.c_float, ctypes.c_float, ctypes.c_float,
                                     vp, vp, vp, vp]
        lib.adt_reduce_sgd_pack.restype = ctypes.c_int
        lib.adt_reduce_sgd_pack.argtypes = [P(GradSegment), ctypes.c_int, P(ctypes.c_void_p), P(ctypes.c_int64),
                                            ctypes.c_int, ctypes.c_float, ctypes.c_float, ctypes.c_float,
                                            vp, vp, vp, vp, vp]
        lib.adt_pack_dyn.restype = ctypes.c_int
        lib.adt_pack_dyn.argtypes = [seg_p, ctypes.c_int, vp, vp, vp, vp]
        lib.adt_unpack_dyn.restype = ctypes.c_int
        lib.adt_unpack_dyn.argtypes = [seg_p, ctypes.c_int, vp, vp, vp]
        lib.adt_sgd_pack_dyn.restype = ctypes.c_int
        lib.adt_sgd_pack_dyn.argtypes = [P(SgdSegment), ctypes.c_int, ctypes.c_float, ctypes.c_float, ctypes.c_float,
                                         vp, vp, vp, vp]
        lib.adt_reduce_sgd_pack_dyn.restype = ctypes.c_int
        lib.adt_reduce_sgd_pack_dyn.argtypes = [P(GradSegment), ctypes.c_int, P(ctypes.c_void_p), P(ctypes.c_int64),
                                                ctypes.c_int, ctypes.c_float, ctypes.c_float, ctypes.c_float,
                                                vp, vp, vp, vp, vp]
        lib.adt_awp_observe.restype = ctypes.c_int
        lib.adt_awp_observe.argtypes = [vp, P(AwpDevice), P(AwpConfig), vp, vp]
        lib.adt_awp_fixup.restype = ctypes.c_int
        lib.adt_awp_fixup.argtypes = [seg_p, seg_p, ctypes.c_int, vp, vp, vp, vp]
        lib.adt_unpack_multi_dyn.restype = ctypes.c_int
        lib.adt_unpack_multi_dyn.argtypes = [seg_p, ctypes.c_int, P(ctypes.c_void_p), ctypes.c_int, vp, vp, vp]
        lib.adt_awp_combine.restype = ctypes.c_int
        lib.adt_awp_combine.argtypes = [vp, ctypes.c_int, vp, ctypes.c_int, vp, vp, vp]
        lib.adt_awp_fixup_pieces.restype = ctypes.c_int
        lib.adt_awp_fixup_pieces.argtypes = [seg_p, seg_p, ctypes.c_int, P(ctypes.c_int32), vp, vp, vp, vp, vp]
        lib.adt_awp_fixup_gather.restype = ctypes.c_int
        lib.adt_awp_fixup_gather.argtypes = [seg_p, ctypes.c_int, P(ctypes.c_int32), P(ctypes.c_void_p), ctypes.c_int,
                                             vp, vp, vp, vp]
        lib.adt_sumsq.restype = ctypes.c_int
        lib.adt_sumsq.argtypes = [seg_p, ctypes.c_int, vp, vp, vp]
        lib.adt_device_sm_count.restype = ctypes.c_int
        lib.adt_device_sm_count.argtypes = [P(ctypes.c_int)]
        lib.adt_pack_host.restype = ctypes.c_int
        lib.adt_pack_host.argtypes = [seg_p, ctypes.c_int, vp, vp, ctypes.c_int]
        lib.adt_host_to_device.restype = ctypes.c_int
        lib.adt_host_to_device.argtypes = [seg_p, seg_p, ctypes.c_int, vp, vp, ctypes.c_uint64, vp, ctypes.c_int,
                                           ctypes.c_uint64, vp]
        lib.adt_host_to_device_ring.restype = ctypes.c_int
        lib.adt_host_to_device_ring.argtypes = [seg_p, seg_p, ctypes.c_int, vp, ctypes.c_uint64, ctypes.c_uint64, vp,
                                                ctypes.c_uint64, vp, ctypes.c_int, vp]
        lib.adt_host_to_device_ex.restype = ctypes.c_int
        lib.adt_host_to_device_ex.argtypes = [seg_p, seg_p, ctypes.c_int, vp, vp, ctypes.c_uint64, vp, ctypes.c_int,
                                              ctypes.c_uint64, ctypes.c_uint32, vp, vp]
        lib.adt_host_threads.restype = ctypes.c_int
        lib.adt_host_threads.argtypes = [P(ctypes.c_int)]
        lib.adt_host_simd.restype = ctypes.c_int
        lib.adt_host_simd.argtypes = []
        lib.adt_sumsq_f64_partials.restype = ctypes.c_int
        lib.adt_sumsq_f64_partials.argtypes = [ctypes.c_uint64, P(ctypes.c_uint64)]
        lib.adt_roundtrip.restype = ctypes.c_int
        lib.adt_roundtrip.argtypes = [seg_p, seg_p, ctypes.c_int, vp, vp, vp, vp, vp]
        lib.adt_roundtrip_max_tiles.restype = ctypes.c_int
        lib.adt_roundtrip_max_tiles.argtypes = [P(ctypes.c_int)]
        lib.adt_sumsq_f64.restype = ctypes.c_int
        lib.adt_sumsq_f64.argtypes = [vp, ctypes.c_uint64, vp, vp, vp]
        if lib.adt_abi_version() != ABI_VERSION:
            raise ImportError(f"libadt ABI {lib.adt_abi_version()} != expected {ABI_VERSION}; rebuild")
        _lib = lib
        return lib


def strerror(status: int) -> str:
    return load().adt_strerror(status).decode()


def check(status: int) -> None:
    """Map a libadt status to the reference's exception types."""
    if status == ADT_OK:
        return
    text = strerror(status)
    if status == ADT_ERR_ROUND_TO:
        raise ValueError(text)
    raise AdtError(status, text)


def segment_array(segs) -> ctypes.Array:
    """[(ptr, count, offset, round_to[, source]), ...] -> adt_segment[]."""
    arr = (Segment * max(1, len(segs)))()
    for i, seg in enumerate(segs):
        ptr, count, offset, r = seg[:4]
        arr[i].weights = ptr
        arr[i].count = count
        arr[i].offset = offset
        arr[i].round_to = r
        arr[i].reserved = seg[4] if len(seg) > 4 else 0
    return arr


def pointer_array(ptrs) -> ctypes.Array:
    arr = (ctypes.c_void_p * max(1, len(ptrs)))()
    for i, p in enumerate(ptrs):
        arr[i] = p
    return arr


def partials_count(seg_arr, nseg: int) -> int:
    out = ctypes.c_uint64(0)
    check(load().adt_partials_count(seg_arr, nseg, ctypes.byref(out)))
    return int(out.value)
