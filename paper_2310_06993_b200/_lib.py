"""ctypes binding of liboptr.so (the C ABI declared in include/optr.h).

The product path has no CPU fallback: importing a device entry point without
the built library raises immediately (build it with
``python -c "import __graft_entry__ as g; g.build()"``).
"""

from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("OPTR_LIB") or os.path.join(_HERE, "liboptr.so")

OPTR_OK = 0
OPTR_EINVAL = 1
OPTR_EEMPTY = 2
OPTR_ECUDA = 3
OPTR_ENOMEM = 4

OPTR_F32 = 0
OPTR_BF16 = 1

OPTR_MASK_NONE = 0
OPTR_MASK_COIN = 1
OPTR_MASK_BITMAP = 2

MAX_WORKERS = 16

# kernel classes of optr_timing_collect (optr.h OPTR_K_*)
K_NAMES = ["prep", "enc_first", "enc_mid", "enc_last", "aggregate", "dec_first", "dec_mid",
           "dec_last", "assemble", "barrier", "other", "enc_mean", "fused", "small"]


class optr_mask_spec(ctypes.Structure):
    _fields_ = [
        ("kind", ctypes.c_int32),
        ("epp", ctypes.c_int32),
        ("seed", ctypes.c_uint64),
        ("drop_prob", ctypes.c_double),
        ("bitmap", ctypes.c_void_p),
        ("stream_offsets", ctypes.c_void_p),
    ]


# every symbol include/optr.h declares: name -> (restype, argtypes)
_vp = ctypes.c_void_p
_i64 = ctypes.c_int64
_u64 = ctypes.c_uint64
_int = ctypes.c_int
SIGNATURES = {
    "optr_derive_seed": (_u64, [_u64, _u64, _u64]),
    "optr_pcg64_output": (_u64, [ctypes.POINTER(_u64), _int, _u64]),
    "optr_next_pow2": (_i64, [_i64]),
    "optr_mask_words": (_i64, [_i64, _int, _int]),
    "optr_masks_host": (_int, [_vp, _i64, _int, _int, _u64, ctypes.c_double, _int]),
    "optr_version": (ctypes.c_char_p, []),
    "optr_coin_packets": (_int, [_u64, _int, _u64, _i64, ctypes.c_double, _vp]),
    "optr_mean_received": (_int, [_vp, _vp, _vp, _int, _int, _i64, _vp, _vp]),
    "optr_ring_cast": (_int, [_vp, _i64, _vp, _vp]),
    "optr_ring_step": (_int, [_vp, _vp, _vp, _i64, _int, _vp]),
    "optr_ring_finish": (_int, [_vp, _int, _i64, _vp, _vp]),
    "optr_packetize": (_int, [_vp, _i64, _int, ctypes.c_uint32, _int, _int, _int, _vp, _i64, _vp]),
    "optr_depacketize": (_int, [_vp, _i64, _i64, _vp, _int, ctypes.c_uint32, _int, _vp, _vp, _i64, _vp, _vp]),
    "optr_rht_signs": (_int, [_vp, _i64, _u64, _vp]),
    "optr_fwht": (_int, [_vp, _i64, _vp]),
    "optr_rht_encode": (_int, [_vp, _int, _i64, _vp, _i64, _u64, _vp]),
    "optr_rht_decode": (_int, [_vp, _vp, _i64, _i64, _u64, _vp, _int, _vp]),
    "optr_fwht_f64": (_int, [_vp, _i64, _vp]),
    "optr_rht_encode_f64": (_int, [_vp, _i64, _vp, _i64, _u64, _vp]),
    "optr_rht_decode_f64": (_int, [_vp, _vp, _i64, _i64, _u64, _vp, _vp]),
    "optr_tar_local_workspace": (ctypes.c_size_t, [_int, _i64, _int, _int]),
    "optr_tar_local": (_int, [ctypes.POINTER(_vp), ctypes.POINTER(_vp), _int, _i64, _int, _int, _u64,
                              _u64, _u64, _int, _int, ctypes.POINTER(optr_mask_spec), _vp,
                              ctypes.c_size_t, _vp, _vp, _vp]),
    "optr_tar_local_async": (_int, [ctypes.POINTER(_vp), ctypes.POINTER(_vp), _int, _i64, _int, _int, _u64,
                                    _u64, _u64, _int, _int, ctypes.POINTER(optr_mask_spec), _vp,
                                    ctypes.c_size_t, _vp, _vp, _int, _vp]),
    "optr_local_join": (_int, [_vp]),
    "optr_comm_create": (_int, [ctypes.POINTER(_vp), _int, _int, _int, _i64, _int]),
    "optr_comm_handle_bytes": (ctypes.c_size_t, []),
    "optr_comm_get_handle": (_int, [_vp, _vp]),
    "optr_comm_open": (_int, [_vp, _vp]),
    "optr_comm_destroy": (_int, [_vp]),
    "optr_tar": (_int, [_vp, _vp, _vp, _i64, _int, _int, _u64, _u64, _u64, _int, _int,
                        ctypes.POINTER(optr_mask_spec), _vp, _vp]),
    "optr_comm_barrier": (_int, [_vp, _vp]),
    "optr_comm_set_fused_grid": (_int, [_vp, _int]),
    "optr_tar_async": (_int, [_vp, _vp, _vp, _i64, _int, _int, _u64, _u64, _u64, _int, _int,
                              ctypes.POINTER(optr_mask_spec), _vp, _vp]),
    "optr_comm_join": (_int, [_vp, _vp]),
    "optr_tar_bounded": (_int, [_vp, _vp, _vp, _i64, _int, _int, _u64, _u64, _u64, _int, _int,
                                ctypes.POINTER(optr_mask_spec), _u64, _vp, _vp, _int, _vp]),
    "optr_fused_unit_entries": (_i64, [_i64, _int]),
    "optr_timing_enable": (_int, [_int]),
    "optr_timing_collect": (_int, [ctypes.POINTER(ctypes.c_double), ctypes.POINTER(_i64), ctypes.POINTER(_i64)]),
    "optr_launch_count": (_i64, []),
    "optr_debug_trace": (_int, [_vp, _i64]),
    "optr_probe_enable_peer": (_int, [_int, _int]),
    "optr_probe_copy": (_int, [_vp, _vp, _i64, _int, _int, _vp]),
}

_lib = None


class LibraryMissing(RuntimeError):
    pass


def lib():
    """Load liboptr.so once; raise loudly if it was not built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise LibraryMissing(
                f"{LIB_PATH} not found: the CUDA library is required (no CPU fallback). "
                "Build it with __graft_entry__.build()."
            )
        l = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            f = getattr(l, name)
            f.restype = res
            f.argtypes = args
        _lib = l
    return _lib


class EmptyReceptionError(RuntimeError):
    """Nothing arrived; the caller should consult the safeguards policy
    (hadamard.py:17-18)."""


def check(rc: int, what: str = "optr") -> None:
    if rc == OPTR_OK:
        return
    if rc == OPTR_EINVAL:
        raise ValueError(f"{what}: invalid argument")
    if rc == OPTR_EEMPTY:
        raise EmptyReceptionError("no transformed entries received")
    raise RuntimeError(f"{what}: CUDA error (status {rc})")


def timing_enable(on: bool) -> None:
    lib().optr_timing_enable(1 if on else 0)


def timing_collect() -> dict:
    """{class name: (total_ms, launches, worker_passes)} since the last collect."""
    ms = (ctypes.c_double * len(K_NAMES))()
    cnt = (ctypes.c_int64 * len(K_NAMES))()
    units = (ctypes.c_int64 * len(K_NAMES))()
    check(lib().optr_timing_collect(ms, cnt, units), "timing_collect")
    return {k: (ms[i], cnt[i], units[i]) for i, k in enumerate(K_NAMES)}


def launch_count() -> int:
    return int(lib().optr_launch_count())
