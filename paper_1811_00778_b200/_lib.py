"""ctypes binding of libhcnn_b200.so (include/hcnn_b200.h).

There is no fallback: if the library is missing or cannot be loaded the
import of any GPU entry point fails loudly.
"""

from __future__ import annotations

import ctypes as C
import os

from .errors import STATUS, BackendError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libhcnn_b200.so")

_lib = None

_SIGS = {
    "hcnn_ctx_create": (C.c_int, [C.POINTER(C.c_void_p), C.c_uint32, C.c_uint32,
                                  C.POINTER(C.c_uint64), C.c_uint64, C.c_uint32, C.c_int]),
    "hcnn_ctx_destroy": (C.c_int, [C.c_void_p]),
    "hcnn_ctx_set_stream": (C.c_int, [C.c_void_p, C.c_void_p]),
    "hcnn_ctx_query": (C.c_int64, [C.c_void_p, C.c_int]),
    "hcnn_ctx_prime": (C.c_uint64, [C.c_void_p, C.c_int, C.POINTER(C.c_uint64)]),
    "hcnn_ctx_set_option": (C.c_int, [C.c_void_p, C.c_int, C.c_int64]),
    "hcnn_ctx_set_workspace_limit": (C.c_int, [C.c_void_p, C.c_size_t]),
    "hcnn_set_relin_key": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int]),
    "hcnn_set_public_key": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int]),
    "hcnn_encrypt": (C.c_int, [C.c_void_p] + [C.c_void_p] * 5 + [C.c_size_t]),
    "hcnn_encrypt_device_msg": (C.c_int, [C.c_void_p] + [C.c_void_p] * 5 + [C.c_size_t]),
    "hcnn_codec_create": (C.c_int, [C.c_uint64, C.c_uint32, C.c_int, C.POINTER(C.c_void_p)]),
    "hcnn_codec_destroy": (C.c_int, [C.c_void_p]),
    "hcnn_codec_encode": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p]),
    "hcnn_codec_decode": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p]),
    "hcnn_ntt64": (C.c_int, [C.c_void_p, C.c_void_p, C.c_size_t, C.c_int, C.c_void_p]),
    "hcnn_set_secret_key": (C.c_int, [C.c_void_p, C.c_void_p]),
    "hcnn_decrypt": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t]),
    "hcnn_alloc": (C.c_int, [C.c_void_p, C.c_size_t, C.POINTER(C.c_void_p)]),
    "hcnn_free": (C.c_int, [C.c_void_p, C.c_void_p]),
    "hcnn_upload_u64": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t]),
    "hcnn_download_u64": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t]),
    "hcnn_sync": (C.c_int, [C.c_void_p]),
    "hcnn_weights_create": (C.c_int, [C.c_void_p, C.c_void_p, C.c_size_t, C.POINTER(C.c_void_p)]),
    "hcnn_weights_destroy": (C.c_int, [C.c_void_p, C.c_void_p]),
    "hcnn_conv": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p] + [C.c_int] * 3
                  + [C.c_void_p] + [C.c_int] * 7),
    "hcnn_fc": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_void_p]),
    "hcnn_pool": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p] + [C.c_int] * 6),
    "hcnn_square": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t]),
    "hcnn_hmult_raw": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t]),
    "hcnn_hmult": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t]),
    "hcnn_relinearize": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t]),
    "hcnn_keygen": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "hcnn_hfir_pack": (C.c_int, [C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p]),
    "hcnn_hfir_unpack": (C.c_int, [C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p]),
    "hcnn_mul_plain": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t]),
    "hcnn_hadd": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t]),
    "hcnn_ntt": (C.c_int, [C.c_void_p, C.c_void_p, C.c_size_t, C.c_uint32, C.c_uint32, C.c_int]),
    "hcnn_release_memory": (C.c_int, [C.c_int]),
    "hcnn_crt_combine": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_size_t, C.c_void_p, C.c_int, C.c_void_p,
                                    C.c_int, C.c_void_p]),
    "hcnn_host_narrow": (C.c_int, [C.c_void_p, C.c_size_t, C.c_size_t, C.c_void_p, C.c_int]),
    "hcnn_host_widen": (C.c_int, [C.c_void_p, C.c_size_t, C.c_size_t, C.c_void_p, C.c_int]),
    "hcnn_profile": (C.c_int, [C.c_void_p, C.c_int]),
    "hcnn_profile_dump": (C.c_int64, [C.c_void_p, C.c_char_p, C.c_size_t]),
    "hcnn_int_peak": (C.c_int, [C.c_int, C.c_int, C.POINTER(C.c_double)]),
    "hcnn_last_error": (C.c_char_p, []),
    "hcnn_version": (C.c_char_p, []),
}

EXPORTED = tuple(_SIGS)


def lib():
    """The loaded library (raises BackendError if it is not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise BackendError(
                f"{LIB_PATH} not built: run `python -m paper_1811_00778_b200.build`"
            )
        handle = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _lib = handle
    return _lib


def check(status: int, what: str = ""):
    if status != 0:
        msg = lib().hcnn_last_error().decode(errors="replace")
        cls = STATUS.get(status, BackendError)
        raise cls(f"{what}: {msg}" if what else msg)
