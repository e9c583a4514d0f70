"""ctypes binding of the in-tree sm_100a library ``_lib/libck32b200.so``.

This is the only way the package computes: there is no CPU or PyTorch
fallback.  If the shared library is missing or cannot be loaded the import
fails loudly.
"""
from __future__ import annotations

import ctypes
import os
from pathlib import Path

PKG = Path(__file__).resolve().parent
LIB_PATH = PKG / "_lib" / "libck32b200.so"

CK_OK, CK_INVALID_ARGUMENT, CK_RUNTIME_ERROR, CK_CUDA_ERROR = 0, 1, 2, 3


class CkCudaError(RuntimeError):
    pass


class ck_prof_stat(ctypes.Structure):
    _fields_ = [("name", ctypes.c_char * 16), ("groups", ctypes.c_uint64), ("launches", ctypes.c_uint64),
                ("ms", ctypes.c_double), ("bytes", ctypes.c_double)]


class ck_params(ctypes.Structure):
    _fields_ = [("n", ctypes.c_uint32), ("l", ctypes.c_uint32), ("alpha", ctypes.c_uint32),
                ("delta_bits", ctypes.c_uint32), ("lazy_rescale", ctypes.c_int32)]


_vp = ctypes.c_void_p
_u32 = ctypes.c_uint32
_i64 = ctypes.c_int64
_u32p = ctypes.POINTER(ctypes.c_uint32)

# name -> argtypes (restype is ck_status = int unless noted)
_SIGS = {
    "ck_context_create": [ctypes.POINTER(ck_params), _u32p, ctypes.c_int, ctypes.POINTER(_vp)],
    "ck_context_destroy": [_vp],
    "ck_generate_basis": [_u32, _u32, _u32, _u32, _u32p],
    "ck_context_primes": [_vp, _u32p],
    "ck_context_counters": [_vp, ctypes.POINTER(ctypes.c_uint64)],
    "ck_context_reset_counters": [_vp],
    "ck_malloc": [_vp, ctypes.c_size_t, ctypes.POINTER(_vp)],
    "ck_free": [_vp, _vp],
    "ck_memcpy_h2d": [_vp, _vp, _vp, ctypes.c_size_t, _vp],
    "ck_memcpy_d2h": [_vp, _vp, _vp, ctypes.c_size_t, _vp],
    "ck_memcpy_d2d": [_vp, _vp, _vp, ctypes.c_size_t, _vp],
    "ck_stream_sync": [_vp, _vp],
    "ck_stream_create": [_vp, ctypes.POINTER(_vp)],
    "ck_stream_destroy": [_vp, _vp],
    "ck_profile": [_vp, ctypes.c_int],
    "ck_profile_read": [_vp, ctypes.POINTER(ck_prof_stat), _u32, ctypes.POINTER(ctypes.c_uint32)],
    "ck_ntt_forward": [_vp, _vp, _u32, _u32p, _vp],
    "ck_intt_inverse": [_vp, _vp, _u32, _u32p, _u32p, _vp],
    "ck_bconv": [_vp, _vp, _u32, _u32p, _vp, _u32, _u32p, _vp],
    "ck_mod_switch": [_vp, _vp, _u32, _u32p, _vp, _u32, _u32, _vp],
    "ck_automorphism": [_vp, _vp, _vp, _u32, _i64, _vp],
    "ck_automorphism_galois": [_vp, _vp, _vp, _u32, _u32, ctypes.c_uint64, ctypes.c_int, _vp],
    "ck_ew_binary": [_vp, ctypes.c_int, _vp, _vp, _vp, _u32, _u32, _vp],
    "ck_ew_mul_const": [_vp, _vp, _u32p, _vp, _u32, _u32, _vp],
    "ck_ew_mul_const_raw": [_vp, _vp, _u32p, _vp, _u32, _u32, _vp],
    "ck_ntt_forward_raw": [_vp, _vp, _u32, _u32p, _vp],
    "ck_intt_inverse_raw": [_vp, _vp, _u32, _u32p, _u32p, _vp],
    "ck_bconv_table": [_vp, _vp, _u32, _u32p, _vp, _u32, _u32p, ctypes.POINTER(ctypes.c_int32), _vp],
    "ck_ew_add": [_vp, _vp, _vp, _vp, _u32, _vp],
    "ck_ew_sub": [_vp, _vp, _vp, _vp, _u32, _vp],
    "ck_ew_mul": [_vp, _vp, _vp, _vp, _u32, _vp],
    "ck_mod_up": [_vp, _u32, _vp, _vp, _vp],
    "ck_key_mult": [_vp, _u32, _vp, _vp, _vp, _vp],
    "ck_mod_down": [_vp, _u32, _vp, _vp, _vp],
    "ck_key_switch": [_vp, _u32, _vp, _vp, _vp, _vp],
    "ck_rescale": [_vp, _u32, _u32, _vp, _vp, _vp],
    "ck_hmult": [_vp, _u32, _u32, _vp, _vp, _vp, _vp, _vp],
    "ck_hrot": [_vp, _u32, _u32, _vp, _i64, _vp, _vp, _vp],
    "ck_hadd": [_vp, _u32, _u32, _vp, _vp, _vp, _vp],
    "ck_padd": [_vp, _u32, _u32, _vp, _vp, _vp, _vp],
    "ck_pmult": [_vp, _u32, _u32, _vp, _vp, _vp, _vp],
    "ck_hoisted_rotations": [_vp, _u32, _vp, _u32, ctypes.POINTER(_i64), ctypes.POINTER(_vp), _vp, _vp],
    "ck_hoisted_rotate_accumulate": [_vp, _u32, _vp, _u32, ctypes.POINTER(_i64), ctypes.POINTER(_vp),
                                     ctypes.POINTER(_vp), _vp, _vp],
    "ck_encode": [_vp, _vp, _u32, ctypes.c_double, _u32, ctypes.c_int, _vp, _vp],
    "ck_decode": [_vp, _vp, _u32, ctypes.c_double, _vp, _vp],
    "ck_decode_rational": [_vp, _vp, _u32, ctypes.c_double, _vp, _u32, _vp, _u32, _vp, _vp],
    "ck_decrypt": [_vp, _u32, _u32, _vp, _vp, _vp, _vp],
    "ck_encrypt_sk": [_vp, _u32, _vp, _vp, _vp, _vp, _vp, _vp],
    "ck_encrypt_pk": [_vp, _u32, _vp, _vp, _vp, _vp, _vp, _vp, _vp],
    "ck_evk_digit": [_vp, _vp, _vp, _vp, _vp, _u32p, ctypes.c_int, _vp, _vp],
    "ck_coeffs_to_eval": [_vp, _vp, _u32, _u32, _vp, _vp],
    "ck_shard_create": [_vp, _u32, _u32, ctypes.POINTER(_vp)],
    "ck_shard_destroy": [_vp],
    "ck_shard_layout": [_vp, _u32, _u32p],
    "ck_shard_modup_begin": [_vp, _u32, _vp, _vp, _vp],
    "ck_shard_modup_keymult": [_vp, _u32, _vp, _vp, _vp, _vp, _vp, _vp],
    "ck_shard_switch_begin": [_vp, ctypes.c_int, _u32, _vp, _vp, _vp],
    "ck_shard_switch_end": [_vp, ctypes.c_int, _u32, _vp, _vp, _vp, _u32, ctypes.c_int32, _i64, _vp, _vp],
    "ck_shard_tensor": [_vp, _u32, _vp, _vp, _vp, _vp, _vp],
    "ck_rng_create": [ctypes.c_uint64, ctypes.POINTER(_vp)],
    "ck_rng_destroy": [_vp],
    "ck_rng_draws": [_vp, ctypes.c_uint64, _vp],
    "ck_sample_gaussian": [_vp, _u32, ctypes.c_double, _vp],
    "ck_sample_ternary": [_vp, _u32, _u32, _vp],
    "ck_sample_uniform": [_vp, _vp, _u32, _u32, _vp],
    "ck_shard_exchange_buffer": [_vp, ctypes.POINTER(_vp), ctypes.POINTER(ctypes.c_uint64)],
    "ck_shard_set_peers": [_vp, ctypes.POINTER(ctypes.c_uint64), _u32],
    "ck_shard_set_timeout": [_vp, ctypes.c_uint64],
    "ck_shard_peer_error": [_vp, _u32p],
    "ck_ipc_get_handle": [_vp, ctypes.POINTER(ctypes.c_ubyte)],
    "ck_ipc_open_handle": [ctypes.POINTER(ctypes.c_ubyte), ctypes.POINTER(_vp)],
    "ck_ipc_close": [_vp],
    "ck_context_params": [_vp, ctypes.POINTER(ck_params)],
    "ck_serialize_basis": [_vp, _vp, ctypes.c_size_t, ctypes.POINTER(ctypes.c_size_t)],
    "ck_deserialize_basis": [_vp, ctypes.c_size_t, ctypes.POINTER(ck_params), _u32p, _u32],
    "ck_serialize_poly": [_vp, _vp, _u32, _u32, ctypes.c_int, ctypes.c_int, _vp, ctypes.c_size_t,
                          ctypes.POINTER(ctypes.c_size_t), _vp],
    "ck_deserialize_poly": [_vp, _vp, ctypes.c_size_t, _vp, _u32, _u32p, _vp],
    "ck_serialize_ciphertext": [_vp, _vp, _u32, ctypes.c_int, _vp, ctypes.c_size_t, _vp, ctypes.c_size_t, _vp,
                                ctypes.c_size_t, ctypes.POINTER(ctypes.c_size_t), _vp],
    "ck_deserialize_ciphertext": [_vp, _vp, ctypes.c_size_t, _vp, _u32, _u32p, ctypes.POINTER(ctypes.c_int), _vp,
                                  ctypes.c_size_t, ctypes.POINTER(ctypes.c_size_t), _vp, ctypes.c_size_t,
                                  ctypes.POINTER(ctypes.c_size_t), _vp],
    "ck_serialize_evk": [_vp, _vp, _u32, ctypes.c_int, _i64, _vp, ctypes.c_size_t, ctypes.POINTER(ctypes.c_size_t),
                         _vp],
    "ck_deserialize_evk": [_vp, _vp, ctypes.c_size_t, _vp, _u32, ctypes.POINTER(ctypes.c_int),
                           ctypes.POINTER(_i64), _u32p, _vp],
}
EXPORTS = sorted(list(_SIGS) + ["ck_last_error", "ck_version", "ck_launch_count"])

_lib = None


def lib():
    """Load (once) and return the native library; raises if it is absent."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise ImportError(f"{LIB_PATH} is not built; run `make -C {PKG}` (or __graft_entry__.build())")
        L = ctypes.CDLL(str(LIB_PATH), mode=os.RTLD_GLOBAL if hasattr(os, "RTLD_GLOBAL") else 0)
        for name, args in _SIGS.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = ctypes.c_int
        L.ck_last_error.restype = ctypes.c_char_p
        L.ck_version.restype = ctypes.c_char_p
        L.ck_launch_count.restype = ctypes.c_uint64
        L.ck_launch_count.argtypes = [_vp]
        _lib = L
    return _lib


def check(status: int) -> None:
    if status == CK_OK:
        return
    msg = lib().ck_last_error().decode()
    if status == CK_INVALID_ARGUMENT:
        raise ValueError(msg)  # std::invalid_argument in the reference
    if status == CK_CUDA_ERROR:
        raise CkCudaError(msg)
    raise RuntimeError(msg)


def call(name: str, *args) -> None:
    check(getattr(lib(), name)(*args))


def u32_array(values):
    vals = [int(v) for v in values]
    return (ctypes.c_uint32 * max(len(vals), 1))(*vals)
