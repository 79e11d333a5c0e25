"""ctypes binding of libhrt_b200.so (the C ABI declared in include/hrt_b200.h).

The shared library is built in-tree (`python -m paper_2212_01543_b200.build`
or `__graft_entry__.build()`); there is no CPU fallback: if the library or a
GPU is missing, every engine entry point raises.
"""

from __future__ import annotations

import ctypes as C
import os

LIB_NAME = "libhrt_b200.so"
LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), LIB_NAME)

HRT_OK, HRT_ERR_INVALID, HRT_ERR_INFERENCE, HRT_ERR_DECODING, HRT_ERR_MEMORY, HRT_ERR_CUDA = range(6)
HRT_DTYPE_F32, HRT_DTYPE_BF16 = 0, 1

# every symbol include/hrt_b200.h declares
EXPORTED = (
    "hrt_create", "hrt_destroy", "hrt_param_count", "hrt_estimate_arena", "hrt_last_error", "hrt_get_stats", "hrt_stream",
    "hrt_synchronize", "hrt_encode", "hrt_start_cache", "hrt_step", "hrt_reorder", "hrt_parallel_logits",
    "hrt_argmax_logprobs", "hrt_translate_batch", "hrt_at_translate_batch", "hrt_set_option", "hrt_phase_times", "hrt_timing_enable",
    "hrt_timing_report", "hrt_timing_read",
)


class HrtConfig(C.Structure):
    _fields_ = [(n, C.c_int32) for n in (
        "d_model", "d_ff", "n_heads", "enc_layers", "dec_layers", "vocab_size", "max_len",
        "max_chunk", "dtype", "max_sentences", "max_beam", "max_src_tokens")]


class HrtStats(C.Structure):
    _fields_ = [(n, C.c_int64) for n in (
        "kernel_launches", "decoder_calls", "arena_bytes", "arena_high_water", "weight_bytes",
        "stage1_row_steps")]


class HrtTranslateOut(C.Structure):
    _fields_ = [("tokens", C.c_void_p), ("lens", C.c_void_p), ("scores", C.c_void_p),
                ("calls", C.c_void_p), ("forced", C.c_void_p)]


_lib = None


class LibraryMissing(RuntimeError):
    pass


def load(path: str | None = None):
    """Load (once) and type the shared library."""
    global _lib
    if _lib is not None:
        return _lib
    p = path or LIB_PATH
    if not os.path.exists(p):
        raise LibraryMissing(
            f"{p} is not built; run `python -m paper_2212_01543_b200.build` (no CPU fallback exists)")
    lib = C.CDLL(p)
    vp, i32, i64, f32p, i32p = C.c_void_p, C.c_int32, C.c_int64, C.POINTER(C.c_float), C.POINTER(C.c_int32)
    sig = {
        "hrt_create": ([C.POINTER(HrtConfig), f32p, i64, i32, C.POINTER(vp)], C.c_int),
        "hrt_destroy": ([vp], None),
        "hrt_param_count": ([C.POINTER(HrtConfig)], i64),
        "hrt_estimate_arena": ([C.POINTER(HrtConfig), C.POINTER(C.c_int64)], C.c_int),
        "hrt_last_error": ([vp], C.c_char_p),
        "hrt_get_stats": ([vp, C.POINTER(HrtStats)], C.c_int),
        "hrt_stream": ([vp], vp),
        "hrt_synchronize": ([vp], C.c_int),
        "hrt_encode": ([vp, i32p, i32p, i32, f32p], C.c_int),
        "hrt_start_cache": ([vp, i32, i32, i32p], C.c_int),
        "hrt_step": ([vp, i32p, i32, f32p], C.c_int),
        "hrt_reorder": ([vp, i32p], C.c_int),
        "hrt_parallel_logits": ([vp, i32p, i32p, C.POINTER(C.c_uint8), i32, i32, i32, i32p, f32p], C.c_int),
        "hrt_argmax_logprobs": ([vp, i32p, i32, i32p, f32p], C.c_int),
        "hrt_translate_batch": ([vp, vp, i32p, i32, i32, i32, i32, C.c_float, i32p,
                                 C.POINTER(HrtTranslateOut), i32], C.c_int),
        "hrt_at_translate_batch": ([vp, vp, i32p, i32, i32, C.c_float, i32p, C.POINTER(HrtTranslateOut), i32],
                                   C.c_int),
        "hrt_set_option": ([vp, C.c_char_p, i32], C.c_int),
        "hrt_phase_times": ([vp, f32p], C.c_int),
        "hrt_timing_report": ([vp, C.c_char_p, i64], C.c_int),
        "hrt_timing_enable": ([vp, C.c_char_p, i32], C.c_int),
        "hrt_timing_read": ([vp, C.POINTER(C.c_double), C.POINTER(C.c_int64), C.POINTER(C.c_double),
                             C.POINTER(C.c_double)], C.c_int),
    }
    for name, (args, res) in sig.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    _lib = lib
    return lib


def exported_symbols(path: str | None = None):
    """Names from EXPORTED that the library actually exports (no GPU needed)."""
    lib = C.CDLL(path or LIB_PATH)
    return [n for n in EXPORTED if hasattr(lib, n)]
