"""B200-native Hybrid-Regressive Translation inference (arXiv 2212.01543).

Drop-in for the reference package's inference path (`hrt.infer`,
`hrt.decoding`): `CudaSession` implements the session protocol and
`hrt_translate` / `hrt_translate_batch` run the fused sm_100a path
(libhrt_b200.so, C ABI in include/hrt_b200.h). No CPU fallback exists.
"""

from .model import (BOS, BOS_K, EOS, EXCLUDED_OUTPUT_IDS, MASK, PAD, HRTModel, ModelConfig, ModelError,
                    init_params, param_layout)
from .engine import (ArenaOverflowError, CudaSession, DecoderCache, DecodingError, Engine, EngineCudaError,
                     EnginePool, InferenceError, estimate_max_bytes)
from .decoding import (Hypothesis, Translation, at_translate, at_translate_batch, build_stage2_input, combined_score,
                       hrt_translate, hrt_translate_batch, skip_at_stage, skip_cmlm_fill, truncate_at_eos)

__version__ = "0.1.0"

__all__ = [
    "PAD", "BOS", "EOS", "MASK", "BOS_K", "EXCLUDED_OUTPUT_IDS",
    "ModelConfig", "ModelError", "HRTModel", "init_params", "param_layout",
    "Engine", "EnginePool", "estimate_max_bytes", "CudaSession", "DecoderCache", "InferenceError", "DecodingError", "ArenaOverflowError",
    "EngineCudaError", "Hypothesis", "Translation", "truncate_at_eos", "build_stage2_input", "combined_score",
    "skip_at_stage", "skip_cmlm_fill", "hrt_translate", "hrt_translate_batch", "at_translate", "at_translate_batch",
]
