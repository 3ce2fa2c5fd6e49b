"""ctypes binding of ``libspecrollout_b200.so`` (declared in
``include/specrollout_b200.h``).

The library is the only compute path: if it is missing, or no CUDA device is
visible, :func:`lib` raises :class:`DeviceError` -- there is no CPU fallback.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

from .errors import ConfigError, DeviceError

LIB_PATH = Path(__file__).resolve().parent / "libspecrollout_b200.so"
if os.environ.get("SR_LIB_PATH"):  # measurement builds only (scripts/gemm_trace.py)
    LIB_PATH = Path(os.environ["SR_LIB_PATH"])

_i32, _i64, _u32, _dbl, _vp = (ctypes.c_int, ctypes.c_int64, ctypes.c_uint32,
                               ctypes.c_double, ctypes.c_void_p)

# name -> argument types (all return int status unless listed in _RESTYPES)
SIGNATURES: dict[str, list] = {
    "sr_version": [],
    "sr_last_error": [],
    "sr_device_sm_count": [],
    "sr_abi_sizes": [_vp, _i32],
    "sr_keyed_tokens": [_i32, _vp, _vp, _i32, _i64, _i32, _vp, _vp],
    "sr_keyed_uniforms": [_i32, _vp, _vp, _i32, _i32, _vp, _vp],
    "sr_verify_windows": [_i32, _vp, _i32, _i32, _i32, _vp, _vp, _vp, _vp, _i32,
                          _vp, _vp, _vp, _vp],
    "sr_ngram_propose": [_i32, _vp, _i64, _vp, _i32, _i32, _i32, _vp, _vp, _vp, _vp],
    "sr_pooled_ngram_propose": [_i32, _vp, _i64, _vp, _i32, _i32, _i32, _vp, _vp, _vp, _vp],
    "sr_gemm": [_i32, _i32, _i32, _i32, _vp, _i32, _vp, _i32, _vp, _i32, _i32, _vp, _i32,
                _vp, _vp],
    "sr_gemm_splits": [_i32, _i32, _i32],
    "sr_set_gemm_swap_max_m": [_i32],
    "sr_paged_attention": [_i32, _vp, _vp, _i32, _i32, _i32, _i32, _i32, _i32, _i32, _i32, _vp, _i32,
                           _vp, _i32, _vp, _i32, _i32, _vp, ctypes.c_uint64, _vp, _vp],
    "sr_set_attention_split": [_i32],
    "sr_set_attention_tc": [_i32],
    "sr_sample_rows": [_vp, _i32, _i32, _i32, _vp, _vp, ctypes.c_uint32, ctypes.c_float, _vp, _vp],
    "sr_model_workspace_bytes": [_vp],
    "sr_model_create": [_vp, _vp],
    "sr_model_destroy": [_vp],
    "sr_model_forward": [_vp, _vp, _vp],
    "sr_model_profile": [_vp, _i32, _vp, _vp],
    "sr_launch_count": [],
    "sr_accept_commit": [_vp, _i32, _i32, _vp, _vp, _vp, _vp, _i64, _vp, _vp, _vp, _i32, _vp, _vp, _vp],
    "sr_synthetic_draft": [_i32, _i32, _vp, _i64, _vp, _vp, _i64, _vp, _vp, _i32, _vp, _vp, _vp],
    "sr_draft_model_batch": [_i32, _i32, _i32, _vp, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp,
                             _vp, _vp, _vp, _vp],
    "sr_accept_rejection": [_i32, _i32, _vp, _vp, _vp, _i64, _vp, _i64, _i32, ctypes.c_float, ctypes.c_uint32,
                            _vp, _i64, _vp, _vp, _vp, _i32, _vp, _vp, _vp, _vp],
    "sr_accept_rejection_workspace_floats": [_i32, _i32],
    "sr_decoupled_draft_prep": [_i32, _vp, _vp, _vp, _vp, _vp, _vp],
    "sr_decoupled_draft_post": [_i32, _i32, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp],
    "sr_decoupled_draft_apply": [_i32, _i32, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp],
    "sr_decoupled_verify_post": [_i32, _i32, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp],
    "sr_decoupled_verify_receive": [_i32, _i32, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp],
    "sr_pack_results": [_i32, _i32, _i32, _vp, _vp, _i64, _vp, _vp, _vp],
    "sr_io_begin": [_i32, _vp, _vp, _vp, _vp, _vp],
    "sr_build_verify_batch": [_i32, _i32, _i32, _vp, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp,
                              _vp, _vp, _vp, _vp, _vp],
}
_RESTYPES = {"sr_last_error": ctypes.c_char_p, "sr_model_workspace_bytes": ctypes.c_uint64,
             "sr_accept_rejection_workspace_floats": ctypes.c_uint64,
             "sr_launch_count": ctypes.c_longlong}


class SeqInfo(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in
                ("q_start", "q_len", "request", "ctx_len", "branch", "pad0", "pad1", "pad2")]
    __slots__ = ()


class ModelDesc(ctypes.Structure):
    """Mirror of ``sr_model_desc`` (include/specrollout_b200.h)."""

    _fields_ = [(n, ctypes.c_int32) for n in
                ("hidden", "intermediate", "layers", "q_heads", "kv_heads", "head_dim", "vocab",
                 "dtype")] + [("rms_eps", ctypes.c_float)] + [
        (n, ctypes.c_int32) for n in
        ("max_pos", "num_pages", "page_size", "max_requests", "max_pages_per_req",
         "max_branches", "window_max", "max_tokens", "max_seqs", "max_key", "logits_capacity")] + [
        (n, ctypes.c_void_p) for n in
        ("embed", "lm_head", "final_norm", "layer_weights", "rope_cos", "rope_sin", "kv_cache",
         "block_table", "window_kv", "workspace")] + [("workspace_bytes", ctypes.c_uint64)]
    __slots__ = ()


class ForwardArgs(ctypes.Structure):
    """Mirror of ``sr_forward_args``."""

    _fields_ = [(n, ctypes.c_int32) for n in
                ("num_tokens", "num_seqs", "max_q_len", "max_key", "output", "num_logit_rows")] + [
        (n, ctypes.c_void_p) for n in
        ("token_ids", "positions", "seqs", "logit_rows", "out", "out_val")] + [
        ("temperature", ctypes.c_float), ("seed", ctypes.c_uint32), ("live_rows", ctypes.c_void_p)]
    __slots__ = ()  # typos in field names raise instead of silently adding attributes

_lib = None


def load(path: os.PathLike | None = None) -> ctypes.CDLL:
    """Load the shared library and bind every declared symbol (no GPU needed)."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = Path(path) if path is not None else LIB_PATH
    if not p.exists():
        raise DeviceError(
            f"CUDA extension not built: {p} is missing "
            "(run `python -m paper_2511_16193_b200.build`)")
    handle = ctypes.CDLL(str(p))
    for name, argtypes in SIGNATURES.items():
        fn = getattr(handle, name)
        fn.argtypes = argtypes
        fn.restype = _RESTYPES.get(name, ctypes.c_int)
    if path is None:
        _lib = handle
    return handle


def lib() -> ctypes.CDLL:
    """The loaded library, after checking that a CUDA device is usable."""
    import torch

    if not torch.cuda.is_available():
        raise DeviceError("no CUDA device visible: the B200 rollout path needs a GPU")
    return load()


def check(status: int, what: str) -> None:
    if status == 0:
        return
    msg = load().sr_last_error().decode(errors="replace")
    if status == 2:
        raise ConfigError(f"{what}: {msg}")
    raise DeviceError(f"{what}: {msg} (status {status})")


def stream_handle(stream=None) -> int:
    """cudaStream_t of ``stream`` (default: torch's current stream)."""
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def ptr(t) -> int:
    return t.data_ptr()
