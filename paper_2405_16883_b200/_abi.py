"""ctypes binding of ``libstc.so`` (declared in ``include/stc.h``).

Every call passes raw device pointers (``tensor.data_ptr()``) and the
caller's current CUDA stream; the library never allocates. Negative return
codes become Python exceptions that mirror the reference's error types
(`ShapeError` / `ValueError` / `RuntimeError`, cf. tensor.py:20, tiling.py:55).
There is no fallback: if the library or a GPU is missing, ``lib()`` raises.
"""

from __future__ import annotations

import ctypes
import os
import threading
from pathlib import Path

import torch

from .tensor import ShapeError

# STC_LIBRARY selects another build of the same ABI (the checked build, tools/run_checked.sh)
_LIB_PATH = Path(os.environ.get("STC_LIBRARY") or Path(__file__).resolve().parent / "libstc.so")
_lock = threading.Lock()
_lib = None

STC_OK = 0
STC_EINVAL = -1
STC_EUNSUPPORTED = -2
STC_ELAUNCH = -3
STC_EWORKSPACE = -4

VARIANT_ROW = 0
VARIANT_MERGE = 1
VARIANT_COLTILE = 2
VARIANTS = {"row": VARIANT_ROW, "merge": VARIANT_MERGE, "coltile": VARIANT_COLTILE}

EPILOGUE_NONE = 0
EPILOGUE_RELU = 1

FSUM_INF_MINUS_INF = 0x7FF8DEAD00000001
FSUM_OVERFLOW = 0x7FF8DEAD00000002

EWISE_UNION = 0
EWISE_INTERSECT = 1

_p = ctypes.c_void_p
_i = ctypes.c_int
_ll = ctypes.c_longlong
_f = ctypes.c_float
_sz = ctypes.c_size_t

# name -> (restype, argtypes); kept in the same order as include/stc.h
SIGNATURES = {
    "stc_abi_version": (_i, []),
    "stc_last_error": (ctypes.c_char_p, []),
    "stc_launch_count": (_ll, []),
    "stc_merge_path_groups": (_ll, [_i, _ll, _i]),
    "stc_merge_path_partition": (_i, [_i, _ll, _p, _i, _p, _p]),
    "stc_coltile_plan_ints": (_ll, [_i, _i, _ll]),
    "stc_coltile_plan": (_i, [_i, _i, _ll, _p, _p, _p, _p, _ll, _p]),
    "stc_merge_interleave": (_i, [_i, _ll, _p, _p, _p, _i, _p, _p, _p]),
    "stc_merge_plan_items_per_group": (_i, [_i, _ll, _i, _i, _i]),
    "stc_spmm_workspace_bytes": (_sz, [_i, _ll, _i, _i, _i, _i]),
    "stc_spmm_csr_f32": (_i, [_i, _i, _i, _p, _p, _p, _ll, _p, _ll, _p, _ll, _p, _ll, _i, _i, _p, _i,
                              _p, _sz, _p]),
    "stc_spmm_csr_batched_f32": (_i, [_i, _i, _i, _i, _p, _p, _p, _ll, _ll, _p, _ll, _ll, _p, _ll, _ll,
                                      _i, _i, _p, _i, _p, _sz, _p]),
    "stc_coo_segments_temp_bytes": (_sz, [_ll]),
    "stc_coo_segments": (_i, [_ll, _p, _p, _p, _p, _p, _sz, _p]),
    "stc_spmm_coo_f32": (_i, [_i, _i, _i, _p, _p, _p, _ll, _p, _ll, _p, _ll, _i, _p, _i, _p, _sz, _p]),
    "stc_sddmm_csr_f32": (_i, [_i, _i, _i, _i, _p, _p, _p, _ll, _p, _ll, _ll, _p, _ll, _ll, _f, _p, _p]),
    "stc_segsoftmax_csr_f32": (_i, [_i, _i, _p, _ll, _p, _p]),
    "stc_sparse_attention_f32": (_i, [_i, _i, _i, _i, _p, _p, _p, _ll, _p, _ll, _ll, _p, _ll, _ll, _p,
                                      _ll, _ll, _f, _p, _ll, _ll, _p, _p, _p]),
    "stc_attention_tiled_workspace_bytes": (_sz, [_i, _i]),
    "stc_sparse_attention_tiled_f32": (_i, [_i, _i, _i, _i, _i, _i, _p, _p, _p, _p, _p, _ll, _p, _ll, _ll, _p, _ll,
                                            _ll, _p, _ll, _ll, _f, _p, _ll, _ll, _p, _sz, _p]),
    "stc_mttkrp_coo3_f32": (_i, [_i, _i, _p, _p, _p, _p, _ll, _i, _p, _ll, _i, _p, _ll, _p, _ll, _i, _p, _i,
                                 _p, _sz, _p]),
    "stc_mttkrp_items_bytes": (_sz, [_ll]),
    "stc_mttkrp_prepare_items": (_i, [_ll, _p, _p, _p, _i, _ll, _i, _ll, _p, _p]),
    "stc_mttkrp_prepared_items_per_group": (_i, [_i, _ll, _i]),
    "stc_mttkrp_coo3_prepared_f32": (_i, [_i, _i, _p, _p, _ll, _i, _p, _ll, _i, _p, _ll, _p, _ll, _p, _i,
                                          _p, _sz, _p]),
    "stc_fsum_segments_f64": (_i, [_ll, _p, _p, _p, _p]),
    "stc_spgemm_products_temp_bytes": (_sz, [_i]),
    "stc_spgemm_products": (_i, [_i, _p, _p, _p, _p, _p, _sz, _p]),
    "stc_spgemm_workspace_bytes": (_sz, [_i, _i, _ll]),
    "stc_spgemm_symbolic": (_i, [_i, _i, _p, _p, _p, _p, _p, _p, _p, _ll, _p, _sz, _p, _p]),
    "stc_spgemm_numeric": (_i, [_i, _i, _p, _p, _p, _p, _p, _p, _ll, _p, _sz, _p, _p, _p, _p]),
    "stc_csr_ewise_temp_bytes": (_sz, [_i]),
    "stc_csr_ewise_symbolic": (_i, [_i, _i, _p, _p, _p, _p, _p, _p, _sz, _p]),
    "stc_csr_ewise_f32": (_i, [_i, _i, _p, _p, _p, _p, _p, _p, _p, _p, _p, _p]),
}


class ExtensionUnavailable(RuntimeError):
    """libstc.so is missing or no CUDA device is present; nothing falls back."""


def load_library(path: Path | None = None) -> ctypes.CDLL:
    """Open the shared object and attach the C signatures (no GPU needed)."""
    path = Path(path) if path is not None else _LIB_PATH
    if not path.exists():
        raise ExtensionUnavailable(
            f"{path} not found: build it with `python -m paper_2405_16883_b200._build` "
            "(the CUDA path has no CPU fallback)"
        )
    lib = ctypes.CDLL(str(path))
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                _lib = load_library()
    return _lib


_cuda_seen = False


def require_cuda(*tensors: torch.Tensor) -> None:
    global _cuda_seen
    if not _cuda_seen:
        if not torch.cuda.is_available():
            raise ExtensionUnavailable("no CUDA device: sparse contractions run only on the GPU")
        _cuda_seen = True
    dev = None
    for t in tensors:
        if t is None:
            continue
        if not t.is_cuda:
            raise ExtensionUnavailable(
                "operand buffers are on the CPU; move the tensor to CUDA (tensor.to('cuda'))"
            )
        if dev is None:
            dev = t.device
        elif t.device != dev:
            raise ValueError(f"operands on different devices ({dev} and {t.device})")


def on_operand_device(fn):
    """Run an op with its operands' device current, so its launches (and the stream handle
    passed to the C ABI) belong to that device even when another device is current."""
    import functools

    @functools.wraps(fn)
    def wrapper(*args, **kwargs):
        dev = next((a.device for a in args if isinstance(a, torch.Tensor) and a.is_cuda), None)
        if dev is not None and dev.index is not None and dev.index != torch.cuda.current_device():
            with torch.cuda.device(dev):
                return fn(*args, **kwargs)
        return fn(*args, **kwargs)

    return wrapper


def check(rc: int, what: str) -> None:
    if rc == STC_OK:
        return
    msg = lib().stc_last_error().decode(errors="replace")
    text = f"{what}: {msg} (code {rc})"
    if rc == STC_EINVAL:
        raise ShapeError(text)
    if rc == STC_EUNSUPPORTED:
        raise ValueError(text)
    raise RuntimeError(text)


def ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def stream_handle() -> int:
    return torch.cuda.current_stream().cuda_stream


def launch_count() -> int:
    """Kernels launched so far by libstc.so in this process."""
    return int(lib().stc_launch_count())
