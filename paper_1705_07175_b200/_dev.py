"""Device-memory plumbing: torch CUDA tensors as buffers, ctypes pointers.

PyTorch provides allocation, streams and graphs only; every computation on
these buffers is one of our own kernels (see _lib.py).  Packed uint64
words live in int64 tensors (same bytes).
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib

_NP2T = {
    np.dtype(np.uint64): torch.int64,
    np.dtype(np.int64): torch.int64,
    np.dtype(np.int32): torch.int32,
    np.dtype(np.uint32): torch.int32,
    np.dtype(np.uint8): torch.uint8,
    np.dtype(np.float32): torch.float32,
    np.dtype(np.float64): torch.float64,
}
_VIEW = {np.dtype(np.uint64): np.int64, np.dtype(np.uint32): np.int32}


def require_cuda():
    if not torch.cuda.is_available():
        raise RuntimeError("paper_1705_07175_b200 runs on a CUDA GPU (sm_100a) only; there is no CPU fallback")


def device() -> torch.device:
    require_cuda()
    return torch.device("cuda", torch.cuda.current_device())


def tdtype(np_dtype) -> torch.dtype:
    return _NP2T[np.dtype(np_dtype)]


def upload(arr: np.ndarray, dev=None) -> torch.Tensor:
    arr = np.ascontiguousarray(arr)
    if not arr.flags.writeable:
        arr = arr.copy()
    v = _VIEW.get(arr.dtype)
    if v is not None:
        arr = arr.view(v)
    return torch.from_numpy(arr).to(dev or device())


def empty(shape, np_dtype, dev=None) -> torch.Tensor:
    return torch.empty(tuple(int(s) for s in shape), dtype=tdtype(np_dtype), device=dev or device())


def zeros(shape, np_dtype, dev=None) -> torch.Tensor:
    return torch.zeros(tuple(int(s) for s in shape), dtype=tdtype(np_dtype), device=dev or device())


def download(t: torch.Tensor, np_dtype) -> np.ndarray:
    a = t.detach().cpu().numpy()
    np_dtype = np.dtype(np_dtype)
    if a.dtype != np_dtype:
        a = a.view(np_dtype)
    return a


def P(t) -> ctypes.c_void_p:
    """Device pointer of a tensor (None -> NULL).

    The tensor is kept alive until the next `_lib.call` returns, so a
    temporary (`P(upload(x))`) cannot be freed and its memory handed to a
    later argument before the kernel that reads it has been enqueued."""
    if t is None:
        return ctypes.c_void_p(0)
    _lib.KEEPALIVE.append(t)
    return ctypes.c_void_p(t.data_ptr())


def stream() -> ctypes.c_void_p:
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def sync():
    torch.cuda.current_stream().synchronize()


def widen_f4(words: torch.Tensor, rows: int, k: int) -> torch.Tensor:
    """Packed +/-1 rows (rows, wpl) on the device -> e2m1 nibbles (rows,
    kpad/2) uint8 for the fp4 tensor-core GEMM (b2_expand_f4)."""
    kpad = int(_lib.raw("b2_f4_kpad")(int(k)))
    out = torch.empty((int(rows), kpad // 2), dtype=torch.uint8, device=words.device)
    wpl = (int(k) + 63) // 64
    _lib.call("b2_expand_f4", P(words), int(rows), wpl, int(k), P(out), stream())
    return out


def tc_weights(words: torch.Tensor, rows: int, k: int, fmt: str | None = None) -> torch.Tensor:
    """Tensor-core weights of packed rows in format `fmt` (default _lib.TC_FORMAT)."""
    return widen_f4(words, rows, k) if (fmt or _lib.TC_FORMAT) == "f4" else widen_i8(words, rows, k)


def widen_i8(words: torch.Tensor, rows: int, k: int, permute: bool = True) -> torch.Tensor:
    """Packed +/-1 rows (rows, wpl) on the device -> int8 (rows, kpad) for the
    tensor-core GEMM (b2_expand_i8)."""
    kpad = int(_lib.raw("b2_i8_kpad")(int(k)))
    out = torch.empty((int(rows), kpad), dtype=torch.int8, device=words.device)
    wpl = (int(k) + 63) // 64
    _lib.call("b2_expand_i8", P(words), int(rows), wpl, int(k), int(bool(permute)), P(out), stream())
    return out
