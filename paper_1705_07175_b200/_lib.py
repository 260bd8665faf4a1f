"""ctypes binding of the C ABI in include/bitnn_b200.h.

The CUDA library is the only compute path: there is no CPU fallback.  If
lib/libbitnn_b200.so is missing this module raises at import time (build it
with ``python -m paper_1705_07175_b200.build``); if no GPU is present, every
op raises when it needs the device.
"""

from __future__ import annotations

import ctypes
import os

from .build import LIB

LIB = os.environ.get("B2_LIB", LIB)  # A/B experiments load an alternative build
if not os.path.exists(LIB):  # pragma: no cover - exercised on broken installs only
    raise ImportError(f"CUDA library {LIB} is missing; run `python -m paper_1705_07175_b200.build` "
                      "(this package has no CPU fallback)")

_so = ctypes.CDLL(LIB)

B2_EINVAL = 1000

vp = ctypes.c_void_p
i64 = ctypes.c_int64
i32 = ctypes.c_int32
cint = ctypes.c_int
f64 = ctypes.c_double


class Thresh(ctypes.Structure):
    """struct b2_thresh (include/bitnn_b200.h)."""

    _fields_ = [("thresh", vp), ("thresh64", vp), ("ge_dir", vp)]


# name -> (restype, argtypes), in header order
SIGNATURES = {
    "b2_version": (ctypes.c_char_p, []),
    "b2_launch_count": (i64, []),
    "b2_set_pdl": (cint, [cint]),
    "b2_pack_lines_f32": (cint, [vp, i64, i64, vp, vp]),
    "b2_unpack_lines_f32": (cint, [vp, i64, i64, vp, vp]),
    "b2_pack_byte_planes": (cint, [vp, i64, i64, vp, vp]),
    "b2_bgemm": (cint, [vp, i64, vp, i64, i64, i32, vp, vp]),
    "b2_bgemv": (cint, [vp, i64, i64, vp, i64, i32, vp, vp]),
    "b2_bitplane_gemv": (cint, [vp, i64, vp, i64, i64, vp, vp]),
    "b2_unroll_packed": (cint, [vp, i64, cint, cint, cint, cint, cint, cint, cint, vp, vp]),
    "b2_conv_correction": (cint, [vp, i64, cint, cint, cint, cint, cint, cint, cint, vp, vp]),
    "b2_conv_scratch_words": (i64, [i64, cint, cint, cint, cint, cint, cint, cint]),
    "b2_conv_forward": (cint, [vp, i64, cint, cint, cint, vp, i64, cint, cint, cint, cint, vp, vp, vp, vp]),
    "b2_add_correction_i32": (cint, [vp, vp, i64, i64, vp]),
    "b2_conv_bn_pack": (cint, [vp, i64, cint, cint, cint, vp, i64, cint, cint, cint, cint, vp, cint, Thresh, vp, vp]),
    "b2_maxpool_i32": (cint, [vp, i64, cint, cint, cint, cint, cint, cint, vp, vp]),
    "b2_threshold_pack": (cint, [vp, cint, i64, i64, i64, Thresh, cint, vp, vp]),
    "b2_bn_affine_f64": (cint, [vp, cint, i64, vp, vp, vp, i64, vp, vp]),
    "b2_bn_calibrate": (cint, [vp, vp, vp, vp, f64, i64, i64, vp, vp, vp, vp, vp]),
    "b2_dense_bn_pack": (cint, [vp, i64, vp, i64, i64, i32, Thresh, vp, vp]),
    "b2_input8_bn_pack": (cint, [vp, i64, i64, vp, i64, Thresh, vp, vp]),
    "b2_byte_conv_bn_pack": (cint, [vp, i64, cint, cint, cint, Thresh, vp, i64, cint, cint, cint, cint, Thresh, vp,
                                    vp]),
    "b2_i8_kpad": (i64, [i64]),
    "b2_expand_i8": (cint, [vp, i64, i64, i64, cint, vp, vp]),
    "b2_tc_bgemm": (cint, [vp, i64, vp, i64, i64, i32, vp, vp]),
    "b2_tc_dense_bn_pack": (cint, [vp, i64, vp, i64, i64, i32, Thresh, vp, vp]),
    "b2_tc_dense_affine_f64": (cint, [vp, i64, vp, i64, i64, i32, vp, vp, vp, vp, vp]),
    "b2_tc_conv_forward": (cint, [vp, i64, cint, cint, cint, vp, i64, cint, cint, cint, cint, vp, vp]),
    "b2_tc_conv_bn_pack": (cint, [vp, i64, cint, cint, cint, vp, i64, cint, cint, cint, cint, cint, Thresh, vp, vp]),
    "b2_tc_input8_bn_pack": (cint, [vp, i64, i64, vp, i64, Thresh, vp, vp]),
    "b2_tc_byte_conv_scratch_bytes": (i64, [i64, cint, cint, cint, cint, cint, cint, cint]),
    "b2_tc_byte_conv_bn_pack": (cint, [vp, i64, cint, cint, cint, Thresh, vp, i64, cint, cint, cint, cint, cint,
                                       Thresh, vp, vp, vp]),
    "b2_f4_kpad": (i64, [i64]),
    "b2_tc_byte_conv_path": (cint, [i64, cint, cint, cint, i64, cint, cint, cint, cint, cint]),
    "b2_tc4_conv_path": (cint, [i64, cint, cint, cint, i64, cint, cint, cint, cint, cint]),
    "b2_expand_f4": (cint, [vp, i64, i64, i64, vp, vp]),
    "b2_f4_cells_row_bytes": (i64, [cint]),
    "b2_expand_f4_cells": (cint, [vp, i64, i64, cint, cint, vp, vp]),
    "b2_tc4_byte_conv_padrow": (cint, [vp, i64, cint, cint, cint, Thresh, vp, i64, cint, cint, cint, cint, Thresh, vp,
                                       vp]),
}
# fp4-weight twins of the tensor-core entry points (same arguments)
for _n in ("bgemm", "dense_bn_pack", "dense_affine_f64", "conv_forward", "conv_bn_pack", "byte_conv_bn_pack"):
    SIGNATURES["b2_tc4_" + _n] = SIGNATURES["b2_tc_" + _n]

# GEMM engine for the shapes both engines support: "tc" (tcgen05 int8 tensor
# cores, the default) or "popc" (LOP3+POPC on the CUDA cores).  The choice
# is measured, not a fallback: DESIGN.md "engine choice" and
# profiles/ hold the ncu evidence; B2_ENGINE=popc exists to reproduce it.
ENGINE = os.environ.get("B2_ENGINE", "tc")
if ENGINE not in ("tc", "popc"):  # pragma: no cover
    raise ValueError(f"B2_ENGINE must be 'tc' or 'popc', got {ENGINE!r}")

# Tensor-core operand format: "f4" (tcgen05 kind::mxf4, packed e2m1 +/-1
# with unit block scales: twice the int8 MMA rate and half the operand
# bytes; the default) or "i8" (kind::i8).  u8-input layers always use i8.
TC_FORMAT = os.environ.get("B2_TC_FORMAT", "f4")
if TC_FORMAT not in ("f4", "i8"):  # pragma: no cover
    raise ValueError(f"B2_TC_FORMAT must be 'f4' or 'i8', got {TC_FORMAT!r}")


def tc_entry(op: str, fmt: str | None = None) -> str:
    """C entry point of tensor-core op `op` for weight format `fmt`."""
    return ("b2_tc4_" if (fmt or TC_FORMAT) == "f4" else "b2_tc_") + op


for _name, (_res, _args) in SIGNATURES.items():
    _fn = getattr(_so, _name)
    _fn.restype = _res
    _fn.argtypes = _args


class CudaOpError(RuntimeError):
    pass


# tensors whose pointers were taken for the call being assembled (see _dev.P)
KEEPALIVE: list = []


def call(name: str, *args) -> int:
    try:
        rc = getattr(_so, name)(*args)
    finally:
        KEEPALIVE.clear()
    if rc != 0:
        if rc == B2_EINVAL:
            raise ValueError(f"{name}: invalid arguments for the CUDA kernel")
        raise CudaOpError(f"{name} failed with cudaError {rc}")
    return rc


def raw(name: str):
    return getattr(_so, name)


def version() -> str:
    return _so.b2_version().decode()


def launch_count() -> int:
    return int(_so.b2_launch_count())


def set_pdl(on: bool) -> bool:
    """Programmatic dependent launch on/off; returns the previous setting."""
    return bool(_so.b2_set_pdl(1 if on else 0))


def exported_symbols() -> list[str]:
    return list(SIGNATURES)
