"""B200-native binary forward pass (Espresso, arXiv 1705.07175).

Drop-in for the packed path of the reference `bitnn` package: same public
names and semantics (`load`, `Network`, `forward`, `classify`, tensors,
layer and GEMM ops), computed by hand-written sm_100a CUDA kernels behind
the C ABI in include/bitnn_b200.h.  Adds `forward_batch` for batched,
multi-GPU inference.  There is no CPU fallback.
"""

from .modelfile import ModelFormatError, ModelSpec, ModelValidationError, load_model, read_model, save_model, write_model
from .network import (Backend, Network, classify, classify_batch, convert, forward, forward_batch, load, model_size,
                      serialize)
from .tensor import Axis, BitPlanes, FloatTensor, PackedTensor, bitplanes, linear_offset, pack, unpack

__version__ = "0.1.0"

__all__ = [
    "Axis", "Backend", "BitPlanes", "FloatTensor", "ModelFormatError", "ModelSpec", "ModelValidationError", "Network",
    "PackedTensor", "bitplanes", "classify", "classify_batch", "convert", "forward", "forward_batch", "linear_offset",
    "load", "load_model", "model_size", "pack", "read_model", "save_model", "serialize", "unpack", "write_model",
    "__version__",
]
