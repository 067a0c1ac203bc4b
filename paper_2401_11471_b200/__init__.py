"""B200-native row-centric convolution training (LR-CNN, arXiv 2401.11471).

The product is the C-ABI library liblrcnn.so (include/lrcnn.h) built from the
CUDA sources in csrc/; `lrcnn` is its thin ctypes binding.
"""
from .lrcnn import Plan, DeviceState, LrcnnError, lib, LIB_PATH  # noqa: F401
