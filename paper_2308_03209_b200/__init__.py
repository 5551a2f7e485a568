"""B200-native CoFree-GNN per-partition training step (arXiv 2308.03209).

The product is libsagecut_cuda.so (csrc/, sm_100a kernels behind the C ABI in
include/sagecut_cuda.h). `sagecut` is the Python mirror of the reference's
`sagecut::` API over that ABI; importing it requires the built library.
"""
import os

PACKAGE_DIR = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PACKAGE_DIR, "libsagecut_cuda.so")
