"""Drive the tensor-core GEMM kernels at products-like shapes for ncu captures.

    ncu --set full -k regex:gemm_f16x3 -c 1 python tools/profile_kernels.py nt
    ncu --set full -k regex:gemm_tn_f16x3 -c 1 python tools/profile_kernels.py tn
"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2308_03209_b200 import sagecut as sc  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "nt"
M = int(sys.argv[2]) if len(sys.argv) > 2 else 1_000_000
rng = np.random.default_rng(0)
if which == "nt":
    A = rng.standard_normal((M, 256), dtype=np.float32)
    B = rng.standard_normal((256, 256), dtype=np.float32)
    for _ in range(2):
        t0 = time.perf_counter()
        sc.debug_gemm(A, B, epi=1)
        print("nt wall", time.perf_counter() - t0)
elif which == "nt512":  # the update GEMM's dual-source shape: [mean | h] U^T (K = 256 + 256)
    A = rng.standard_normal((M, 256), dtype=np.float32)
    A2 = rng.standard_normal((M, 256), dtype=np.float32)
    B = rng.standard_normal((256, 256), dtype=np.float32)
    B2 = rng.standard_normal((256, 256), dtype=np.float32)
    for _ in range(2):
        t0 = time.perf_counter()
        sc.debug_gemm(A, B, A2=A2, B2=B2)
        print("nt512 wall", time.perf_counter() - t0)
elif which == "tn512":  # the update layer's dU = dh^T [mean | h] shape (N2 = 512)
    A = rng.standard_normal((M, 256), dtype=np.float32)
    B = rng.standard_normal((M, 256), dtype=np.float32)
    B2 = rng.standard_normal((M, 256), dtype=np.float32)
    for _ in range(2):
        t0 = time.perf_counter()
        sc.debug_gemm_tn(A, B, B2)
        print("tn512 wall", time.perf_counter() - t0)
else:
    A = rng.standard_normal((M, 256), dtype=np.float32)
    B = rng.standard_normal((M, 256), dtype=np.float32)
    for _ in range(2):
        t0 = time.perf_counter()
        sc.debug_gemm_tn(A, B)
        print("tn wall", time.perf_counter() - t0)
