"""oracle/_ref: the reference built behind the Eigen shim.

Checks that the step-wise harness (oracle/ref_harness.cpp) used to dump the
goldens is the reference's own train_cofree, bit for bit.
"""
import ctypes as C
import os

import numpy as np
import pytest

from cpu_libs import REF_SO, reference

pytestmark = pytest.mark.skipif(not os.path.exists(REF_SO), reason="oracle/_ref not built")


def test_harness_equals_train_cofree():
    R = reference()
    g = R.graph_sbm(200, 4, 0.15, 0.01, 8, 0.3, 7)
    part = g.partition("random", 8, 3)
    hidden = np.array([16, 16], np.int32)
    for f32 in (0, 1):
        for de in (0, 1):
            t = part.trainer([16, 16], lr=0.01, dropedge=bool(de), seed=1, f32=bool(f32), workers=3)
            losses = [t.step(e)[0] for e in range(6)]
            theta = t.params()
            out = np.zeros(t.nparam)
            L, G, M = np.zeros(6), np.zeros(6), np.zeros(18)
            fn = R.lib.ref_train_cofree
            audit = np.zeros(7, np.uint64)
            fn.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_double, C.c_int, C.c_int, C.c_int,
                           C.c_int, C.c_double, C.c_uint64, C.c_int, C.c_int, C.c_int] + [C.c_void_p] * 5
            st = fn(g.h, part.h, hidden.ctypes.data, 2, 0.01, 0, 0, de, 10, 0.5, 1, f32, 1, 6,
                    out.ctypes.data, L.ctypes.data, G.ctypes.data, M.ctypes.data, audit.ctypes.data)
            assert st == 0
            # TrainResult::audit: p * |theta| gradient floats per epoch, no embeddings (trainer.hpp:303-309)
            assert audit[:6].tolist() == [8 * t.nparam] * 6 and audit[6] == 0
            np.testing.assert_array_equal(theta, out)
            np.testing.assert_array_equal(losses, L)
