"""Golden fixtures for the multi-label path and the reference's analytic helpers,
from the REAL reference (oracle/_ref/libsagecut_ref.so, see make_golden.py).

    make -C oracle && python tests/golden/make_golden_multilabel.py

multilabel.npz:
  Y                       the 200 x 5 0/1 target matrix attached to sbm200
                          (SbmSpec{200,4,0.15,0.01,8,0.3,7}) via Graph::multilabels
  traj_*                  5-step train_cofree trajectory, loss = bce against Y
                          (nn.hpp:348-378), p = 8 random vertex cut (seed 3),
                          DropEdge on, f32; eval = micro-F1 per split (trainer.cpp:72-87)
  eval_model_*            the reference's evaluate (trainer.cpp:101-112) of the
                          final f64 model on each split mask
  mc_eval_*               evaluate on the multi-class sbm200 (accuracy)
  comm_*, erf_*, ilb_*    comm_volume / expected_rf_random / imbalance_lower_bound
  audit                   TrainResult::audit of a 3-epoch train_cofree (p*|theta| per epoch, embeddings)
"""
from __future__ import annotations

import ctypes as C
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
os.environ["SAGECUT_REF_NO_BLAS"] = "1"
sys.path.insert(0, os.path.dirname(HERE))
from cpu_libs import reference  # noqa: E402

sys.path.insert(0, HERE)
from make_golden import trajectory  # noqa: E402


def multilabel_targets(labels, C_=5, seed=11):
    """Deterministic 0/1 targets: column y(v) mod C set, plus Bernoulli(0.3) noise."""
    rng = np.random.default_rng(seed)
    y = (rng.random((len(labels), C_)) < 0.3).astype(np.float32)
    y[np.arange(len(labels)), labels % C_] = 1.0
    return y


def main():
    R = reference()
    out = {}
    gs = R.graph_sbm(200, 4, 0.15, 0.01, 8, 0.3, 7)
    labels = gs.labels()
    Y = multilabel_targets(labels)
    gs.set_multilabels(Y)
    out["Y"] = Y
    part = gs.partition("random", 8, 3)
    t = trajectory(part, "traj_", 5, hidden=[16, 16], lr=0.01, loss="bce", dropedge=True, seed=1, f32=True)
    out.update(t)
    tr, va, te = gs.masks()
    theta = t["traj_params"][-1]
    for name, m in (("train", tr), ("val", va), ("test", te)):
        out[f"eval_model_{name}"] = np.float64(gs.evaluate(theta, [16, 16], m))
    # multi-class evaluate on a fresh sbm200 with the golden init model
    gm = R.graph_sbm(200, 4, 0.15, 0.01, 8, 0.3, 7)
    init = R.init_params(8, [16, 16], 4, 1, f32=True)
    out["mc_init"] = init
    for name, m in zip(("train", "val", "test"), gm.masks()):
        out[f"mc_eval_{name}"] = np.float64(gm.evaluate(init, [16, 16], m))
    # analytic helpers
    cv = [("cofree", 8, 521984, 3, 256, 0), ("halo_sync_model", 4, 8320, 2, 32, 1234), ("cofree", 1, 7, 0, 0, 0)]
    out["comm_args"] = np.array([[0 if c[0] == "cofree" else 1] + list(c[1:]) for c in cv], np.int64)
    out["comm_out"] = np.array([R.comm_volume(*c) for c in cv], np.uint64)
    erf = [(2, 1), (7, 1), (2, 2), (4, 500), (1, 3), (4, 0), (8, 13), (16, 100)]
    out["erf_args"] = np.array(erf, np.int64)
    out["erf_out"] = np.array([R.expected_rf_random(*a) for a in erf])
    ilb = [(2, 3, 1), (8, 5, 5), (1, 10, 2), (8, 1000, 3), (3, 7, 2)]
    out["ilb_args"] = np.array(ilb, np.int64)
    out["ilb_out"] = np.array([R.imbalance_lower_bound(*a) for a in ilb])
    # TrainResult::audit of the reference's own train_cofree
    gc = R.graph_sbm(200, 4, 0.15, 0.01, 8, 0.3, 7)
    pc = gc.partition("random", 8, 3)
    hidden = np.array([16, 16], np.int32)
    tt = pc.trainer([16, 16], lr=0.01, seed=1)
    params = np.zeros(tt.nparam)
    L, G, M = np.zeros(3), np.zeros(3), np.zeros(9)
    audit = np.zeros(4, np.uint64)
    fn = R.lib.ref_train_cofree
    fn.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_double, C.c_int, C.c_int, C.c_int,
                   C.c_int, C.c_double, C.c_uint64, C.c_int, C.c_int, C.c_int] + [C.c_void_p] * 5
    st = fn(gc.h, pc.h, hidden.ctypes.data, 2, 0.01, 0, 0, 0, 10, 0.5, 1, 1, 1, 3, params.ctypes.data,
            L.ctypes.data, G.ctypes.data, M.ctypes.data, audit.ctypes.data)
    assert st == 0
    out["audit"] = audit
    out["audit_params"] = np.int64(tt.nparam)
    np.savez_compressed(os.path.join(HERE, "multilabel.npz"), **out)
    print("multilabel.npz", os.path.getsize(os.path.join(HERE, "multilabel.npz")))


if __name__ == "__main__":
    main()
