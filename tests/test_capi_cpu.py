"""CPU-side checks of libsagecut_cuda.so: it loads, exports every symbol the
C header declares, and its host-only entry points (substream, select_mask,
param_count) agree with the oracle. No kernel is launched here."""
import ctypes
import os
import re

import numpy as np
import pytest

from cpu_libs import oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "sagecut_cuda.h")
LIB = os.path.join(ROOT, "paper_2308_03209_b200", "libsagecut_cuda.so")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(sc_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    assert os.path.exists(LIB), "build libsagecut_cuda.so first (__graft_entry__.build())"
    lib = ctypes.CDLL(LIB)
    syms = declared_symbols()
    assert len(syms) >= 45
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing


def test_host_entry_points_match_oracle():
    from paper_2308_03209_b200 import sagecut as sc
    O = oracle()
    for seed in (0, 1, 7, 2**63 + 5):
        for tag in ("init", "dropedge", "partition.random"):
            assert sc.substream(seed, tag) == O.substream(seed, tag)
            assert sc.substream(seed, tag, 3) == O.substream(seed, tag, 3)
            assert sc.substream(seed, tag, 3, 9) == O.substream(seed, tag, 3, 9)
    for part in range(8):
        for epoch in range(10):
            for k in (1, 3, 10):
                assert sc.select_mask(1, part, epoch, k) == O.select_mask(1, part, epoch, k)
    assert sc.param_count(100, [256, 256, 256], 47) == 521984  # SURVEY §8 S3 |theta|
    assert sc.param_count(602, [256, 256], 41) == 580864       # S2
    assert sc.param_count(64, [32, 32], 4) == 8320             # S1
    assert len(O.init_params(64, [32, 32], 4, 0)) == 8320


def test_train_config_validation_messages():
    from paper_2308_03209_b200 import sagecut as sc
    cfg = sc.TrainConfig(layers=2, hidden=[8, 8, 8])
    with pytest.raises(ValueError, match="hidden dims must match"):
        cfg.validate()
    with pytest.raises(ValueError, match="learning rate"):
        sc.TrainConfig(learning_rate=0.0).validate()
    with pytest.raises(ValueError, match="drop_ratio"):
        sc.TrainConfig(use_dropedge=True, drop_ratio=1.0).validate()
