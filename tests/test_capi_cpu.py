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


def _ckpt_lib():
    lib = ctypes.CDLL(LIB)
    lib.sc_save_checkpoint_params.argtypes = [ctypes.c_void_p, ctypes.c_int32, ctypes.c_void_p, ctypes.c_int32,
                                              ctypes.c_int32, ctypes.c_char_p]
    lib.sc_load_checkpoint_params.argtypes = [ctypes.c_char_p, ctypes.c_void_p, ctypes.c_int64,
                                              ctypes.POINTER(ctypes.c_int64)]
    lib.sc_last_error.restype = ctypes.c_char_p
    return lib


def test_checkpoint_params_round_trip_and_format(tmp_path):
    """CFCK layout (checkpoint.cpp:44-84) through the host-only entry points: magic, u64 L,
    per layer message + update, then the head, each u64 rows, u64 cols, row-major f64."""
    import struct
    from paper_2308_03209_b200 import sagecut as sc
    lib = _ckpt_lib()
    in_dim, hidden, classes = 5, [4, 3], 2
    n = sc.param_count(in_dim, hidden, classes)
    theta = np.random.default_rng(0).standard_normal(n).astype(np.float32)
    h = np.array(hidden, np.int32)
    path = str(tmp_path / "p.ckpt")
    assert lib.sc_save_checkpoint_params(theta.ctypes.data, in_dim, h.ctypes.data, 2, classes, path.encode()) == 0
    raw = open(path, "rb").read()
    assert raw[:4] == b"CFCK" and struct.unpack("<Q", raw[4:12])[0] == 2
    shapes, off = [], 12
    while off < len(raw):
        r, c = struct.unpack("<QQ", raw[off:off + 16])
        shapes.append((r, c))
        off += 16 + 8 * r * c
    assert off == len(raw)
    assert sum(r * c for r, c in shapes) == n and len(shapes) == 5 and shapes[-1][0] == classes
    cnt = ctypes.c_int64()
    assert lib.sc_load_checkpoint_params(path.encode(), None, 0, ctypes.byref(cnt)) == 0 and cnt.value == n
    back = np.zeros(n, np.float32)
    assert lib.sc_load_checkpoint_params(path.encode(), back.ctypes.data, n, ctypes.byref(cnt)) == 0
    np.testing.assert_array_equal(back, theta)
    assert lib.sc_load_checkpoint_params(path.encode(), back.ctypes.data, n - 1, ctypes.byref(cnt)) != 0


@pytest.mark.parametrize("corrupt", ["magic", "layers", "shape", "truncated"])
def test_checkpoint_corrupt_files_rejected(tmp_path, corrupt):
    """Corrupt headers fail with an error, without allocating from the bogus sizes."""
    import struct
    from paper_2308_03209_b200 import sagecut as sc
    lib = _ckpt_lib()
    n = sc.param_count(3, [2], 2)
    theta = np.ones(n, np.float32)
    h = np.array([2], np.int32)
    path = tmp_path / "c.ckpt"
    assert lib.sc_save_checkpoint_params(theta.ctypes.data, 3, h.ctypes.data, 1, 2, str(path).encode()) == 0
    raw = bytearray(path.read_bytes())
    if corrupt == "magic":
        raw[:4] = b"XXXX"
    elif corrupt == "layers":
        raw[4:12] = struct.pack("<Q", 2**62)
    elif corrupt == "shape":
        raw[12:28] = struct.pack("<QQ", 2**40, 2**20)
    else:
        raw = raw[:-5]
    path.write_bytes(bytes(raw))
    cnt = ctypes.c_int64()
    assert lib.sc_load_checkpoint_params(str(path).encode(), None, 0, ctypes.byref(cnt)) != 0
    msg = lib.sc_last_error().decode()
    assert ("bad magic" if corrupt == "magic" else "truncated") in msg
