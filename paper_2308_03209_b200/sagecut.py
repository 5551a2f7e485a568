"""Python mirror of the reference's `sagecut` API over libsagecut_cuda.so.

Every public name follows the reference C++ API it replaces (cited per item);
all compute runs in the sm_100a kernels of libsagecut_cuda.so behind the C ABI
declared in include/sagecut_cuda.h. There is no CPU fallback: importing this
module without the built library, or calling it without a CUDA device, raises.

Used by tests/ (parity against the oracle) and bench.py. The C++ facade for
C++ callers of the reference is include/sagecut_b200.hpp.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# SC_LIB: load another build of the same library (A/B timing of kernel variants)
LIB_PATH = os.environ.get("SC_LIB") or os.path.join(_HERE, "libsagecut_cuda.so")

SC_OK, SC_EINVAL, SC_ERUNTIME, SC_EINTERNAL, SC_ECUDA, SC_ENCCL = range(6)


class CudaError(RuntimeError):
    pass


class NcclError(RuntimeError):
    pass


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback)")
    return C.CDLL(LIB_PATH)


_lib = _load()
_vp = C.c_void_p
_pp = C.POINTER(C.c_void_p)
_i32, _i64, _u64, _f64 = C.c_int32, C.c_int64, C.c_uint64, C.c_double


def _sig(name, args, res=C.c_int):
    if os.environ.get("SC_LIB") and not hasattr(_lib, name):
        return None  # A/B timing against an older build (SC_LIB): entry points it lacks stay unbound
    f = getattr(_lib, name)
    f.argtypes = args
    f.restype = res
    return f


_sig("sc_last_error", [], C.c_char_p)
_sig("sc_version", [], C.c_char_p)
_sig("sc_ctx_create", [C.c_int, _pp])
_sig("sc_ctx_destroy", [_vp])
_sig("sc_ctx_sync", [_vp])
_sig("sc_ctx_launch_count", [_vp], _i64)
_sig("sc_ctx_timer_start", [_vp])
_sig("sc_ctx_timer_stop", [_vp, C.POINTER(_f64)])
_sig("sc_build_graph", [_vp, _i32, _vp, _i64, _pp, C.POINTER(_i64), C.POINTER(_i64)])
_sig("sc_build_graph_dev", [_vp, _i32, _vp, _i64, _pp, C.POINTER(_i64), C.POINTER(_i64)])
_sig("sc_graph_set_data", [_vp, _vp, _i32, _vp, _i32, _vp, _vp, _vp])
_sig("sc_graph_set_features", [_vp, _vp, C.c_int])
_sig("sc_graph_set_feature_rows", [_vp, _i64, _i64, _vp, C.c_int])
_sig("sc_graph_set_multilabels", [_vp, _vp, _i32])
_sig("sc_load_graph", [_vp, C.c_char_p, _i32, _i32, _pp, C.POINTER(_i64), C.POINTER(_i64)])
_sig("sc_read_edge_list", [C.c_char_p, _i32, _vp, _i64, C.POINTER(_i64), C.POINTER(_i32)])
_sig("sc_load_features", [C.c_char_p, _i32, _vp, _i64, C.POINTER(_i64), C.POINTER(_i64)])
_sig("sc_load_labels", [C.c_char_p, _i32, _vp, _vp, _i64, C.POINTER(_i32), C.POINTER(_i32)])
_sig("sc_load_masks", [C.c_char_p, _i32, _vp, _vp, _vp])
_sig("sc_save_edge_list", [_vp, C.c_char_p])
_sig("sc_save_features", [C.c_char_p, _vp, _i64, _i64, _i32])
_sig("sc_save_labels", [C.c_char_p, _i32, _vp, _vp, _i32])
_sig("sc_save_masks", [C.c_char_p, _i32, _vp, _vp, _vp])
_sig("sc_graph_set_part_ownership", [_vp, _i32, _i32])
_sig("sc_vcut_part_held", [_vp, _i32, C.POINTER(_i32)])
EXCHANGE_FN = C.CFUNCTYPE(_i32, _vp, _i32, _i32, _i32, _vp, _vp, _i64)
_sig("sc_trainer_set_exchange", [_vp, EXCHANGE_FN, _vp])
_sig("sc_graph_info", [_vp, C.POINTER(_i32), C.POINTER(_i64), C.POINTER(_i32), C.POINTER(_i32)])
_sig("sc_graph_copy_edges", [_vp, _vp])
_sig("sc_graph_copy_csr", [_vp, _vp, _vp, _vp, _vp])
_sig("sc_graph_destroy", [_vp])
_sig("sc_partition_random", [_vp, _i32, _u64, _pp])
_sig("sc_partition_dbh", [_vp, _i32, _u64, _pp])
_sig("sc_build_vertex_cut", [_vp, _i32, _vp, _pp])
_sig("sc_vcut_num_parts", [_vp, C.POINTER(_i32)])
_sig("sc_vcut_assignment", [_vp, _vp])
_sig("sc_vcut_part_sizes", [_vp, _i32, C.POINTER(_i64), C.POINTER(_i64)])
_sig("sc_vcut_part_copy", [_vp, _i32] + [_vp] * 8)
_sig("sc_replication_stats", [_vp, _vp, C.POINTER(_f64), C.POINTER(_f64), C.POINTER(_f64), C.POINTER(_i64)])
_sig("sc_vcut_destroy", [_vp])
_sig("sc_partition_ne", [_vp, _i32, _u64, _f64, _pp])
_sig("sc_partition_edge_cut_greedy", [_vp, _i32, _u64, _vp])
_sig("sc_edge_cut_from_assignment", [_vp, _i32, _vp, _vp, C.POINTER(_i64), _vp, _vp, _vp, _vp])
_sig("sc_edge_cut_to_vertex_cut", [_vp, _i32, _vp, _u64, _pp])
_sig("sc_vcut_warnings", [_vp, C.c_char_p, _i64, C.POINTER(_i64)])
_sig("sc_save_partition", [_vp, C.c_char_p, _i32])
_sig("sc_load_partition", [_vp, C.c_char_p, _pp])
_sig("sc_save_edge_cut", [_vp, _i32, _vp, C.c_char_p])
_sig("sc_trainer_save_checkpoint", [_vp, C.c_char_p])
_sig("sc_trainer_load_checkpoint", [_vp, C.c_char_p])


class _EpochMetricsC(C.Structure):
    _fields_ = [("epoch", _i32), ("train_loss", _f64), ("train_metric", _f64), ("val_metric", _f64),
                ("test_metric", _f64), ("grad_norm", _f64), ("comm_floats", _u64)]


_sig("sc_write_metrics_jsonl", [C.c_char_p, _i32, _vp])
_sig("sc_compute_weights", [_vp, _i32, _vp])
_sig("sc_precompute_masks", [_vp, _i64, _i32, _f64, _u64, _vp])
_sig("sc_select_mask", [_u64, _u64, _u64, _i32], _i32)
_sig("sc_substream", [_u64, C.c_char_p, _i32, _u64, _u64], _u64)
_sig("sc_param_count", [_i32, _vp, _i32, _i32], _i64)
_sig("sc_init_params", [_vp, _i32, _vp, _i32, _i32, _u64, _vp])


class _TrainConfigC(C.Structure):
    _fields_ = [("layers", _i32), ("hidden", _vp), ("learning_rate", _f64), ("loss", _i32), ("reweight", _i32),
                ("use_dropedge", _i32), ("dropedge_k", _i32), ("drop_ratio", _f64), ("seed", _u64),
                ("deterministic", _i32), ("gemm", _i32)]


_sig("sc_trainer_create", [_vp, _vp, _vp, C.POINTER(_TrainConfigC), _i32, _i32, _pp])
_sig("sc_nccl_unique_id", [_vp])
_sig("sc_trainer_init_comm", [_vp, _vp])
_sig("sc_trainer_emulate_rank", [_vp])
_sig("sc_trainer_step", [_vp, _i32, C.POINTER(_f64), C.POINTER(_f64)])
_sig("sc_trainer_step_async", [_vp, _i32])
_sig("sc_trainer_stage_features", [_vp, _vp, _i32])
_sig("sc_trainer_last", [_vp, C.POINTER(_f64), C.POINTER(_f64)])
_sig("sc_trainer_param_count", [_vp, C.POINTER(_i64)])
for _n in ("sc_trainer_get_params", "sc_trainer_set_params", "sc_trainer_get_grads"):
    _sig(_n, [_vp, _vp])
_sig("sc_trainer_get_part_grads", [_vp, _i32, _vp])
_sig("sc_trainer_get_part_logits", [_vp, _i32, _vp])
_sig("sc_trainer_get_part_loss", [_vp, _i32, C.POINTER(_f64)])
_sig("sc_trainer_get_part_mask", [_vp, _i32, C.POINTER(_i32)])
_sig("sc_trainer_evaluate", [_vp, C.POINTER(_f64), C.POINTER(_f64), C.POINTER(_f64)])
_sig("sc_trainer_profile", [_vp, _i32])
_sig("sc_trainer_evaluate_mask", [_vp, _vp, C.POINTER(_f64)])
_sig("sc_evaluate", [_vp, _vp, _vp, _vp, _i32, _vp, C.POINTER(_f64)])
_sig("sc_trainer_comm_audit", [_vp, C.POINTER(_u64), C.POINTER(_u64)])
_sig("sc_trainer_fallback_count", [_vp, C.POINTER(_i64)])
_sig("sc_trainer_memory_mode", [_vp, C.POINTER(C.c_int32), C.POINTER(_i64)])
_sig("sc_comm_volume", [_i32, _i32, _u64, _u64, _u64, _u64, C.POINTER(_u64), C.POINTER(_u64), C.POINTER(_u64)])
_sig("sc_expected_rf_random", [_i32, _i64, C.POINTER(_f64)])
_sig("sc_imbalance_lower_bound", [_i32, _i64, _i64, C.POINTER(_f64)])
_sig("sc_trainer_kernel_times", [_vp, C.POINTER(C.c_char_p), C.POINTER(_f64), C.POINTER(_f64), _i32,
                                 C.POINTER(_i32)])
_sig("sc_trainer_kernel_flops", [_vp, C.POINTER(_f64), _i32, C.POINTER(_i32)])
_sig("sc_trainer_destroy", [_vp])
_sig("sc_debug_gemm", [_vp, _i32, _i64, _i32, _i32, _vp, _i64, _i64, _vp, _vp, _i64, _i32, _i32, _vp, _i64, _vp,
                       _i64, _i32, _i32, _vp, _vp])


_sig("sc_debug_gemm_tn", [_vp, _i32, _i64, _vp, _i32, _vp, _i32, _vp, _i64, _i32, _vp, _vp])
_sig("sc_debug_gemm_tn_dual", [_vp, _i64, _vp, _i32, _vp, _i32, _vp, _i32, _vp, _i32, _vp, _vp])


def debug_gemm_tn_dual(A1, A2, B1, B2, ctx: Optional["Context"] = None):
    """Kernel-level hook of the dual weight-gradient launch: (A1^T [B1 | B2], A2^T B2)."""
    ctx = ctx or default_context()
    A1, A2, B1, B2 = (np.ascontiguousarray(x, np.float32) for x in (A1, A2, B1, B2))
    M = A1.shape[0]
    C1 = np.zeros((A1.shape[1], B1.shape[1] + B2.shape[1]), np.float32)
    C2 = np.zeros((A2.shape[1], B2.shape[1]), np.float32)
    _check(_lib.sc_debug_gemm_tn_dual(ctx.h, M, _ptr(A1), A1.shape[1], _ptr(A2), A2.shape[1], _ptr(B1), B1.shape[1],
                                      _ptr(B2), B2.shape[1], _ptr(C1), _ptr(C2)), "debug_gemm_tn_dual")
    return C1, C2


_sig("sc_debug_spmm", [_vp, _i32, _i64, _i32, _vp, _vp, _vp, _i64, _vp, _vp, _vp, _vp])
_sig("sc_trainer_debug_buffer", [_vp, C.c_char_p, _i32, _vp, _i64])


def debug_spmm(bwd, offsets, nbrs, eids, src, edge_mask=None, msg=None, ctx: Optional["Context"] = None):
    """The aggregation kernels alone (nn.hpp:209-230 / 277-288) on host arrays; see sc_debug_spmm.
    bwd: 0 mean (inv * sum), 1 transposed with the ReLU gate of msg, 2 sum of inv[nbr]-scaled rows,
    3 msg + inv * sum (the projected top layer's two aggregations)."""
    ctx = ctx or default_context()
    off = np.ascontiguousarray(offsets, np.int64)
    nb = np.ascontiguousarray(nbrs, np.int32)
    ei = np.ascontiguousarray(eids, np.int32)
    x = np.ascontiguousarray(src, np.float32)
    n, H = len(off) - 1, x.shape[1]
    out = np.empty((n, H), np.float32)
    mk = None if edge_mask is None else np.ascontiguousarray(edge_mask, np.uint8)
    ms = None if msg is None else np.ascontiguousarray(msg, np.float32)
    _check(_lib.sc_debug_spmm(ctx.h, int(bwd), n, H, _ptr(off), _ptr(nb), _ptr(ei), 0 if mk is None else mk.size,
                              _ptr(mk), _ptr(x), _ptr(ms), _ptr(out)), "debug_spmm")
    return out


def debug_gemm_tn(A, B1, B2=None, rows2=None, simt=False, ctx: Optional["Context"] = None) -> np.ndarray:
    """Kernel-level hook: C = A^T [B1 | B2[rows2]] (weight-gradient shape, K = rows)."""
    ctx = ctx or default_context()
    A = np.ascontiguousarray(A, np.float32)
    B1 = np.ascontiguousarray(B1, np.float32)
    M, N1 = A.shape
    N2a = B1.shape[1]
    b2p, b2r, n2b = None, 0, 0
    if B2 is not None:
        B2 = np.ascontiguousarray(B2, np.float32)
        b2p, b2r, n2b = B2, B2.shape[0], B2.shape[1]
    r2 = None if rows2 is None else np.ascontiguousarray(rows2, np.int32)
    C = np.zeros((N1, N2a + n2b), np.float32)
    _check(_lib.sc_debug_gemm_tn(ctx.h, 1 if simt else 0, M, _ptr(A), N1, _ptr(B1), N2a, _ptr(b2p), b2r, n2b,
                                 _ptr(r2), _ptr(C)), "debug_gemm_tn")
    return C


def debug_gemm(A1, B1, b1_nn=False, rows1=None, A2=None, B2=None, b2_nn=False, epi=0, scale=None, simt=False,
               N=None, ctx: Optional["Context"] = None) -> np.ndarray:
    """Kernel-level hook: C = A1[rows1] op(B1) (+ A2 op(B2)), epilogue 0/1(relu)/2(row scale)."""
    ctx = ctx or default_context()
    A1 = np.ascontiguousarray(A1, np.float32)
    B1 = np.ascontiguousarray(B1, np.float32)
    K1 = B1.shape[0] if b1_nn else B1.shape[1]
    N = N or (B1.shape[1] if b1_nn else B1.shape[0])
    r1 = None if rows1 is None else np.ascontiguousarray(rows1, np.int32)
    M = len(r1) if r1 is not None else A1.shape[0]
    K2, A2p, B2p, lda2, ldb2 = 0, None, None, 0, 0
    if A2 is not None:
        A2 = np.ascontiguousarray(A2, np.float32)
        B2 = np.ascontiguousarray(B2, np.float32)
        K2 = B2.shape[0] if b2_nn else B2.shape[1]
        A2p, B2p, lda2, ldb2 = A2, B2, A2.shape[1], B2.shape[1]
    sc = None if scale is None else np.ascontiguousarray(scale, np.float32)
    C = np.zeros((M, N), np.float32)
    _check(_lib.sc_debug_gemm(ctx.h, 1 if simt else 0, M, N, K1, _ptr(A1), A1.shape[0], A1.shape[1], _ptr(r1),
                              _ptr(B1), B1.shape[1], int(b1_nn), K2, _ptr(A2p), lda2, _ptr(B2p), ldb2, int(b2_nn),
                              epi, _ptr(sc), _ptr(C)), "debug_gemm")
    return C


def _check(status: int, what: str = ""):
    if status == SC_OK:
        return
    msg = _lib.sc_last_error().decode()
    exc = {SC_EINVAL: ValueError, SC_ERUNTIME: RuntimeError, SC_EINTERNAL: AssertionError, SC_ECUDA: CudaError,
           SC_ENCCL: NcclError}.get(status, RuntimeError)
    raise exc(f"{what}: {msg}" if what else msg)


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(_vp)


def version() -> str:
    return _lib.sc_version().decode()


# ---------------------------------------------------------------------------
class Context:
    """One CUDA device + stream + scratch (sc_ctx)."""

    def __init__(self, device: int = 0):
        h = _vp()
        _check(_lib.sc_ctx_create(device, C.byref(h)), "sc_ctx_create")
        self.h = h
        self.device = device

    def sync(self):
        _check(_lib.sc_ctx_sync(self.h))

    def launch_count(self) -> int:
        return int(_lib.sc_ctx_launch_count(self.h))

    def timer_start(self):
        _check(_lib.sc_ctx_timer_start(self.h))

    def timer_stop(self) -> float:
        ms = _f64()
        _check(_lib.sc_ctx_timer_stop(self.h, C.byref(ms)))
        return ms.value

    def close(self):
        if getattr(self, "h", None):
            _lib.sc_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        self.close()


_default_ctx: Optional[Context] = None


def default_context() -> Context:
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = Context(int(os.environ.get("LOCAL_RANK", "0")) if os.environ.get("SC_DEVICE") is None
                               else int(os.environ["SC_DEVICE"]))
    return _default_ctx


@dataclass
class ValidationReport:  # graph.hpp:43-48
    dropped_self_loops: int = 0
    merged_duplicate_edges: int = 0


class Graph:
    """sagecut::Graph (graph.hpp:53-80), device resident."""

    def __init__(self, handle, ctx: Context):
        self.h, self.ctx = handle, ctx
        n, m, d, c = _i32(), _i64(), _i32(), _i32()
        _check(_lib.sc_graph_info(self.h, C.byref(n), C.byref(m), C.byref(d), C.byref(c)))
        self.num_nodes, self._m, self.dim, self.num_classes = n.value, m.value, d.value, c.value
        self.multilabel = False

    def num_edges(self) -> int:
        return self._m

    def edges(self) -> np.ndarray:
        out = np.zeros((self._m, 2), np.int32)
        _check(_lib.sc_graph_copy_edges(self.h, _ptr(out)))
        return out

    def csr(self):
        off = np.zeros(self.num_nodes + 1, np.int64)
        nb = np.zeros(2 * self._m, np.int32)
        ei = np.zeros(2 * self._m, np.int32)
        dg = np.zeros(self.num_nodes, np.int32)
        _check(_lib.sc_graph_copy_csr(self.h, _ptr(off), _ptr(nb), _ptr(ei), _ptr(dg)))
        return off, nb, ei, dg

    def degrees(self) -> np.ndarray:
        dg = np.zeros(self.num_nodes, np.int32)
        _check(_lib.sc_graph_copy_csr(self.h, None, None, None, _ptr(dg)))
        return dg

    def set_data(self, features, labels, num_classes, train_mask, val_mask, test_mask, dim: Optional[int] = None):
        """features: n x d array, or None with `dim` given (a zero matrix to fill with set_feature_rows)."""
        if features is None:
            if not dim or dim < 1:
                raise ValueError("set_data: features=None needs dim")
            f, d = None, int(dim)
        else:
            f = np.ascontiguousarray(features, np.float32)
            if f.ndim != 2 or f.shape[0] != self.num_nodes:
                raise ValueError("set_data: features must be num_nodes x d")
            d = f.shape[1]
        lab = np.ascontiguousarray(labels, np.int32)
        tr, va, te = (np.ascontiguousarray(x, np.uint8) for x in (train_mask, val_mask, test_mask))
        _check(_lib.sc_graph_set_data(self.h, _ptr(f), d, _ptr(lab), int(num_classes), _ptr(tr), _ptr(va),
                                      _ptr(te)), "set_data")
        self.dim, self.num_classes = d, int(num_classes)
        self.multilabel = False

    def set_feature_rows(self, row0: int, rows=None, device_ptr: Optional[int] = None, num_rows: int = 0):
        """Write feature rows [row0, row0 + k): from a host array `rows` (k x d), or k = num_rows rows
        at a device pointer."""
        if device_ptr is not None:
            _check(_lib.sc_graph_set_feature_rows(self.h, int(row0), int(num_rows), _vp(device_ptr), 1),
                   "set_feature_rows")
        else:
            f = np.ascontiguousarray(rows, np.float32)
            if f.ndim != 2 or f.shape[1] != self.dim:
                raise ValueError("set_feature_rows: rows must be k x d")
            _check(_lib.sc_graph_set_feature_rows(self.h, int(row0), f.shape[0], _ptr(f), 0), "set_feature_rows")

    def set_part_ownership(self, rank: int, world: int):
        """Vertex cuts built after this hold only the parts this rank trains (i % world == rank)."""
        _check(_lib.sc_graph_set_part_ownership(self.h, rank, world), "set_part_ownership")

    def set_multilabels(self, targets):
        """Graph::multilabels (graph.hpp:64): n x C of 0/1; the graph then trains with bce
        and evaluates with micro-F1 (trainer.cpp:72-87)."""
        y = np.ascontiguousarray(targets, np.float32)
        if y.ndim != 2 or y.shape[0] != self.num_nodes:
            raise ValueError("set_multilabels: targets must be num_nodes x C")
        _check(_lib.sc_graph_set_multilabels(self.h, _ptr(y), y.shape[1]), "set_multilabels")
        self.num_classes = y.shape[1]
        self.multilabel = True

    def set_features(self, features, device_ptr: Optional[int] = None, host_ptr: Optional[int] = None):
        """Replace the n x d feature matrix (same shape) from a numpy array, a host
        pointer (pinned memory -> async DMA), or a device pointer."""
        if device_ptr is not None:
            _check(_lib.sc_graph_set_features(self.h, _vp(device_ptr), 1))
        elif host_ptr is not None:
            _check(_lib.sc_graph_set_features(self.h, _vp(host_ptr), 0))
        else:
            f = np.ascontiguousarray(features, np.float32)
            _check(_lib.sc_graph_set_features(self.h, _ptr(f), 0))

    def __del__(self):
        if getattr(self, "h", None):
            _lib.sc_graph_destroy(self.h)
            self.h = None


def build_graph(num_nodes: int, raw_edges, ctx: Optional[Context] = None):
    """build_graph (graph.cpp:8-64) on the device -> (Graph, ValidationReport)."""
    ctx = ctx or default_context()
    raw = np.ascontiguousarray(raw_edges, np.int32).reshape(-1, 2)
    h = _vp()
    sl, du = _i64(), _i64()
    _check(_lib.sc_build_graph(ctx.h, int(num_nodes), _ptr(raw), len(raw), C.byref(h), C.byref(sl), C.byref(du)),
           "build_graph")
    return Graph(h, ctx), ValidationReport(sl.value, du.value)


def load_graph(path: str, num_nodes: Optional[int] = None, strict: bool = False, ctx: Optional[Context] = None):
    """load_graph (graph_io.cpp:41-80) -> (Graph, ValidationReport)."""
    ctx = ctx or default_context()
    h, sl, dp = _vp(), _i64(), _i64()
    _check(_lib.sc_load_graph(ctx.h, os.fsencode(path), -1 if num_nodes is None else num_nodes, int(strict),
                              C.byref(h), C.byref(sl), C.byref(dp)), "load_graph")
    return Graph(h, ctx), ValidationReport(sl.value, dp.value)


def read_edge_list(path: str, num_nodes: Optional[int] = None):
    """load_graph's parse alone (host only): (raw pairs [m, 2] in file order, node count)."""
    m, n = _i64(), _i32()
    nn = -1 if num_nodes is None else num_nodes
    _check(_lib.sc_read_edge_list(os.fsencode(path), nn, None, 0, C.byref(m), C.byref(n)), "load_graph")
    uv = np.zeros((m.value, 2), np.int32)
    _check(_lib.sc_read_edge_list(os.fsencode(path), nn, _ptr(uv), m.value, C.byref(m), C.byref(n)), "load_graph")
    return uv, n.value


def load_features(path: str, expected_nodes: int) -> np.ndarray:  # graph_io.cpp:82-160
    r, c = _i64(), _i64()
    _check(_lib.sc_load_features(os.fsencode(path), expected_nodes, None, 0, C.byref(r), C.byref(c)), "load_features")
    out = np.zeros((r.value, c.value), np.float32)
    _check(_lib.sc_load_features(os.fsencode(path), expected_nodes, _ptr(out), out.size, C.byref(r), C.byref(c)),
           "load_features")
    return out


def load_labels(path: str, num_nodes: int):
    """load_labels (graph_io.cpp:188-242) -> (class ids or None, 0/1 targets or None, num_classes)."""
    nc, ml = _i32(), _i32()
    _check(_lib.sc_load_labels(os.fsencode(path), num_nodes, None, None, 0, C.byref(nc), C.byref(ml)), "load_labels")
    if ml.value:
        y = np.zeros((num_nodes, nc.value), np.float32)
        _check(_lib.sc_load_labels(os.fsencode(path), num_nodes, None, _ptr(y), y.size, C.byref(nc), C.byref(ml)),
               "load_labels")
        return None, y, nc.value
    lab = np.zeros(num_nodes, np.int32)
    _check(_lib.sc_load_labels(os.fsencode(path), num_nodes, _ptr(lab), None, 0, C.byref(nc), C.byref(ml)),
           "load_labels")
    return lab, None, nc.value


def load_masks(path: str, num_nodes: int):  # graph_io.cpp:256-283
    tr, va, te = (np.zeros(num_nodes, np.uint8) for _ in range(3))
    _check(_lib.sc_load_masks(os.fsencode(path), num_nodes, _ptr(tr), _ptr(va), _ptr(te)), "load_masks")
    return tr, va, te


def save_edge_list(g: "Graph", path: str):  # graph_io.cpp:75-80
    _check(_lib.sc_save_edge_list(g.h, os.fsencode(path)), "save_edge_list")


def save_features(features, path: str, binary: bool = False):  # graph_io.cpp:162-186
    f = np.ascontiguousarray(features, np.float32)
    _check(_lib.sc_save_features(os.fsencode(path), _ptr(f), f.shape[0], f.shape[1], int(binary)), "save_features")


def save_labels(path: str, labels=None, targets=None):  # graph_io.cpp:244-254
    if targets is not None:
        y = np.ascontiguousarray(targets, np.float32)
        _check(_lib.sc_save_labels(os.fsencode(path), y.shape[0], None, _ptr(y), y.shape[1]), "save_labels")
    else:
        lab = np.ascontiguousarray(labels, np.int32)
        _check(_lib.sc_save_labels(os.fsencode(path), lab.size, _ptr(lab), None, 0), "save_labels")


def save_masks(path: str, train, val, test):  # graph_io.cpp:285-296
    tr, va, te = (np.ascontiguousarray(x, np.uint8) for x in (train, val, test))
    _check(_lib.sc_save_masks(os.fsencode(path), tr.size, _ptr(tr), _ptr(va), _ptr(te)), "save_masks")


def build_graph_device(num_nodes: int, raw_dev_ptr: int, m_raw: int, ctx: Optional[Context] = None):
    """build_graph from a raw int32 [m][2] edge list already in device memory."""
    ctx = ctx or default_context()
    h = _vp()
    sl, du = _i64(), _i64()
    _check(_lib.sc_build_graph_dev(ctx.h, int(num_nodes), _vp(raw_dev_ptr), int(m_raw), C.byref(h), C.byref(sl),
                                   C.byref(du)), "build_graph")
    return Graph(h, ctx), ValidationReport(sl.value, du.value)


@dataclass
class PartSubgraph:  # partition.hpp:14-31
    nodes: np.ndarray
    edges: np.ndarray
    edge_global_ids: np.ndarray
    local_degrees: np.ndarray
    adj_offsets: np.ndarray
    adj_neighbors: np.ndarray
    adj_edge_ids: np.ndarray
    global_to_local: np.ndarray

    def num_local_nodes(self) -> int:
        return len(self.nodes)


@dataclass
class ReplicationStats:  # partition.hpp:50-56
    rf: float
    per_node_rf: np.ndarray
    edge_balance: float
    node_balance: float
    duplicated_nodes: int


class VertexCutPartition:
    """sagecut::VertexCutPartition (partition.hpp:35-40); parts stay on the device,
    `part(i)` copies one PartSubgraph to the host for inspection."""

    def __init__(self, handle, g: Graph):
        self.h, self.g = handle, g
        p = _i32()
        _check(_lib.sc_vcut_num_parts(self.h, C.byref(p)))
        self.num_parts = p.value

    @property
    def edge_assignment(self) -> np.ndarray:
        out = np.zeros(self.g.num_edges(), np.int32)
        _check(_lib.sc_vcut_assignment(self.h, _ptr(out)))
        return out

    def part_sizes(self, i: int):
        nl, ne = _i64(), _i64()
        _check(_lib.sc_vcut_part_sizes(self.h, i, C.byref(nl), C.byref(ne)))
        return nl.value, ne.value

    def part(self, i: int) -> PartSubgraph:
        nl, ne = self.part_sizes(i)
        s = PartSubgraph(np.zeros(nl, np.int32), np.zeros((ne, 2), np.int32), np.zeros(ne, np.int32),
                         np.zeros(nl, np.int32), np.zeros(nl + 1, np.int64), np.zeros(2 * ne, np.int32),
                         np.zeros(2 * ne, np.int32), np.zeros(self.g.num_nodes, np.int32))
        _check(_lib.sc_vcut_part_copy(self.h, i, _ptr(s.nodes), _ptr(s.edges), _ptr(s.edge_global_ids),
                                      _ptr(s.local_degrees), _ptr(s.adj_offsets), _ptr(s.adj_neighbors),
                                      _ptr(s.adj_edge_ids), _ptr(s.global_to_local)))
        return s

    def part_held(self, i: int) -> bool:
        x = _i32()
        _check(_lib.sc_vcut_part_held(self.h, i, C.byref(x)))
        return bool(x.value)

    @property
    def parts(self) -> List[PartSubgraph]:
        return [self.part(i) for i in range(self.num_parts)]

    @property
    def warnings(self) -> List[str]:  # VertexCutPartition::warnings (partition.hpp:36)
        need = _i64()
        _check(_lib.sc_vcut_warnings(self.h, None, 0, C.byref(need)))
        buf = C.create_string_buffer(int(need.value))
        _check(_lib.sc_vcut_warnings(self.h, buf, len(buf), C.byref(need)))
        w = buf.value.decode()
        return w.split("\n") if w else []

    def __del__(self):
        if getattr(self, "h", None):
            _lib.sc_vcut_destroy(self.h)
            self.h = None


def partition_random(g: Graph, num_parts: int, seed: int) -> VertexCutPartition:  # partition.cpp:92
    h = _vp()
    _check(_lib.sc_partition_random(g.h, num_parts, seed, C.byref(h)), "partition_random")
    return VertexCutPartition(h, g)


def partition_dbh(g: Graph, num_parts: int, seed: int) -> VertexCutPartition:  # partition.cpp:102
    h = _vp()
    _check(_lib.sc_partition_dbh(g.h, num_parts, seed, C.byref(h)), "partition_dbh")
    return VertexCutPartition(h, g)


def partition_ne(g: Graph, num_parts: int, seed: int, balance_slack: float = 1.1) -> VertexCutPartition:
    """partition_ne (partition.cpp:116-201): same assignment as the reference, O(E log E)."""
    h = _vp()
    _check(_lib.sc_partition_ne(g.h, num_parts, seed, float(balance_slack), C.byref(h)), "partition_ne")
    return VertexCutPartition(h, g)


@dataclass
class EdgeCutPartition:  # partition.hpp:41-52
    num_parts: int
    node_assignment: np.ndarray
    kept_edges: List[np.ndarray]
    cut_edges: np.ndarray
    halo_sets: List[np.ndarray]

    def total_halo(self) -> int:
        return int(sum(len(h) for h in self.halo_sets))


def edge_cut_from_assignment(g: Graph, num_parts: int, node_assignment) -> EdgeCutPartition:  # partition.cpp:203
    na = np.ascontiguousarray(node_assignment, np.int32)
    if len(na) != g.num_nodes:
        raise ValueError("node assignment length does not match node count")
    kept = np.zeros(max(num_parts, 1), np.int64)
    halo = np.zeros(max(num_parts, 1), np.int64)
    ncut = _i64()
    _check(_lib.sc_edge_cut_from_assignment(g.h, num_parts, _ptr(na), _ptr(kept), C.byref(ncut), _ptr(halo), None,
                                            None, None), "edge_cut_from_assignment")
    kept_ids = np.zeros(g.num_edges() - ncut.value, np.int32)
    cut = np.zeros(ncut.value, np.int32)
    nodes = np.zeros(int(halo.sum()), np.int32)
    _check(_lib.sc_edge_cut_from_assignment(g.h, num_parts, _ptr(na), _ptr(kept), C.byref(ncut), _ptr(halo),
                                            _ptr(kept_ids), _ptr(cut), _ptr(nodes)), "edge_cut_from_assignment")
    kb = np.concatenate([[0], np.cumsum(kept[:num_parts])])
    hb = np.concatenate([[0], np.cumsum(halo[:num_parts])])
    return EdgeCutPartition(num_parts, na, [kept_ids[kb[i]:kb[i + 1]] for i in range(num_parts)], cut,
                            [nodes[hb[i]:hb[i + 1]] for i in range(num_parts)])


def partition_edge_cut_greedy(g: Graph, num_parts: int, seed: int) -> EdgeCutPartition:  # partition.cpp:233
    na = np.zeros(g.num_nodes, np.int32)
    _check(_lib.sc_partition_edge_cut_greedy(g.h, num_parts, seed, _ptr(na)), "partition_edge_cut_greedy")
    return edge_cut_from_assignment(g, num_parts, na)


def edge_cut_to_vertex_cut(g: Graph, ec: EdgeCutPartition, seed: int) -> VertexCutPartition:  # partition.cpp:280
    na = np.ascontiguousarray(ec.node_assignment, np.int32)
    if len(na) != g.num_nodes:
        raise ValueError("edge cut does not match graph")
    h = _vp()
    _check(_lib.sc_edge_cut_to_vertex_cut(g.h, ec.num_parts, _ptr(na), seed, C.byref(h)), "edge_cut_to_vertex_cut")
    return VertexCutPartition(h, g)


def save_partition(part: VertexCutPartition, path: str, weights: Optional[str] = None):
    """save_partition (partition_io.cpp:12-29); `weights` names a reweight scheme to embed."""
    _check(_lib.sc_save_partition(part.h, os.fsencode(path), -1 if weights is None else _SCHEMES[weights]),
           "save_partition")


def load_partition(path: str, g: Graph) -> VertexCutPartition:  # partition_io.cpp:31-56
    h = _vp()
    _check(_lib.sc_load_partition(g.h, os.fsencode(path), C.byref(h)), "load_partition")
    return VertexCutPartition(h, g)


def save_edge_cut(g: Graph, ec: "EdgeCutPartition", path: str):  # partition_io.cpp:58-68
    na = np.ascontiguousarray(ec.node_assignment, np.int32)
    _check(_lib.sc_save_edge_cut(g.h, ec.num_parts, _ptr(na), os.fsencode(path)), "save_edge_cut")


def write_metrics_jsonl(metrics, path: str):
    """write_metrics_jsonl (trainer.cpp:126-140); metrics: EpochMetrics-like objects or dicts."""
    rows = (_EpochMetricsC * max(len(metrics), 1))()
    for i, m in enumerate(metrics):
        get = (lambda k: m[k]) if isinstance(m, dict) else (lambda k: getattr(m, k))
        rows[i] = _EpochMetricsC(int(get("epoch")), float(get("train_loss")), float(get("train_metric")),
                                 float(get("val_metric")), float(get("test_metric")), float(get("grad_norm")),
                                 int(get("comm_floats")))
    _check(_lib.sc_write_metrics_jsonl(os.fsencode(path), len(metrics), C.cast(rows, _vp)), "write_metrics_jsonl")


def build_vertex_cut(g: Graph, num_parts: int, edge_assignment) -> VertexCutPartition:  # partition.cpp:22
    a = np.ascontiguousarray(edge_assignment, np.int32)
    if len(a) != g.num_edges():
        raise ValueError("edge assignment length does not match edge count")
    h = _vp()
    _check(_lib.sc_build_vertex_cut(g.h, num_parts, _ptr(a), C.byref(h)), "build_vertex_cut")
    return VertexCutPartition(h, g)


def replication_stats(part: VertexCutPartition, g: Graph) -> ReplicationStats:  # partition.cpp:310
    rfv = np.zeros(g.num_nodes, np.int32)
    rf, eb, nb = _f64(), _f64(), _f64()
    dup = _i64()
    _check(_lib.sc_replication_stats(part.h, _ptr(rfv), C.byref(rf), C.byref(eb), C.byref(nb), C.byref(dup)))
    return ReplicationStats(rf.value, rfv, eb.value, nb.value, dup.value)


_SCHEMES = {"dar": 0, "vanilla_inv": 1, "none": 2}
_LOSSES = {"softmax_ce": 0, "bce": 1}


@dataclass
class NodeWeights:  # reweight.hpp:15-19
    scheme: str
    per_part: List[np.ndarray]


def compute_weights(scheme: str, g: Graph, part: VertexCutPartition) -> NodeWeights:  # reweight.cpp:73
    if scheme not in _SCHEMES:
        raise ValueError(f"unknown reweight scheme: {scheme}")
    sizes = [part.part_sizes(i)[0] for i in range(part.num_parts)]
    out = np.zeros(sum(sizes), np.float64)
    _check(_lib.sc_compute_weights(part.h, _SCHEMES[scheme], _ptr(out)), "compute_weights")
    res, k = [], 0
    for s in sizes:
        res.append(out[k:k + s].copy())
        k += s
    return NodeWeights(scheme, res)


@dataclass
class DropEdgeMaskSet:  # dropedge.hpp:13-18
    num_masks: int
    ratio: float
    seed: int
    masks: np.ndarray  # [K, num_edges] uint8


def precompute_masks(num_edges: int, num_masks: int, ratio: float, seed: int,
                     ctx: Optional[Context] = None) -> DropEdgeMaskSet:  # dropedge.cpp:9
    ctx = ctx or default_context()
    out = np.zeros(max(num_edges * max(num_masks, 0), 1), np.uint8)
    _check(_lib.sc_precompute_masks(ctx.h, num_edges, num_masks, ratio, seed, _ptr(out)), "precompute_masks")
    return DropEdgeMaskSet(num_masks, ratio, seed, out[:num_edges * num_masks].reshape(num_masks, num_edges))


def select_mask(seed: int, part_index: int, epoch: int, num_masks: int) -> int:  # trainer.hpp:261-266
    if num_masks < 1:
        raise ValueError("select_mask: need at least one mask")
    return int(_lib.sc_select_mask(seed, part_index, epoch, num_masks))


def substream(seed: int, tag: str, *idx: int) -> int:  # rng.hpp:94-103
    a = idx[0] if len(idx) > 0 else 0
    b = idx[1] if len(idx) > 1 else 0
    return int(_lib.sc_substream(seed, tag.encode(), len(idx), a, b))


def param_count(in_dim: int, hidden: Sequence[int], num_classes: int) -> int:
    h = np.ascontiguousarray(hidden, np.int32)
    return int(_lib.sc_param_count(in_dim, _ptr(h), len(h), num_classes))


def make_sage_model(in_dim: int, hidden: Sequence[int], num_classes: int, seed: int,
                    ctx: Optional[Context] = None) -> np.ndarray:  # nn.hpp:73-102 (float)
    ctx = ctx or default_context()
    h = np.ascontiguousarray(hidden, np.int32)
    out = np.zeros(param_count(in_dim, hidden, num_classes), np.float32)
    _check(_lib.sc_init_params(ctx.h, in_dim, _ptr(h), len(h), num_classes, seed, _ptr(out)), "make_sage_model")
    return out


@dataclass
class TrainConfig:  # trainer.hpp:20-33
    layers: int = 2
    hidden: List[int] = field(default_factory=lambda: [32])
    epochs: int = 100
    learning_rate: float = 0.01
    loss: str = "softmax_ce"
    reweight: str = "dar"
    use_dropedge: bool = False
    dropedge_k: int = 10
    drop_ratio: float = 0.5
    seed: int = 0
    precision: str = "f32"
    workers: int = 1
    # B200 knobs
    deterministic: bool = True
    gemm: str = "auto"  # "auto" (tcgen05 where supported) | "simt"

    def resolved_hidden(self) -> List[int]:  # trainer.cpp:12-19
        if self.layers == 0:
            return []
        if len(self.hidden) == 1:
            return [self.hidden[0]] * self.layers
        if len(self.hidden) != self.layers:
            raise ValueError("hidden dims must match layer count (or be a single value)")
        return list(self.hidden)

    def validate(self):  # trainer.cpp:21-36
        if self.layers < 0:
            raise ValueError("layers must be >= 0")
        if self.epochs < 0:
            raise ValueError("epochs must be >= 0")
        if not self.learning_rate > 0.0:
            raise ValueError("learning rate must be > 0")
        if self.workers < 1:
            raise ValueError("workers must be >= 1")
        if self.layers > 0 and not self.hidden:
            raise ValueError("hidden dims required for layers > 0")
        if any(h < 1 for h in self.hidden):
            raise ValueError("hidden dims must be positive")
        if self.use_dropedge:
            if self.dropedge_k < 1:
                raise ValueError("dropedge_k must be >= 1")
            if not 0.0 <= self.drop_ratio < 1.0:
                raise ValueError("drop_ratio must lie in [0, 1)")
        if self.precision != "f32":
            raise ValueError("sagecut_cuda trains in f32 (the reference's Precision::f32)")
        self.resolved_hidden()


@dataclass
class EpochMetrics:  # trainer.hpp:38-46
    epoch: int
    train_loss: float
    train_metric: float = 0.0
    val_metric: float = 0.0
    test_metric: float = 0.0
    grad_norm: float = 0.0
    comm_floats: int = 0


class CoFreeTrainer:
    """The state of train_cofree_impl (trainer.hpp:202-313) on one rank."""

    def __init__(self, g: Graph, part: VertexCutPartition, config: TrainConfig, rank: int = 0, world: int = 1,
                 nccl_id: Optional[bytes] = None, _defer_comm: bool = False):
        config.validate()
        self.g, self.part, self.config = g, part, config
        self.hidden = np.ascontiguousarray(config.resolved_hidden(), np.int32)
        c = _TrainConfigC(len(self.hidden), self.hidden.ctypes.data if len(self.hidden) else None,
                          config.learning_rate, _LOSSES[config.loss], _SCHEMES[config.reweight],
                          int(config.use_dropedge), config.dropedge_k, config.drop_ratio, config.seed,
                          int(config.deterministic), 1 if config.gemm == "simt" else 0)
        h = _vp()
        _check(_lib.sc_trainer_create(g.ctx.h, g.h, part.h, C.byref(c), rank, world, C.byref(h)), "train_cofree")
        self.h = h
        n = _i64()
        _check(_lib.sc_trainer_param_count(self.h, C.byref(n)))
        self.param_count = n.value
        self.rank, self.world = rank, world
        if world > 1 and nccl_id is None and not _defer_comm:
            raise ValueError("world > 1 needs the rank-0 NCCL unique id (or set_exchange with _defer_comm=True)")
        if nccl_id is not None:  # (world == 1 too: a single-rank communicator runs the exchange path)
            buf = (C.c_uint8 * 128).from_buffer_copy(nccl_id)
            _check(_lib.sc_trainer_init_comm(self.h, buf), "init_comm")

    def set_exchange(self, allgather):
        """Host transport for the gradient exchange instead of NCCL: allgather(kind, round, bucket, send: bytes)
        must return the world ranks' byte strings concatenated in rank order (kind 0: one f32 gradient
        bucket, 1: the round's f64 partition losses). None restores NCCL."""
        if allgather is None:
            self._xfn = None
            _check(_lib.sc_trainer_set_exchange(self.h, EXCHANGE_FN(), None))
            return

        def cb(_user, kind, rnd, bucket, send, recv, nbytes):
            try:
                out = allgather(kind, rnd, bucket, C.string_at(send, nbytes))
                C.memmove(recv, out, len(out))
                return 0
            except Exception as e:  # noqa: BLE001 (reported through the status code)
                self._xerr = e
                return 1

        self._xfn = EXCHANGE_FN(cb)  # keep the trampoline alive
        _check(_lib.sc_trainer_set_exchange(self.h, self._xfn, None))

    def emulate_rank(self):
        """Time this rank's share of the world-size job on one GPU: exchanges skipped, the other
        ranks' gradient slots stay zero (timing / memory only)."""
        _check(_lib.sc_trainer_emulate_rank(self.h), "emulate_rank")

    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = (C.c_uint8 * 128)()
        _check(_lib.sc_nccl_unique_id(buf), "nccl_unique_id")
        return bytes(buf)

    def step(self, epoch: int):
        loss, gn = _f64(), _f64()
        _check(_lib.sc_trainer_step(self.h, epoch, C.byref(loss), C.byref(gn)), "step")
        return loss.value, gn.value

    def stage_features(self, features=None, host_ptr: Optional[int] = None, device_ptr: Optional[int] = None):
        """Copy the next step's features (n x d) while the current step runs; the next step() uses them."""
        if device_ptr is not None:
            _check(_lib.sc_trainer_stage_features(self.h, _vp(device_ptr), 1), "stage_features")
        elif host_ptr is not None:
            _check(_lib.sc_trainer_stage_features(self.h, _vp(host_ptr), 0), "stage_features")
        else:
            f = np.ascontiguousarray(features, np.float32)
            if f.shape != (self.g.num_nodes, self.g.dim):
                raise ValueError("stage_features: features must be num_nodes x d")
            self._staged = f  # keep the host buffer alive until the copy has run
            _check(_lib.sc_trainer_stage_features(self.h, _ptr(f), 0), "stage_features")

    def save_checkpoint(self, path: str):  # checkpoint.cpp:44-57 (model as SageModel<double>)
        _check(_lib.sc_trainer_save_checkpoint(self.h, os.fsencode(path)), "save_checkpoint")

    def load_checkpoint(self, path: str):  # checkpoint.cpp:59-84
        _check(_lib.sc_trainer_load_checkpoint(self.h, os.fsencode(path)), "load_checkpoint")

    def step_async(self, epoch: int):
        _check(_lib.sc_trainer_step_async(self.h, epoch), "step")

    def last(self):
        loss, gn = _f64(), _f64()
        _check(_lib.sc_trainer_last(self.h, C.byref(loss), C.byref(gn)), "step")
        return loss.value, gn.value

    def params(self) -> np.ndarray:
        out = np.zeros(self.param_count, np.float32)
        _check(_lib.sc_trainer_get_params(self.h, _ptr(out)))
        return out

    def set_params(self, theta):
        t = np.ascontiguousarray(theta, np.float32)
        if t.size != self.param_count:
            raise ValueError("set_params: wrong parameter count")
        _check(_lib.sc_trainer_set_params(self.h, _ptr(t)))

    def grads(self) -> np.ndarray:
        out = np.zeros(self.param_count, np.float32)
        _check(_lib.sc_trainer_get_grads(self.h, _ptr(out)))
        return out

    def part_grads(self, i: int) -> np.ndarray:
        out = np.zeros(self.param_count, np.float32)
        _check(_lib.sc_trainer_get_part_grads(self.h, i, _ptr(out)))
        return out

    def part_logits(self, i: int) -> np.ndarray:
        nl = self.part.part_sizes(i)[0]
        out = np.zeros((nl, self.g.num_classes), np.float32)
        _check(_lib.sc_trainer_get_part_logits(self.h, i, _ptr(out)))
        return out

    def part_loss(self, i: int) -> float:
        x = _f64()
        _check(_lib.sc_trainer_get_part_loss(self.h, i, C.byref(x)))
        return x.value

    def part_mask(self, i: int) -> int:
        x = _i32()
        _check(_lib.sc_trainer_get_part_mask(self.h, i, C.byref(x)))
        return x.value

    def evaluate(self):
        a, b, c = _f64(), _f64(), _f64()
        _check(_lib.sc_trainer_evaluate(self.h, C.byref(a), C.byref(b), C.byref(c)), "evaluate")
        return a.value, b.value, c.value

    def evaluate_mask(self, mask) -> float:
        """evaluate (trainer.cpp:101-112) of the current model over one split mask."""
        m = np.ascontiguousarray(mask, np.uint8)
        if m.size != self.g.num_nodes:
            raise ValueError("evaluate: mask length != node count")
        x = _f64()
        _check(_lib.sc_trainer_evaluate_mask(self.h, _ptr(m), C.byref(x)), "evaluate")
        return x.value

    def comm_audit(self):
        """CommAudit of the last step (trainer.hpp:61-76): (gradient floats, embedding floats)."""
        a, b = _u64(), _u64()
        _check(_lib.sc_trainer_comm_audit(self.h, C.byref(a), C.byref(b)))
        return a.value, b.value

    def fallback_count(self) -> int:
        """GEMMs that fell back to the fp32 SIMT kernels on the tensor-core path (0 on TMA-friendly shapes)."""
        x = _i64()
        _check(_lib.sc_trainer_fallback_count(self.h, C.byref(x)))
        return x.value

    def memory_mode(self) -> dict:
        """Device memory layout the trainer chose for this graph (compact activations, shared caches)."""
        f, b = C.c_int32(), _i64()
        _check(_lib.sc_trainer_memory_mode(self.h, C.byref(f), C.byref(b)))
        return {"compact_activations": bool(f.value & 1), "shared_x0": bool(f.value & 2),
                "shared_logits": bool(f.value & 4), "arena_gb": round(b.value / 1e9, 2)}

    def debug_buffer(self, name: str, layer: int, dst_ptr: int, nbytes: int):
        """Device-to-device copy of a trainer activation buffer (the last local partition's cache)."""
        _check(_lib.sc_trainer_debug_buffer(self.h, name.encode(), layer, _vp(dst_ptr), nbytes), "debug_buffer")

    def profile(self, enable: bool = True):
        _check(_lib.sc_trainer_profile(self.h, int(enable)))

    def kernel_times(self):
        cnt = _i32()
        _check(_lib.sc_trainer_kernel_times(self.h, None, None, None, 0, C.byref(cnt)))
        k = cnt.value
        names = (C.c_char_p * k)()
        ms = (_f64 * k)()
        by = (_f64 * k)()
        _check(_lib.sc_trainer_kernel_times(self.h, names, ms, by, k, C.byref(cnt)))
        return {names[i].decode(): (ms[i], by[i]) for i in range(k)}

    def kernel_flops(self):
        """{group: algorithmic GEMM flops of the last step} (2MNK; fp16x3 issues 3x that on the MMAs)."""
        names = list(self.kernel_times())
        fl = (_f64 * max(len(names), 1))()
        cnt = _i32()
        _check(_lib.sc_trainer_kernel_flops(self.h, fl, len(names), C.byref(cnt)))
        return {n: fl[i] for i, n in enumerate(names)}

    def close(self):
        if getattr(self, "h", None):
            _lib.sc_trainer_destroy(self.h)
            self.h = None

    def __del__(self):
        self.close()


@dataclass
class CommAudit:  # trainer.hpp:61-67
    gradient_floats_per_epoch: List[int] = field(default_factory=list)
    embedding_floats: int = 0


@dataclass
class CommReport:  # trainer.hpp:48-53
    mode: str
    floats_per_iteration: int
    gradient_floats: int
    embedding_floats: int


def comm_volume(mode: str, num_parts: int, param_count: int, num_layers: int, hidden_dim: int,
                total_halo: int) -> CommReport:  # trainer.cpp:38-49
    a, b, c = _u64(), _u64(), _u64()
    _check(_lib.sc_comm_volume({"cofree": 0, "halo_sync_model": 1}[mode], num_parts, param_count, num_layers,
                               hidden_dim, total_halo, C.byref(a), C.byref(b), C.byref(c)), "comm_volume")
    return CommReport(mode, a.value, b.value, c.value)


def expected_rf_random(num_parts: int, degree: int) -> float:  # partition.cpp:344-349
    x = _f64()
    _check(_lib.sc_expected_rf_random(num_parts, degree, C.byref(x)), "expected_rf_random")
    return x.value


def imbalance_lower_bound(num_parts: int, max_degree: int, min_degree: int) -> float:  # partition.cpp:351-362
    x = _f64()
    _check(_lib.sc_imbalance_lower_bound(num_parts, max_degree, min_degree, C.byref(x)), "imbalance_lower_bound")
    return x.value


def evaluate(model, g: Graph, mask, hidden: Sequence[int]) -> float:
    """evaluate (trainer.cpp:101-112): full-graph metric of a flat model (for_each_matrix
    order; hidden = the resolved per-layer dims) over one split mask, forward-only on the device."""
    theta = np.ascontiguousarray(model, np.float32)
    h = np.ascontiguousarray(hidden, np.int32)
    m = np.ascontiguousarray(mask, np.uint8)
    if m.size != g.num_nodes:
        raise ValueError("evaluate: mask length != node count")
    if theta.size != param_count(g.dim, list(h), g.num_classes):
        raise ValueError("evaluate: model does not match the graph's dims")
    x = _f64()
    _check(_lib.sc_evaluate(g.ctx.h, g.h, _ptr(theta), _ptr(h) if h.size else None, h.size, _ptr(m), C.byref(x)),
           "evaluate")
    return x.value


@dataclass
class TrainResult:  # trainer.hpp:71-75
    model: np.ndarray
    metrics: List[EpochMetrics]
    audit: CommAudit = field(default_factory=CommAudit)


def train_full_graph(g: Graph, config: TrainConfig, evaluate: bool = True) -> TrainResult:
    """train_full_graph (trainer.hpp:164-200): the whole graph as one partition — every edge in
    part 0, local ids = global ids, unit loss weights on the train mask, no DropEdge — through the
    same device trainer (the reference's p = 1 degeneracy, test_trainer.cpp:69-79)."""
    from dataclasses import replace
    part = build_vertex_cut(g, 1, np.zeros(g.num_edges(), np.int32))
    cfg = replace(config, reweight="none", use_dropedge=False)
    res = train_cofree(g, part, cfg, evaluate)
    for m in res.metrics:
        m.comm_floats = 0  # nothing is exchanged (trainer.hpp:197)
    return res


def train_cofree(g: Graph, part: VertexCutPartition, config: TrainConfig, evaluate: bool = True) -> TrainResult:
    """train_cofree (trainer.cpp:119 / trainer.hpp:202-313): per-epoch step, Adam,
    and (like the reference) a full-graph evaluation after every epoch."""
    t = CoFreeTrainer(g, part, config)
    metrics = []
    audit = CommAudit()
    for epoch in range(config.epochs):
        loss, gn = t.step(epoch)
        audit.gradient_floats_per_epoch.append(t.comm_audit()[0])
        tr, va, te = t.evaluate() if evaluate else (0.0, 0.0, 0.0)
        metrics.append(EpochMetrics(epoch, loss, tr, va, te, gn, part.num_parts * t.param_count))
    return TrainResult(t.params(), metrics, audit)
