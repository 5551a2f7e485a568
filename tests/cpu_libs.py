"""ctypes front-end for the two CPU checkers — TEST INFRASTRUCTURE ONLY.

* ``oracle/liboracle.so``          — the CPU restatement (prefix ``or_``)
* ``oracle/_ref/libsagecut_ref.so`` — the unmodified reference sources compiled
  behind oracle/eigen_shim (prefix ``ref_``)

Both export the same flat C ABI (oracle/sagecut_oracle.h), so one wrapper
drives either. Only tests/, __graft_entry__.smoke() and bench.py's reference
leg import this module.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_SO = os.path.join(ROOT, "oracle", "liboracle.so")
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libsagecut_ref.so")

_p = C.c_void_p
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")


def _ptr_or_null(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


@dataclass
class PartArrays:
    nodes: np.ndarray
    edges: np.ndarray  # [m_i, 2] local endpoints
    edge_gids: np.ndarray
    local_deg: np.ndarray
    offsets: np.ndarray
    nbrs: np.ndarray
    eids: np.ndarray
    g2l: np.ndarray


class CpuLib:
    """One of the CPU checkers behind its flat C ABI."""

    def __init__(self, path: str, prefix: str):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle`")
        self.path = path
        self.lib = C.CDLL(path)
        self.pre = prefix
        L, f = self.lib, self._f
        f("last_error").restype = C.c_char_p
        f("mix64").restype = C.c_uint64
        f("mix64").argtypes = [C.c_uint64]
        f("substream").restype = C.c_uint64
        f("substream").argtypes = [C.c_uint64, C.c_char_p, C.c_int, C.c_uint64, C.c_uint64]
        f("rng_draws").argtypes = [C.c_uint64, C.c_int, C.c_uint64, C.c_int64, _p, _p]
        f("graph_build").restype = _p
        f("graph_build").argtypes = [C.c_int32, _i32p, C.c_int64]
        f("graph_sbm").restype = _p
        f("graph_sbm").argtypes = [C.c_int32, C.c_int, C.c_double, C.c_double, C.c_int, C.c_double, C.c_uint64]
        f("graph_free").argtypes = [_p]
        f("graph_num_nodes").restype = C.c_int32
        f("graph_num_nodes").argtypes = [_p]
        f("graph_num_edges").restype = C.c_int64
        f("graph_num_edges").argtypes = [_p]
        f("graph_edges").argtypes = [_p, _i32p]
        f("graph_csr").argtypes = [_p, _i32p, _i32p, _i32p, _i32p]
        f("graph_features").argtypes = [_p, _f64p]
        f("graph_labels").argtypes = [_p, _i32p]
        f("graph_masks").argtypes = [_p, _u8p, _u8p, _u8p]
        f("graph_set_data").argtypes = [_p, _f32p, C.c_int, _i32p, C.c_int, _u8p, _u8p, _u8p]
        f("graph_set_multilabels").argtypes = [_p, _f32p, C.c_int]
        f("evaluate").argtypes = [_p, _f64p, _i32p, C.c_int, _u8p, C.POINTER(C.c_double)]
        f("comm_volume").argtypes = [C.c_int, C.c_int, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, _u64p]
        f("expected_rf_random").argtypes = [C.c_int, C.c_int64, C.POINTER(C.c_double)]
        f("imbalance_lower_bound").argtypes = [C.c_int, C.c_int64, C.c_int64, C.POINTER(C.c_double)]
        if prefix == "or_":
            f("spmm").argtypes = [C.c_int, C.c_int64, C.c_int32, _p, _p, _p, _p, _p, _p, _p, C.c_int]
            f("spmm").restype = None
        f("partition").restype = _p
        f("partition").argtypes = [_p, C.c_int, C.c_int, C.c_uint64]
        f("partition_ne").restype = _p
        f("partition_ne").argtypes = [_p, C.c_int, C.c_uint64, C.c_double, C.c_char_p, C.c_int64]
        f("edge_cut_greedy").argtypes = [_p, C.c_int, C.c_uint64, _i32p]
        f("edge_cut_stats").argtypes = [_p, C.c_int, _i32p, _p, _p, _p, _p, _p]
        f("edge_cut_to_vertex_cut").restype = _p
        f("edge_cut_to_vertex_cut").argtypes = [_p, C.c_int, _i32p, C.c_uint64]
        f("build_vertex_cut").restype = _p
        f("build_vertex_cut").argtypes = [_p, C.c_int, _i32p]
        f("partition_free").argtypes = [_p]
        f("partition_assignment").argtypes = [_p, _i32p]
        f("part_sizes").argtypes = [_p, C.c_int, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
        f("part_arrays").argtypes = [_p, C.c_int] + [_i32p] * 7 + [_p]
        f("replication_stats").argtypes = [_p, _p, _i32p, C.POINTER(C.c_double), C.POINTER(C.c_double),
                                           C.POINTER(C.c_double), C.POINTER(C.c_int64)]
        f("weights").argtypes = [_p, _p, C.c_int, _f64p]
        f("precompute_masks").argtypes = [C.c_int64, C.c_int, C.c_double, C.c_uint64, _u8p]
        f("select_mask").argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, C.c_int]
        f("init_params").restype = C.c_int64
        f("init_params").argtypes = [C.c_int, _i32p, C.c_int, C.c_int, C.c_uint64, C.c_int, _p]
        f("trainer_new").restype = _p
        f("trainer_new").argtypes = [_p, _p, _i32p, C.c_int, C.c_double, C.c_int, C.c_int, C.c_int, C.c_int,
                                     C.c_double, C.c_uint64, C.c_int, C.c_int]
        f("trainer_free").argtypes = [_p]
        f("trainer_step").argtypes = [_p, C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_double)]
        f("trainer_param_count").restype = C.c_int64
        f("trainer_param_count").argtypes = [_p]
        for name in ("trainer_params", "trainer_gathered"):
            f(name).argtypes = [_p, _f64p]
        f("trainer_set_params").argtypes = [_p, _f64p]
        f("trainer_part_grads").argtypes = [_p, C.c_int, _f64p]
        f("trainer_part_logits").argtypes = [_p, C.c_int, _f64p]
        f("trainer_part_loss").restype = C.c_double
        f("trainer_part_loss").argtypes = [_p, C.c_int]
        f("trainer_part_mask").argtypes = [_p, C.c_int]
        f("trainer_eval").argtypes = [_p] + [C.POINTER(C.c_double)] * 3
        f("trainer_time_part_step").restype = C.c_double
        f("trainer_time_part_step").argtypes = [_p, C.c_int, C.c_int, C.c_int]
        del L

    def _f(self, name):
        return getattr(self.lib, self.pre + name)

    def _check(self, status, what):
        if status != 0:
            msg = self._f("last_error")().decode()
            raise {1: ValueError, 2: RuntimeError}.get(status, AssertionError)(f"{what}: {msg}")

    def _checked_handle(self, h, what):
        if not h:
            raise ValueError(f"{what}: {self._f('last_error')().decode()}")
        return h

    # ---- rng ----
    def mix64(self, x):
        return int(self._f("mix64")(x))

    def substream(self, seed, tag, *idx):
        a = idx[0] if len(idx) > 0 else 0
        b = idx[1] if len(idx) > 1 else 0
        return int(self._f("substream")(seed, tag.encode(), len(idx), a, b))

    def rng_draws(self, seed, kind, n, arg=0):
        """kind: 0 next_u64, 1 next_below(arg), 2 next_double, 3 next_gaussian."""
        u = np.zeros(n, np.uint64)
        d = np.zeros(n, np.float64)
        self._f("rng_draws")(seed, kind, arg, n, u.ctypes.data_as(C.c_void_p), d.ctypes.data_as(C.c_void_p))
        return u if kind in (0, 1) else d

    # ---- analytic models (trainer.cpp:38-49, partition.cpp:344-362) ----
    def comm_volume(self, mode, p, params, layers, hidden, halo):
        out = np.zeros(3, np.uint64)
        self._check(self._f("comm_volume")({"cofree": 0, "halo_sync_model": 1}[mode], p, params, layers, hidden,
                                           halo, out), "comm_volume")
        return [int(x) for x in out]

    def expected_rf_random(self, p, degree):
        x = C.c_double()
        self._check(self._f("expected_rf_random")(p, degree, C.byref(x)), "expected_rf_random")
        return x.value

    def imbalance_lower_bound(self, p, max_d, min_d):
        x = C.c_double()
        self._check(self._f("imbalance_lower_bound")(p, max_d, min_d, C.byref(x)), "imbalance_lower_bound")
        return x.value

    def spmm(self, bwd, offsets, nbrs, eids, mask, src, msg=None, threads=8):
        """The restatement's masked mean aggregation (nn.hpp:209-230) or its transpose (:277-288)."""
        assert self.pre == "or_"
        off = np.ascontiguousarray(offsets, np.int64)
        nb = np.ascontiguousarray(nbrs, np.int32)
        ei = np.ascontiguousarray(eids, np.int32)
        src = np.ascontiguousarray(src, np.float32)
        n, H = len(off) - 1, src.shape[1]
        out = np.empty((n, H), np.float32)
        mk = None if mask is None else np.ascontiguousarray(mask, np.uint8)
        ms = None if msg is None else np.ascontiguousarray(msg, np.float32)
        self._f("spmm")(int(bwd), n, H, off.ctypes.data, nb.ctypes.data, ei.ctypes.data, _ptr_or_null(mk),
                        src.ctypes.data, _ptr_or_null(ms), out.ctypes.data, threads)
        return out

    # ---- graphs ----
    def graph_build(self, n, uv):
        uv = np.ascontiguousarray(uv, np.int32).reshape(-1, 2)
        return Graph(self, self._checked_handle(self._f("graph_build")(n, uv, len(uv)), "build_graph"))

    def graph_sbm(self, n, classes, p_in, p_out, d, noise, seed):
        h = self._f("graph_sbm")(n, classes, p_in, p_out, d, noise, seed)
        return Graph(self, self._checked_handle(h, "gen_homophilic_sbm"))

    # ---- dropedge / init ----
    def precompute_masks(self, m, k, ratio, seed):
        out = np.zeros(k * m, np.uint8)
        self._check(self._f("precompute_masks")(m, k, ratio, seed, out), "precompute_masks")
        return out.reshape(k, m)

    def select_mask(self, seed, part, epoch, k):
        return int(self._f("select_mask")(seed, part, epoch, k))

    def init_params(self, in_dim, hidden, classes, seed, f32=True):
        h = np.asarray(hidden, np.int32)
        n = self._f("init_params")(in_dim, h, len(h), classes, seed, int(f32), None)
        if n < 0:
            raise ValueError(self._f("last_error")().decode())
        out = np.zeros(n, np.float64)
        self._f("init_params")(in_dim, h, len(h), classes, seed, int(f32), out.ctypes.data_as(C.c_void_p))
        return out


class Graph:
    def __init__(self, lib: CpuLib, handle):
        self.lib, self.h = lib, handle

    def __del__(self):
        try:
            self.lib._f("graph_free")(self.h)
        except Exception:
            pass

    @property
    def n(self):
        return int(self.lib._f("graph_num_nodes")(self.h))

    @property
    def m(self):
        return int(self.lib._f("graph_num_edges")(self.h))

    def edges(self):
        out = np.zeros((self.m, 2), np.int32)
        self.lib._f("graph_edges")(self.h, out.reshape(-1))
        return out

    def csr(self):
        off = np.zeros(self.n + 1, np.int32)
        nb = np.zeros(2 * self.m, np.int32)
        ei = np.zeros(2 * self.m, np.int32)
        dg = np.zeros(self.n, np.int32)
        self.lib._f("graph_csr")(self.h, off, nb, ei, dg)
        return off, nb, ei, dg

    def features(self, d):
        out = np.zeros(self.n * d, np.float64)
        self.lib._f("graph_features")(self.h, out)
        return out.reshape(self.n, d)

    def labels(self):
        out = np.zeros(self.n, np.int32)
        self.lib._f("graph_labels")(self.h, out)
        return out

    def masks(self):
        t, v, s = (np.zeros(self.n, np.uint8) for _ in range(3))
        self.lib._f("graph_masks")(self.h, t, v, s)
        return t, v, s

    def set_data(self, features, labels, classes, train, val, test):
        feats = np.ascontiguousarray(features, np.float32)
        self.lib._check(self.lib._f("graph_set_data")(
            self.h, feats.reshape(-1), feats.shape[1], np.ascontiguousarray(labels, np.int32), classes,
            np.ascontiguousarray(train, np.uint8), np.ascontiguousarray(val, np.uint8),
            np.ascontiguousarray(test, np.uint8)), "set_data")

    def set_multilabels(self, y):
        y = np.ascontiguousarray(y, np.float32)
        self.lib._check(self.lib._f("graph_set_multilabels")(self.h, y.reshape(-1), y.shape[1]), "set_multilabels")

    def evaluate(self, theta, hidden, mask):
        """evaluate (trainer.cpp:101-112) of a flat f64 model over one mask."""
        x = C.c_double()
        self.lib._check(self.lib._f("evaluate")(self.h, np.ascontiguousarray(theta, np.float64),
                                                np.ascontiguousarray(hidden, np.int32), len(hidden),
                                                np.ascontiguousarray(mask, np.uint8), C.byref(x)), "evaluate")
        return x.value

    def partition(self, algo, p, seed):
        algo_id = {"random": 0, "dbh": 1, "ne": 2, "ec2vc": 3}[algo]
        h = self.lib._f("partition")(self.h, algo_id, p, seed)
        return Partition(self, self.lib._checked_handle(h, f"partition_{algo}"), p)

    def partition_ne(self, p, seed, slack=1.1):
        """partition_ne with its warnings (partition.cpp:116-201)."""
        buf = C.create_string_buffer(1 << 16)
        h = self.lib._f("partition_ne")(self.h, p, seed, slack, buf, len(buf))
        part = Partition(self, self.lib._checked_handle(h, "partition_ne"), p)
        w = buf.value.decode()
        return part, (w.split("\n") if w else [])

    def edge_cut_greedy(self, p, seed):
        """partition_edge_cut_greedy's node assignment (partition.cpp:233-278)."""
        out = np.zeros(self.n, np.int32)
        self.lib._check(self.lib._f("edge_cut_greedy")(self.h, p, seed, out), "edge_cut_greedy")
        return out

    def edge_cut(self, p, node_assign):
        """edge_cut_from_assignment (partition.cpp:203-231): kept counts, cut edges, halo sets."""
        na = np.ascontiguousarray(node_assign, np.int32)
        kept = np.zeros(p, np.int64)
        halo = np.zeros(p, np.int64)
        ncut = C.c_int64()
        f = self.lib._f("edge_cut_stats")
        self.lib._check(f(self.h, p, na, kept.ctypes.data_as(_p), C.byref(ncut), halo.ctypes.data_as(_p), None, None),
                        "edge_cut_stats")
        cut = np.zeros(ncut.value, np.int32)
        nodes = np.zeros(int(halo.sum()), np.int32)
        self.lib._check(f(self.h, p, na, kept.ctypes.data_as(_p), C.byref(ncut), halo.ctypes.data_as(_p),
                          cut.ctypes.data_as(_p), nodes.ctypes.data_as(_p)), "edge_cut_stats")
        bounds = np.concatenate([[0], np.cumsum(halo)])
        return kept, cut, [nodes[bounds[i]:bounds[i + 1]] for i in range(p)]

    def edge_cut_to_vertex_cut(self, p, node_assign, seed):
        h = self.lib._f("edge_cut_to_vertex_cut")(self.h, p, np.ascontiguousarray(node_assign, np.int32), seed)
        return Partition(self, self.lib._checked_handle(h, "edge_cut_to_vertex_cut"), p)

    def build_vertex_cut(self, p, assign):
        h = self.lib._f("build_vertex_cut")(self.h, p, np.ascontiguousarray(assign, np.int32))
        return Partition(self, self.lib._checked_handle(h, "build_vertex_cut"), p)


class Partition:
    def __init__(self, g: Graph, handle, p):
        self.g, self.lib, self.h, self.p = g, g.lib, handle, p

    def __del__(self):
        try:
            self.lib._f("partition_free")(self.h)
        except Exception:
            pass

    def assignment(self):
        out = np.zeros(self.g.m, np.int32)
        self.lib._f("partition_assignment")(self.h, out)
        return out

    def sizes(self, i):
        nl, ne = C.c_int64(), C.c_int64()
        self.lib._f("part_sizes")(self.h, i, C.byref(nl), C.byref(ne))
        return nl.value, ne.value

    def part(self, i) -> PartArrays:
        nl, ne = self.sizes(i)
        a = PartArrays(np.zeros(nl, np.int32), np.zeros((ne, 2), np.int32), np.zeros(ne, np.int32),
                       np.zeros(nl, np.int32), np.zeros(nl + 1, np.int32), np.zeros(2 * ne, np.int32),
                       np.zeros(2 * ne, np.int32), np.zeros(self.g.n, np.int32))
        self.lib._f("part_arrays")(self.h, i, a.nodes, a.edges.reshape(-1), a.edge_gids, a.local_deg, a.offsets,
                                   a.nbrs, a.eids, a.g2l.ctypes.data_as(C.c_void_p))
        return a

    def stats(self):
        rfv = np.zeros(self.g.n, np.int32)
        rf, eb, nb = C.c_double(), C.c_double(), C.c_double()
        dup = C.c_int64()
        self.lib._check(self.lib._f("replication_stats")(self.h, self.g.h, rfv, C.byref(rf), C.byref(eb),
                                                          C.byref(nb), C.byref(dup)), "replication_stats")
        return dict(per_node_rf=rfv, rf=rf.value, edge_balance=eb.value, node_balance=nb.value,
                    duplicated_nodes=dup.value)

    def weights(self, scheme):
        sid = {"dar": 0, "vanilla_inv": 1, "none": 2}[scheme]
        total = sum(self.sizes(i)[0] for i in range(self.p))
        out = np.zeros(total, np.float64)
        self.lib._check(self.lib._f("weights")(self.g.h, self.h, sid, out), "weights")
        res, k = [], 0
        for i in range(self.p):
            nl = self.sizes(i)[0]
            res.append(out[k:k + nl].copy())
            k += nl
        return res

    def trainer(self, hidden, lr=0.01, loss="softmax_ce", reweight="dar", dropedge=False, k=10, ratio=0.5,
                seed=0, f32=True, workers=1):
        h = np.asarray(hidden, np.int32)
        t = self.lib._f("trainer_new")(self.g.h, self.h, h, len(h), lr, {"softmax_ce": 0, "bce": 1}[loss],
                                       {"dar": 0, "vanilla_inv": 1, "none": 2}[reweight], int(dropedge), k,
                                       ratio, seed, int(f32), workers)
        return Trainer(self, self.lib._checked_handle(t, "trainer"))


class Trainer:
    def __init__(self, part: Partition, handle):
        self.part, self.lib, self.h = part, part.lib, handle
        self.nparam = int(self.lib._f("trainer_param_count")(self.h))

    def __del__(self):
        try:
            self.lib._f("trainer_free")(self.h)
        except Exception:
            pass

    def step(self, epoch):
        loss, gn = C.c_double(), C.c_double()
        self.lib._check(self.lib._f("trainer_step")(self.h, epoch, C.byref(loss), C.byref(gn)), "step")
        return loss.value, gn.value

    def params(self):
        out = np.zeros(self.nparam, np.float64)
        self.lib._f("trainer_params")(self.h, out)
        return out

    def set_params(self, theta):
        self.lib._f("trainer_set_params")(self.h, np.ascontiguousarray(theta, np.float64))

    def gathered(self):
        out = np.zeros(self.nparam, np.float64)
        self.lib._f("trainer_gathered")(self.h, out)
        return out

    def part_grads(self, i):
        out = np.zeros(self.nparam, np.float64)
        self.lib._f("trainer_part_grads")(self.h, i, out)
        return out

    def part_logits(self, i, classes):
        nl = self.part.sizes(i)[0]
        out = np.zeros(nl * classes, np.float64)
        self.lib._f("trainer_part_logits")(self.h, i, out)
        return out.reshape(nl, classes)

    def part_loss(self, i):
        return float(self.lib._f("trainer_part_loss")(self.h, i))

    def part_mask(self, i):
        return int(self.lib._f("trainer_part_mask")(self.h, i))

    def eval(self):
        a, b, c = C.c_double(), C.c_double(), C.c_double()
        self.lib._f("trainer_eval")(self.h, C.byref(a), C.byref(b), C.byref(c))
        return a.value, b.value, c.value

    def time_part_step(self, i, epoch, reps=1):
        return float(self.lib._f("trainer_time_part_step")(self.h, i, epoch, reps))


def oracle() -> CpuLib:
    return CpuLib(ORACLE_SO, "or_")


def reference() -> CpuLib:
    return CpuLib(REF_SO, "ref_")
