"""The aggregation kernels at every row width the trainer uses (nn.hpp:222-230 / 277-288), bitwise
against the oracle's restatement (float sums in CSR order, then * inv) on a vertex-cut partition with
a DropEdge mask: rows of H <= 128 floats and <= 64 CSR slots run several per warp
(spmm_narrow_kernel, e.g. the projected top layer's Cp = 48), longer rows and wider H a warp per row
(spmm_kernel; 40 rows of ~150 slots here). A hub row above kHeavySlots (4096 CSR slots) takes the
segmented path (ordered segment partials: tolerance); every other row is bitwise."""
import os

import numpy as np
import pytest

from cpu_libs import oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def part0():
    from paper_2308_03209_b200 import sagecut as sc
    rng = np.random.default_rng(5)
    n, m = 60_000, 500_000
    uv = rng.integers(0, n, size=(m, 2), dtype=np.int32)
    hub = np.stack([np.zeros(12000, np.int32), rng.integers(1, n, size=12000, dtype=np.int32)], axis=1)
    # rows above the narrow kernel's 64 CSR slots but below the hub threshold: the warp-per-row pass
    mid = np.stack([np.repeat(np.arange(1, 41, dtype=np.int32), 300), rng.integers(41, n, size=40 * 300, dtype=np.int32)],
                   axis=1)
    g, _ = sc.build_graph(n, np.concatenate([uv, hub, mid]))
    part = sc.partition_random(g, 2, 0)
    a = part.part(0)
    masks = sc.precompute_masks(len(a.edges), 3, 0.5, 11)
    return sc, a, masks.masks[1]


@pytest.mark.parametrize("H", [8, 12, 16, 20, 32, 48, 64, 100, 256])
def test_spmm_widths_bitwise(part0, H):
    sc, a, mask = part0
    O = oracle()
    rng = np.random.default_rng(H)
    n = len(a.nodes)
    deg = np.diff(a.adj_offsets)
    light = deg <= 4096
    assert (~light).sum() >= 1  # the hub row takes the segmented path
    src = rng.standard_normal((n, H), dtype=np.float32)
    msg = np.maximum(rng.standard_normal((n, H), dtype=np.float32), 0)
    for bwd in (0, 1):
        got = sc.debug_spmm(bwd, a.adj_offsets, a.adj_neighbors, a.adj_edge_ids, src, edge_mask=mask,
                            msg=msg if bwd else None)
        ref = O.spmm(bwd, a.adj_offsets, a.adj_neighbors, a.adj_edge_ids, mask, src, msg=msg if bwd else None,
                     threads=os.cpu_count() or 8)
        assert int((got[light] != ref[light]).sum()) == 0, (H, bwd)
        d = np.abs(got[~light] - ref[~light]).max() / np.abs(ref[~light]).max()
        assert d <= 1e-5, (H, bwd, d)


@pytest.mark.parametrize("H", [8, 12, 48, 64, 128])
def test_projected_top_layer_sums_bitwise(part0, H):
    """The projected top layer's two aggregations (sc_debug_spmm modes 2 / 3): the backward's
    sum_kept inv[nbr] src[nbr] and the forward's addend + inv * sum_kept src[nbr], bitwise against the
    oracle's restatement on inv-scaled rows (inv = 1 / masked degree in fp32, as inv_degree)."""
    sc, a, mask = part0
    O = oracle()
    rng = np.random.default_rng(100 + H)
    n = len(a.nodes)
    off = a.adj_offsets
    light = np.diff(off) <= 4096
    cs = np.concatenate([[0], np.cumsum(mask[a.adj_edge_ids].astype(np.int64))])
    deg = cs[off[1:]] - cs[off[:-1]]  # kept CSR slots per row (masked_degrees, nn.hpp:174-188)
    inv = np.where(deg > 0, np.float32(1) / np.maximum(deg, 1).astype(np.float32), np.float32(0)).astype(np.float32)
    src = rng.standard_normal((n, H), dtype=np.float32)
    add = rng.standard_normal((n, H), dtype=np.float32)
    ones = np.ones((n, H), np.float32)
    got = sc.debug_spmm(2, off, a.adj_neighbors, a.adj_edge_ids, src, edge_mask=mask)
    ref = O.spmm(1, off, a.adj_neighbors, a.adj_edge_ids, mask, (src * inv[:, None]).astype(np.float32), msg=ones,
                 threads=os.cpu_count() or 8)
    assert int((got[light] != ref[light]).sum()) == 0, H
    assert np.abs(got[~light] - ref[~light]).max() / np.abs(ref[~light]).max() <= 1e-5
    got = sc.debug_spmm(3, off, a.adj_neighbors, a.adj_edge_ids, src, edge_mask=mask, msg=add)
    ref = add + O.spmm(0, off, a.adj_neighbors, a.adj_edge_ids, mask, src, threads=os.cpu_count() or 8)
    assert int((got[light] != ref[light]).sum()) == 0, H
    assert np.abs(got[~light] - ref[~light]).max() / np.abs(ref[~light]).max() <= 1e-5
