"""The aggregation kernels at every row width the trainer uses (nn.hpp:222-230 / 277-288), bitwise
against the oracle's restatement (float sums in CSR order, then * inv) on a vertex-cut partition with
a DropEdge mask: H = 8 .. 64 run several rows per warp (spmm_narrow_kernel, e.g. the projected top
layer's Cp = 48), H = 100 .. 256 a warp per row (spmm_kernel). A hub row above kHeavySlots (4096 CSR
slots) takes the segmented path (ordered segment partials: tolerance); every other row is bitwise."""
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
    g, _ = sc.build_graph(n, np.concatenate([uv, hub]))
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
