"""fp64 PyTorch restatement of one partition's training step — TEST
INFRASTRUCTURE ONLY (a checker for shapes the C oracle cannot finish in seconds).

sage_forward / softmax_ce_loss / bce_loss / sage_backward of the reference
(proj/include/sagecut/nn.hpp:192-293, 317-378) in float64, on any torch device
(the headline-scale parity tests run it on the GPU next to the trainer, which
it never touches: inputs come from the library's C ABI as host arrays).
Validated against the oracle restatement's f64 mode in
tests/test_torch_ref_cpu.py (<= 1e-12). The aggregation is a cuSPARSE /
torch sparse CSR product: in f64 the summation order is immaterial at the
1e-6 level these checks resolve.
"""
from __future__ import annotations

import numpy as np
import torch


def unflatten(theta, d, hidden, C):
    """Flat for_each_matrix vector -> [(W_l, U_l)], head (nn.hpp:73-102 order, row-major)."""
    mats, k, inp = [], 0, d
    for h in hidden:
        W = theta[k:k + h * inp].reshape(h, inp)
        k += h * inp
        U = theta[k:k + h * (h + inp)].reshape(h, h + inp)
        k += h * (h + inp)
        mats.append((W, U))
        inp = h
    head = theta[k:k + C * inp].reshape(C, inp)
    return mats, head


def kept_adjacency(offsets, nbrs, eids, mask, n, device, dtype):
    """Symmetric 0/1 CSR of the kept slots (nn.hpp:222-230 / 277-288) and inv = 1/masked degree."""
    off = torch.as_tensor(np.asarray(offsets, np.int64), device=device)
    nb = torch.as_tensor(np.asarray(nbrs, np.int64), device=device)
    if mask is not None:
        keep = torch.as_tensor(np.asarray(mask, np.bool_), device=device)[torch.as_tensor(
            np.asarray(eids, np.int64), device=device)]
        deg = torch.zeros(n, dtype=torch.int64, device=device)
        rows = torch.repeat_interleave(torch.arange(n, device=device), off[1:] - off[:-1])
        deg.index_add_(0, rows, keep.to(torch.int64))
        nb = nb[keep]
        off = torch.cat([torch.zeros(1, dtype=torch.int64, device=device), torch.cumsum(deg, 0)])
    else:
        deg = off[1:] - off[:-1]
    A = torch.sparse_csr_tensor(off, nb, torch.ones(nb.numel(), dtype=dtype, device=device), size=(n, n))
    inv = torch.where(deg > 0, 1.0 / deg.clamp(min=1).to(dtype), torch.zeros((), dtype=dtype, device=device))
    return A, inv


def partition_step(theta, d, hidden, C, offsets, nbrs, eids, mask, x0, w, normalizer, labels=None, targets=None,
                   loss="softmax_ce", relu_masks=None, device="cpu", dtype=torch.float64, keep_pre=False):
    """One partition's forward + loss + backward. Returns dict with logits, loss (float), grads (flat,
    for_each_matrix order, numpy f64) and, if keep_pre, the pre-activations. relu_masks (optional list of
    bool tensors, one per layer): use these ReLU decisions in the backward instead of pre > 0 (to separate
    the effect of pre-activations that land on the other side of 0 from rounding)."""
    th = torch.as_tensor(np.asarray(theta, np.float64), device=device).to(dtype)
    mats, head = unflatten(th, d, hidden, C)
    n = x0.shape[0]
    A, inv = kept_adjacency(offsets, nbrs, eids, mask, n, device, dtype)
    h = torch.as_tensor(np.asarray(x0), device=device).to(dtype)
    inputs, pres, means = [], [], []
    for W, U in mats:  # nn.hpp:217-236
        inputs.append(h)
        pre = h @ W.T
        msg = pre.clamp(min=0)
        mean = (A @ msg) * inv[:, None]
        H = W.shape[0]
        h = mean @ U[:, :H].T + h @ U[:, H:].T
        pres.append(pre)
        means.append(mean)
        del msg
    emb = h
    logits = emb @ head.T
    wt = torch.as_tensor(np.asarray(w, np.float64), device=device).to(dtype)
    sc = (wt / normalizer)[:, None]
    if loss == "softmax_ce":  # nn.hpp:317-345
        y = torch.as_tensor(np.asarray(labels, np.int64), device=device)
        lse = torch.logsumexp(logits, dim=1)
        zy = logits.gather(1, y[:, None])[:, 0]
        total = float((wt * (lse - zy)).sum()) / normalizer
        G = torch.softmax(logits, dim=1)
        G[torch.arange(n, device=device), y] -= 1.0
        G = sc * G
    else:  # nn.hpp:348-378
        t = torch.as_tensor(np.asarray(targets), device=device).to(dtype)
        sp = logits.clamp(min=0) + torch.log1p(torch.exp(-logits.abs()))
        total = float((wt[:, None] * (sp - logits * t)).sum()) / normalizer
        G = sc * (torch.sigmoid(logits) - t)
    G = torch.where(wt[:, None] == 0, torch.zeros_like(G), G)
    grads_head = G.T @ emb  # nn.hpp:259-260
    dh = G @ head
    gW, gU = [None] * len(mats), [None] * len(mats)
    for l in range(len(mats) - 1, -1, -1):  # nn.hpp:262-291
        W, U = mats[l]
        H = W.shape[0]
        h_in, mean, pre = inputs[l], means[l], pres[l]
        gU[l] = torch.cat([dh.T @ mean, dh.T @ h_in], dim=1)
        dmean = dh @ U[:, :H]
        ddir = dh @ U[:, H:]
        dmsg = A @ (dmean * inv[:, None])  # the scatter of nn.hpp:277-286 on the symmetric kept adjacency
        gate = relu_masks[l] if relu_masks is not None else (pre > 0)
        dz = gate.to(dtype) * dmsg
        gW[l] = dz.T @ h_in
        dh = ddir + dz @ W
    flat = []
    for l in range(len(mats)):
        flat += [gW[l].reshape(-1), gU[l].reshape(-1)]
    flat.append(grads_head.reshape(-1))
    out = {"logits": logits, "loss": total, "grads": torch.cat(flat).double().cpu().numpy()}
    if keep_pre:
        out["pre"] = pres
    return out


def matrix_slices(d, hidden, C):
    """[(name, start, stop)] of every parameter matrix in the flat vector."""
    out, k, inp = [], 0, d
    for l, h in enumerate(hidden):
        out.append((f"W{l}", k, k + h * inp))
        k += h * inp
        out.append((f"U{l}", k, k + h * (h + inp)))
        k += h * (h + inp)
        inp = h
    out.append(("head", k, k + C * inp))
    return out
