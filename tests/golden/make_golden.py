"""Generate the golden fixtures that pin the CPU oracle (run in the build container).

1. fedavg_ref.npz — outputs of the REFERENCE's own ``coserve.launcher.fedavg`` and
   ``AdapterParams.zeros`` (/root/reference/pkg/src/coserve/launcher.py:28-80), imported from the
   read-only reference tree, on seeded random client sets.  oracle.fedavg must reproduce them
   bit for bit.
2. lora_autograd.npz — an INDEPENDENT formulation of the LoRA projection's forward and gradients:
   torch float64 autograd through ``y = x W^T + round_bf16(s x A^T) B^T`` (straight-through
   rounding), with the gradients taken by autograd instead of the oracle's hand-written
   formulas.  The reference itself has no LoRA arithmetic, so this is the strongest
   available pin for the restatement ("parity unpinned" for LoRA numerics).

Usage: python tests/golden/make_golden.py   (writes next to this file)
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SRC = "/root/reference/pkg/src"


def make_fedavg():
    sys.path.insert(0, REF_SRC)
    from coserve.launcher import AdapterParams, fedavg  # the reference implementation

    out = {}
    rng = np.random.default_rng(20261017)
    cases = [(1, 64, 64, 8), (2, 64, 64, 8), (3, 64, 64, 8), (5, 16, 32, 4), (3, 8, 8, 2)]
    for ci, (k, d, l, r) in enumerate(cases):
        clients = [AdapterParams(rng.normal(size=(d, r)), rng.normal(size=(r, l))) for _ in range(k)]
        mean = fedavg(clients)
        out[f"case{ci}_k"] = np.array(k)
        for j, c in enumerate(clients):
            out[f"case{ci}_b{j}"] = c.b_mat
            out[f"case{ci}_a{j}"] = c.a_mat
        out[f"case{ci}_mean_b"] = mean.b_mat
        out[f"case{ci}_mean_a"] = mean.a_mat
    z = AdapterParams.zeros(64, 48, 8)
    out["zeros_b_shape"] = np.array(z.b_mat.shape)
    out["zeros_a_shape"] = np.array(z.a_mat.shape)
    np.savez_compressed(os.path.join(HERE, "fedavg_ref.npz"), **out)


def bf16_bits(x: np.ndarray) -> np.ndarray:
    import torch
    return torch.from_numpy(np.ascontiguousarray(x, np.float32)).to(torch.bfloat16).view(
        torch.int16).numpy().view(np.uint16)


def from_bits(b: np.ndarray) -> np.ndarray:
    return (b.astype(np.uint32) << 16).view(np.float32)


def make_lora(seed: int, out: dict):
    import torch

    g = np.random.default_rng(seed)
    K, subs, r, r_pad, n_ad = 64, (64, 32, 32), 8, 16, 3
    N = sum(subs)
    R = len(subs) * r_pad
    T_tr, T_inf = 24, 8
    T = T_tr + T_inf
    row_ad = np.array([1] * T_tr + [0, 2, 2, 1, 0, 0, 2, 1], np.int32)  # train adapter 1
    X = from_bits(bf16_bits(g.standard_normal((T, K)).astype(np.float32)))
    W = from_bits(bf16_bits(0.05 * g.standard_normal((N, K)).astype(np.float32)))
    A = np.zeros((n_ad, R, K), np.float32)
    B = np.zeros((n_ad, N, r_pad), np.float32)
    bnd = np.cumsum([0] + list(subs))
    for a in range(n_ad):
        for s in range(len(subs)):
            A[a, s * r_pad:s * r_pad + r] = from_bits(bf16_bits(
                g.uniform(-0.2, 0.2, (r, K)).astype(np.float32)))
            B[a, bnd[s]:bnd[s + 1], :r] = from_bits(bf16_bits(
                0.1 * g.standard_normal((subs[s], r)).astype(np.float32)))
    scale = np.array([2.0, 1.5, 3.0], np.float32)
    dY = from_bits(bf16_bits(g.standard_normal((T_tr, N)).astype(np.float32)))

    class RoundBF16(torch.autograd.Function):
        @staticmethod
        def forward(ctx, x):
            return x.float().to(torch.bfloat16).to(torch.float64)

        @staticmethod
        def backward(ctx, gy):
            return gy

    t = torch.from_numpy
    x = t(X).double()
    w = t(W).double()
    ta = 1  # trained adapter
    A_t = t(A[ta]).double().requires_grad_(True)
    B_t = t(B[ta]).double().requires_grad_(True)
    x_tr = x[:T_tr].clone().requires_grad_(True)
    Y = torch.zeros(T, N, dtype=torch.float64)
    for row in range(T):
        a = int(row_ad[row])
        xa = x_tr[row] if row < T_tr else x[row]
        Aa = A_t if a == ta else t(A[a]).double()
        Ba = B_t if a == ta else t(B[a]).double()
        H = RoundBF16.apply(float(scale[a]) * (xa @ Aa.T))
        y = xa @ w.T
        parts = []
        for s in range(len(subs)):
            parts.append(y[bnd[s]:bnd[s + 1]] + H[s * r_pad:(s + 1) * r_pad] @ Ba[bnd[s]:bnd[s + 1]].T)
        Y[row] = torch.cat(parts)
    loss = (Y[:T_tr] * t(dY).double()).sum()  # upstream gradient dY for the training rows
    loss.backward()
    p = f"s{seed}_"
    out[p + "X"] = bf16_bits(X)
    out[p + "W"] = bf16_bits(W)
    out[p + "A"] = bf16_bits(A)
    out[p + "B"] = bf16_bits(B)
    out[p + "dY"] = bf16_bits(dY)
    out[p + "scale"] = scale
    out[p + "row_ad"] = row_ad
    out[p + "meta"] = np.array([K, r, r_pad, n_ad, T_tr, ta] + list(subs), np.int64)
    out[p + "Y"] = Y.detach().numpy()
    out[p + "dX"] = x_tr.grad.numpy()
    out[p + "dA"] = A_t.grad.numpy()   # [R, K]
    out[p + "dB"] = B_t.grad.numpy()   # [N, r_pad]


def make_ce(out: dict):
    """3. ce_autograd.npz — torch float64 F.cross_entropy (mean over non-ignored rows,
    ignore_index=-100) and its autograd gradient w.r.t. the logits: an independent formulation
    pinning oracle.cross_entropy (the reference has no loss arithmetic, perf.py:92-126)."""
    import torch
    g = np.random.default_rng(7)
    for T, V in ((6, 40), (33, 512)):
        z = (g.standard_normal((T, V)) * 3).astype(np.float32)
        y = g.integers(0, V, T).astype(np.int64)
        y[1] = -100  # an ignored row
        zt = torch.tensor(z, dtype=torch.float64, requires_grad=True)
        loss = torch.nn.functional.cross_entropy(zt, torch.tensor(y), ignore_index=-100)
        loss.backward()
        out[f"ce_{T}x{V}_logits"] = z
        out[f"ce_{T}x{V}_labels"] = y
        out[f"ce_{T}x{V}_loss"] = np.float64(loss.item())
        out[f"ce_{T}x{V}_dlogits"] = zt.grad.numpy()


if __name__ == "__main__":
    ce = {}
    make_ce(ce)
    np.savez_compressed(os.path.join(HERE, "ce_autograd.npz"), **ce)
    make_fedavg()
    lo = {}
    for seed in (0, 1):
        make_lora(seed, lo)
    np.savez_compressed(os.path.join(HERE, "lora_autograd.npz"), **lo)
    for f in ("fedavg_ref.npz", "lora_autograd.npz", "ce_autograd.npz"):
        print(f, os.path.getsize(os.path.join(HERE, f)), "bytes")
