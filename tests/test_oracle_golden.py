"""CPU: the oracle against its golden fixtures (tests/golden, made by make_golden.py).

* fedavg / adapter layout: bit-exact against outputs of the reference's own launcher.fedavg and
  AdapterParams.zeros (/root/reference/pkg/src/coserve/launcher.py:28-80).
* LoRA forward/backward: against an independent torch-float64-autograd formulation.  Y, dB, dX
  and dA share the oracle's rounding points exactly (rel 1e-12; the backward's dH is exact, as
  the device's bf16 hi+lo pair carries it); the single-rounding variant (dh_mode="bf16") is
  shown to miss SURVEY §8(c)'s 1e-3 on dA, which is why the device does not use it.
* the reference's own FedAvg property tests (tests/test_launcher.py:41-82) re-run on the oracle.
"""

import os

import numpy as np
import pytest

import oracle

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _rel(a, b):
    return float(np.linalg.norm(np.asarray(a, np.float64) - b) / max(np.linalg.norm(b), 1e-300))


def test_bf16_rounding_matches_torch():
    import torch
    g = np.random.default_rng(0)
    x = np.concatenate([g.standard_normal(10000).astype(np.float32) * 10 ** g.uniform(-8, 8, 10000)
                        .astype(np.float32), np.array([0.0, -0.0, 1e38, -1e38, 65504.0], np.float32)])
    ref = torch.from_numpy(x).to(torch.bfloat16).float().numpy()
    assert np.array_equal(oracle.bf16_round(x), ref)


def test_fedavg_matches_reference_bitwise():
    d = np.load(os.path.join(GOLD, "fedavg_ref.npz"))
    ci = 0
    while f"case{ci}_k" in d:
        k = int(d[f"case{ci}_k"])
        clients = [(d[f"case{ci}_b{j}"], d[f"case{ci}_a{j}"]) for j in range(k)]
        b, a = oracle.fedavg(clients)
        assert np.array_equal(b, d[f"case{ci}_mean_b"]) and np.array_equal(a, d[f"case{ci}_mean_a"])
        ci += 1
    assert ci == 5
    # adapter layout convention: b_mat (d, r), a_mat (r, l)
    assert tuple(d["zeros_b_shape"]) == (64, 8) and tuple(d["zeros_a_shape"]) == (8, 48)


def test_fedavg_reference_properties():
    """The reference's FedAvg tests (tests/test_launcher.py:41-82) on the oracle."""
    g = np.random.default_rng(3)

    def ad(d=8, l=8, r=2):
        return g.normal(size=(d, r)), g.normal(size=(r, l))

    one = ad()
    out = oracle.fedavg([one])
    assert out[0] is one[0] and out[1] is one[1]  # single client: same objects back
    z = (np.zeros((4, 2)), np.zeros((2, 4)))
    t = (np.full((4, 2), 2.0), np.full((2, 4), 2.0))
    b, a = oracle.fedavg([z, t])
    assert np.all(b == 1.0) and np.all(a == 1.0)
    with pytest.raises(oracle.AggregationError, match="client 1"):
        oracle.fedavg([ad(d=8), ad(d=4)])
    for _ in range(200):
        k = int(g.integers(1, 6))
        cl = [ad(4, 4, 2) for _ in range(k)]
        b, a = oracle.fedavg(cl)
        perm = [cl[i] for i in g.permutation(k)]
        b2, a2 = oracle.fedavg(perm)
        assert np.allclose(b, b2, atol=1e-12) and np.allclose(a, a2, atol=1e-12)
        st = np.stack([c[0] for c in cl])
        assert np.all(b <= st.max(0) + 1e-12) and np.all(b >= st.min(0) - 1e-12)


@pytest.mark.parametrize("seed", [0, 1])
def test_lora_oracle_vs_autograd(seed):
    d = np.load(os.path.join(GOLD, "lora_autograd.npz"))
    p = f"s{seed}_"
    meta = d[p + "meta"]
    K, r, r_pad, n_ad, T_tr, ta = (int(v) for v in meta[:6])
    subs = tuple(int(v) for v in meta[6:])
    f = lambda k: oracle.bits_to_f32(d[p + k])  # noqa: E731
    X, W, A, B, dY = f("X"), f("W"), f("A"), f("B"), f("dY")
    scale, row_ad = d[p + "scale"], d[p + "row_ad"]
    Y, H16 = oracle.lora_forward(X, W, A, B, scale, row_ad, subs, r_pad)
    assert _rel(Y, d[p + "Y"]) < 1e-12
    dX, dB, dAT, _ = oracle.lora_backward(dY, X[:T_tr], H16[:T_tr], W, A[ta], B[ta],
                                          float(scale[ta]), subs, r_pad)
    assert _rel(dB, d[p + "dB"]) < 1e-12
    assert _rel(dAT.T, d[p + "dA"]) < 1e-12
    assert _rel(dX, d[p + "dX"]) < 1e-12
    # the single-rounding variant stays within bf16 output tolerance on dX, not 1e-3 on dA
    dX1, _, dAT1, _ = oracle.lora_backward(dY, X[:T_tr], H16[:T_tr], W, A[ta], B[ta],
                                           float(scale[ta]), subs, r_pad, dh_mode="bf16")
    assert _rel(dX1, d[p + "dX"]) < 4e-3
    assert 1e-4 < _rel(dAT1.T, d[p + "dA"]) < 1e-2


def test_adamw_matches_torch():
    import torch
    g = np.random.default_rng(1)
    p0 = g.standard_normal((16, 8)).astype(np.float32)
    st = oracle.AdamWState(np.zeros_like(p0), np.zeros_like(p0))
    tp = torch.nn.Parameter(torch.from_numpy(p0.copy()))
    opt = torch.optim.AdamW([tp], lr=1e-3, weight_decay=0.01, foreach=False)
    p = p0
    for _ in range(5):
        gr = g.standard_normal((16, 8)).astype(np.float32)
        p = oracle.adamw_step(p, gr, st, lr=1e-3, wd=0.01)
        tp.grad = torch.from_numpy(gr)
        opt.step()
    assert np.allclose(p, tp.detach().numpy(), rtol=1e-6, atol=1e-7)


@pytest.mark.parametrize("shape", ["6x40", "33x512"])
def test_cross_entropy_oracle_vs_autograd(shape):
    """oracle.cross_entropy (K7's restatement) against torch float64 F.cross_entropy + autograd
    (tests/golden/make_golden.py, ignore_index rows included)."""
    d = np.load(os.path.join(GOLD, "ce_autograd.npz"))
    z, y = d[f"ce_{shape}_logits"], d[f"ce_{shape}_labels"]
    loss_rows, mean, dz = oracle.cross_entropy(z, y)
    assert abs(mean - float(d[f"ce_{shape}_loss"])) < 1e-12
    np.testing.assert_allclose(dz, d[f"ce_{shape}_dlogits"], rtol=0, atol=1e-14)
    assert loss_rows[1] == 0.0 and np.all(dz[1] == 0.0)  # the ignored row


def test_paged_attention_oracle_vs_torch_sdpa():
    """oracle.paged_attention (K8's restatement) against torch float64 scaled_dot_product_attention
    on the same sequences laid out contiguously: a causal prefill sequence and decode rows with
    GQA (torch's reference attention, an independent formulation; the reference has none)."""
    import torch
    import torch.nn.functional as F
    g = np.random.default_rng(3)
    H, KV, D, page = 4, 2, 128, 8
    lens = [5, 19]  # sequence 0: decode row at position 4; sequence 1: prefill rows 0..18
    npg = [(n + page - 1) // page for n in lens]
    n_pages = sum(npg) + 2
    perm = g.permutation(n_pages)
    bt = np.zeros((2, max(npg)), np.int32)
    bt[0, :npg[0]] = perm[:npg[0]]
    bt[1, :npg[1]] = perm[npg[0]:npg[0] + npg[1]]
    kc = g.standard_normal((n_pages, KV, page, D))
    vc = g.standard_normal((n_pages, KV, page, D))
    row_seq = [0] + [1] * lens[1]
    row_pos = [lens[0] - 1] + list(range(lens[1]))
    q = g.standard_normal((len(row_seq), H * D))
    got = oracle.paged_attention(q, kc, vc, bt, row_seq, row_pos, H, KV)

    def contiguous(s):
        j = np.arange(lens[s])
        return (torch.tensor(kc[bt[s][j // page], :, j % page]),
                torch.tensor(vc[bt[s][j // page], :, j % page]))
    # decode row: attends to all 5 tokens of sequence 0
    K0, V0 = contiguous(0)
    qd = torch.tensor(q[0]).view(H, 1, D)
    ref0 = F.scaled_dot_product_attention(qd, K0.permute(1, 0, 2).repeat_interleave(H // KV, 0),
                                          V0.permute(1, 0, 2).repeat_interleave(H // KV, 0))
    np.testing.assert_allclose(got[0], ref0.reshape(-1).numpy(), rtol=1e-10, atol=1e-10)
    # prefill rows: causal over sequence 1
    K1, V1 = contiguous(1)
    qp = torch.tensor(q[1:]).view(lens[1], H, D).permute(1, 0, 2)
    ref1 = F.scaled_dot_product_attention(qp, K1.permute(1, 0, 2).repeat_interleave(H // KV, 0),
                                          V1.permute(1, 0, 2).repeat_interleave(H // KV, 0),
                                          is_causal=True)
    np.testing.assert_allclose(got[1:], ref1.permute(1, 0, 2).reshape(lens[1], -1).numpy(),
                               rtol=1e-10, atol=1e-10)


def test_causal_attention_oracle_vs_torch_autograd():
    """Pin K9's oracle (oracle.causal_attention fwd + bwd, packed causal sequences, GQA) against
    torch float64 autograd of softmax attention written independently (masked full matrices)."""
    import numpy as np
    import torch
    import oracle
    g = np.random.default_rng(3)
    lens, H, Hk, D = [5, 1, 9], 4, 2, 16
    T = sum(lens)
    seq = np.concatenate([[0], np.cumsum(lens)])
    q = g.standard_normal((T, H * D))
    k = g.standard_normal((T, Hk * D))
    v = g.standard_normal((T, Hk * D))
    do = g.standard_normal((T, H * D))
    out, lse2, (dq, dk, dv) = oracle.causal_attention(q, k, v, seq, H, Hk, dout=do)
    tq, tk, tv = (torch.tensor(a, requires_grad=True) for a in (q, k, v))
    seg = np.repeat(np.arange(len(lens)), lens)
    allowed = torch.tensor((seg[:, None] == seg[None, :]) & (np.arange(T)[:, None] >= np.arange(T)[None, :]))
    outs = []
    for h in range(H):
        hk = h // (H // Hk)
        s = tq[:, h * D:(h + 1) * D] @ tk[:, hk * D:(hk + 1) * D].T * D ** -0.5
        s = s.masked_fill(~allowed, float("-inf"))
        outs.append(torch.softmax(s, dim=1) @ tv[:, hk * D:(hk + 1) * D])
        if h == 0:
            lse_h0 = torch.logsumexp(s, dim=1) / np.log(2.0)
    o = torch.cat(outs, dim=1)
    o.backward(torch.tensor(do))
    assert np.allclose(out, o.detach().numpy(), atol=1e-12)
    assert np.allclose(lse2[0], lse_h0.detach().numpy(), atol=1e-12)
    for a, t in ((dq, tq), (dk, tk), (dv, tv)):
        assert np.allclose(a, t.grad.numpy(), atol=1e-10)
