"""Kernel-level numerics on the B200: each collm kernel against a plain PyTorch fp32 computation
of the same op on the same bf16 inputs (the layer-level parity against the oracle is in
test_gpu_parity.py).  Tolerances: bf16 outputs |err| <= 1e-2*max|ref| + 1e-3 (one bf16 rounding
of the output plus fp32 summation-order differences); fp32 outputs rel. Frobenius <= 1e-4."""

import math

import pytest
import torch

pytestmark = pytest.mark.gpu


def _bf(*shape, scale=1.0, gen=None):
    return (torch.randn(*shape, generator=gen) * scale).to(torch.bfloat16).cuda()


def _close_bf16(out, ref):
    err = (out.float() - ref).abs().max().item()
    tol = 1e-2 * ref.abs().max().item() + 1e-3
    assert err <= tol, f"max err {err} > tol {tol}"


@pytest.fixture(scope="module", autouse=True)
def lib():
    from paper_2604_16400_b200 import _lib, build
    build.build()
    return _lib.load()


GEMM_VARIANTS = [("1", "dp"), ("1", "hybrid"), ("2", "dp"), ("2", "hybrid"), ("2", "split2"),
                 ("2", "dp", "2"), ("2", "hybrid", "2"), ("2", "split2", "2"), ("2", "dp", "3")]


@pytest.fixture(params=GEMM_VARIANTS, ids=lambda v: f"cg{v[0]}-{v[1]}" + (f"-mc{v[2]}" if len(v) > 2 else ""))
def gemm_variant(request, monkeypatch):
    """Force each kernel variant (CTA or CTA-pair tiles; data-parallel, stream-K, or split-2
    where every tile's K is halved over two CTA pairs that swap half-tile partials — shapes
    with too many tiles for split-2 fall back to the cost model's choice; mc2: 4-CTA clusters of
    two pairs halving K (split-2 over DSMEM); mc3: 4-CTA clusters of two pairs on adjacent N tiles
    multicasting their shared A boxes)."""
    monkeypatch.setenv("COLLM_GEMM_CG", request.param[0])
    monkeypatch.setenv("COLLM_GEMM_SCHED", request.param[1])
    monkeypatch.setenv("COLLM_GEMM_MC", request.param[2] if len(request.param) > 2 else "1")
    return request.param


@pytest.mark.parametrize("M,N,K,bn", [(128, 256, 64, 256), (200, 384, 320, 0), (77, 136, 200, 128),
                                      (1024, 4096, 4096, 0), (512, 1024, 12288, 128),
                                      (300, 688, 256, 128)])
def test_gemm_plain(M, N, K, bn, gemm_variant):
    from paper_2604_16400_b200 import ops
    g = torch.Generator().manual_seed(M * 7 + N)
    A = _bf(M, K, gen=g)
    B = _bf(N, K, scale=0.05, gen=g)
    Y = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    ops.gemm_lora(A, B, Y, bn=bn)
    torch.cuda.synchronize()
    _close_bf16(Y, A.float() @ B.float().t())


@pytest.mark.parametrize("r_pad,n_sub,bn", [(16, 1, 256), (16, 3, 128), (32, 1, 128), (64, 2, 256),
                                            (48, 1, 128)])
def test_gemm_lora_slots(r_pad, n_sub, bn, gemm_variant):
    """Forward-style LoRA K-extension: multiple slots per tile, per-sub H column offsets."""
    from paper_2604_16400_b200 import ops
    g = torch.Generator().manual_seed(r_pad * 31 + n_sub)
    M, K = 600, 256
    TM = 256  # slot-plan granularity
    n_each = 256 if bn == 256 else 128
    N = n_each * n_sub
    n_ad = 5
    R = r_pad * n_sub
    A = _bf(M, K, gen=g)
    W = _bf(N, K, scale=0.05, gen=g)
    # tile slots: tile0 adapters [0, 3], tile1 [3, 1, 4], tile2 [2]
    row_ad = torch.tensor([0] * 100 + [3] * 60 + [1] * 50 + [4] * 46 + [2] * 44 + [1] * 200 +
                          [0] * 30 + [4] * 70, dtype=torch.int32)
    tiles_adapters = []
    for m in range(math.ceil(M / TM)):
        seen = []
        for a in row_ad[m * TM:(m + 1) * TM].tolist():
            if a not in seen:
                seen.append(a)
        tiles_adapters.append(seen)
    tsp = [0]
    slots = []
    for s in tiles_adapters:
        slots += s
        tsp.append(len(slots))
    H = torch.randn(M, R, generator=g).to(torch.bfloat16)
    Hslots = torch.zeros(len(slots) * TM, R, dtype=torch.bfloat16)
    for t in range(M):
        m = t // TM
        s = tsp[m] + tiles_adapters[m].index(int(row_ad[t]))
        Hslots[s * TM + t % TM] = H[t]
    LB = (torch.randn(n_ad, N, r_pad, generator=g) * 0.1).to(torch.bfloat16)
    Y = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    sub_n = [i * n_each for i in range(n_sub + 1)]
    sub_h = [i * r_pad for i in range(n_sub)]
    ops.gemm_lora(A, W, Y, Hslots=Hslots.cuda(), h_rows=Hslots.shape[0],
                  LB=LB.cuda().view(n_ad * N, r_pad), lb_rows=n_ad * N,
                  tile_slot_ptr=torch.tensor(tsp, dtype=torch.int32).cuda(),
                  slot_adapter=torch.tensor(slots, dtype=torch.int32).cuda(), lora_rank=r_pad,
                  lb_rows_per_adapter=N, sub_n_start=sub_n, sub_h_col=sub_h, bn=bn)
    torch.cuda.synchronize()
    ref = A.float().cpu() @ W.float().cpu().t()
    for t in range(M):
        a = int(row_ad[t])
        for s in range(n_sub):
            cols = slice(sub_n[s], sub_n[s + 1])
            ref[t, cols] += H[t, sub_h[s]:sub_h[s] + r_pad].float() @ LB[a, cols].float().t()
    _close_bf16(Y.cpu(), ref)


@pytest.mark.parametrize("R,K", [(16, 512), (32, 520), (48, 4096), (64, 688), (112, 11008)])
def test_shrink(R, K):
    """K1 over ragged 16-row tiles (incl. a 1-row tile), K = 520 (not a multiple of 16) up to
    11008, rank groups of 8..64 — against a CPU fp32 reference; two launches are bitwise
    identical (fixed in-cluster reduction order)."""
    from paper_2604_16400_b200 import ops
    g = torch.Generator().manual_seed(R)
    T, n_ad = 150, 4
    X = _bf(T, K, gen=g)
    A = _bf(n_ad, R, K, scale=0.05, gen=g)
    scale = torch.tensor([1.0, 2.0, 0.5, 3.0]).cuda()
    seg = [0, 40, 41, 90, 150]
    seg_ad = [2, 0, 3, 1]
    tiles = []
    for s in range(len(seg_ad)):
        for r in range(seg[s], seg[s + 1], 16):
            tiles.append((r, min(16, seg[s + 1] - r), seg_ad[s]))
    tt = torch.tensor(tiles, dtype=torch.int32).cuda()
    groups = [(i, min(64, R - i), 0, K) for i in range(0, R, 64)]
    H32 = torch.zeros(T, R, device="cuda")
    H16 = torch.zeros(T, R, dtype=torch.bfloat16, device="cuda")
    ops.lora_shrink(X, A, tt, len(tiles), scale, groups, R, H32=H32, H16=H16)
    H32b = torch.zeros_like(H32)
    ops.lora_shrink(X, A, tt, len(tiles), scale, groups, R, H32=H32b)
    torch.cuda.synchronize()
    assert torch.equal(H32, H32b)
    ref = torch.zeros(T, R)
    for s in range(len(seg_ad)):
        a = seg_ad[s]
        rows = slice(seg[s], seg[s + 1])
        ref[rows] = scale[a].item() * (X[rows].float().cpu() @ A[a].float().cpu().t())
    rel = (H32.cpu() - ref).norm() / ref.norm()
    assert rel < 1e-4, rel
    _close_bf16(H16.cpu(), ref)


@pytest.mark.parametrize("R,K,n_ctas,dh,n_ad", [(16, 512, 2, False, 5), (48, 4096, 16, False, 5),
                                                (96, 1024, 8, False, 5), (192, 5120, 16, False, 5),
                                                (16, 1024, 8, False, 40), (48, 2048, 16, False, 40),
                                                (48, 11008, 8, True, 5), (192, 2048, 4, True, 5),
                                                # the whole GPU (large passes): many split-K parts
                                                (48, 4096, 148, False, 5), (16, 1024, 148, False, 40),
                                                (192, 2048, 148, True, 5)])
def test_shrink_tc(R, K, n_ctas, dh, n_ad):
    """K1 on the rank-space partition (collm_lora_shrink_tc: TMA k-block boxes -> tcgen05 ->
    TMEM): items of <= 128 rows merged from ragged 16-row tiles (1-row tile, a base-only
    segment, a >128-row run, rows crossing a 256-row slot tile), fused rank groups up to 192,
    K up to 11008; per-sub K ranges with one adapter (the dH shape, ``dh``).  H32 vs an fp32
    reference (rel <= 1e-4), H16 / H16lo pair, Hslots (own slot = H16, other slots of the row's
    256-row tile = 0), bitwise repeatable."""
    import numpy as np
    from paper_2604_16400_b200 import ops, segments
    g = torch.Generator().manual_seed(R + K)
    if dh:
        seg, seg_ad = [0, 300], [3]
    elif n_ad == 5:
        seg, seg_ad = [0, 40, 41, 90, 150, 160, 430], [2, 0, 3, -1, 1, 4]
    else:  # many short runs of consecutive (and skipped) ids: windows stack several adapters
        ids = [i for i in range(n_ad) if i % 7 != 3]
        lens = [1 + (i * 5) % 11 for i in range(len(ids))]
        seg = [0] + list(np.cumsum(lens))
        seg_ad = ids
    T = seg[-1]
    X = _bf(T, K, gen=g)
    A = _bf(n_ad, R, K, scale=0.05, gen=g)
    scale = torch.tensor([0.25 * (1 + i % 7) for i in range(n_ad)]).cuda()
    host = segments.plan_segments(seg, seg_ad)
    if dh:  # per-sub K ranges (N ranges of the fused projection), one group per sub
        n_sub = 3 if R % 3 == 0 else 2
        rp = R // n_sub
        bnd = [0] + [K * (s + 1) // n_sub // 64 * 64 for s in range(n_sub - 1)] + [K]
        groups = [(s * rp, rp, bnd[s], bnd[s + 1]) for s in range(n_sub)]
    else:
        groups = [(0, R, 0, K)]
    tc = ops.shrink_tc_groups(groups)
    assert tc is not None
    items, ptr = segments.plan_shrink_windows(host, tc[0][1], n_ctas)
    it_d = torch.from_numpy(items).cuda()
    ptr_d = torch.from_numpy(ptr).cuda()
    H32 = torch.zeros(T, R, device="cuda")
    H16 = torch.zeros(T, R, dtype=torch.bfloat16, device="cuda")
    H16lo = torch.zeros(T, R, dtype=torch.bfloat16, device="cuda")
    dp = segments.DevicePlan(host, "cuda", tc_ctas=0)  # (its device row_adapter / slot tables)
    torch.cuda.synchronize()
    n_slots = host.n_slots
    Hs = torch.full((max(1, n_slots) * 256, R), 7.0, dtype=torch.bfloat16, device="cuda")
    kw = dict(H32=H32, H16=H16, H16lo=H16lo)
    if not dh:
        kw.update(Hslots=Hs, slot_of_row=dp.slot_of_row, tile_slot_ptr=dp.tile_slot_ptr)
    ra = dp.row_adapter
    a_stride = 0 if dh else None
    Ad = A[seg_ad[0]] if dh else A  # dH: one adapter's B_t^T-like [R, K] operand
    ops.lora_shrink_tc(X, Ad, it_d, ptr_d, n_ctas, ra, scale, tc, R, a_stride=a_stride, **kw)
    H32b = torch.zeros_like(H32)
    ops.lora_shrink_tc(X, Ad, it_d, ptr_d, n_ctas, ra, scale, tc, R, a_stride=a_stride, H32=H32b)
    torch.cuda.synchronize()
    assert torch.equal(H32, H32b)
    ref = torch.zeros(T, R)
    Xc, Ac = X.float().cpu(), A.float().cpu()
    for s in range(len(seg_ad)):
        a = seg_ad[s]
        if a < 0:
            continue
        rows = slice(seg[s], seg[s + 1])
        for ro, nr, klo, khi in groups:
            ref[rows, ro:ro + nr] = scale[a].item() * (Xc[rows, klo:khi] @ Ac[a, ro:ro + nr, klo:khi].t())
    has = torch.tensor(np.repeat(np.array(seg_ad) >= 0, np.diff(seg)))
    rel = (H32.cpu()[has] - ref[has]).norm() / ref.norm()
    assert rel < 1e-4, rel
    _close_bf16(H16.cpu()[has], ref[has])
    pair = H16.cpu().double() + H16lo.cpu().double()
    assert torch.allclose(pair[has], H32.cpu().double()[has], rtol=1e-5, atol=1e-7)
    if not dh:
        tsp = host.tile_slot_ptr
        slot_of_row = dp.slot_of_row.cpu().numpy()
        Hs_c = Hs.cpu()
        for t in range(T):
            m = t // 256
            for sl in range(tsp[m], tsp[m + 1]):
                got = Hs_c[sl * 256 + t % 256]
                want = H16.cpu()[t] if (has[t] and sl == slot_of_row[t]) else torch.zeros(R, dtype=torch.bfloat16)
                assert torch.equal(got, want), (t, sl)


@pytest.fixture(params=[1, 0], ids=["tcgen05", "mma"])
def reduce_impl(request):
    from paper_2604_16400_b200 import ops
    prev = ops.reduce_impl()
    ops.set_reduce_impl(request.param)
    yield request.param
    ops.set_reduce_impl(prev)


@pytest.mark.parametrize("T,P,Q,tsplit,v2,accum", [
    (1, 64, 16, 1, False, False), (300, 200, 48, 1, True, False), (513, 384, 8, 4, False, True),
    (1000, 128, 64, 8, True, True), (4096, 256, 24, 2, True, False), (129, 520, 40, 2, False, False)])
def test_reduce_store_grad_vs_fp32(reduce_impl, T, P, Q, tsplit, v2, accum):
    """K5 grad mode against fp32 torch: ragged T (1, 129, 513 — not whole 128-row chunks), P not
    a multiple of the 128-row tile, Q not a multiple of 16, the V2 (bf16 lo half) operand,
    accumulation into an existing grad, T splits; a second launch is bitwise identical."""
    from paper_2604_16400_b200 import _lib, ops
    g = torch.Generator().manual_seed(T + P + Q)
    U = _bf(T, P + 16, gen=g)
    V = _bf(T, Q + 24, gen=g)
    V2 = (_bf(T, Q + 24, gen=g).float() * 1e-3).to(torch.bfloat16) if v2 else None
    init = torch.randn(P, Q + 4, generator=g).cuda()
    outs = []
    for _ in range(2):
        grad = init.clone() if accum else torch.zeros(P, Q + 4, device="cuda")
        grp = ops.reduce_group(U, V, u_off=16, P=P, v_off=8, Q=Q, ldc=Q + 4, c_col_off=4, grad=grad,
                               V2=V2)
        ops.lora_reduce(T, [grp], _lib.MODE_STORE_GRAD, accum_in=accum, grad_scale=0.5,
                        tsplit=tsplit)
        torch.cuda.synchronize()
        outs.append(grad)
    Vf = V[:, 8:8 + Q].float() + (V2[:, 8:8 + Q].float() if v2 else 0)
    ref = 0.5 * U[:, 16:16 + P].float().t() @ Vf
    got = outs[0][:, 4:]
    if accum:
        ref = ref + init[:, 4:]
    assert torch.equal(outs[0][:, :4], init[:, :4] if accum else torch.zeros_like(init[:, :4]))
    rel = ((got - ref).norm() / ref.norm()).item()
    assert rel < 1e-5, rel
    assert torch.equal(outs[0], outs[1])


def test_reduce_many_tensors_falls_back(reduce_impl):
    """More distinct U / V tensors than the tcgen05 K5 maps in one launch (16 groups, 48 tensors):
    the launch still runs (mma.sync kernel) and matches fp32 torch."""
    from paper_2604_16400_b200 import _lib, ops
    g = torch.Generator().manual_seed(11)
    T = 200
    groups, refs, grads, keep = [], [], [], []
    for i in range(16):
        U, V, V2 = _bf(T, 64, gen=g), _bf(T, 16, gen=g), _bf(T, 16, scale=1e-3, gen=g)
        keep += [U, V, V2]  # the group table holds raw pointers
        grad = torch.zeros(64, 16, device="cuda")
        groups.append(ops.reduce_group(U, V, P=64, Q=16, ldc=16, grad=grad, V2=V2))
        refs.append(U.float().t() @ (V.float() + V2.float()))
        grads.append(grad)
    ops.lora_reduce(T, groups, _lib.MODE_STORE_GRAD)
    torch.cuda.synchronize()
    for got, ref in zip(grads, refs):
        assert ((got - ref).norm() / ref.norm()).item() < 1e-5


def test_reduce_adamw(reduce_impl):
    from paper_2604_16400_b200 import _lib, ops
    g = torch.Generator().manual_seed(5)
    T, P, Q = 300, 200, 48
    U = _bf(T, P + 8, gen=g)
    V = _bf(T, Q + 16, gen=g)
    grad = torch.zeros(P, Q, device="cuda")
    grp = ops.reduce_group(U, V, u_off=8, P=P, v_off=16, Q=Q, ldc=Q, grad=grad)
    ops.lora_reduce(T, [grp], _lib.MODE_STORE_GRAD)
    torch.cuda.synchronize()
    ref = U[:, 8:8 + P].float().t() @ V[:, 16:16 + Q].float()
    rel = ((grad - ref).norm() / ref.norm()).item()
    assert rel < 1e-5, rel
    # fused AdamW from the same reduction, two groups in one launch (second: different T-split)
    master = torch.randn(P, Q, generator=g).cuda()
    m = torch.zeros_like(master)
    v = torch.zeros_like(master)
    same = torch.empty(P, Q, dtype=torch.bfloat16, device="cuda")
    trans = torch.empty(Q, P, dtype=torch.bfloat16, device="cuda")
    master2 = torch.randn(64, 16, generator=g).cuda()
    m2, v2 = torch.zeros_like(master2), torch.zeros_like(master2)
    trans2 = torch.empty(16, 64, dtype=torch.bfloat16, device="cuda")
    lr, b1, b2, eps, wd = 1e-3, 0.9, 0.999, 1e-8, 0.01
    p_ref = master.clone()
    p2_ref = master2.clone()
    groups = [ops.reduce_group(U, V, u_off=8, P=P, v_off=16, Q=Q, ldc=Q, master=master, m=m, v=v,
                               out_same=same, out_trans=trans, ld_trans=P),
              ops.reduce_group(U, V, u_off=0, P=64, v_off=0, Q=16, ldc=16, master=master2, m=m2,
                               v=v2, out_trans=trans2, ld_trans=64)]
    ops.lora_reduce(T, groups, _lib.MODE_ADAMW,
                    adamw=torch.tensor([lr, b1, b2, eps, wd, 1 - b1, 1 - b2]).cuda(), tsplit=3)
    torch.cuda.synchronize()
    for pr, gr, got in ((p_ref, ref.cuda(), master),
                        (p2_ref, (U[:, :64].float().t() @ V[:, :16].float()).cuda(), master2)):
        pr.mul_(1 - lr * wd)
        m_ref = (1 - b1) * gr
        v_ref = (1 - b2) * gr * gr
        pr -= (lr / (1 - b1)) * m_ref / (v_ref.sqrt() / math.sqrt(1 - b2) + eps)
        assert torch.allclose(got, pr, rtol=1e-5, atol=1e-6)
    assert torch.equal(same, master.to(torch.bfloat16))
    assert torch.equal(trans, master.to(torch.bfloat16).t())
    assert torch.equal(trans2, master2.to(torch.bfloat16).t())


@pytest.mark.parametrize("T,V", [(1, 512), (7, 4096), (64, 32000), (5, 128256)])
def test_cross_entropy_vs_oracle(T, V):
    """K7 against the oracle (float64 on the same bf16 logits): per-row loss and the mean to fp32
    precision, dlogits to bf16 rounding; an ignored row; the arrival counter is restored so a
    second launch is bitwise identical."""
    import numpy as np

    import oracle
    from paper_2604_16400_b200 import ops
    g = torch.Generator().manual_seed(T * 131 + V)
    z = (torch.randn(T, V, generator=g) * 4).to(torch.bfloat16).cuda()
    y = torch.randint(0, V, (T,), generator=g, dtype=torch.int32)
    if T > 1:
        y[T // 2] = -1
    y = y.cuda()
    loss_rows = torch.empty(T, dtype=torch.float32, device="cuda")
    mean = torch.empty(1, dtype=torch.float32, device="cuda")
    counter = torch.zeros(1, dtype=torch.int32, device="cuda")
    dz = torch.empty(T, V, dtype=torch.bfloat16, device="cuda")
    n_valid = int((y >= 0).sum().item())
    ops.cross_entropy(z, y, V, loss_rows=loss_rows, loss_mean=mean, counter=counter, dlogits=dz,
                      grad_scale=1.0 / n_valid)
    torch.cuda.synchronize()
    ref_rows, ref_mean, ref_dz = oracle.cross_entropy(z.float().cpu().numpy(), y.cpu().numpy())
    np.testing.assert_allclose(loss_rows.cpu().numpy(), ref_rows, rtol=2e-6, atol=2e-5)
    assert abs(mean.item() - ref_mean) <= 2e-6 * abs(ref_mean) + 1e-6
    _close_bf16(dz, torch.from_numpy(ref_dz).float().cuda())
    assert counter.item() == 0
    first = (loss_rows.clone(), mean.clone(), dz.clone())
    ops.cross_entropy(z, y, V, loss_rows=loss_rows, loss_mean=mean, counter=counter, dlogits=dz,
                      grad_scale=1.0 / n_valid)
    torch.cuda.synchronize()
    for a, b in zip(first, (loss_rows, mean, dz)):
        assert torch.equal(a, b)


@pytest.mark.parametrize("n_heads,n_kv", [(4, 4), (4, 2), (8, 2), (8, 1)])
def test_paged_attention_vs_oracle(n_heads, n_kv):
    """K8 over a shuffled paged KV cache: decode rows with contexts 1..700 (multi-split, split
    boundary 256/257), a prefill segment (causal, positions 0..n-1) and GQA — against the float64
    oracle (bf16 output tolerance); two launches bitwise identical (split combine order fixed,
    counters restored)."""
    import numpy as np

    import oracle
    from paper_2604_16400_b200 import ops
    g = torch.Generator().manual_seed(n_heads * 10 + n_kv)
    D, page = 128, 16
    ctxs = [1, 37, 256, 257, 700]          # decode sequences (context length incl. the new token)
    prefill = 23                           # one prefill sequence: rows at positions 0..22
    seq_lens = ctxs + [prefill]
    pages_per = [(n + page - 1) // page for n in seq_lens]
    n_pages = sum(pages_per) + 5
    perm = torch.randperm(n_pages, generator=g)
    bt = torch.zeros(len(seq_lens), max(pages_per), dtype=torch.int32)
    o = 0
    for s, npg in enumerate(pages_per):
        bt[s, :npg] = perm[o:o + npg].to(torch.int32)
        o += npg
    kc = (torch.randn(n_pages, n_kv, page, D, generator=g)).to(torch.bfloat16)
    vc = (torch.randn(n_pages, n_kv, page, D, generator=g)).to(torch.bfloat16)
    row_seq = [s for s in range(len(ctxs))] + [len(ctxs)] * prefill
    row_pos = [n - 1 for n in ctxs] + list(range(prefill))
    T = len(row_seq)
    q = (torch.randn(T, n_heads * D, generator=g) * 2).to(torch.bfloat16)
    out = torch.empty(T, n_heads * D, dtype=torch.bfloat16, device="cuda")
    args = dict(n_heads=n_heads, n_kv_heads=n_kv, max_ctx=max(seq_lens))
    rs = torch.tensor(row_seq, dtype=torch.int32).cuda()
    rp = torch.tensor(row_pos, dtype=torch.int32).cuda()
    ops.paged_attention(q.cuda(), kc.cuda(), vc.cuda(), bt.cuda(), rs, rp, out, **args)
    torch.cuda.synchronize()
    ref = oracle.paged_attention(q.float().numpy(), kc.float().numpy(), vc.float().numpy(),
                                 bt.numpy(), row_seq, row_pos, n_heads, n_kv)
    _close_bf16(out, torch.from_numpy(ref).float().cuda())
    out2 = torch.empty_like(out)
    ops.paged_attention(q.cuda(), kc.cuda(), vc.cuda(), bt.cuda(), rs, rp, out2, **args)
    torch.cuda.synchronize()
    assert torch.equal(out, out2)
    assert np.isfinite(out.float().cpu().numpy()).all()


@pytest.mark.parametrize("lens,n_heads,n_kv", [([512], 4, 4), ([1, 63, 64, 65, 200], 4, 2),
                                               ([130, 7, 300], 8, 2), ([1024], 2, 1),
                                               ([1] * 40 + [3, 17, 90] + [1] * 30, 4, 1),
                                               ([129, 1, 255, 384, 2], 4, 4),
                                               ([300, 5, 700], 8, 1), ([2048, 1000], 4, 1),
                                               # > 2 x 148 (tile, head) items: every persistent
                                               # CTA walks several items (Q / O / dQ buffers wrap)
                                               ([1500, 7, 1200, 1389], 16, 4)])
@pytest.mark.parametrize("impl", [1, 0], ids=["tcgen05", "mma"])
def test_flash_attention_vs_oracle(lens, n_heads, n_kv, impl):
    """K9: causal attention of packed sequences (ragged lengths incl. 1, tile boundaries 63/64/65,
    many 1-row decode sequences sharing tiles with short prefills, GQA G = 1/2/4) forward + backward against the float64 oracle; q/k/v are column views of one
    fused q|k|v buffer as in the step; the backward is bitwise repeatable."""
    import numpy as np
    import oracle
    from paper_2604_16400_b200 import ops
    g = torch.Generator().manual_seed(sum(lens) + n_heads)
    D = 128
    T = sum(lens)
    seq = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    W = (n_heads + 2 * n_kv) * D
    qkv = _bf(T, W, gen=g)
    q, k, v = qkv[:, :n_heads * D], qkv[:, n_heads * D:(n_heads + n_kv) * D], qkv[:, (n_heads + n_kv) * D:]
    dout = _bf(T, n_heads * D, gen=g)
    out = torch.zeros(T, n_heads * D, dtype=torch.bfloat16, device="cuda")
    lse = torch.zeros(n_heads, T, device="cuda")
    rows = ops.seq_rows(seq, "cuda")
    kw = dict(T=T, n_heads=n_heads, n_kv_heads=n_kv)
    prev = ops.flash_impl()
    ops.set_flash_impl(impl)
    try:
        ops.flash_attention(q, k, v, out, lse, *rows, **kw)
        dqkv = torch.zeros_like(qkv)
        dq, dk, dv = (dqkv[:, :n_heads * D], dqkv[:, n_heads * D:(n_heads + n_kv) * D],
                      dqkv[:, (n_heads + n_kv) * D:])
        delta = torch.zeros(n_heads, T, device="cuda")
        ops.flash_attention_bwd(q, k, v, out, dout, lse, delta, dq, dk, dv, *rows, **kw)
        dqkv2 = torch.zeros_like(qkv)
        ops.flash_attention_bwd(q, k, v, out, dout, lse, delta, dqkv2[:, :n_heads * D],
                                dqkv2[:, n_heads * D:(n_heads + n_kv) * D],
                                dqkv2[:, (n_heads + n_kv) * D:], *rows, **kw)
        torch.cuda.synchronize()
    finally:
        ops.set_flash_impl(prev)
    assert torch.equal(dqkv, dqkv2)
    f = lambda t: t.float().cpu().numpy()  # noqa: E731
    ref, lse_ref, (dq_r, dk_r, dv_r) = oracle.causal_attention(f(q), f(k), f(v), seq, n_heads, n_kv,
                                                               dout=f(dout))
    for got, want, what in ((f(out), ref, "out"), (f(dq), dq_r, "dq"), (f(dk), dk_r, "dk"),
                            (f(dv), dv_r, "dv")):
        err = np.abs(got - want).max()
        assert err <= 1e-2 * np.abs(want).max() + 1e-3, (what, err)
        rel = np.linalg.norm(got - want) / np.linalg.norm(want)
        assert rel <= 1e-2, (what, rel)
    assert np.abs(lse.cpu().numpy() - lse_ref).max() <= 1e-3
