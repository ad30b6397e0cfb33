"""GPU: the whole co-batched step (ReplicaStack) — stream overlap and CUDA-graph replay must not
change a single bit of the outputs or of the optimizer state (all kernels are deterministic and
the side-stream schedule only reorders independent work), and the stack's projections match the
oracle layer by layer."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _config(cfg_key):
    """A BASELINE config, optionally cut to its first layers ('llama2-7b:2')."""
    import dataclasses

    from paper_2604_16400_b200.configs import CONFIGS
    key, _, layers = cfg_key.partition(":")
    cfg = CONFIGS[key]
    if layers:
        cfg = dataclasses.replace(cfg, model=dataclasses.replace(cfg.model, layers=int(layers)))
    return cfg


def _stack(overlap, cfg_key="tiny", seed=0, mode="pdl"):
    from paper_2604_16400_b200.replica import ReplicaStack
    cfg = _config(cfg_key)
    st = ReplicaStack(cfg, "cuda", seed=seed)
    st.overlap = overlap
    st.overlap_mode = mode
    plan = st.plan(*cfg.batch(0))
    st.allocate(plan, distinct_synthetic=True)
    return st, plan


def _state(st):
    out = [st._acts["X"][-1].clone()]
    for p in st.projections():
        t = p.train_state
        out += [t.master_B.clone(), t.master_AT.clone(), p.A[t.adapter].clone(), p.B[t.adapter].clone()]
    return out


@pytest.mark.parametrize("cfg_key", ["tiny", "llama2-7b:2", "llama3-8b:1", "llama2-13b:1"])
def test_overlap_and_graph_bitwise(cfg_key):
    """At the tiny shape and at the real 7B/8B/13B shapes (few layers): the two-stream overlap
    (shrink || its GEMM's main loop, flag-signalled LoRA stages; K5 on the side stream) and CUDA
    graph replay give bitwise the serialized results — and never deadlock (a GEMM waiting on a
    shrink that cannot start would trap after the timeout)."""
    ref, plan = _stack(False, cfg_key)
    for _ in range(2):
        ref.run_step(plan)
    torch.cuda.synchronize()
    want = _state(ref)
    del ref

    ov, plan = _stack(True, cfg_key)
    for _ in range(2):
        ov.run_step(plan)
    torch.cuda.synchronize()
    got = _state(ov)
    for a, b in zip(want, got):
        assert torch.equal(a, b)
    del ov

    gr, plan = _stack(True, cfg_key)
    gr.run_step(plan)  # eager step 1 (sizes workspaces)
    gr.capture(plan)
    gr.replay()        # step 2 via the graph
    torch.cuda.synchronize()
    for a, b in zip(want, _state(gr)):
        assert torch.equal(a, b)


def test_stack_forward_matches_oracle():
    """Last layer's q|k|v of the tiny stack against the oracle on the stack's own buffers (the
    per-projection output scratch holds the last layer's result)."""
    import oracle
    st, plan = _stack(True)
    st.run_step(plan, optimizer_step=False)
    torch.cuda.synchronize()
    L = len(st.layers)
    proj = st.layers[L - 1][0]
    X = st._acts["X"][L - 1][: plan.n_rows].float().cpu().numpy()
    row_ad = plan.device.row_adapter.cpu().numpy()
    Y_ref, _ = oracle.lora_forward(X, proj.W.float().cpu().numpy(), proj.A.float().cpu().numpy(),
                                   proj.B.float().cpu().numpy(), proj.scale.cpu().numpy(), row_ad,
                                   proj.spec.subs, proj.spec.r_pad)
    Y = st._acts["Y"][proj.spec.name][: plan.n_rows].float().cpu().numpy()
    err = np.abs(Y - Y_ref).max()
    assert err <= 1e-2 * np.abs(Y_ref).max() + 1e-3


def test_stack_backward_matches_oracle():
    """The stack's training-row backward through the overlapped step — dH shrinks, dX GEMMs and
    the per-layer batched K5 launch (STORE_GRAD mode) — against the oracle on the stack's own
    buffers, for every projection of the first and last layer of the tiny stack."""
    import oracle
    st, plan = _stack(True)
    st.run_step(plan, optimizer_step=False)
    torch.cuda.synchronize()
    a = st._acts
    L = len(st.layers)
    Ttr = plan.n_train
    f = lambda t: t.float().cpu().numpy().astype(np.float64)  # noqa: E731
    for l in (0, L - 1):
        for proj in st.layers[l]:
            name = proj.spec.name
            t = proj.train_state.adapter
            X = a["X"][l] if name in ("qkv", "q", "k", "v", "gate_up", "gate", "up") else \
                (a["Xo"][l] if name == "o" else a["Xd"][l])
            dY = (a["dY_top"] if l == L - 1 else a["dX_first"][l + 1]) if name == "down" \
                else a["dY"][l][name]
            H16 = proj._H16[:Ttr]
            dH16, dH16lo = proj._dH16[:Ttr], proj._dH16lo[:Ttr]
            # dB from the oracle formula on the device's H16; dA^T on the device's dH hi + lo
            _, dB_ref, _, dH_ref = oracle.lora_backward(
                f(dY), f(X[:Ttr]), f(H16), f(proj.W), f(proj.A[t]), f(proj.B[t]),
                float(proj.scale[t]), proj.spec.subs, proj.spec.r_pad, dx_rows=[0])
            dAT_ref = f(X[:Ttr]).T @ (f(dH16) + f(dH16lo))
            # the hi + lo pair carries the exact dH to fp32 accuracy (not one bf16 rounding)
            pair = f(dH16) + f(dH16lo)
            rel = np.linalg.norm(pair - dH_ref) / max(np.linalg.norm(dH_ref), 1e-30)
            assert rel < 1e-4, f"layer {l} {name} dH hi+lo: rel err {rel}"
            gB, gAT = f(proj.train_state.grad_B), f(proj.train_state.grad_AT)
            for got, ref, what in ((gB, dB_ref, "dB"), (gAT, dAT_ref, "dA^T")):
                rel = np.linalg.norm(got - ref) / max(np.linalg.norm(ref), 1e-30)
                assert rel < 1e-4, f"layer {l} {name} {what}: rel err {rel}"
            # the device's hi half is the bf16 rounding of the exact dH (summation order aside)
            err = np.abs(f(dH16) - dH_ref).max()
            assert err <= 1e-2 * np.abs(dH_ref).max() + 1e-6, f"layer {l} {name} dH: {err}"


@pytest.mark.parametrize("cfg_key", ["tiny", "llama2-7b:1"])
def test_flag_overlap_mode_bitwise(cfg_key):
    """The two-stream variant of the overlap (shrink on a side stream, the GEMM's LoRA stages
    wait on a device flag carrying the step generation) gives bitwise the serialized results."""
    ref, plan = _stack(False, cfg_key)
    for _ in range(2):
        ref.run_step(plan)
    torch.cuda.synchronize()
    want = _state(ref)
    del ref
    fl, plan = _stack(True, cfg_key, mode="flag")
    fl.run_step(plan)
    fl.capture(plan)
    fl.replay()
    torch.cuda.synchronize()
    for a, b in zip(want, _state(fl)):
        assert torch.equal(a, b)


def test_lm_head_loss_and_top_gradient():
    """The LM head on the training rows (K2 logits, K7 CE, K3 dX): the step's loss equals the
    oracle CE of the bf16 logits of the stack's final hidden rows, and dY_top = dlogits . W."""
    import numpy as np

    import oracle
    from paper_2604_16400_b200.replica import ReplicaStack
    cfg = _config("tiny")
    st = ReplicaStack(cfg, "cuda", seed=3, lm_head=True)
    plan = st.plan(*cfg.batch(0))
    a = st.allocate(plan, distinct_synthetic=True)
    st.run_step(plan, optimizer_step=False)
    torch.cuda.synchronize()
    Ttr, L = plan.n_train, cfg.model.layers
    Xtop = a["X"][L][:Ttr].float().cpu().numpy()
    Wh = st.head.W.float().cpu().numpy()
    logits = oracle.bf16_round(Xtop @ Wh.T)
    rows, mean, dz = oracle.cross_entropy(logits, a["labels"].cpu().numpy())
    assert abs(st.last_loss() - mean) <= 1e-3 * abs(mean)
    dX_ref = oracle.bf16_round(dz) @ Wh
    got = a["dY_top"].float().cpu().numpy()
    err = np.abs(got - dX_ref).max()
    assert err <= 1e-2 * np.abs(dX_ref).max() + 1e-6, err


def test_adapter_pager_paging_is_exact():
    """registry.AdapterPager: adapters stored in pinned host memory and paged into device slots
    by async copies give bitwise the same forward as adapters set in place; LRU eviction never
    touches the pinned (trainable) slot nor a slot the current request needs; save/load
    round-trips the reference layout exactly."""
    import os
    import tempfile

    from paper_2604_16400_b200.registry import AdapterPager
    ref, plan = _stack(False, "tiny", seed=5)
    n = ref.cfg.n_adapters
    ref.run_step(plan, backward=False)
    torch.cuda.synchronize()
    want = ref._acts["X"][-1].clone()
    # a second stack whose inference adapters come from the pager's host store
    st, plan2 = _stack(False, "tiny", seed=6)
    for p_ref, p in zip(ref.projections(), st.projections()):
        p.W.copy_(p_ref.W)
        p.refresh_transpose()
    pager = AdapterPager(st)
    projs = list(ref.projections())
    for a in range(n):
        pager.register(f"tenant{a}", [p.get_adapter(a) for p in projs])
    t = ref.cfg.train_adapter
    for p_ref, p in zip(projs, st.projections()):  # the pinned trainable slot: set in place
        p.A[t].copy_(p_ref.A[t])
        p.B[t].copy_(p_ref.B[t])
        p.scale[t:t + 1].copy_(p_ref.scale[t:t + 1])
    slots = pager.ensure([f"tenant{a}" for a in range(n) if a != t])
    assert slots == {f"tenant{a}": a for a in range(n) if a != t}
    st._acts["X"][0].copy_(ref._acts["X"][0])
    st.run_step(plan2, backward=False)
    pager.mark_used(range(n))
    torch.cuda.synchronize()
    assert torch.equal(st._acts["X"][-1], want)
    # eviction: a new adapter takes the least recently used pageable slot
    pager.register("new", [p.get_adapter((t + 1) % n) for p in projs])
    order = [f"tenant{a}" for a in range(n) if a != t]
    pager.ensure(order[1:])                 # touch all but the first -> it is the LRU
    got = pager.ensure(["new"])["new"]
    assert got == int(order[0][len("tenant"):]) and got != t
    assert f"tenant{got}" not in pager.slot_of
    torch.cuda.synchronize()
    for p_src, p in zip(projs, st.projections()):
        assert torch.equal(p.A[got], p_src.A[(t + 1) % n]) and torch.equal(p.B[got], p_src.B[(t + 1) % n])
        assert torch.equal(p.A[t], p_src.A[t])
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "a.pt")
        pager.save("tenant1", path)
        pager.load("copy", path)
    for (A0, B0, s0), (A1, B1, s1) in zip(pager.host["tenant1"], pager.host["copy"]):
        assert torch.equal(A0, A1) and torch.equal(B0, B1) and torch.equal(s0, s1)


@pytest.mark.parametrize("cfg_key,mode", [("tiny", "pdl"), ("tiny", "flag"), ("llama3-8b:1", "pdl")])
def test_stack_attention_matches_oracle(cfg_key, mode):
    """ReplicaStack(attention=True): K9 sits between q|k|v and o in the step — its output is o's
    input, its backward turns o's dX into q|k|v's dY.  Layer 0 (the last layer of the backward)
    against the float64 oracle: the attention output over every sequence of the pass (training
    sequences + each request's rows), and q|k|v's dY over the training sequences; two passes are
    bitwise identical (GQA at Llama-3-8B: 32 query / 8 kv heads)."""
    import numpy as np
    import oracle
    from paper_2604_16400_b200.replica import ReplicaStack
    cfg = _config(cfg_key)
    if cfg_key.startswith("llama3"):  # keep the oracle cheap: fewer rows than the full config
        import dataclasses
        cfg = dataclasses.replace(cfg, train_batch=2, train_seq=256)
    st = ReplicaStack(cfg, "cuda", seed=0, attention=True)
    st.overlap = True
    st.overlap_mode = mode
    train, items = cfg.batch(0)
    if cfg_key.startswith("llama3"):
        items = items[:6]
    plan = st.plan(train, items)
    st.allocate(plan, distinct_synthetic=True)
    st.run_step(plan, optimizer_step=False)
    torch.cuda.synchronize()
    a = st._acts
    T, Ttr = plan.n_rows, plan.n_train
    seq = np.asarray(plan.attn_seq)
    H, Hk = st.n_heads, st.n_kv_heads
    f = lambda t: t.float().cpu().numpy()  # noqa: E731
    q, k, v = (f(t) for t in st._qkv_views(a["Yqkv"][0][:T]))
    out_ref, _ = oracle.causal_attention(q, k, v, seq, H, Hk)
    got = f(a["Xo"][0][:T])
    assert np.abs(got - out_ref).max() <= 1e-2 * np.abs(out_ref).max() + 1e-3
    seq_tr = seq[seq <= Ttr]
    _, _, (dq, dk, dv) = oracle.causal_attention(q[:Ttr], k[:Ttr], v[:Ttr], seq_tr, H, Hk,
                                                 dout=f(a["dX"]["o"][:Ttr]))
    ref = np.concatenate([dq, dk, dv], axis=1)
    gotd = f(a["dqkv"][0][:Ttr])
    assert np.abs(gotd - ref).max() <= 1e-2 * np.abs(ref).max() + 1e-3
    assert np.linalg.norm(gotd - ref) / np.linalg.norm(ref) <= 1e-2
    first = (a["Xo"][0].clone(), a["dqkv"][0].clone(), a["X"][-1].clone())
    st.run_step(plan, optimizer_step=False)
    torch.cuda.synchronize()
    for x, y in zip(first, (a["Xo"][0], a["dqkv"][0], a["X"][-1])):
        assert torch.equal(x, y)
