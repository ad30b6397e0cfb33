"""GPU parity of the unified PEFT projection (the hot path, through the C ABI) against the CPU
oracle on identical seeded inputs.

Tolerances (stated here):
  * segment indexing (row_adapter, slot_of_row, tile slots): bit-exact;
  * Y and dX (bf16 out, fp32 accumulation): |err|_inf <= 1e-2 * |ref|_inf + 1e-3, and relative
    Frobenius <= 4e-3;
  * H16 / dH16 (bf16 intermediates): relative Frobenius <= 4e-3;
  * dB, dA^T (fp32 gradients): relative Frobenius <= 1e-3;
  * AdamW master weights after one step on the device gradient: |err| <= 1e-6 + 1e-5 |w|.
"""

import numpy as np
import pytest
import torch

import oracle
from tests.helpers import mixed_items, projection_inputs, rng

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _build():
    from paper_2604_16400_b200 import _lib, build
    build.build()
    _lib.load()


def _t(a, dtype=torch.bfloat16):
    return torch.from_numpy(np.ascontiguousarray(a)).to("cuda", dtype)


def _rel(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def _check_bf16_out(out, ref):
    out = np.asarray(out, np.float64)
    err = np.abs(out - ref).max()
    tol = 1e-2 * np.abs(ref).max() + 1e-3
    assert err <= tol, (err, tol)
    assert _rel(out, ref) <= 4e-3, _rel(out, ref)


CASES = [
    # name, K, subs, rank, n_adapters, T_tr, n_decode, n_prefill, base_rows, seed
    ("tiny_qkv", 256, (256, 256, 256), 8, 4, 128, 16, 0, 0, 0),
    ("tiny_up", 256, (688,), 8, 4, 128, 16, 0, 0, 1),
    ("tiny_down", 688, (256,), 8, 4, 128, 16, 0, 0, 2),
    ("ragged_mixed", 512, (256, 256), 16, 6, 96, 23, 7, 3, 3),
    ("rank32_prefill", 384, (384,), 32, 3, 64, 5, 9, 0, 4),
    ("rank64_gateup", 256, (512, 512), 64, 5, 160, 40, 4, 2, 5),
    ("no_train", 256, (256,), 16, 4, 0, 30, 3, 1, 6),
]


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_projection_fwd_bwd(case):
    from paper_2604_16400_b200 import segments
    from paper_2604_16400_b200.domain import InferenceItem, RowRole, TrainItem
    from paper_2604_16400_b200.layer import (AdamWConfig, LoraProjection, OptimizerState,
                                             ProjectionSpec)

    name, K, subs, rank, n_ad, T_tr, n_dec, n_pre, n_base, seed = case
    g = rng(seed)
    items = mixed_items(g, n_ad, n_dec, n_pre, base_rows=n_base)
    train = (0, T_tr) if T_tr else None
    seg_start, seg_ad, seg_role, row_req, row_pos = oracle.build_rows(train, items)
    T = seg_start[-1]

    # ---- K0: host build + device expansion, bit-exact against the oracle
    mb = segments.build_mixed_batch(
        TrainItem(0, 1, T_tr) if T_tr else None,
        [InferenceItem(rid, ad, n, RowRole(role)) for rid, ad, n, role in items])
    assert list(mb.seg_start) == seg_start and list(mb.seg_adapter) == seg_ad
    assert list(mb.seg_role) == seg_role and list(mb.row_request) == row_req
    hp = segments.plan_segments(mb.seg_start, mb.seg_adapter)
    plan = segments.DevicePlan(hp)
    row_ad = oracle.expand_segments(seg_start, seg_ad)
    tsp, slots = oracle.tile_slots(row_ad)
    assert np.array_equal(hp.tile_slot_ptr, tsp) and np.array_equal(hp.slot_adapter, slots)
    assert np.array_equal(hp.shrink_tiles, oracle.shrink_tiles(seg_start, seg_ad))
    torch.cuda.synchronize()
    assert np.array_equal(plan.row_adapter.cpu().numpy(), row_ad)
    assert np.array_equal(plan.slot_of_row.cpu().numpy(), oracle.slot_of_row(row_ad, tsp, slots))

    # ---- forward
    spec = ProjectionSpec(name, K, subs, rank, alpha=16.0)
    inp = projection_inputs(g, T, T_tr, K, subs, rank, spec.r_pad, n_ad)
    proj = LoraProjection(spec, n_ad)
    proj.W.copy_(_t(inp["W"]))
    proj.refresh_transpose()
    proj.A.copy_(_t(inp["A"]))
    proj.B.copy_(_t(inp["B"]))
    proj.scale.copy_(_t(inp["scale"], torch.float32))
    X = _t(inp["X"])
    Y, cache = proj.forward(X, plan, n_train=T_tr)
    torch.cuda.synchronize()
    Y_ref, H16_ref = oracle.lora_forward(inp["X"], inp["W"], inp["A"], inp["B"], inp["scale"],
                                         row_ad, subs, spec.r_pad)
    _check_bf16_out(Y.float().cpu().numpy(), Y_ref)
    assert _rel(cache.H16[:T].float().cpu().numpy(), H16_ref) <= 4e-3
    if not T_tr:
        return

    # ---- backward (gradients stored, no optimizer)
    tp = segments.DevicePlan(segments.uniform_plan(T_tr, 0))
    proj.make_trainable(0)
    dY = _t(inp["dY"])
    dX = proj.backward(dY, cache, tp)
    torch.cuda.synchronize()
    st = proj.train_state
    dX_ref, dB_ref, dAT_ref, dH16_ref = oracle.lora_backward(
        inp["dY"], inp["X"][:T_tr], H16_ref[:T_tr], inp["W"], inp["A"][0], inp["B"][0],
        float(inp["scale"][0]), subs, spec.r_pad)
    _check_bf16_out(dX.float().cpu().numpy(), dX_ref)
    assert _rel(st.grad_B.cpu().numpy(), dB_ref) <= 1e-3
    assert _rel(st.grad_AT.cpu().numpy(), dAT_ref) <= 1e-3

    # ---- fused AdamW on the same backward (fresh state) vs the oracle's AdamW on the device grad
    gB = st.grad_B.cpu().numpy().copy()
    gAT = st.grad_AT.cpu().numpy().copy()
    proj.make_trainable(0)
    st = proj.train_state
    mB0 = st.master_B.cpu().numpy().copy()
    mAT0 = st.master_AT.cpu().numpy().copy()
    opt = AdamWConfig(lr=1e-3, weight_decay=0.01)
    ostate = OptimizerState(opt)
    ostate.advance()
    proj.backward(dY, cache, tp, optimizer=ostate, need_dx=False)
    torch.cuda.synchronize()
    for master0, grad, dev, r in ((mB0, gB, st.master_B, "B"), (mAT0, gAT, st.master_AT, "AT")):
        ost = oracle.AdamWState(np.zeros_like(master0), np.zeros_like(master0))
        ref = oracle.adamw_step(master0, grad, ost, lr=opt.lr, wd=opt.weight_decay)
        got = dev.cpu().numpy()
        assert np.all(np.abs(got - ref) <= 1e-6 + 1e-5 * np.abs(ref)), r
    # bf16 working copies follow the masters in every layout
    bnd = spec.sub_bounds
    mB = st.master_B.cpu()
    assert torch.equal(proj.B[0].cpu(), mB.to(torch.bfloat16))
    assert torch.equal(proj.A[0].cpu(), st.master_AT.cpu().t().to(torch.bfloat16))
    assert torch.equal(st.AT16.cpu(), st.master_AT.cpu().to(torch.bfloat16))
    rp = spec.r_pad
    for s in range(len(subs)):
        assert torch.equal(st.BT16[s * rp:(s + 1) * rp, bnd[s]:bnd[s + 1]].cpu(),
                           mB[bnd[s]:bnd[s + 1]].t().to(torch.bfloat16))


def test_deterministic_repeat():
    """Two identical passes give bitwise-identical outputs and gradients (no float atomics)."""
    from paper_2604_16400_b200 import segments
    from paper_2604_16400_b200.layer import LoraProjection, ProjectionSpec
    g = rng(11)
    items = mixed_items(g, 4, 50, 6)
    seg_start, seg_ad, *_ = oracle.build_rows((1, 256), items)
    T = seg_start[-1]
    spec = ProjectionSpec("det", 1024, (512, 512), 16, 32.0)
    inp = projection_inputs(g, T, 256, 1024, spec.subs, 16, spec.r_pad, 4)
    proj = LoraProjection(spec, 4)
    proj.W.copy_(_t(inp["W"]))
    proj.refresh_transpose()
    proj.A.copy_(_t(inp["A"]))
    proj.B.copy_(_t(inp["B"]))
    proj.scale.copy_(_t(inp["scale"], torch.float32))
    plan = segments.DevicePlan(segments.plan_segments(seg_start, seg_ad))
    tp = segments.DevicePlan(segments.uniform_plan(256, 1))
    proj.make_trainable(1)
    outs = []
    for _ in range(2):
        Y, cache = proj.forward(_t(inp["X"]), plan, n_train=256)
        dX = proj.backward(_t(inp["dY"]), cache, tp)
        torch.cuda.synchronize()
        outs.append((Y.clone(), dX.clone(), proj.train_state.grad_B.clone(),
                     proj.train_state.grad_AT.clone()))
    for a, b in zip(*outs):
        assert torch.equal(a, b)
