"""GPU parity of many-adapter decode tiles: every row of a 256-row slot tile
is a decode row of a DIFFERENT adapter, so the tile carries 256 LoRA slots (the GEMM folds
256 x r rank columns into its accumulator as extra k-stages and the shrink fills 255 zero slots
per row).  Ranks 16 and 64, fused sub-projections, 256 + 44 rows (a second, partial tile), with
and without training rows, and through the rank-space partition — Y / H16 against the oracle with
the stated tolerances (tests/test_gpu_parity.py)."""

import numpy as np
import pytest
import torch

import oracle
from tests.helpers import projection_inputs, rng

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _build():
    from paper_2604_16400_b200 import _lib, build
    build.build()
    _lib.load()


def _t(a, dtype=torch.bfloat16):
    return torch.from_numpy(np.ascontiguousarray(a)).to("cuda", dtype)


def _rel(a, b):
    return float(np.linalg.norm(np.asarray(a, np.float64) - b) / max(np.linalg.norm(b), 1e-30))


@pytest.mark.parametrize("rank,T_tr,rank_sms,fused", [(16, 0, 0, False), (64, 0, 0, False),
                                                    (16, 64, 0, False), (16, 64, 16, False),
                                                    (16, 0, 0, True), (64, 64, 0, True)])
def test_many_adapter_decode(rank, T_tr, rank_sms, fused, monkeypatch):
    """fused=False: tiles with > 32 slots skip the GEMM's fused expand and take the per-row
    expand kernel (collm_lora_expand_rows); fused=True forces the fused expand everywhere."""
    monkeypatch.setenv("COLLM_EXPAND_ROWS_SLOTS", "100000" if fused else "32")
    from paper_2604_16400_b200 import ops, segments
    from paper_2604_16400_b200.domain import InferenceItem, RowRole, TrainItem
    from paper_2604_16400_b200.layer import LoraProjection, ProjectionSpec
    ops.set_rank_sms(rank_sms)
    try:
        g = rng(rank + T_tr)
        n_ad = 300
        K, subs = 512, (256, 256)
        # 300 decode rows, adapters a permutation: every row of the first 256-row tile (after the
        # training rows) has its own adapter
        perm = g.permutation(n_ad)
        items = [(i, int(perm[i]), 1, 2) for i in range(n_ad)]
        train = (int(perm[0]), T_tr) if T_tr else None
        seg_start, seg_ad, *_ = oracle.build_rows(train, items)
        T = seg_start[-1]
        mb = segments.build_mixed_batch(
            TrainItem(int(perm[0]), 1, T_tr) if T_tr else None,
            [InferenceItem(rid, ad, n, RowRole(role)) for rid, ad, n, role in items])
        hp = segments.plan_segments(mb.seg_start, mb.seg_adapter)
        slots_per_tile = np.diff(hp.tile_slot_ptr)
        assert slots_per_tile.max() >= 190, slots_per_tile
        plan = segments.DevicePlan(hp)
        assert (plan.n_expand_tiles > 0) != fused
        spec = ProjectionSpec("many", K, subs, rank, alpha=16.0)
        inp = projection_inputs(g, T, T_tr, K, subs, rank, spec.r_pad, n_ad)
        proj = LoraProjection(spec, n_ad)
        proj.W.copy_(_t(inp["W"]))
        proj.refresh_transpose()
        proj.A.copy_(_t(inp["A"]))
        proj.B.copy_(_t(inp["B"]))
        proj.scale.copy_(_t(inp["scale"], torch.float32))
        Y, cache = proj.forward(_t(inp["X"]), plan, n_train=T_tr)
        torch.cuda.synchronize()
        row_ad = oracle.expand_segments(seg_start, seg_ad)
        Y_ref, H16_ref = oracle.lora_forward(inp["X"], inp["W"], inp["A"], inp["B"], inp["scale"],
                                             row_ad, subs, spec.r_pad)
        out = Y.float().cpu().numpy()
        err = np.abs(out - Y_ref).max()
        assert err <= 1e-2 * np.abs(Y_ref).max() + 1e-3, err
        assert _rel(out, Y_ref) <= 4e-3
        assert _rel(cache.H16[:T].float().cpu().numpy(), H16_ref) <= 4e-3
    finally:
        ops.set_rank_sms(0)
