"""CPU: host logic of the path — batch composition (K0), the native host planner, the C-ABI
library surface, the domain types, the configs and the FLOP/byte accounting."""

import ctypes as C
import os
import re

import numpy as np
import pytest

import oracle
from tests.helpers import mixed_items, rng

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_2604_16400_b200 import _lib, build
    build.build()
    return _lib.load()


# ------------------------------------------------------------------ C ABI surface
def test_header_symbols_exported(lib):
    from paper_2604_16400_b200 import _lib
    header = open(os.path.join(ROOT, "include", "collm.h")).read()
    declared = set(re.findall(r"^\s*(?:int|size_t|const char\*)\s+(collm_\w+)\(", header, re.M))
    assert len(declared) >= 11
    for name in declared:
        assert hasattr(lib, name), name
        assert name in _lib.SIGNATURES, f"{name} has no ctypes signature"
    assert set(_lib.SIGNATURES) <= declared
    assert lib.collm_version() >= 1


def test_reduce_group_struct_matches_header():
    from paper_2604_16400_b200 import _lib
    header = open(os.path.join(ROOT, "include", "collm.h")).read()
    body = header[header.index("typedef struct {"):header.index("} collm_reduce_group;")]
    fields = re.findall(r"(\w+)\s*[,;]", re.sub(r"/\*.*?\*/", "", body, flags=re.S))
    names = [f[0] for f in _lib.ReduceGroup._fields_]
    assert fields == names
    assert C.sizeof(_lib.ReduceGroup) == 9 * 8 + 12 * 4


def test_status_mapping(lib):
    from paper_2604_16400_b200 import _lib
    from paper_2604_16400_b200.domain import ConfigurationError
    bad = (C.c_int32 * 3)(0, 5, 4)  # unsorted segment table
    ad = (C.c_int32 * 2)(0, 1)
    st = lib.collm_plan_segments(bad, ad, 2, 4, None, None, 0, None, None, 0, None)
    assert st == _lib.COLLM_EINVAL and b"segment" in lib.collm_last_error()
    with pytest.raises(ConfigurationError):
        _lib.check(st, "collm_plan_segments")


# ------------------------------------------------------------------ K0: batch composition
@pytest.mark.parametrize("seed", range(6))
def test_segments_bit_exact(lib, seed):
    from paper_2604_16400_b200 import segments
    from paper_2604_16400_b200.domain import InferenceItem, RowRole, TrainItem
    g = rng(100 + seed)
    n_ad = int(g.integers(1, 40))
    items = mixed_items(g, n_ad, int(g.integers(0, 300)), int(g.integers(0, 30)),
                        prefill_len=(2, 200), base_rows=int(g.integers(0, 5)))
    T_tr = int(g.integers(0, 3)) * int(g.integers(1, 300))
    if not items and not T_tr:
        T_tr = 7
    train_ad = int(g.integers(0, n_ad))
    ref = oracle.build_rows((train_ad, T_tr) if T_tr else None, items)
    mb = segments.build_mixed_batch(
        TrainItem(train_ad, 1, T_tr) if T_tr else None,
        [InferenceItem(rid, ad, n, RowRole(role)) for rid, ad, n, role in items])
    assert (list(mb.seg_start), list(mb.seg_adapter), list(mb.seg_role), list(mb.row_request),
            list(mb.row_pos)) == tuple(ref)
    hp = segments.plan_segments(mb.seg_start, mb.seg_adapter)
    row_ad = oracle.expand_segments(ref[0], ref[1])
    tsp, slots = oracle.tile_slots(row_ad)
    assert np.array_equal(hp.tile_slot_ptr, tsp)
    assert np.array_equal(hp.slot_adapter, slots)
    assert np.array_equal(hp.shrink_tiles, oracle.shrink_tiles(ref[0], ref[1]))


def test_batch_validation():
    from paper_2604_16400_b200 import segments
    from paper_2604_16400_b200.domain import ConfigurationError, InferenceItem, RowRole, TrainItem
    with pytest.raises(ConfigurationError):
        segments.build_mixed_batch(None, [])
    with pytest.raises(ConfigurationError):
        segments.build_mixed_batch(None, [InferenceItem(1, 0, 1), InferenceItem(1, 1, 1)])
    with pytest.raises(ConfigurationError):
        InferenceItem(3, 0, 2, RowRole.DECODE)  # a decode step is one row
    with pytest.raises(ConfigurationError):
        TrainItem(-1, 1, 4)


# ------------------------------------------------------------------ domain mirror
def test_domain_mirrors_reference():
    from paper_2604_16400_b200 import domain
    with pytest.raises(domain.ConfigurationError, match="deadline"):
        domain.Request(1, 2.0, 1.0, 5)
    with pytest.raises(domain.ConfigurationError, match="output_tokens"):
        domain.Request(1, 1.0, 2.0, 0)
    with pytest.raises(domain.ConfigurationError):
        domain.BatchConfig(-1, 0)
    ref_src = "/root/reference/pkg/src"
    if not os.path.isdir(ref_src):
        pytest.skip("reference not mounted")
    import sys
    sys.path.insert(0, ref_src)
    try:
        from coserve import domain as ref
    finally:
        sys.path.remove(ref_src)
    for name in ("ConfigurationError", "InvariantViolation"):
        assert issubclass(getattr(domain, name), getattr(ref, name).__mro__[1])
    for cls in ("Request", "BatchConfig"):
        assert [f for f in getattr(domain, cls).__dataclass_fields__] == \
            [f for f in getattr(ref, cls).__dataclass_fields__]


# ------------------------------------------------------------------ configs and accounting
def test_configs_batches():
    from paper_2604_16400_b200.configs import CONFIGS
    from paper_2604_16400_b200.segments import build_mixed_batch
    expect = {"tiny": (144, 128), "llama2-7b": (1024, 512), "llama2-13b": (16640, 16384)}
    for key, (T, Ttr) in expect.items():
        mb = build_mixed_batch(*CONFIGS[key].batch(0))
        assert (mb.n_rows, mb.n_train_rows) == (T, Ttr), key
    mb = build_mixed_batch(*CONFIGS["llama3-8b"].batch(0))
    assert mb.n_train_rows == 8192 and 10000 < mb.n_infer_rows < 25000
    # 7B: 32 adapters, every adapter serves 1..32 rows
    mb = build_mixed_batch(*CONFIGS["llama2-7b"].batch(0))
    counts = np.bincount(oracle.expand_segments(list(mb.seg_start), list(mb.seg_adapter))[512:],
                         minlength=32)
    assert counts.sum() == 512 and counts.min() >= 1 and counts.max() <= 32


def test_flop_accounting_matches_survey():
    from paper_2604_16400_b200.configs import CONFIGS
    cfg = CONFIGS["llama2-7b"]
    per_row = cfg.model.flops_per_row()
    assert abs(per_row / 1e9 - 12.95) < 0.01  # 12.95 GFLOP per token (7B)
    step = per_row * (1024 + 512)
    assert abs(step / 1e12 - 19.89) < 0.01      # 19.89 TFLOP per 7B step
    specs = cfg.projections
    assert [s.name for s in specs] == ["qkv", "o", "gate_up", "down"]
    assert sum(2 * s.in_features * s.out_features for s in specs) * 32 == per_row


@pytest.mark.parametrize("n_ctas", [2, 8, 16])
def test_plan_shrink_items(lib, n_ctas):
    """collm_plan_shrink_items (host): the <=16-row shrink tiles merge into items of consecutive
    rows of ONE adapter (never across adapters or base-only runs, never above max_rows), every
    row is covered exactly once, the class is the smallest box height holding the item, and the
    longest-first assignment keeps the CTA loads within one item of each other."""
    import numpy as np
    from paper_2604_16400_b200 import segments
    g = np.random.default_rng(n_ctas)
    lens = g.integers(1, 300, 40)
    ads = g.integers(-1, 12, 40)
    ads[1:][ads[1:] == ads[:-1]] = 12  # break equal neighbours (the planner merges runs anyway)
    seg = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    host = segments.plan_segments(seg, ads)
    for mr in (128, 32):
        items, ptr = segments.plan_shrink_items(host, n_ctas, max_rows=mr)
        assert ptr[0] == 0 and ptr[-1] == len(items) and np.all(np.diff(ptr) >= 0)
        row_ad = np.repeat(ads, lens)
        covered = np.zeros(seg[-1], np.int32)
        for r0, n, a, cls in items:
            assert 1 <= n <= mr and (16 << cls) >= n and (cls == 0 or (16 << (cls - 1)) < n)
            assert np.all(row_ad[r0:r0 + n] == a)
            covered[r0:r0 + n] += 1
        assert np.all(covered == 1)
        cost = [(16 << c) + 64 if a >= 0 else 1 for _, _, a, c in items]
        loads = [sum(cost[ptr[c]:ptr[c + 1]]) for c in range(n_ctas)]
        assert max(loads) - min(loads) <= max(cost)
