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


@pytest.mark.parametrize("n_ctas,nr", [(2, 16), (8, 48), (16, 32), (16, 256)])
def test_plan_shrink_windows(lib, n_ctas, nr):
    """collm_plan_shrink_windows (host): units are 128-row windows x runs of consecutive adapter
    ids whose span rounded to 2^c keeps 2^c * nr <= 256; every (row, adapter) of the batch is in
    exactly one unit's window and adapter range, base-only rows in a zero unit; the longest-first
    assignment keeps the CTA loads within one unit of each other."""
    import numpy as np
    from paper_2604_16400_b200 import segments
    g = np.random.default_rng(n_ctas + nr)
    lens = g.integers(1, 300, 40)
    ads = g.integers(-1, 24, 40)
    seg = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    host = segments.plan_segments(seg, ads)
    chunks, ptr = segments.plan_shrink_windows(host, nr, n_ctas)
    assert ptr[0] == 0 and ptr[-1] == len(chunks) and np.all(np.diff(ptr) >= 0)
    row_ad = np.repeat(ads, lens)
    T = int(seg[-1])
    covered = np.zeros(T, np.int32)
    # every unit's parts 0..S-1 appear exactly once, with one first-chunk id per unit
    parts = {}
    for r0, n, a, c, S, part, c0, u in chunks:
        parts.setdefault(u, []).append((part, S, c0))
    for u, ps in parts.items():
        assert sorted(p for p, _, _ in ps) == list(range(ps[0][1])) and len({c0 for *_, c0 in ps}) == 1
    units = [tuple(ch[:4]) for ch in chunks if ch[5] == 0]
    for r0, n, a, c in units:
        assert r0 % 128 == 0 and n == min(128, T - r0)
        rows = np.arange(r0, r0 + n)
        if a < 0:
            mine = rows[row_ad[rows] < 0]
        else:
            assert (1 << c) * nr <= 256 and (1 << c) <= 16
            mine = rows[(row_ad[rows] >= a) & (row_ad[rows] < a + (1 << c))]
            assert a in set(row_ad[rows])
        covered[mine] += 1
    assert np.all(covered == 1)
    cost = [((128 + (1 << c) * nr) // S + (8 if S > 1 else 0)) if a >= 0 else 1
            for _, _, a, c, S, *_ in chunks]
    loads = [sum(cost[ptr[c]:ptr[c + 1]]) for c in range(n_ctas)]
    assert max(loads) - min(loads) <= max(cost)


def test_reduce_tsplit_rules(monkeypatch):
    """K5 split choice (host side of collm_lora_reduce): the tcgen05 stream splits T only when the
    static share per CTA would be unbalanced by > 8 % and every part keeps >= 8 whole 128-row
    chunks (BASELINE shapes: 7B / 8B whole tiles, 13B two parts); the mma.sync kernel fills one
    wave of 3 CTAs per SM."""
    import torch

    from paper_2604_16400_b200 import ops
    monkeypatch.setattr(ops, "num_sms", lambda device=None: 148)
    dev = torch.device("cpu")
    monkeypatch.setattr(ops, "reduce_impl", lambda: 1)
    assert ops.reduce_tsplit(512, 514, dev) == 1        # 7B: 4 chunks per tile
    assert ops.reduce_tsplit(8192, 576, dev) == 1       # 8B: 3.89 tiles per CTA, balanced
    assert ops.reduce_tsplit(16384, 644, dev) == 2      # 13B: 4.35 -> 8.70 units per CTA
    assert ops.reduce_tsplit(100, 3, dev) == 1          # one chunk
    for T, tiles in ((4096, 10), (70000, 300), (2048, 148)):
        ts = ops.reduce_tsplit(T, tiles, dev)
        chunks = -(-T // 128)
        assert 1 <= ts <= chunks and (ts == 1 or chunks >= 8 * ts)
    monkeypatch.setattr(ops, "reduce_impl", lambda: 0)
    assert ops.reduce_tsplit(512, 514, dev) == 1
    assert ops.reduce_tsplit(4096, 8, dev) == min(3 * 148 // 8, 4096 // 32 // 3, 128)


def test_shrink_tc_selection_by_rows():
    """Passes of >= SHRINK_TC_MIN_ROWS rows take K1' on the whole GPU, smaller passes keep the
    mma.sync K1, a rank-space partition always takes K1' on its SMs (BASELINE: 7B 1024 rows -> K1,
    8B 26985 / 13B 16640 rows -> K1' on 148 CTAs)."""
    from paper_2604_16400_b200 import segments
    m = segments.SHRINK_TC_MIN_ROWS
    assert segments.default_tc_ctas(1024, 0, 148) == (148 if m <= 1024 else 0)
    assert segments.default_tc_ctas(max(m, 16640), 0, 148) == 148
    assert segments.default_tc_ctas(max(m, 16640), 0, 147) == 146
    assert segments.default_tc_ctas(100, 16, 148) == 16
