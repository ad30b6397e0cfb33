"""Time the K1 shrink alone on the Llama-2-7B step's shapes (CUDA events, inputs > L2 rotated).
Env COLLM_SHRINK_CTAS_PER_SM varies the K-split target."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2604_16400_b200 import ops, segments  # noqa: E402
from paper_2604_16400_b200.configs import CONFIGS  # noqa: E402

cfg = CONFIGS[os.environ.get("CFG", "llama2-7b")]
TC = int(os.environ.get("TC", "0"))  # rank-space partition size: collm_lora_shrink_tc
if TC and TC <= 64:
    ops.set_rank_sms(TC)
mb = segments.build_mixed_batch(*cfg.batch(0))
plan = segments.DevicePlan(segments.plan_segments(mb.seg_start, mb.seg_adapter), tc_ctas=TC)
tplan = segments.DevicePlan(segments.uniform_plan(mb.n_train_rows, mb.train_adapter), tc_ctas=TC)
T, Ttr = mb.n_rows, mb.n_train_rows
scale = torch.full((cfg.n_adapters,), 2.0, device="cuda")
res = []
ONLY = os.environ.get("ONLY")
for name, K, R, fwd, subs in (("fwd qkv", 4096, 48, True, 1), ("fwd o", 4096, 16, True, 1),
                              ("fwd gate_up", 4096, 32, True, 1), ("fwd down", 11008, 16, True, 1),
                              ("dH qkv", 12288, 48, False, 3), ("dH o", 4096, 16, False, 1),
                              ("dH gate_up", 22016, 32, False, 2), ("dH down", 4096, 16, False, 1)):
    reps = 6
    if ONLY and name != ONLY:
        continue
    if fwd:
        Xs = [torch.randn(T, K, device="cuda").to(torch.bfloat16) for _ in range(reps)]
        A = torch.randn(cfg.n_adapters, R, K, device="cuda").to(torch.bfloat16)
        H16 = torch.empty(T, R, device="cuda", dtype=torch.bfloat16)
        Hs = torch.empty(max(1, plan.n_slots) * 256, R, device="cuda", dtype=torch.bfloat16)
        groups = [(g, min(64, R - g), 0, K) for g in range(0, R, 64)]

        def run(i):
            if TC:
                g = ops.shrink_tc_groups(groups)
                ops.lora_shrink_tc(Xs[i % reps], A, *plan.tc_units(g[0][1]), TC, plan.row_adapter,
                                   scale, g, R, H16=H16, Hslots=Hs, slot_of_row=plan.slot_of_row,
                                   tile_slot_ptr=plan.tile_slot_ptr)
                return
            ops.lora_shrink(Xs[i % reps], A, plan.shrink_tiles, plan.n_shrink_tiles, scale, groups, R,
                            H16=H16, Hslots=Hs, slot_of_row=plan.slot_of_row,
                            tile_slot_ptr=plan.tile_slot_ptr)
        nbytes = 2 * T * K + 2 * len({a for a in mb.seg_adapter if a >= 0}) * R * K
    else:
        Xs = [torch.randn(Ttr, K, device="cuda").to(torch.bfloat16) for _ in range(reps)]
        BT = torch.randn(R, K, device="cuda").to(torch.bfloat16)
        H16 = torch.empty(Ttr, R, device="cuda", dtype=torch.bfloat16)
        H16lo = torch.empty(Ttr, R, device="cuda", dtype=torch.bfloat16) \
            if os.environ.get("NO_LO") != "1" else None
        n = K // subs
        rp = R // subs
        groups = [(s * rp, rp, s * n, (s + 1) * n) for s in range(subs)]

        def run(i):
            if TC:
                g = ops.shrink_tc_groups(groups)
                ops.lora_shrink_tc(Xs[i % reps], BT, *tplan.tc_units(g[0][1]), TC, tplan.row_adapter,
                                   scale, g, R, a_stride=0, H16=H16, H16lo=H16lo)
                return
            ops.lora_shrink(Xs[i % reps], BT, tplan.shrink_tiles, tplan.n_shrink_tiles, scale, groups,
                            R, a_stride=0, H16=H16, H16lo=H16lo)
        nbytes = 2 * Ttr * K + 2 * R * K
    for i in range(3):
        run(i)
    torch.cuda.synchronize()
    n = 30
    g = torch.cuda.CUDAGraph()  # replay removes the Python launch overhead between kernels
    st = torch.cuda.Stream()
    st.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(st), torch.cuda.graph(g, stream=st):
        for i in range(n):
            run(i)
    torch.cuda.current_stream().wait_stream(st)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / n * 1e3
    res.append((name, us, nbytes / us / 1e6))
print(f"TC={TC}: " +
      "  ".join(f"{n} {us:.1f}us {tb:.2f}TB/s" for n, us, tb in res))
