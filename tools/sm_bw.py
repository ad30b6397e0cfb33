"""Per-SM HBM streaming bandwidth (tools/sm_bw.cu): GB/s for W SMs pulling a 2 GB buffer by
bulk-copy rings (stages x chunk bytes in flight per SM) and by LDG.128.  usage: sm_bw.py"""
import ctypes
import os

import torch

here = os.path.dirname(os.path.abspath(__file__))
so = os.path.join(here, "sm_bw.so")
lib = ctypes.CDLL(so)
buf = torch.empty(2 << 30, dtype=torch.uint8, device="cuda")
buf.random_(0, 255)
sink = torch.zeros(4, dtype=torch.int64, device="cuda")
st = torch.cuda.current_stream()
total = 1 << 30


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e-3


def bw(ctas, cl, stages, chunk, pieces=1, box_rows=0, box_kb=0):
    per = (total // ctas) // chunk * chunk
    if box_rows:
        per = (total // ctas) // (8192 * 256) * (8192 * 256)
    t = timed(lambda: lib.run_bw(ctypes.c_void_p(buf.data_ptr()), ctypes.c_longlong(per),
                                 ctas, cl, stages, chunk, ctypes.c_void_p(sink.data_ptr()),
                                 ctypes.c_void_p(st.cuda_stream), pieces, box_rows, box_kb))
    return per * ctas / t / 1e9


for P, cw, stages, chunk in ((1, 1, 6, 32768), (2, 1, 6, 32768), (3, 1, 6, 32768), (4, 1, 4, 49152),
                           (1, 4, 6, 32768), (2, 4, 6, 32768), (1, 1, 3, 65536), (3, 1, 3, 65536),
                           (4, 1, 12, 16384), (1, 1, 12, 16384)):
    per = (total // 16) // chunk * chunk
    t = timed(lambda: lib.run_multiprod(ctypes.c_void_p(buf.data_ptr()), ctypes.c_longlong(per), 16, stages,
                                        chunk, P, cw, ctypes.c_void_p(sink.data_ptr()), ctypes.c_void_p(st.cuda_stream)))
    g = per * 16 / t / 1e9
    print(f"producers={P} consumers={cw} ring {stages}x{chunk // 1024}KB: {g:7.1f} GB/s ({g / 16:6.1f}/SM)")
