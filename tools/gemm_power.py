"""SM clock and board power while one GEMM shape runs back to back for ~2 s: collm (auto) vs
cuBLAS.  Tells whether a shape is power/clock-bound (sw_power_cap) and at what clock each
implementation runs.  usage: gemm_power.py M N K [seconds]"""
import os
import subprocess
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2604_16400_b200 import ops  # noqa: E402

M, N, K = (int(x) for x in sys.argv[1:4])
secs = float(sys.argv[4]) if len(sys.argv) > 4 else 2.0
A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
Ws = [torch.randn(N, K, device="cuda").to(torch.bfloat16) for _ in range(3)]
Y = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)


def graph_of(fn, reps=30):
    for i in range(3):
        fn(i)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    st = torch.cuda.Stream()
    st.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(st), torch.cuda.graph(g, stream=st):
        for i in range(reps):
            fn(i)
    torch.cuda.current_stream().wait_stream(st)
    return g, reps


def measure(name, fn):
    g, reps = graph_of(fn)
    g.replay()
    torch.cuda.synchronize()
    smi = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,clocks_throttle_reasons.active",
                            "--format=csv,noheader,nounits", "-lms", "50"], stdout=subprocess.PIPE, text=True)
    time.sleep(0.2)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t_end = time.time() + secs
    n = 0
    e0.record()
    while time.time() < t_end:
        g.replay()
        n += 1
        if n % 20 == 0:
            torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    smi.terminate()
    out = smi.communicate()[0].strip().splitlines()
    rows = [r.split(",") for r in out if r.strip()]
    clk = sorted(float(r[0]) for r in rows[4:-2]) or [0]
    pw = sorted(float(r[1]) for r in rows[4:-2]) or [0]
    us = e0.elapsed_time(e1) / (n * reps) * 1e3
    print(f"{name:8s} {us:7.1f} us/launch {2 * M * N * K / (us * 1e-6) / 1e12:6.0f} TF/s  "
          f"sm clock median {clk[len(clk) // 2]:.0f} MHz  power median {pw[len(pw) // 2]:.0f} W  "
          f"reasons {sorted({r[2].strip() for r in rows})}")


measure("collm", lambda i: ops.gemm_lora(A, Ws[i % 3], Y))
measure("cublas", lambda i: torch.matmul(A, Ws[i % 3].t(), out=Y))
