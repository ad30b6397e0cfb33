"""Ours vs cuBLAS (torch.matmul) per GEMM shape of the BASELINE configs' steps: base projection
GEMMs (no LoRA stages; the forward of all rows and the dX of the training rows), graph-replayed
over rotating weights (inputs > L2), CUDA events.  Writes a markdown table to stdout.

  python tools/gemm_table.py [llama2-7b llama3-8b llama2-13b]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2604_16400_b200 import _lib, ops  # noqa: E402
from paper_2604_16400_b200.configs import CONFIGS  # noqa: E402
from paper_2604_16400_b200.segments import build_mixed_batch  # noqa: E402


def graph_us(fn, reps):
    for i in range(2):
        fn(i)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    st = torch.cuda.Stream()
    st.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(st), torch.cuda.graph(g, stream=st):
        for i in range(reps):
            fn(i)
    torch.cuda.current_stream().wait_stream(st)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


def main():
    _lib.load()
    keys = sys.argv[1:] or ["llama2-7b", "llama3-8b", "llama2-13b"]
    print("| config | GEMM | M x N x K | ours us | ours TFLOP/s | cuBLAS us | cuBLAS TFLOP/s | ours / cuBLAS time |")
    print("|---|---|---|---|---|---|---|---|")
    for key in keys:
        cfg = CONFIGS[key]
        mb = build_mixed_batch(*cfg.batch(0))
        T, Ttr = mb.n_rows, mb.n_train_rows
        for sp in cfg.projections:
            K, N = sp.in_features, sp.out_features
            for what, M, n, k in (("fwd " + sp.name, T, N, K), ("dX " + sp.name, Ttr, K, N)):
                if M == 0:
                    continue
                nrot = max(2, min(4, int(3e9 // (2 * n * k))))
                Ws = [torch.randn(n, k, device="cuda").to(torch.bfloat16) for _ in range(nrot)]
                A = torch.randn(M, k, device="cuda").to(torch.bfloat16)
                Y = torch.empty(M, n, device="cuda", dtype=torch.bfloat16)
                reps = 20 if M * n * k < 1e11 else 6
                ours = graph_us(lambda i: ops.gemm_lora(A, Ws[i % nrot], Y), reps)
                cub = graph_us(lambda i: torch.matmul(A, Ws[i % nrot].t(), out=Y), reps)
                fl = 2 * M * n * k
                print(f"| {key} | {what} | {M} x {n} x {k} | {ours:.1f} | {fl / ours / 1e6:.0f} | "
                      f"{cub:.1f} | {fl / cub / 1e6:.0f} | {ours / cub:.3f} |", flush=True)
                del Ws, A, Y
                torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
