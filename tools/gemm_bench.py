"""Time the collm GEMM alone on Llama-7B projection shapes (CUDA events) for several forced
kernel variants.  VARIANTS="cg:bn:sched,..." (default: auto + all pure variants)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2604_16400_b200 import ops  # noqa: E402

SHAPES = [("qkv", 1024, 12288, 4096), ("o", 1024, 4096, 4096), ("gate_up", 1024, 22016, 4096),
          ("down", 1024, 4096, 11008), ("dX_qkv", 512, 4096, 12288), ("dX_o", 512, 4096, 4096),
          ("dX_gu", 512, 4096, 22016), ("dX_down", 512, 11008, 4096)]
if os.environ.get("TINY"):
    SHAPES = [("t256", 256, 256, 64), ("t256k4k", 256, 256, 4096), ("t512x4kx64", 512, 4096, 64)]
if os.environ.get("BIG"):
    SHAPES = SHAPES + [("big", 4096, 8192, 8192), ("big2", 8192, 8192, 8192)]
DEFAULT = "auto,1:256:dp,1:128:dp,1:256:hybrid,2:256:dp,2:128:dp,2:256:hybrid,2:128:hybrid"


def set_variant(v):
    for k in ("COLLM_GEMM_CG", "COLLM_GEMM_BN", "COLLM_GEMM_SCHED", "COLLM_GEMM_MC"):
        os.environ.pop(k, None)
    os.environ.pop("COLLM_GEMM_LEAN", None)
    if v.endswith("+lean"):
        os.environ["COLLM_GEMM_LEAN"] = "1"
        v = v[:-5]
    if v != "auto":
        cg, bn, sc, *mc = v.split(":")
        os.environ.update(COLLM_GEMM_CG=cg, COLLM_GEMM_BN=bn, COLLM_GEMM_SCHED=sc)
        if mc:
            os.environ["COLLM_GEMM_MC"] = mc[0]


def main():
    variants = os.environ.get("VARIANTS", DEFAULT).split(",")
    res = {}
    for name, M, N, K in SHAPES:
        A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
        Ws = [torch.randn(N, K, device="cuda").to(torch.bfloat16) for _ in range(3)]
        Y = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
        reps = 30

        def graph_time(fn):
            """us per launch of fn(i) over `reps` launches replayed from one CUDA graph (no host
            launch overhead between kernels)."""
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
            g.replay()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            g.replay()
            e1.record()
            torch.cuda.synchronize()
            return e0.elapsed_time(e1) / reps * 1e3

        for v in variants:
            set_variant(v)
            us = graph_time(lambda i: ops.gemm_lora(A, Ws[i % 3], Y))
            res[(name, v)] = (us, 2 * M * N * K / (us * 1e-6) / 1e12)
        # cuBLAS (torch.matmul) on the same shape, same W rotation (the library baseline)
        us = graph_time(lambda i: torch.matmul(A, Ws[i % 3].t(), out=Y))
        res[(name, "cublas")] = (us, 2 * M * N * K / (us * 1e-6) / 1e12)
    variants = variants + ["cublas"]
    print(f"{'shape':8s} " + " ".join(f"{v:>14s}" for v in variants))
    for name, *_ in SHAPES:
        print(f"{name:8s} " + " ".join(f"{res[(name, v)][0]:7.1f}/{res[(name, v)][1]:5.0f}" for v in variants))


if __name__ == "__main__":
    main()
