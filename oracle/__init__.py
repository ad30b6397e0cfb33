"""CPU oracle for the co-batched LoRA layer — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline / reference arm may
import this package, and only as the checker (or the timed CPU baseline), never as the product
path.  The product path is ``paper_2604_16400_b200`` over ``libcollm.so`` and has no CPU fallback.

Parity status:
  * fedavg / adapter layout / round averaging: PINNED — checked bit-for-bit against fixtures
    produced by importing the reference (``tests/golden/make_golden.py``).
  * LoRA forward/backward/AdamW numerics: PARITY UNPINNED against the reference — the reference
    (a discrete-event simulator) contains no LoRA arithmetic.  The restatement follows
    PAPER.md:359-366 (W_pre frozen, dW = B.A, B (d x r), A (r x l)) and launcher.py:28-47 (adapter
    layout), and is cross-checked against an independent torch-autograd float64 formulation
    committed as golden vectors.
"""

from .lora_oracle import *  # noqa: F401,F403
