"""Debug: bitwise repeatability of the step (same mode twice) and across modes."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from tests.test_gpu_stack import _stack, _state  # noqa: E402

key = sys.argv[1] if len(sys.argv) > 1 else "llama3-8b:1"
steps = int(os.environ.get("STEPS", "2"))
bwd = os.environ.get("BWD", "1") == "1"


def run(overlap):
    st, plan = _stack(overlap, key)
    for _ in range(steps):
        st.run_step(plan, backward=bwd)
    torch.cuda.synchronize()
    out = _state(st)
    del st
    return out


res = {}
for name, ov in (("serial-a", False), ("serial-b", False), ("overlap-a", True), ("overlap-b", True)):
    res[name] = run(ov)
base = res["serial-a"]
for name, st in res.items():
    diffs = [i for i, (a, b) in enumerate(zip(base, st)) if not torch.equal(a, b)]
    print(f"{key} steps={steps} bwd={bwd} {name}: {'identical' if not diffs else 'DIFF in tensors ' + str(diffs[:8])}", flush=True)
