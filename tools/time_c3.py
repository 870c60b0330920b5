"""Config 3 "3b" timing: matmul_b then matmul_a as two calls and as one
tt_linalg_chain2 launch (CUDA events, device-resident operands)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2011_01805_b200 as tt  # noqa: E402
from paper_2011_01805_b200 import configs  # noqa: E402

c3 = configs.config3()
S = tt.Session(8192, 8)
T = {k: tt.pack(c3.tensors[k], tt.parse_shape(v), S) for k, v in c3.shapes.items()
     if k in ("A3", "Bt3", "C3")}


def timeit(fn, reps=50):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


two = timeit(lambda: tt.matmul_a(T["A3"], tt.matmul_b(T["Bt3"], T["C3"])))
one_b = timeit(lambda: tt.matmul_b(T["Bt3"], T["C3"]))
r1 = tt.matmul_b(T["Bt3"], T["C3"])
one_a = timeit(lambda: tt.matmul_a(T["A3"], r1))
ch = timeit(lambda: tt.linalg_chain("matmul_b", T["Bt3"], T["C3"], "matmul_a", T["A3"]))
alg = 4864 * 8192 * 8
print(f"two calls {two:.1f} us  (matmul_b {one_b:.1f}, matmul_a {one_a:.1f})  chain {ch:.1f} us"
      f"  -> {alg / ch / 1e3:.0f} GB/s = {alg / ch / 1e3 / 8000:.3f} of 8 TB/s")
