"""Runs the small configs (1, 2, 4) a few times -- for ncu launch lists."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2011_01805_b200 as tt  # noqa: E402
from paper_2011_01805_b200 import configs  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "c1"
if which == "c1":
    c1 = configs.config1()
    S = tt.Session(512, 8)
    sA = tt.parse_shape(c1.shapes["A"])
    A, B = tt.pack(c1.tensors["A"], sA, S), tt.pack(c1.tensors["B"], sA, S)
    for _ in range(3):
        tt.tt_mul_sum(A, B, 2)
elif which == "c2":
    c2 = configs.config2()
    S = tt.Session(8192, 8)
    M = tt.pack(c2.tensors["M"], tt.parse_shape(c2.shapes["M"]), S)
    V = tt.pack(c2.tensors["V"], tt.parse_shape(c2.shapes["V"]), S)
    for _ in range(3):
        tt.matvec_a(M, V)
elif which == "c4f":  # one call per layer (tt_mul_sum_affine), as the bench
    c4 = configs.config4(True)
    S = tt.Session(8192, 8)
    T = {k: tt.pack(c4.tensors[k], tt.parse_shape(v), S) for k, v in c4.shapes.items()}
    for _ in range(2):
        h = tt.tt_mul_sum_affine(T["W1t"], T["X"], 1, T["b1"], square=True)
        tt.tt_mul_sum_affine(T["W2"], h, 2, T["b2"])
else:
    c4 = configs.config4(True)
    S = tt.Session(8192, 8)
    T = {k: tt.pack(c4.tensors[k], tt.parse_shape(v), S) for k, v in c4.shapes.items()}
    for _ in range(2):
        h = tt.tt_add(tt.tt_mul_sum(T["W1t"], T["X"], 1), T["b1"])
        h = tt.tt_mul(h, h)
        tt.tt_add(tt.tt_mul_sum(T["W2"], h, 2), T["b2"])
torch.cuda.synchronize()
print("ok")
