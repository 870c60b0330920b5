"""One config-3 '3b' chain (matmul_b then matmul_a) after warm-up: a target for
`ncu --set full` capturing the chain's four kernels (two GEMM folds, two trees)."""
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
for _ in range(3):
    r = tt.matmul_a(T["A3"], tt.matmul_b(T["Bt3"], T["C3"]))
torch.cuda.synchronize()
print("done")
