"""Times the unfused elementwise product tt_mul(X, W) and tt_add(X, X) on the
config-5 tensors (CUDA events): 16 GiB in (+ broadcast W), 16 GiB out."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2011_01805_b200 as tt  # noqa: E402
from paper_2011_01805_b200 import configs  # noqa: E402

S = tt.Session(16384, 8)
sx, sw = tt.parse_shape(configs.C5_X_SHAPE), tt.parse_shape(configs.C5_W_SHAPE)
x = torch.empty(configs.C5_DIMS, dtype=torch.float64, device="cuda")
tt.fill_uniform(S, x, configs.C5_SEED_X, -1.0, 1.0)
w = torch.empty((1, 2048, 512), dtype=torch.float64, device="cuda")
tt.fill_uniform(S, w, configs.C5_SEED_W, -1.0, 1.0)
X, W = tt.pack(x, sx, S), tt.pack(w, sw, S)
del x
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for name, fn, nbytes in (("mul X*W", lambda: tt.tt_mul(X, W), 2 * 2**34 + 2**27),
                         ("add X+X", lambda: tt.tt_add(X, X), 2 * 2**34)):
    fn()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(5):
        fn()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(f"{name}: {ms:.3f} ms = {nbytes / ms / 1e6:.0f} GB/s")
