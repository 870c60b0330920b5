"""Duration of the first config-5 dim-1 launch after a synchronize, against the GPU's idle time
before it (CUDA events around single launches)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2011_01805_b200 as tt  # noqa: E402

S = tt.Session(16384, 8)
sx = tt.parse_shape("[2048/16,2048/32,512/32]")
sw = tt.parse_shape("[*/16,2048/32,512/32]")
x = torch.empty((2048, 2048, 512), dtype=torch.float64, device="cuda")
w = torch.empty((1, 2048, 512), dtype=torch.float64, device="cuda")
tt.fill_uniform(S, x, 5, -1.0, 1.0)
tt.fill_uniform(S, w, 6, -1.0, 1.0)
X, W = tt.pack(x, sx, S), tt.pack(w, sw, S)
del x
for idle_ms in (0, 0, 1, 5, 20, 100):
    for _ in range(3):
        for k in (1, 2, 3):
            tt.tt_mul_sum(X, W, k)
    torch.cuda.synchronize()
    if idle_ms:
        time.sleep(idle_ms / 1e3)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
    ev[0].record()
    for i in range(4):
        tt.tt_mul_sum(X, W, 1)
        ev[i + 1].record()
    torch.cuda.synchronize()
    print(f"idle {idle_ms:3d} ms: dim-1 launches " + " ".join(f"{ev[i].elapsed_time(ev[i + 1]):.3f}" for i in range(4)))
