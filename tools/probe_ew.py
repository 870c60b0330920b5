"""Config-5 broadcast elementwise (X * W, W broadcast along dim 1), paired vs unpaired items."""
import os
import sys
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


def ev(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / reps


nb = (2 * sx.tile_count() + sw.tile_count()) * 16384 * 8
for name, fn in (("X * W", lambda: tt.tt_mul(X, W)), ("W * X", lambda: tt.tt_mul(W, X)),
                 ("X + W", lambda: tt.tt_add(X, W)), ("X + X", lambda: tt.tt_add(X, X))):
    ms = ev(fn)
    print(f"TT_EW_PAIR={os.environ.get('TT_EW_PAIR', '1')} {name}: {ms:.3f} ms = {nb / ms / 1e6:.0f} GB/s")
