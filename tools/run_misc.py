"""Bandwidth of the remaining tile passes on config-5-sized data (CUDA events):
tt_sum over each dim (unfused), rotate (tile primitive), clean_unknowns and
replicate_dim on a '?' result."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2011_01805_b200 as tt  # noqa: E402
from paper_2011_01805_b200 import configs  # noqa: E402

S = tt.Session(16384, 8)
sx = tt.parse_shape(configs.C5_X_SHAPE)
x = torch.empty(configs.C5_DIMS, dtype=torch.float64, device="cuda")
tt.fill_uniform(S, x, configs.C5_SEED_X, -1.0, 1.0)
X = tt.pack(x, sx, S)
del x
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def timeit(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


G = 2 ** 34
for k, out_tiles in ((1, 1024), (2, 2048), (3, 8192)):
    ms = timeit(lambda: tt.tt_sum(X, k))
    nb = G + out_tiles * 16384 * 8
    print(f"tt_sum dim {k}: {ms:.3f} ms = {nb / ms / 1e6:.0f} GB/s")
ms = timeit(lambda: tt.tiles_rotate(S, X.data(), 5))
print(f"rotate (all tiles, r=5): {ms:.3f} ms = {2 * G / ms / 1e6:.0f} GB/s")
R = tt.tt_sum(X, 3)  # [2048/16,2048/32,1?/32]: 8192 tiles with '?'
ms = timeit(lambda: tt.clean_unknowns(R), 10)
nb = 2 * 8192 * 16384 * 8
print(f"clean_unknowns (8192 tiles): {ms:.3f} ms = {nb / ms / 1e6:.0f} GB/s")
C = tt.clean_unknowns(R)
ms = timeit(lambda: tt.replicate_dim(C, 3), 10)
print(f"replicate_dim 3 (8192 tiles, 5 levels): {ms:.3f} ms = {nb / ms / 1e6:.0f} GB/s")
