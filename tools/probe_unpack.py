"""Config-5 unpack (16 GiB of tiles -> 16 GiB dense) against pack, CUDA events."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2011_01805_b200 as tt  # noqa: E402

S = tt.Session(16384, 8)
sx = tt.parse_shape("[2048/16,2048/32,512/32]")
x = torch.empty((2048, 2048, 512), dtype=torch.float64, device="cuda")
tt.fill_uniform(S, x, 5, -1.0, 1.0)
X = tt.pack(x, sx, S)


def ev(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / reps


nb = 2 * x.numel() * 8
for name, fn in (("pack", lambda: tt.pack(x, sx, S)), ("unpack_device", lambda: tt.unpack_device(X))):
    ms = ev(fn)
    print(f"{name}: {ms:.3f} ms = {nb / ms / 1e6:.0f} GB/s")
y = tt.unpack_device(X)
print("round trip bitwise:", bool(torch.equal(x, y)))
# a partial-tile shape (padding on every dim) through the same kernels
sp = tt.parse_shape("[2000/16,2040/32,500/32]")
xp = torch.empty((2000, 2040, 500), dtype=torch.float64, device="cuda")
tt.fill_uniform(S, xp, 7, -1.0, 1.0)
XP = tt.pack(xp, sp, S)
nbp = xp.numel() * 8 + sp.tile_count() * 16384 * 8
for name, fn in (("pack (padded)", lambda: tt.pack(xp, sp, S)), ("unpack (padded)", lambda: tt.unpack_device(XP))):
    ms = ev(fn)
    print(f"{name}: {ms:.3f} ms = {nbp / ms / 1e6:.0f} GB/s")
print("round trip bitwise:", bool(torch.equal(xp, tt.unpack_device(XP))))
