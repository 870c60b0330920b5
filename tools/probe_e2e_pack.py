"""Where the e2e step's time goes: one plain H2D of the config-5 dense input against
tt.pack() of the pinned host tensor (slabs, copy overlapped) at several slab sizes."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2011_01805_b200 as tt  # noqa: E402
from paper_2011_01805_b200 import tiletensor as T  # noqa: E402

S = tt.Session(16384, 8)
sx = tt.parse_shape("[2048/16,2048/32,512/32]")
x = torch.empty((2048, 2048, 512), dtype=torch.float64, device="cuda")
tt.fill_uniform(S, x, 5, -1.0, 1.0)
host = x.to("cpu").pin_memory()
del x
torch.cuda.empty_cache()
d = torch.empty(host.numel(), dtype=torch.float64, device="cuda")


def timed(fn, reps=2):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e3


nb = host.numel() * 8
ms = timed(lambda: d.copy_(host.reshape(-1), non_blocking=True))
print(f"plain H2D of {nb / 2**30:.0f} GiB: {ms:.1f} ms = {nb / ms / 1e6:.1f} GB/s")
del d
torch.cuda.empty_cache()
for slab in (64, 128, 256, 512, 1024):
    T._STAGED_SLAB = slab << 20
    ms = timed(lambda: tt.pack(host, sx, S))
    print(f"tt.pack(pinned host), {slab} MiB slabs: {ms:.1f} ms = {nb / ms / 1e6:.1f} GB/s")
