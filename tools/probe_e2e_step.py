"""Per-call wall clock of the bench's e2e step (config 5 from pinned host buffers)."""
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
X = tt.pack(x, sx, S)   # the bench keeps its resident copy as well
host_x = x.to("cpu").pin_memory()
host_w = w.to("cpu").pin_memory()
torch.cuda.empty_cache()


def step(log):
    def lap(name, t0):
        torch.cuda.synchronize()
        log.append((name, (time.perf_counter() - t0) * 1e3))
    t = time.perf_counter(); Xh = tt.pack(host_x, sx, S); lap("pack X", t)
    t = time.perf_counter(); Wh = tt.pack(host_w, sw, S); lap("pack W", t)
    for k in (1, 2, 3):
        t = time.perf_counter(); r = tt.tt_mul_sum(Xh, Wh, k); lap(f"mul_sum {k}", t)
        t = time.perf_counter(); res = tt.unpack(r); lap(f"unpack {k}", t)
    t = time.perf_counter(); del Xh, Wh, r, res; lap("release", t)


for i in range(3):
    log = []
    t0 = time.perf_counter()
    step(log)
    print(f"step {i}: {(time.perf_counter() - t0) * 1e3:.1f} ms  " + "  ".join(f"{n} {v:.1f}" for n, v in log))


def plain():
    Xh = tt.pack(host_x, sx, S)
    Wh = tt.pack(host_w, sw, S)
    for k in (1, 2, 3):
        res = tt.unpack(tt.tt_mul_sum(Xh, Wh, k))


plain()
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(3):
    plain()
torch.cuda.synchronize()
print(f"unsynchronised step: {(time.perf_counter() - t0) / 3 * 1e3:.1f} ms")
