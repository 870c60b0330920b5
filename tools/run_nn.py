"""Times cryptonets_infer (paper_2011_01805_b200/nn.py) on the CryptoNets network:
batch packed (tile [1,1,s], every scalar a tile of s samples) and tiled
([32,256,1]-style), CUDA events around the whole call."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2011_01805_b200 as tt  # noqa: E402
from paper_2011_01805_b200 import nn  # noqa: E402

net = nn.cryptonets_network(42)
for s, tile, n in ((8192, (1, 1, 8192), 8192), (8192, (32, 256, 1), 1), (8192, (8, 16, 64), 64)):
    S = tt.Session(s, 8)
    batch = np.random.default_rng(1).uniform(0, 1, size=(784, n))
    if "--device" in sys.argv:  # batch already resident on the GPU: no H2D in the timed calls
        batch = torch.from_numpy(batch).cuda()
    nn.cryptonets_infer(net, batch, tile, S)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    reps = 3
    for _ in range(reps):
        r = nn.cryptonets_infer(net, batch, tile, S)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / reps
    print(f"tile {tile} batch {n}: {dt * 1e3:.2f} ms per call ({n / dt:.0f} samples/s), "
          f"rot={r.cost.rotations} mul={r.cost.multiplications}")
if "--compiled" in sys.argv:
    S = tt.Session(8192, 8)
    batch = torch.from_numpy(np.random.default_rng(1).uniform(0, 1, size=(784, 8192))).cuda()
    comp = nn.CompiledBatchPacked(net, S)
    comp.infer(batch)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(10):
        r = comp.infer(batch)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / 10
    print(f"compiled batch packed 8192: {dt * 1e3:.3f} ms per call ({8192 / dt:.0f} samples/s)")
if "--compiled" in sys.argv:
    S = tt.Session(8192, 8)
    comp = nn.CompiledTiled(net, (32, 256, 1), S)
    one = np.random.default_rng(1).uniform(0, 1, size=(784, 1))
    comp.infer(one)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(10):
        r = comp.infer(one)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / 10
    print(f"compiled tiled (32, 256, 1), 1 sample: {dt * 1e3:.3f} ms per call")

