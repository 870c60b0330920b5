"""Times pack / unpack of the config-5 tensor (16 GiB) with CUDA events."""
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
torch.cuda.synchronize()
if "--heat" in sys.argv:  # the bench's order: fused products first
    W = tt.pack(torch.empty((1, 2048, 512), dtype=torch.float64, device="cuda").uniform_(),
                tt.parse_shape(configs.C5_W_SHAPE), S)
    for _ in range(int(sys.argv[sys.argv.index("--heat") + 1])):
        for k in (1, 2, 3):
            tt.tt_mul_sum(X, W, k)
    torch.cuda.synchronize()
    if "--empty" in sys.argv:
        torch.cuda.empty_cache()
    print("allocated GiB", torch.cuda.memory_allocated() / 2**30, "reserved", torch.cuda.memory_reserved() / 2**30)
if "--heat2" in sys.argv:  # sustained pack load first
    for _ in range(40):
        tt.pack(x, sx, S)
    torch.cuda.synchronize()
if "--alloc" in sys.argv:  # keep the previous result alive: a different output block each time
    keep = [tt.pack(x, sx, S)]
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for name, fn in (("pack", lambda: tt.pack(x, sx, S)), ("unpack", lambda: tt.unpack_device(X))):
    fn()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(5):
        fn()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(f"{name}: {ms:.3f} ms = {2 * 2**34 / ms / 1e6:.0f} GB/s")
