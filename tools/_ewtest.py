import sys, time
sys.path.insert(0, "/root/repo")
import torch
import paper_2011_01805_b200 as tt
from paper_2011_01805_b200 import configs
S = tt.Session(configs.C5_SLOTS, 8)
sx, sw = tt.parse_shape(configs.C5_X_SHAPE), tt.parse_shape(configs.C5_W_SHAPE)
x = torch.empty(configs.C5_DIMS, dtype=torch.float64, device="cuda")
w = torch.empty((1, 2048, 512), dtype=torch.float64, device="cuda")
tt.fill_uniform(S, x, configs.C5_SEED_X, -1.0, 1.0); tt.fill_uniform(S, w, configs.C5_SEED_W, -1.0, 1.0)
X, W = tt.pack(x, sx, S), tt.pack(w, sw, S)
del x
torch.cuda.synchronize()
for i in range(5):
    t0 = time.perf_counter(); r = tt.tt_mul(X, W); t1 = time.perf_counter(); torch.cuda.synchronize(); t2 = time.perf_counter()
    print(i, "fast" if r._block is not None else "slow", f"host {(t1-t0)*1e3:.2f} ms total {(t2-t0)*1e3:.2f} ms", hex(r._p))
    del r
for i in range(3):
    t0 = time.perf_counter(); r = tt.tt_add(X, X); t1 = time.perf_counter(); torch.cuda.synchronize(); t2 = time.perf_counter()
    print("add", i, "fast" if r._block is not None else "slow", f"host {(t1-t0)*1e3:.2f} ms total {(t2-t0)*1e3:.2f} ms", hex(r._p))
    del r
