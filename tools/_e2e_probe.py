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
hx = x.cpu().pin_memory(); hw = w.cpu().pin_memory()
del x; torch.cuda.empty_cache()
def tm(label, fn, n=2):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n): r = fn()
    torch.cuda.synchronize()
    print(f"{label}: {(time.perf_counter()-t0)/n*1e3:.1f} ms"); return r
X = tm("pack(host_x) staged", lambda: tt.pack(hx, sx, S))
T = tt.tiletensor
old = T._STAGED_MIN; T._STAGED_MIN = 1 << 62
tm("pack(host_x) one piece", lambda: tt.pack(hx, sx, S))
T._STAGED_MIN = old
W = tm("pack(host_w)", lambda: tt.pack(hw, sw, S))
tm("3 mul_sum", lambda: [tt.tt_mul_sum(X, W, k) for k in (1, 2, 3)])
rs = [tt.tt_mul_sum(X, W, k) for k in (1, 2, 3)]
tm("3 unpack+D2H", lambda: [tt.unpack(r) for r in rs])
def step():
    Xh = tt.pack(hx, sx, S); Wh = tt.pack(hw, sw, S)
    return [tt.unpack(tt.tt_mul_sum(Xh, Wh, k)) for k in (1, 2, 3)]
tm("e2e step", step, 3)
for k, r in zip((1, 2, 3), rs):
    tm(f"unpack_device dim{k} {tt.format_shape(r.shape())}", lambda: tt.unpack_device(r), 5)
    d = tt.unpack_device(r)
    tm(f"  D2H {d.numel()*8/2**20:.0f} MiB pageable", lambda: d.cpu(), 5)
    hp = torch.empty(d.shape, dtype=d.dtype).pin_memory()
    tm(f"  D2H pinned", lambda: hp.copy_(d), 5)
