"""Runs the config-3 '3b' chain (matmul_b then matmul_a) a few times -- for
ncu launch lists and kernel captures of the tile-matmul path.  With --time,
prints the mean chain time from CUDA events (after warm-up)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2011_01805_b200 as tt  # noqa: E402
from paper_2011_01805_b200 import configs  # noqa: E402

args = [a for a in sys.argv[1:] if not a.startswith("--")]
reps = int(args[0]) if args else 3
if len(args) > 1:
    tt.set_kernel_path(args[1])
c3 = configs.config3()
S = tt.Session(8192, 8)
T = {k: tt.pack(c3.tensors[k], tt.parse_shape(v), S) for k, v in c3.shapes.items()
     if k in ("A3", "Bt3", "C3")}


def chain():
    s1 = tt.matmul_b(T["Bt3"], T["C3"])
    return tt.matmul_a(T["A3"], s1)


for _ in range(reps):
    r = chain()
torch.cuda.synchronize()
if "--time" in sys.argv:
    n = 50
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        r = chain()
    e1.record()
    torch.cuda.synchronize()
    print(f"c3b chain: {e0.elapsed_time(e1) / n * 1e3:.1f} us")
    s1 = tt.matmul_b(T["Bt3"], T["C3"])
    for name, fn in (("matmul_b", lambda: tt.matmul_b(T["Bt3"], T["C3"])),
                     ("matmul_a", lambda: tt.matmul_a(T["A3"], s1))):
        fn()
        e0.record()
        for _ in range(n):
            fn()
        e1.record()
        torch.cuda.synchronize()
        print(f"  {name}: {e0.elapsed_time(e1) / n * 1e3:.1f} us")
if "--timeline" in sys.argv:
    # per-kernel durations and the idle gaps between them (CUPTI via the torch
    # profiler): how much of the chain is launch / ramp rather than kernel time
    from torch.profiler import ProfilerActivity, profile
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        r = chain()
    g.replay()
    torch.cuda.synchronize()
    for mode in ("api", "graph"):
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            for _ in range(20):
                if mode == "api":
                    r = chain()
                else:
                    g.replay()
            torch.cuda.synchronize()
        ev = sorted((e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA
                     and "Memcpy" not in e.name and "Memset" not in e.name),
                    key=lambda e: e.time_range.start)
        per = len(ev) // 20
        rows = {}
        for i in range(per, len(ev)):  # skip the first chain
            e, prev = ev[i], ev[i - 1]
            k = i % per
            d = rows.setdefault(k, [e.name[:60], 0.0, 0.0, 0])
            d[1] += e.time_range.end - e.time_range.start
            d[2] += e.time_range.start - prev.time_range.end
            d[3] += 1
        print(f"[{mode}] kernels per chain: {per}")
        tot_k = tot_g = 0.0
        for k in sorted(rows):
            name, dur, gap, c = rows[k]
            tot_k += dur / c
            tot_g += gap / c
            print(f"  {dur / c:7.2f} us  gap-before {gap / c:6.2f} us  {name}")
        print(f"  kernels {tot_k:.1f} us + gaps {tot_g:.1f} us per chain")
if "--host" in sys.argv:
    import time
    import cProfile
    import pstats
    t0 = time.perf_counter()
    for _ in range(200):
        r = chain()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    print(f"host: {(t1 - t0) / 200 * 1e6:.1f} us per chain (enqueue only)")
    pr = cProfile.Profile()
    pr.enable()
    for _ in range(200):
        r = chain()
    pr.disable()
    torch.cuda.synchronize()
    pstats.Stats(pr).sort_stats("tottime").print_stats(6)
    from paper_2011_01805_b200 import _abi
    L = tt.tiletensor.lib()
    fn = L.tt_linalg_product
    acc = [0.0, 0]

    def timed(*a):
        t = time.perf_counter()
        r = fn(*a)
        acc[0] += time.perf_counter() - t
        acc[1] += 1
        return r

    class Proxy:
        def __getattr__(self, n):
            return timed if n == "tt_linalg_product" else getattr(L, n)

    orig = tt.tiletensor.lib
    tt.tiletensor.lib = lambda: Proxy()
    for _ in range(200):
        r = chain()
    torch.cuda.synchronize()
    tt.tiletensor.lib = orig
    print(f"tt_linalg_product: {acc[0] / acc[1] * 1e6:.1f} us per call")
print("ok", tt.format_shape(r.shape()))
