"""Per-kernel timeline of the small config chains (CUPTI via the torch profiler),
API calls and CUDA-graph replay.  Usage: python tools/timeline.py c1 c2 c3 c4 ...

Prints, per chain, each kernel's mean duration and the idle gap before it, plus the
chain's CUDA-event time -- where the time of a latency-scale chain goes."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_2011_01805_b200 as tt  # noqa: E402
from paper_2011_01805_b200 import configs  # noqa: E402


def chains():
    out = {}
    c1 = configs.config1()
    S1 = tt.Session(512, 8)
    A = tt.pack(c1.tensors["A"], tt.parse_shape(c1.shapes["A"]), S1)
    B = tt.pack(c1.tensors["B"], tt.parse_shape(c1.shapes["B"]), S1)
    out["c1"] = lambda: tt.tt_mul_sum(A, B, 2)
    c2 = configs.config2()
    S2 = tt.Session(8192, 8)
    M = tt.pack(c2.tensors["M"], tt.parse_shape(c2.shapes["M"]), S2)
    V = tt.pack(c2.tensors["V"], tt.parse_shape(c2.shapes["V"]), S2)
    out["c2"] = lambda: tt.matvec_a(M, V)
    c3 = configs.config3()
    S3 = tt.Session(8192, 8)
    T3 = {k: tt.pack(c3.tensors[k], tt.parse_shape(c3.shapes[k]), S3) for k in ("A3", "Bt3", "C3")}
    out["c3"] = lambda: tt.matmul_a(T3["A3"], tt.matmul_b(T3["Bt3"], T3["C3"]))
    T3.update({k: tt.pack(c3.tensors[k], tt.parse_shape(c3.shapes[k]), S3) for k in ("B3", "Ct3")})
    out["c3a"] = lambda: tt.tt_mul_sum(tt.replicate_dim(tt.clean_unknowns(
        tt.matmul_a(T3["A3"], T3["B3"])), 2), T3["Ct3"], 3)
    out["c3af"] = lambda: tt.tt_mul_sum(tt.replicate_dim(
        tt.tt_mul_sum_clean(T3["A3"], T3["B3"], 2), 2), T3["Ct3"], 3)
    c4 = configs.config4(True)
    S4 = tt.Session(8192, 8)
    T4 = {k: tt.pack(c4.tensors[k], tt.parse_shape(v), S4) for k, v in c4.shapes.items()}

    def c4_chain():
        h = tt.tt_add(tt.tt_mul_sum(T4["W1t"], T4["X"], 1), T4["b1"])
        h = tt.tt_mul(h, h)
        return tt.tt_add(tt.tt_mul_sum(T4["W2"], h, 2), T4["b2"])
    out["c4"] = c4_chain
    out["c4f"] = lambda: tt.tt_mul_sum_affine(
        T4["W2"], tt.tt_mul_sum_affine(T4["W1t"], T4["X"], 1, T4["b1"], square=True), 2, T4["b2"])
    return out


def timeline(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    api_us = e0.elapsed_time(e1) / reps * 1e3
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        fn()
    torch.cuda.current_stream().wait_stream(side)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    g.replay()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    graph_us = e0.elapsed_time(e1) / reps * 1e3
    print(f"  chain: api {api_us:.1f} us, graph replay {graph_us:.1f} us")
    for mode in ("api", "graph"):
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            for _ in range(reps):
                fn() if mode == "api" else g.replay()
            torch.cuda.synchronize()
        ev = sorted((e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA
                     and "Memcpy" not in e.name and "Memset" not in e.name),
                    key=lambda e: e.time_range.start)
        per = len(ev) // reps
        rows = {}
        for i in range(per, len(ev)):
            e, prev = ev[i], ev[i - 1]
            d = rows.setdefault(i % per, [e.name[:70], 0.0, 0.0, 0])
            d[1] += e.time_range.end - e.time_range.start
            d[2] += e.time_range.start - prev.time_range.end
            d[3] += 1
        print(f"  [{mode}] kernels per chain: {per}")
        tk = tg = 0.0
        for k in sorted(rows):
            name, dur, gap, c = rows[k]
            tk += dur / c
            tg += gap / c
            print(f"    {dur / c:8.2f} us  gap-before {gap / c:6.2f} us  {name}")
        print(f"    kernels {tk:.1f} us + gaps {tg:.1f} us")


if __name__ == "__main__":
    want = [a for a in sys.argv[1:] if not a.startswith("-")] or ["c1", "c2", "c3", "c4"]
    cs = chains()
    for name in want:
        print(name)
        timeline(cs[name])
