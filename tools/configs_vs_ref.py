"""Per-config comparison with the reference's CPU path (BASELINE.json configs 1-4):
the reference's own op chain (oracle/_ref, all host threads, its two-step
tt_sum(tt_mul(...)) bodies) against this package's GPU chain through the Python
API (device-resident operands; CUDA events) and as a CUDA-graph replay, checking
that both give the same tiles bit for bit.  Prints a markdown table.

Usage (GPU box): python tools/configs_vs_ref.py [reps]"""
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2011_01805_b200 as tt  # noqa: E402
from oracle_lib import load_ref  # noqa: E402
from paper_2011_01805_b200 import configs  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
ref = load_ref()
if ref is None:
    sys.exit("oracle/_ref/libttref.so not built")
threads = min(64, os.cpu_count() or 1)
ref.lib.ref_set_threads(threads)


def cpu_time(fn, n):
    fn()
    t0 = time.perf_counter()
    for _ in range(n):
        r = fn()
    return (time.perf_counter() - t0) / n, r


def gpu_time(fn, n):
    # ~0.2 s of warm-up: the GPU idled (and may have clocked down) during the
    # CPU timing just before
    t0 = time.perf_counter()
    while time.perf_counter() - t0 < 0.2:
        fn()
        torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        r = fn()
    e1.record()
    torch.cuda.synchronize()
    api = e0.elapsed_time(e1) / n / 1e3
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
    for _ in range(n):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return api, e0.elapsed_time(e1) / n / 1e3, r


def same(a, b):
    return np.array_equal(np.ascontiguousarray(a).view(np.uint64), np.ascontiguousarray(b).view(np.uint64))


# GPU timings first, the reference's after: its host thread pool would
# otherwise compete with the Python thread that enqueues the GPU work
c1, c2, c3, c4 = configs.config1(), configs.config2(), configs.config3(), configs.config4(False)
sh1 = {k: tt.parse_shape(v) for k, v in c1.shapes.items()}
sh2 = {k: tt.parse_shape(v) for k, v in c2.shapes.items()}
sh3 = {k: tt.parse_shape(v) for k, v in c3.shapes.items()}
sh4 = {k: tt.parse_shape(v) for k, v in c4.shapes.items()}
gpu = {}
S = tt.Session(512, 8)
T = {k: tt.pack(c1.tensors[k], sh1[k], S) for k in sh1}
gpu["c1"] = gpu_time(lambda: tt.tt_mul_sum(T["A"], T["B"], 2), reps * 10)
del T
torch.cuda.empty_cache()
S = tt.Session(8192, 8)
T = {k: tt.pack(c2.tensors[k], sh2[k], S) for k in sh2}
gpu["c2"] = gpu_time(lambda: tt.matvec_a(T["M"], T["V"]), reps * 5)
del T
torch.cuda.empty_cache()
T = {k: tt.pack(c3.tensors[k], sh3[k], S) for k in ("A3", "Bt3", "C3")}
gpu["c3"] = gpu_time(lambda: tt.matmul_a(T["A3"], tt.matmul_b(T["Bt3"], T["C3"])), reps)
del T
torch.cuda.empty_cache()
T = {k: tt.pack(c4.tensors[k], sh4[k], S) for k in sh4}
gpu["c4"] = gpu_time(lambda: tt.tt_mul_sum_affine(
    T["W2"], tt.tt_mul_sum_affine(T["W1t"], T["X"], 1, T["b1"], square=True), 2, T["b2"]), reps)
del T
torch.cuda.synchronize()

cpu = {}
P = {k: ref.pack(c1.tensors[k], sh1[k], 512) for k in sh1}
cpu["c1"] = cpu_time(lambda: ref.mul_sum(sh1["A"], P["A"], sh1["B"], P["B"], 512, 2), 200)
s = 8192
P = {k: ref.pack(c2.tensors[k], sh2[k], s) for k in sh2}
cpu["c2"] = cpu_time(lambda: ref.linalg(0, sh2["M"], P["M"], sh2["V"], P["V"], s), 5)
P = {k: ref.pack(c3.tensors[k], sh3[k], s) for k in ("A3", "Bt3", "C3")}


def ref_c3():
    s1, t1, _ = ref.linalg(3, sh3["Bt3"], P["Bt3"], sh3["C3"], P["C3"], s)
    return ref.linalg(2, sh3["A3"], P["A3"], s1, t1, s)


cpu["c3"] = cpu_time(ref_c3, 1)
P = {k: ref.pack(c4.tensors[k], sh4[k], s) for k in sh4}


def ref_c4():
    s1, t1, _ = ref.mul_sum(sh4["W1t"], P["W1t"], sh4["X"], P["X"], s, 1)
    s2, t2, _ = ref.elementwise(0, s1, t1, sh4["b1"], P["b1"], s)
    s3, t3, _ = ref.elementwise(1, s2, t2, s2, t2, s)
    s4, t4, _ = ref.mul_sum(sh4["W2"], P["W2"], s3, t3, s, 2)
    return ref.elementwise(0, s4, t4, sh4["b2"], P["b2"], s)


cpu["c4"] = cpu_time(ref_c4, 1)
names = {"c1": "c1 mul + sum dim 2, [100/16,200/32] (512 slots)",
         "c2": "c2 matvec_a 1024x4096 (8192 slots)",
         "c3": "c3 A(512x1024) B(1024x768) C(768x256), '3b' chain (8192 slots)",
         "c4": "c4 FC 784->100, square, FC 100->10, 4096 samples (8192 slots)"}
rows = []
for k in ("c1", "c2", "c3", "c4"):
    api, graph, r = gpu[k]
    t_cpu, (rs, rt, _) = cpu[k]
    rows.append((names[k], t_cpu, api, graph, same(r.tiles(), rt)))

print(f"reference CPU path: oracle/_ref (the reference's headers compiled here), "
      f"{threads} host threads; GPU: one B200, operands resident\n")
print("| config | reference CPU | GPU, API call | GPU, graph replay | speed-up (API) | tiles bit-equal |")
print("|---|---|---|---|---|---|")
for name, c, a, g, ok in rows:
    print(f"| {name} | {c * 1e3:.3f} ms | {a * 1e6:.1f} us | {g * 1e6:.1f} us | {c / a:.0f}x | {ok} |")
