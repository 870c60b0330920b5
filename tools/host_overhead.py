"""Host-side cost of one small op through the Python API (config 1 mul+sum):
enqueue time per call and a cProfile breakdown.  For tuning the wrapper."""
import cProfile
import pstats
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2011_01805_b200 as tt  # noqa: E402
from paper_2011_01805_b200 import configs  # noqa: E402

c1 = configs.config1()
S = tt.Session(512, 8)
sA = tt.parse_shape(c1.shapes["A"])
A, B = tt.pack(c1.tensors["A"], sA, S), tt.pack(c1.tensors["B"], sA, S)
for _ in range(50):
    tt.tt_mul_sum(A, B, 2)
torch.cuda.synchronize()
n = 2000
t0 = time.perf_counter()
for _ in range(n):
    tt.tt_mul_sum(A, B, 2)
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"enqueue {1e6 * (t1 - t0) / n:.1f} us/op, with drain {1e6 * (t2 - t0) / n:.1f} us/op")
c2 = configs.config2()
S2 = tt.Session(8192, 8)
M = tt.pack(c2.tensors["M"], tt.parse_shape(c2.shapes["M"]), S2)
V = tt.pack(c2.tensors["V"], tt.parse_shape(c2.shapes["V"]), S2)
for _ in range(20):
    tt.matvec_a(M, V)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(500):
    tt.matvec_a(M, V)
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"c2 matvec_a enqueue {1e6 * (t1 - t0) / 500:.1f} us/op, with drain {1e6 * (t2 - t0) / 500:.1f} us/op")
lib = tt.tiletensor.lib()
import ctypes  # noqa: E402
t0 = time.perf_counter()
for _ in range(n):
    S.handle
t1 = time.perf_counter()
print(f"Session.handle {1e6 * (t1 - t0) / n:.2f} us")
t0 = time.perf_counter()
for _ in range(n):
    S.empty_tiles(7)
t1 = time.perf_counter()
print(f"empty_tiles {1e6 * (t1 - t0) / n:.2f} us")
# the bare C call with prebuilt arguments
so = tt.CShape()
ch = ctypes.c_int64()
out = S.empty_tiles(7)
ca, cb = A.shape().to_c(), B.shape().to_c()
pa, pb, po = ctypes.c_void_p(A.data().data_ptr()), ctypes.c_void_p(B.data().data_ptr()), \
    ctypes.c_void_p(out.data_ptr())
h = S.handle
f = lib.tt_mul_sum
t0 = time.perf_counter()
for _ in range(n):
    f(h, ctypes.byref(ca), pa, 8, ctypes.byref(cb), pb, 8, 2, -1, ctypes.byref(so), po,
      ctypes.byref(ch))
t1 = time.perf_counter()
torch.cuda.synchronize()
print(f"bare tt_mul_sum C call {1e6 * (t1 - t0) / n:.2f} us")
g = lib.tt_tiles_binary
t0 = time.perf_counter()
for _ in range(n):
    g(h, 1, pa, pa, po, 1, None, None, None)
t1 = time.perf_counter()
torch.cuda.synchronize()
print(f"bare tt_tiles_binary (1 small-param launch) {1e6 * (t1 - t0) / n:.2f} us")
pr = cProfile.Profile()
pr.enable()
for _ in range(n):
    tt.tt_mul_sum(A, B, 2)
pr.disable()
torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
