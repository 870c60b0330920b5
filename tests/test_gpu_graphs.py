"""The device passes are CUDA-graph capturable: ops launch on torch's current
stream (Session binds it per call), so a warmed-up chain captured with
torch.cuda.graph replays bit-identically -- how a caller removes host launch
overhead from small, repeated chains (configs 1-4).  Launch-parameter caches
(occupancy, smem opt-in, schedules) are filled by the warm-up, so nothing
host-synchronous runs during capture."""
import numpy as np
import pytest
import torch

import paper_2011_01805_b200 as tt
from paper_2011_01805_b200 import configs

pytestmark = pytest.mark.gpu


def _bits(t):
    return t.detach().cpu().numpy().view(np.uint64)


def test_capture_and_replay_config1(gpu):
    c1 = configs.config1()
    S = tt.Session(512, 8)
    sA = tt.parse_shape(c1.shapes["A"])
    A, B = tt.pack(c1.tensors["A"], sA, S), tt.pack(c1.tensors["B"], sA, S)
    want = tt.tt_mul_sum(A, B, 2).data().clone()
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        for _ in range(3):
            tt.tt_mul_sum(A, B, 2)  # warm-up on the capture stream
    torch.cuda.current_stream().wait_stream(side)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        r = tt.tt_mul_sum(A, B, 2)
    for _ in range(3):
        r.data().zero_()
        g.replay()
        torch.cuda.synchronize()
        assert np.array_equal(_bits(r.data()), _bits(want))


def test_capture_matmul_chain(gpu):
    """The c3-shaped chain (GEMM fold with the session work queue + tree passes)."""
    rng = np.random.default_rng(12)
    S = tt.Session(8192, 8)
    shapes = {"Bt": "[48/16,64/32,*/16]", "C": "[48/16,*/32,40/16]", "A": "[40/16,64/32,*/16]"}
    T = {}
    for k, v in shapes.items():
        sh = tt.parse_shape(v)
        T[k] = tt.TileTensor(sh, rng.uniform(-1, 1, size=(sh.tile_count(), 8192)), S)

    def chain():
        return tt.matmul_a(T["A"], tt.matmul_b(T["Bt"], T["C"]))
    want = chain().data().clone()
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        for _ in range(3):
            chain()
    torch.cuda.current_stream().wait_stream(side)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        r = chain()
    for _ in range(4):
        g.replay()
        torch.cuda.synchronize()
        assert np.array_equal(_bits(r.data()), _bits(want))
