"""The Python small-op fast path and the session tile cache (tt_tiles_alloc /
tt_tiles_release): results are never aliased while alive, a released block is
reused on the same stream only, a torch view from data() keeps its block alive,
and under CUDA-graph capture results are torch allocations."""
import numpy as np
import pytest
import torch

import paper_2011_01805_b200 as tt
from golden_cases import bitwise_equal

pytestmark = pytest.mark.gpu


@pytest.fixture
def setup(gpu):
    S = tt.Session(512, 8)
    sh = tt.parse_shape("[100/16,200/32]")
    rng = np.random.default_rng(3)
    a, b, c = (tt.pack(rng.standard_normal((100, 200)), sh, S) for _ in range(3))
    return S, a, b, c


def test_live_results_are_not_aliased(setup):
    S, a, b, c = setup
    r0 = tt.tt_mul_sum(a, b, 2)           # first call: slow path (C-ABI shape round trip)
    want_ab, want_ac = r0.tiles(), tt.tt_mul_sum(a, c, 2).tiles()
    r1 = tt.tt_mul_sum(a, b, 2)           # fast path from here on
    r2 = tt.tt_mul_sum(a, c, 2)
    assert r1._p != r2._p != r0._p
    assert bitwise_equal(r1.tiles(), want_ab) and bitwise_equal(r2.tiles(), want_ac)
    assert r1._block is not None and r2._block is not None


def test_released_block_is_reused_on_its_stream_only(setup):
    S, a, b, _ = setup
    tt.tt_mul_sum(a, b, 2)
    r = tt.tt_mul_sum(a, b, 2)
    p = r._p
    del r
    r = tt.tt_mul_sum(a, b, 2)
    assert r._p == p                      # same stream: the cached block again
    keep = r
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        r2 = tt.tt_mul_sum(a, b, 2)       # other stream: a different block
        assert r2._p != keep._p
        want = r2.tiles()
    torch.cuda.current_stream().wait_stream(side)
    assert bitwise_equal(keep.tiles(), want)


def test_data_view_keeps_the_block(setup):
    S, a, b, _ = setup
    tt.tt_mul_sum(a, b, 2)
    r = tt.tt_mul_sum(a, b, 2)
    want = r.tiles()
    view = r.data()
    p = r._p
    del r
    other = tt.tt_mul_sum(a, b, 2)        # must not get the block the view still holds
    assert other._p != p
    assert bitwise_equal(view.cpu().numpy(), want)


def test_graph_capture_uses_torch_memory(setup):
    S, a, b, _ = setup
    tt.tt_mul_sum(a, b, 2)
    want = tt.tt_mul_sum(a, b, 2).tiles()
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        for _ in range(2):
            tt.tt_mul_sum(a, b, 2)
    torch.cuda.current_stream().wait_stream(side)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        r = tt.tt_mul_sum(a, b, 2)
    assert r._block is None               # a torch tensor from the graph's pool
    g.replay()
    torch.cuda.synchronize()
    assert bitwise_equal(r.tiles(), want)


def test_errors_on_the_fast_path(setup):
    S, a, b, _ = setup
    tt.tt_mul_sum(a, b, 2)
    low = tt.TileTensor(a.shape(), a.data(), S, chain=0)
    with pytest.raises(tt.DepthExhaustedError):   # still checked in C on the fast path
        tt.tt_mul_sum(low, b, 2)
    S2 = tt.Session(512, 8)
    other = tt.TileTensor(b.shape(), b.data(), S2)
    with pytest.raises(ValueError):
        tt.tt_mul_sum(a, other, 2)
