"""cryptonets_infer on the GPU ops (paper_2011_01805_b200/nn.py) against the
reference's own cryptonets_infer (oracle/_ref): identical logits bit for bit
and identical cost counters for every tile choice of the reference's small
conv + fc network, the batch-packed branch (one tt_batch_affine pass per
layer), the paper-scale counts for tile [32,256,1] and the error contracts
(tests/test_nn.cpp:162-245 restated)."""
import numpy as np
import pytest

import paper_2011_01805_b200 as tt
from paper_2011_01805_b200 import nn

pytestmark = pytest.mark.gpu

SMALL = ("input h=6 w=6\n"
         "conv filters=2 kh=3 kw=3 stride=2 pad=1\n"
         "act square\n"
         "fc in=18 out=4\n"
         "act square\n"
         "fc in=4 out=3\n")


def _cost(c):
    return (c.additions, c.multiplications, c.mask_multiplications, c.rotations, c.bootstraps,
            c.power_of_two_rotations)


def _same(got, want):
    return np.array_equal(np.ascontiguousarray(got).view(np.uint64),
                          np.ascontiguousarray(want).view(np.uint64))


def test_every_tile_choice_matches_reference(gpu, ref):
    net = nn.parse_network(SMALL, "", 44)
    rng = np.random.default_rng(331)
    s = 64
    t3 = 1
    while t3 <= s:
        t1 = 1
        while t1 * t3 <= s:
            tile = (t1, s // (t1 * t3), t3)
            batch = rng.uniform(-1, 1, size=(36, t3))
            S = tt.Session(s, 8)
            got = nn.cryptonets_infer(net, batch, tile, S)
            want, wc = ref.nn_run(1, SMALL, 44, batch, tile, s, 8)
            assert _same(got.logits, want), tile
            assert _cost(got.cost) == _cost(wc), tile
            np.testing.assert_allclose(got.logits, nn.nn_forward(net, batch), rtol=1e-6, atol=1e-9)
            t1 *= 2
        t3 *= 2


def test_batch_packed_branch(gpu, ref):
    net = nn.parse_network(SMALL, "", 43)
    rng = np.random.default_rng(317)
    for s, n in ((64, 64), (64, 5), (1024, 1000)):
        batch = rng.uniform(-1, 1, size=(36, n))
        S = tt.Session(s, 8)
        got = nn.cryptonets_infer(net, batch, (1, 1, s), S)
        want, wc = ref.nn_run(1, SMALL, 43, batch, (1, 1, s), s, 8)
        assert got.cost.rotations == 0
        assert _same(got.logits, want)
        assert _cost(got.cost) == _cost(wc)


def test_paper_scale_counts(gpu, ref):
    net = nn.cryptonets_network(42)
    batch = np.random.default_rng(313).uniform(-1, 1, size=(784, 1))
    S = tt.Session(8192, 8)
    got = nn.cryptonets_infer(net, batch, (32, 256, 1), S)
    assert (got.cost.multiplications, got.cost.rotations, got.cost.additions,
            got.cost.bootstraps) == (32, 89, 113, 0)
    want, wc = ref.nn_run(1, nn.CRYPTONETS_SPEC, 42, batch, (32, 256, 1), 8192, 8)
    assert _same(got.logits, want)
    assert _cost(got.cost) == _cost(wc)


def test_cryptonets_batch_packed_full(gpu, ref):
    """The paper's network, batch packed (every scalar a tile of 1024 samples)."""
    net = nn.cryptonets_network(9)
    batch = np.random.default_rng(9).uniform(0, 1, size=(784, 1024))
    S = tt.Session(1024, 8)
    got = nn.cryptonets_infer(net, batch, (1, 1, 1024), S)
    want, wc = ref.nn_run(1, nn.CRYPTONETS_SPEC, 9, batch, (1, 1, 1024), 1024, 8)
    assert _same(got.logits, want)
    assert _cost(got.cost) == _cost(wc)


def test_compiled_batch_packed(gpu, ref):
    """CompiledBatchPacked (layers uploaded once) equals the reference's
    cryptonets_infer bit for bit, call after call, device or host batches;
    a too-shallow session fails on the same layer with the same message."""
    import torch
    net = nn.cryptonets_network(9)
    S = tt.Session(1024, 8)
    comp = nn.CompiledBatchPacked(net, S)
    rng = np.random.default_rng(19)
    for n in (1024, 300):
        batch = rng.uniform(0, 1, size=(784, n))
        want, wc = ref.nn_run(1, nn.CRYPTONETS_SPEC, 9, batch, (1, 1, 1024), 1024, 8)
        for b in (batch, torch.from_numpy(batch).cuda()):
            got = comp.infer(b)
            assert _same(got.logits, want)
            assert _cost(got.cost) == _cost(wc)
    small = nn.parse_network(SMALL, "", 43)
    S2 = tt.Session(64, 8)
    c2 = nn.CompiledBatchPacked(small, S2)
    batch = rng.uniform(-1, 1, size=(36, 64))
    want, wc = ref.nn_run(1, SMALL, 43, batch, (1, 1, 64), 64, 8)
    got = c2.infer(batch)
    assert _same(got.logits, want) and _cost(got.cost) == _cost(wc)
    shallow = tt.Session(64, 2)
    with pytest.raises(tt.DepthExhaustedError) as e1:
        nn.cryptonets_infer(small, batch, (1, 1, 64), shallow)
    with pytest.raises(tt.DepthExhaustedError) as e2:
        nn.CompiledBatchPacked(small, shallow).infer(batch)
    assert str(e1.value) == str(e2.value)
    with pytest.raises(tt.ShapeError):
        comp.infer(rng.uniform(0, 1, size=(783, 10)))
    comp.close()


def test_error_contracts(gpu):
    net = nn.parse_network(SMALL, "", 45)
    rng = np.random.default_rng(337)
    S = tt.Session(64, 8)
    small = nn.cryptonets_infer(net, rng.uniform(-1, 1, size=(36, 3)), (2, 4, 8), S)
    assert small.logits.shape == (3, 3)
    with pytest.raises(tt.ShapeError):
        nn.cryptonets_infer(net, rng.uniform(size=(36, 9)), (2, 4, 8), S)
    with pytest.raises(tt.ShapeError):
        nn.cryptonets_infer(net, rng.uniform(size=(36, 1)), (2, 4, 4), S)
    shallow = tt.Session(64, 2)
    for tile in ((2, 32, 1), (1, 1, 64)):
        with pytest.raises(tt.DepthExhaustedError, match="layer"):
            nn.cryptonets_infer(net, rng.uniform(size=(36, 1)), tile, shallow)
    pooled = nn.parse_network("input h=4 w=4\nfc in=16 out=4\npool mean window=2\n", "", 1)
    with pytest.raises(tt.ShapeError):
        nn.cryptonets_infer(pooled, rng.uniform(size=(16, 1)), (2, 8, 1), tt.Session(16, 8))


def test_lifted_batch_limit(gpu, ref):
    """lift_batch_limit: a batch of n > t3 samples (several external batch
    tiles; several s-sized chunks when batch packed) gives, sample for
    sample, the reference's logits for t3-sized chunks, bit for bit."""
    net = nn.parse_network(SMALL, "", 44)
    rng = np.random.default_rng(4321)
    for tile in ((2, 4, 8), (4, 2, 8), (1, 1, 64)):
        s = tile[0] * tile[1] * tile[2]
        t3 = tile[2]
        n = 3 * t3 + 5
        batch = rng.uniform(-1, 1, size=(36, n))
        S = tt.Session(s, 8)
        with pytest.raises(tt.ShapeError):
            nn.cryptonets_infer(net, batch, tile, S)
        got = nn.cryptonets_infer(net, batch, tile, S, lift_batch_limit=True)
        want = np.concatenate([ref.nn_run(1, SMALL, 44, batch[:, k:k + t3], tile, s, 8)[0]
                               for k in range(0, n, t3)], axis=1)
        assert _same(got.logits, want), tile


def test_compiled_tiled(gpu, ref):
    """CompiledTiled (weights / biases packed once) equals the reference's
    cryptonets_infer bit for bit across calls and tile choices."""
    net = nn.parse_network(SMALL, "", 44)
    rng = np.random.default_rng(4242)
    s = 64
    for tile in ((2, 32, 1), (4, 4, 4), (8, 1, 8)):
        S = tt.Session(s, 8)
        comp = nn.CompiledTiled(net, tile, S)
        for _ in range(3):
            batch = rng.uniform(-1, 1, size=(36, tile[2]))
            got = comp.infer(batch)
            want, wc = ref.nn_run(1, SMALL, 44, batch, tile, s, 8)
            assert _same(got.logits, want), tile
            assert _cost(got.cost) == _cost(wc), tile
    cn = nn.cryptonets_network(42)
    S = tt.Session(8192, 8)
    comp = nn.CompiledTiled(cn, (32, 256, 1), S)
    for seed in (1, 2):
        batch = np.random.default_rng(seed).uniform(-1, 1, size=(784, 1))
        got = comp.infer(batch)
        want = nn.cryptonets_infer(cn, batch, (32, 256, 1), S)
        assert _same(got.logits, want.logits) and _cost(got.cost) == _cost(want.cost)
    with pytest.raises(tt.ShapeError):
        nn.CompiledTiled(cn, (1, 1, 8192), S)
