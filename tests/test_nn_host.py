"""Host side of the nn layer (inc/nn.hpp mirror in paper_2011_01805_b200/nn.py):
seeded parameters, the plaintext forward pass, im2col, the network and tensor
text formats and the bootstrap bound -- bit-exact against the reference
compiled here (oracle/_ref) where it applies, and the reference's own KATs
(tests/test_nn.cpp) restated.  No GPU needed."""
import numpy as np
import pytest

from paper_2011_01805_b200 import nn
from paper_2011_01805_b200.tiletensor import ShapeError

SMALL = ("input h=6 w=6\n"
         "conv filters=2 kh=3 kw=3 stride=2 pad=1\n"
         "act square\n"
         "fc in=18 out=4\n"
         "act square\n"
         "fc in=4 out=3\n")


def _params(net):
    out = []
    for layer in net.layers:
        if isinstance(layer, (nn.ConvLayer, nn.FcLayer)):
            out += [np.asarray(layer.weights).reshape(-1), np.asarray(layer.bias).reshape(-1)]
    return np.concatenate(out)


@pytest.mark.parametrize("spec,seed", [(SMALL, 44), (nn.CRYPTONETS_SPEC, 7), ("fc in=5 out=3\n", 0)])
def test_seeded_parameters_match_reference(ref, spec, seed):
    got = _params(nn.parse_network(spec, "", seed))
    want = ref.nn_params(spec, seed)
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))


@pytest.mark.parametrize("spec,seed,features", [(SMALL, 45, 36), (nn.CRYPTONETS_SPEC, 42, 784)])
def test_nn_forward_matches_reference_bitwise(ref, spec, seed, features):
    rng = np.random.default_rng(seed)
    batch = rng.uniform(-1, 1, size=(features, 5))
    got = nn.nn_forward(nn.parse_network(spec, "", seed), batch)
    want, _ = ref.nn_run(0, spec, seed, batch)
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))


def test_im2col_kats():
    rng = np.random.default_rng(301)
    x = rng.uniform(-1, 1, size=(4, 4))
    m1 = nn.im2col(x, 2, 2, 2, 0)
    assert m1.shape == (4, 4)
    assert list(m1[0]) == [x[0, 0], x[0, 1], x[1, 0], x[1, 1]]
    assert m1[3, 0] == x[2, 2]
    single = nn.im2col(x, 1, 1, 1, 0)
    assert single.shape == (16, 1) and np.array_equal(single.reshape(-1), x.reshape(-1))
    assert nn.im2col(np.zeros((28, 28)), 5, 5, 2, 1).shape[0] == 169
    with pytest.raises(ShapeError):
        nn.im2col(x, 6, 6, 1, 0)
    # im2col times the flattened filter is the direct convolution
    for h in range(2, 7):
        for kh in range(1, min(3, h) + 1):
            for stride in (1, 2):
                for pad in (0, 1):
                    img = rng.uniform(-1, 1, size=(h, h))
                    f = rng.uniform(-1, 1, size=(kh, kh))
                    gh = (h + 2 * pad - kh) // stride + 1
                    padded = np.pad(img, pad)
                    direct = np.array([[np.sum(padded[gy * stride:gy * stride + kh,
                                                      gx * stride:gx * stride + kh] * f)
                                        for gx in range(gh)] for gy in range(gh)])
                    prod = (nn.im2col(img, kh, kh, stride, pad) @ f.reshape(-1)).reshape(gh, gh)
                    np.testing.assert_allclose(prod, direct, rtol=1e-12, atol=1e-12)


def test_network_parsing(tmp_path):
    for bad in ("fc in=4\n", "act relu\n", "# nothing\n", "conv2d x=1\n"):
        with pytest.raises(RuntimeError):
            nn.parse_network(bad, "", 1)
    net = nn.cryptonets_network(7)
    assert len(net.layers) == 5 and net.input_size() == 784
    assert net.layers[0].filters == 5 and net.layers[2].inp == 845
    assert np.array_equal(net.layers[2].weights, nn.cryptonets_network(7).layers[2].weights)
    (tmp_path / "w.tensor").write_text("shape: 2 3\n1 2 3\n4 5 6\n")
    (tmp_path / "b.tensor").write_text("shape: 2\n10 20\n")
    net = nn.parse_network("fc in=3 out=2 weights=w.tensor bias=b.tensor\n", str(tmp_path), 1)
    assert np.array_equal(net.layers[0].weights, [[1, 2, 3], [4, 5, 6]])
    assert np.array_equal(nn.nn_forward(net, np.ones((3, 1))), [[16.0], [35.0]])
    with pytest.raises(RuntimeError):
        nn.parse_network("fc in=3 out=2 weights=nope.tensor\n", str(tmp_path), 1)
    with pytest.raises(RuntimeError):
        nn.parse_network("fc in=4 out=2 weights=w.tensor\n", str(tmp_path), 1)
    pooled = nn.parse_network("input h=4 w=4\nfc in=16 out=4\npool mean window=2\n", "", 1)
    assert len(pooled.layers) == 2
    with pytest.raises(ShapeError):
        nn.nn_forward(pooled, np.ones((16, 1)))


def test_tensor_text_round_trip():
    rng = np.random.default_rng(5)
    for shape in ((3,), (2, 5), (2, 3, 4)):
        t = rng.normal(size=shape)
        t.reshape(-1)[0] = -0.0
        back = nn.read_tensor(nn.write_tensor(t))
        assert back.shape == t.shape
        assert np.array_equal(back.view(np.uint64), t.view(np.uint64))
    assert nn.write_tensor(np.array([[1.0, 0.1]])) == "shape: 1 2\n1 0.10000000000000001\n"
    with pytest.raises(RuntimeError):
        nn.read_tensor("1 2 3\n")
    with pytest.raises(RuntimeError):
        nn.read_tensor("shape: 2\n1 x\n")
