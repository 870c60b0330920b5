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


def test_bootstrap_lower_bound():
    G = nn.FilterGroup
    groups = [G(32, 3, 50, 18), G(32, 5, 50, 16)]
    assert nn.bootstrap_lower_bound(groups, 3) == 1088
    assert nn.bootstrap_lower_bound(groups, 4) == 816
    assert nn.bootstrap_lower_bound([G(1, 3, 50, 18)], 3) == 18
    assert nn.bootstrap_lower_bound([G(1, 2, 2, 100)], 1) == 12
    with pytest.raises(ValueError):
        nn.bootstrap_lower_bound(groups, 0)
    prev = nn.bootstrap_lower_bound(groups, 1)
    assert prev == 3264
    for d in range(2, 65):
        b = nn.bootstrap_lower_bound(groups, d)
        assert b <= prev
        if 3264 % d == 0:
            assert b * d == 3264
        prev = b


# ---- plan checker (nn.hpp:534-700) ------------------------------------------------------

REF_PLAN = "/root/reference/proj/tests/data/cnn_train_plan.txt"


def _steps_text(steps):
    out = []
    for st in steps:
        parts = [f"step {st.name}", f"op={st.op}"] + [f"in={x}" for x in st.inputs]
        if st.output:
            parts.append(f"out={st.output}")
        parts.append(f"chain={st.chain_before}:{st.chain_after}")
        out.append(" ".join(parts))
    return "\n".join(out) + "\n"


def test_plan_checker_kats():
    P = nn.PlanStep
    steps = [P(f"mul{i + 1}", "mul", ["[4/4]", "[4/4]"], "[4/4]", 3 - i, 2 - i) for i in range(4)]
    rep = nn.validate_plan(steps, nn.BackendConfig(4, 3))
    assert not rep.ok and len(rep.issues) == 1 and rep.issues[0].step == 4
    assert not rep.issues[0].info
    cfg = nn.BackendConfig(4, 3)
    assert not nn.validate_plan([P("mul", "mul", ["[4/4]", "[4/4]"], "[4/4]", 3, 3)], cfg).ok
    assert not nn.validate_plan([P("add", "add", ["[5/4]", "[6/4]"], "[6/4]", 3, 3)], cfg).ok
    assert not nn.validate_plan([P("x", "add", ["[5/"], "[5/4]", 1, 1)], cfg).ok
    assert not nn.validate_plan([P("boot", "bootstrap", ["[4/4]"], "[4/4]", 0, 2)], cfg).ok
    assert nn.validate_plan([], cfg).ok
    bridge = P("conv", "mul", ["[18,*/32,150/256,255]", "[1,32/32,150/256]"],
               "[18,32/32,150/256,255]", 4, 3)
    rep = nn.validate_plan([bridge], nn.BackendConfig(8192, 4))
    assert rep.ok and len(rep.issues) == 1 and rep.issues[0].info
    for bad in ("step s1 in=[4/4] out=[4/4] chain=1:1\n",
                "step s1 op=add in=[4/4] out=[4/4] chain=11\n", "op=add\n", "step s1 op=add bogus\n"):
        with pytest.raises(RuntimeError):
            nn.parse_plan(bad)
    assert len(nn.parse_plan("# c\nstep s1 op=add in=[4/4] in=[4/4] out=[4/4] chain=1:1\n")) == 1


def test_plan_reports_match_reference(ref):
    import os
    import random
    texts = []
    if os.path.exists(REF_PLAN):
        texts.append(open(REF_PLAN).read())
    rng = random.Random(99)
    shapes = ["[4/4]", "[5/4]", "[6/4]", "[*/4,8/2]", "[3/2,*/4]", "[5/", "[2,3/4]", "[8/8,1?/2]",
              "[1,32/32,150/256]", "[18,*/32,150/256,255]"]
    ops = ["add", "sub", "mul", "square", "mask", "scale", "sum", "matmul", "rotate", "reshape",
           "concat", "bridge", "bootstrap"]
    for _ in range(60):
        steps = []
        for k in range(rng.randint(0, 8)):
            cb = rng.randint(-1, 5)
            steps.append(nn.PlanStep(f"s{k}", rng.choice(ops),
                                     [rng.choice(shapes) for _ in range(rng.randint(0, 3))],
                                     rng.choice(shapes + [""]), cb, cb - rng.randint(-1, 2)))
        texts.append(_steps_text(steps))
    for text in texts:
        for depth in (3, 4):
            want = ref.validate_plan(text, 8192, depth)
            got = nn.validate_plan(nn.parse_plan(text), nn.BackendConfig(8192, depth)).to_text()
            assert got == want, text
