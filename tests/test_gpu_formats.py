"""Packed tile files and dense text tensors (paper_2011_01805_b200/formats.py):
exact text for a known packing, bit-exact round trips of GPU-packed tensors
(replicated, '?'-carrying and relaxed shapes), and the error contracts of the
reference CLI's read_tiles_file (tools/tiletensor_main.cpp:76-128)."""
import numpy as np
import pytest

import paper_2011_01805_b200 as tt
from paper_2011_01805_b200 import formats

pytestmark = pytest.mark.gpu


def test_known_tile_file_text(gpu):
    S = tt.Session(4, 8)
    t = tt.pack(np.array([1.0, 2.0, 3.0]), tt.parse_shape("[3/2,*/2]"), S)
    assert formats.write_tiles(t) == ("shape: [3/2,*/2]\nslots: 4\n"
                                      "tile: 1 1 2 2\ntile: 3 3 0 0\n")


def test_round_trips_are_bit_exact(gpu):
    rng = np.random.default_rng(77)
    S = tt.Session(16, 8)
    for text in ("[5/4,7/4]", "[*/4,9/4]", "[6/2,*3/8]"):
        shape = tt.parse_shape(text)
        t = tt.pack(rng.normal(size=shape.tensor_extents()), shape, S)
        back = formats.read_tiles(formats.write_tiles(t), S)
        assert back.shape() == t.shape()
        assert np.array_equal(back.tiles().view(np.uint64), t.tiles().view(np.uint64))
    # a '?' result (sum) and a relaxed shape keep their flags
    a = tt.pack(rng.normal(size=(5, 7)), tt.parse_shape("[5/4,7/4]"), S)
    r = tt.tt_sum(a, 2)
    back = formats.read_tiles(formats.write_tiles(r), S)
    assert back.shape() == r.shape() and back.shape().has_unknown()
    assert np.array_equal(back.tiles().view(np.uint64), r.tiles().view(np.uint64))
    relaxed = tt.TileTensorShape(tt.parse_shape("[3/2,2/2]").dims(), True)
    rt = tt.pack(rng.normal(size=(3, 2)), relaxed, tt.Session(8, 8))
    text = formats.write_tiles(rt)
    assert "relaxed: true\n" in text
    assert formats.read_tiles(text, tt.Session(8, 8)).shape().relaxed()


def test_dense_text_round_trip_through_unpack(gpu):
    rng = np.random.default_rng(3)
    S = tt.Session(16, 8)
    x = rng.normal(size=(6, 5))
    t = tt.pack(x, tt.parse_shape("[6/4,5/4]"), S)
    back = formats.read_tensor(formats.write_tensor(tt.unpack(t)))
    assert np.array_equal(back.view(np.uint64), x.view(np.uint64))


def test_tile_file_errors(gpu):
    S = tt.Session(4, 8)
    with pytest.raises(RuntimeError, match="slots"):
        formats.read_tiles("shape: [2/2,*/2]\nslots: 8\n", S)
    with pytest.raises(RuntimeError, match="no shape"):
        formats.read_tiles("slots: 4\n", S)
    with pytest.raises(RuntimeError, match="unrecognized"):
        formats.read_tiles("shape: [2/2,*/2]\nbogus 1\n", S)
