"""pack() of a pinned host tensor in slabs with the host-to-device copy
overlapped (tiletensor._pack_staged): the tiles equal one pack() of the whole
device-resident tensor bit for bit -- whole slabs, a partial last slab, padded
last external row, replicated / relaxed shapes falling back to one piece."""
import numpy as np
import pytest
import torch

import paper_2011_01805_b200 as tt
from golden_cases import bitwise_equal
from paper_2011_01805_b200 import tiletensor as T

pytestmark = pytest.mark.gpu


@pytest.fixture
def small_slabs(monkeypatch):
    monkeypatch.setattr(T, "_STAGED_MIN", 1 << 10)
    monkeypatch.setattr(T, "_STAGED_SLAB", 7 << 10)


@pytest.mark.parametrize("text,s", [("[100/4,30/8,5/2]", 64), ("[37/8,20/16]", 128),
                                    ("[64/16,64/32]", 512)])
def test_staged_pack_bitwise(gpu, small_slabs, text, s):
    sh = tt.parse_shape(text)
    S = tt.Session(s, 8)
    rng = np.random.default_rng(11)
    dense = rng.standard_normal(sh.tensor_extents())
    host = torch.from_numpy(dense).pin_memory()
    want = tt.pack(torch.from_numpy(dense).cuda(), sh, S)
    got = tt.pack(host, sh, S)
    assert bitwise_equal(got.tiles(), want.tiles())


def test_staged_pack_full_size_path(gpu):
    # above the default threshold: 64 Mi values = 512 MiB -> slabs of 512 MiB rows
    sh = tt.parse_shape("[8192/16,8192/32]")
    S = tt.Session(512, 8)
    x = torch.arange(8192 * 8192, dtype=torch.float64).reshape(8192, 8192)
    host = x.pin_memory()
    got = tt.pack(host, sh, S)
    want = tt.pack(x.cuda(), sh, S)
    assert torch.equal(got.data(), want.data())
