"""The bench's N > 1 step (config 5 as named, strong scaling) with two ranks on
the one B200, over gloo (NCCL refuses two ranks on one device; a functional
check of the multi-rank data path, not a measurement).

`bench.py --gpus 2` is launched under torchrun exactly as the driver does for
N = 2, with TT_BENCH_BACKEND=gloo and `--dump`: each rank writes slabs of its
results (first / middle / last external rows of its dim-2 and dim-3 results,
columns l2 = 0 / 31 / 63 of the dim-1 result, all-reduced and chained).  The
slabs are compared with the CPU oracle on the matching input slabs of the one
global X [2048,2048,512]:

* dims 2 and 3 (local sums): bitwise;
* dim 1 via the exact chain (sharding.chain_mul_sum): bitwise;
* dim 1 via the all-reduce of the partial sums: <= 1e-12 relative (the
  cross-rank addition re-associates the reference's left fold,
  tile_tensor.hpp:313-330).
"""
import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

import paper_2011_01805_b200 as tt
from golden_cases import bitwise_equal
from paper_2011_01805_b200 import configs

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
ROOT = Path(__file__).resolve().parents[1]
S5 = configs.C5_SLOTS


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.fixture(scope="module")
def run(tmp_path_factory, gpu):
    out = tmp_path_factory.mktemp("mr")
    # TT_BENCH_HOST_GIB: pretend a 20 GiB host so the e2e leg stages half of
    # each rank's 8 GiB slab (the x_slab_fraction < 1 path)
    env = dict(os.environ, TT_BENCH_BACKEND="gloo", OMP_NUM_THREADS="4", TT_BENCH_HOST_GIB="20")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           str(ROOT / "bench.py"), "--gpus", "2", "--steps", "1", "--warmup", "3",
           "--skip-extra", "--e2e-steps", "1", "--skip-cpu", "--dump", str(out)]
    proc = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=1500)
    assert proc.returncode == 0, proc.stderr[-3000:]
    lines = [ln for ln in proc.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, proc.stdout[-2000:]
    return json.loads(lines[0]), [np.load(out / f"rank{r}.npz") for r in (0, 1)]


def test_bench_line_is_config5_as_named(run):
    line, _ = run
    assert line["n_gpus"] == 2 and line["scaling"] == "strong"
    assert line["config"]["global_x"] == [2048, 2048, 512]
    assert line["config"]["x_tiles_total"] == 131072
    assert line["roofline"]["x_tiles_per_rank"] == 65536
    assert "error" not in line["ops"]["mul_sum_dim1_chain"]
    assert line["value"] > 0 and line["gpu_launches"] > 0
    e2e = line["e2e"]
    assert e2e["x_slab_fraction"] == 0.5, e2e
    assert e2e["h2d_bytes_per_step"] == (512 * 2048 * 512 + 2048 * 512) * 8  # half of 1024 rows + W


def _row_shape(rows):
    return tt.TileTensorShape([tt.DimSpec(rows, 1, 16), tt.DimSpec(2048, 1, 32), tt.DimSpec(512, 1, 32)])


@pytest.fixture(scope="module")
def w_tiles(oracle):
    return oracle.pack(configs.c5_w(), tt.parse_shape(configs.C5_W_SHAPE), S5)


def test_local_dims_bitwise(run, oracle, w_tiles):
    _, ranks = run
    sw = tt.parse_shape(configs.C5_W_SHAPE)
    ss = _row_shape(16)
    assert tuple(ranks[0]["begin"]) == (0, 64) and tuple(ranks[1]["begin"]) == (64, 128)
    for blob in ranks:
        for dim, name in ((2, "dim2"), (3, "dim3")):
            for tag in ("first", "mid", "last"):
                row = int(blob[f"{name}_{tag}_row"][0])   # global external row of dim 1
                px = oracle.pack(configs.c5_x_slab(slice(16 * row, 16 * row + 16)), ss, S5)
                _, want, _ = oracle.mul_sum(ss, px, sw, w_tiles, S5, dim)
                assert bitwise_equal(blob[f"{name}_{tag}"], want), (name, tag, row)


def test_dim1_chain_bitwise_allreduce_1e12(run, oracle):
    _, ranks = run
    last = ranks[1]          # the chain's result lives on the last rank
    ss2 = tt.TileTensorShape([tt.DimSpec(2048, 1, 16), tt.DimSpec(32, 1, 32), tt.DimSpec(512, 1, 32)])
    sw2 = tt.TileTensorShape([tt.DimSpec(1, 16, 16), tt.DimSpec(32, 1, 32), tt.DimSpec(512, 1, 32)])
    for tag in ("first", "mid", "last"):
        l2 = int(last[f"dim1_{tag}_l2"][0])
        cols = slice(32 * l2, 32 * l2 + 32)
        px = oracle.pack(configs.c5_x_slab(slice(None), cols), ss2, S5)
        pw = oracle.pack(configs.c5_w(cols), sw2, S5)
        _, want, _ = oracle.mul_sum(ss2, px, sw2, pw, S5, 1)
        assert bitwise_equal(last[f"dim1chain_{tag}"], want), tag
        for blob in ranks:   # the all-reduced result is replicated on every rank
            got = blob[f"dim1_{tag}"]
            assert np.array_equal(got, ranks[0][f"dim1_{tag}"])
            assert oracle.max_rel_diff(got, want) < 1e-12, tag
