"""Multi-rank path on CPU: world_size 2 over gloo (127.0.0.1).

Each rank plans its shard (tt_shard_plan in the native library), builds its
slab of a seeded global tensor, runs the reduction locally (oracle compute:
no GPU here) and, for a sum over the sharded dim, all-reduces the partial
tiles.  Results are compared with the single-process oracle on the whole
tensor: bitwise for sums over other dims, 1e-12 relative for the sum over the
sharded dim (the cross-rank addition re-associates the left fold).
"""
import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parents[1]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


GLOBAL_X = "[64/4,8/2,6/2]"   # ext [16, 4, 3], 16-slot tiles
GLOBAL_W = "[*/4,8/2,6/2]"
S = 16


def _worker(rank, world, port, out_dir):
    sys.path.insert(0, str(ROOT))
    sys.path.insert(0, str(ROOT / "tests"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle_lib import Oracle
    from paper_2011_01805_b200 import configs, parse_shape, sharding
    oracle = Oracle()
    sx, sw = parse_shape(GLOBAL_X), parse_shape(GLOBAL_W)
    plan = sharding.plan(sx, 1, world, rank)
    assert sharding.operand_plan(sw, plan) is None  # W broadcasts along dim 1
    xd = configs.uniform(64 * 8 * 6, 21, -1, 1).reshape(64, 8, 6)[plan.dense_slices()]
    wd = configs.uniform(8 * 6, 22, -1, 1).reshape(1, 8, 6)
    tx = oracle.pack(xd, plan.local_shape, S)
    tw = oracle.pack(wd, sw, S)
    wt = torch.from_numpy(tw.copy())
    sharding.broadcast_operand(wt)  # every rank holds W whole
    results = {}
    for dim in (1, 2, 3):
        def mul_sum(a, b, k):
            so, out, _ = oracle.mul_sum(plan.local_shape, a, sw, b, S, k)
            return torch.from_numpy(out.copy())
        r, sharded = sharding.sharded_mul_sum(tx, wt.numpy(), dim, plan, mul_sum, lambda t: t)
        results[f"dim{dim}"] = r.numpy()
        results[f"dim{dim}_sharded"] = np.array(sharded)
    # the bench's form: the dim-1 all-reduce in flight (async) while the
    # other dims are computed, waited on before use -- same values
    def mul_sum1(a, b, k):
        so, out, _ = oracle.mul_sum(plan.local_shape, a, sw, b, S, k)
        return torch.from_numpy(out.copy())
    part = mul_sum1(tx, wt.numpy(), 1)
    work = sharding.allreduce_partial(part, async_op=True)
    assert work is not None
    _ = mul_sum1(tx, wt.numpy(), 2)
    work.wait()
    results["dim1_async"] = part.numpy()
    results["begin"] = np.array(plan.begin)
    results["end"] = np.array(plan.end)
    np.savez(Path(out_dir) / f"rank{rank}.npz", **results)
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gloo(tmp_path, oracle):
    world = 2
    mp.start_processes(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world,
                       join=True, start_method="spawn")
    from paper_2011_01805_b200 import configs, parse_shape
    sx, sw = parse_shape(GLOBAL_X), parse_shape(GLOBAL_W)
    xd = configs.uniform(64 * 8 * 6, 21, -1, 1).reshape(64, 8, 6)
    wd = configs.uniform(8 * 6, 22, -1, 1).reshape(1, 8, 6)
    tx, tw = oracle.pack(xd, sx, S), oracle.pack(wd, sw, S)
    ranks = [np.load(tmp_path / f"rank{r}.npz") for r in range(world)]
    assert [int(r["begin"]) for r in ranks] == [0, 8] and [int(r["end"]) for r in ranks] == [8, 16]
    for dim in (1, 2, 3):
        so, want, _ = oracle.mul_sum(sx, tx, sw, tw, S, dim)
        if dim == 1:  # spans ranks: all-reduced, replicated on every rank
            for r in ranks:
                assert not bool(r["dim1_sharded"])
                got = r["dim1"]
                assert np.array_equal(r["dim1_async"].view(np.uint64), got.view(np.uint64))
                assert got.shape == want.shape
                assert oracle.max_rel_diff(got, want) < 1e-12
                # the meaningful (replicated) values agree with the dense sum
                dense = oracle.dense_sum(oracle.dense_elementwise(1, xd, wd), 1)
                assert oracle.max_rel_diff(oracle.unpack(so, S, got), dense) < 1e-12
        else:  # local: concatenation of the rank results == single-process, bitwise
            got = np.concatenate([r[f"dim{dim}"] for r in ranks])
            assert np.array_equal(got.view(np.uint64), want.view(np.uint64))


def test_plan_covers_every_tile():
    from paper_2011_01805_b200 import parse_shape, sharding
    for text, world in [("[2048/16,2048/32,512/32]", 8), ("[100/16,200/32]", 3), ("[5/2,7/4]", 4)]:
        shape = parse_shape(text)
        plans = [sharding.plan(shape, 1, world, r) for r in range(world)]
        assert plans[0].begin == 0 and plans[-1].end == shape.external_extents()[0]
        assert sum(p.local_tiles() for p in plans if p.end > p.begin) == shape.tile_count()
        rows = [p.row_slice for p in plans if p.end > p.begin]
        assert rows[0].start == 0 and rows[-1].stop == shape.dim(0).n
        for a, b in zip(rows, rows[1:]):
            assert a.stop == b.start


def _chain_worker(rank, world, port, out_dir):
    """chain_mul_sum over gloo: the fold is a numpy left fold (acc = P0, then
    acc + P_l in order; each np op is one correctly rounded IEEE operation,
    like the GPU kernel's __dadd_rn / __dmul_rn), the finish is the oracle's
    tt_sum on the accumulated tiles viewed with fold_shape."""
    sys.path.insert(0, str(ROOT))
    sys.path.insert(0, str(ROOT / "tests"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle_lib import Oracle
    from paper_2011_01805_b200 import configs, fold_shape, parse_shape, sharding
    oracle = Oracle()
    sx, sw = parse_shape(GLOBAL_X), parse_shape(GLOBAL_W)
    plan = sharding.plan(sx, 1, world, rank)
    xd = configs.uniform(64 * 8 * 6, 21, -1, 1).reshape(64, 8, 6)[plan.dense_slices()]
    wd = configs.uniform(8 * 6, 22, -1, 1).reshape(1, 8, 6)
    tx = oracle.pack(xd, plan.local_shape, S)
    tw = oracle.pack(wd, sw, S)
    n_o = 4 * 3
    fshape = fold_shape(sx, sw, 1)

    def fold(x, w, dim, rng, init):
        lo, hi = rng
        xs = x.reshape(-1, n_o, S)[:, lo:hi]
        ws = w.reshape(n_o, S)[lo:hi]
        if init is None:
            acc, start = xs[0] * ws, 1
        else:
            acc, start = init.numpy().copy(), 0
        for l in range(start, xs.shape[0]):
            acc = acc + xs[l] * ws
        return torch.from_numpy(np.ascontiguousarray(acc))

    def finish(parts):
        acc = np.concatenate([p.numpy() for p in parts])
        so, out, _ = oracle.sum(fshape, acc, S, 1)
        return out

    res = sharding.chain_mul_sum(tx, tw, 1, plan, fold, finish, n_o,
                                 lambda k: torch.empty((k, S), dtype=torch.float64), chunks=5)
    if rank == world - 1:
        np.save(Path(out_dir) / "chain.npy", res)
    else:
        assert res is None
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_chain_is_bitwise_exact(tmp_path, oracle, world):
    """The exact cross-rank sum: ranks continue each other's left-fold
    accumulators in chunks, so the sum over the sharded dim equals the
    single-process oracle bit for bit (the all-reduce path only to 1e-12)."""
    mp.start_processes(_chain_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world,
                       join=True, start_method="spawn")
    from paper_2011_01805_b200 import configs, parse_shape
    sx, sw = parse_shape(GLOBAL_X), parse_shape(GLOBAL_W)
    xd = configs.uniform(64 * 8 * 6, 21, -1, 1).reshape(64, 8, 6)
    wd = configs.uniform(8 * 6, 22, -1, 1).reshape(1, 8, 6)
    tx, tw = oracle.pack(xd, sx, S), oracle.pack(wd, sw, S)
    so, want, _ = oracle.mul_sum(sx, tx, sw, tw, S, 1)
    got = np.load(tmp_path / "chain.npy")
    assert got.shape == want.shape
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))
