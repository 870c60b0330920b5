"""Sharding of external tile indices across GPUs (north-star item 5).

One process per GPU.  A tile tensor is block-partitioned along one external
dimension (`shard_dim`, 1-based): rank r owns external indices
[begin_r, end_r) of that dim, i.e. the dense slab of rows
[begin_r * t, min(n, end_r * t)).  Because every output tile of an
elementwise op or of a sum over another dim depends only on operand tiles at
the same external index (or the broadcast index l mod e,
tile_tensor.hpp:260-265), those ops run locally with NO communication and
the results stay sharded, bit-identical to the single-GPU result.

Only a sum over `shard_dim` itself spans ranks.  Two ways:

* `sharded_mul_sum`: each rank runs the fused fold + rotate-and-sum on its
  slab and the partial results are summed with one NCCL all-reduce over
  NVLink (torch.distributed, backend "nccl").  The cross-rank addition
  re-associates the reference's left fold: within 1e-12 relative (north
  star), not bitwise.
* `chain_mul_sum`: the ranks form a chain along `shard_dim`.  Rank r
  continues the left-fold accumulators of rank r-1 over its own slab
  (`tt_mul_fold` with an initial accumulator) and passes them on; the last
  rank runs the in-tile rotate-and-sum once.  This is the reference's own
  association, so the result is bit-identical to one GPU.  The output tiles
  are split into chunks that flow down the chain back to back (NCCL
  send / recv are stream-ordered), so the ranks overlap: the chain costs
  (chunks + ranks - 1) / chunks of one slab's fold plus the point-to-point
  transfers of the accumulators.

The compute backend is injectable (`ops`): on GPUs it is this package's
CUDA path; the CPU gloo tests drive the same planning and collective logic
with the oracle as compute.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Any, Callable, Optional

from .tiletensor import DimSpec, TileTensorShape, shard_plan


@dataclass(frozen=True)
class ShardPlan:
    global_shape: TileTensorShape
    local_shape: TileTensorShape
    shard_dim: int           # 1-based
    world: int
    rank: int
    begin: int               # external tile index range [begin, end)
    end: int

    @property
    def row_slice(self) -> slice:
        """Dense rows of `shard_dim` this rank holds."""
        d = self.global_shape.dim(self.shard_dim - 1)
        lo = self.begin * d.t
        return slice(lo, min(d.used(), self.end * d.t))

    def dense_slices(self) -> tuple:
        sl = [slice(None)] * self.global_shape.rank()
        sl[self.shard_dim - 1] = self.row_slice
        return tuple(sl)

    def local_tiles(self) -> int:
        return self.local_shape.tile_count()


def plan(global_shape: TileTensorShape, shard_dim: int, world: int, rank: int) -> ShardPlan:
    b, e, local = shard_plan(global_shape, shard_dim, world, rank)
    return ShardPlan(global_shape, local, shard_dim, world, rank, b, e)


def operand_plan(op_shape: TileTensorShape, x_plan: ShardPlan) -> Optional[ShardPlan]:
    """How a second operand follows X's sharding: None when it broadcasts
    (fully replicated, one external tile) along shard_dim -- then every rank
    holds it whole -- else the same block partition."""
    d = op_shape.dim(x_plan.shard_dim - 1)
    if d.n == 1 and (d.d + d.t - 1) // d.t == 1:
        return None
    return plan(op_shape, x_plan.shard_dim, x_plan.world, x_plan.rank)


def _dist():
    import torch.distributed as dist
    return dist if dist.is_available() and dist.is_initialized() else None


def allreduce_partial(data, group=None, async_op: bool = False):
    """Sum a rank-partial result over all ranks in place (NCCL on GPUs).
    async_op: return the collective's work handle (None when there is nothing
    to reduce) so independent kernels can run while it is in flight; the
    caller waits on it before using `data`."""
    dist = _dist()
    if dist is not None and dist.get_world_size(group) > 1:
        return dist.all_reduce(data, op=dist.ReduceOp.SUM, group=group, async_op=async_op)
    return None


def broadcast_operand(data, src: int = 0, group=None) -> None:
    """Replicate an operand that every rank needs whole (e.g. W)."""
    dist = _dist()
    if dist is not None and dist.get_world_size(group) > 1:
        dist.broadcast(data, src=src, group=group)


def _p2p_staged(dist, group) -> bool:
    """gloo moves point-to-point messages through host memory only: device
    tensors are staged through a host copy (the functional multi-rank check
    on one GPU); NCCL sends device memory directly over NVLink."""
    return dist.get_backend(group) == "gloo"


def _send(dist, t, dst, group):
    if _p2p_staged(dist, group) and getattr(t, "is_cuda", False):
        t = t.cpu()
    dist.send(t, dst=dst, group=group)


def _recv_into(dist, t, src, group):
    if _p2p_staged(dist, group) and getattr(t, "is_cuda", False):
        h = t.new_empty(t.shape, device="cpu")
        dist.recv(h, src=src, group=group)
        t.copy_(h)
    else:
        dist.recv(t, src=src, group=group)


def sharded_mul_sum(x_local, w_local, dim: int, x_plan: ShardPlan,
                    mul_sum: Callable[[Any, Any, int], Any],
                    data_of: Callable[[Any], Any], group=None):
    """tt_sum(tt_mul(X, W), dim) on a sharded X.

    dim != shard_dim: local fused op, result sharded like X (no traffic).
    dim == shard_dim: local fused op over the slab, then one all-reduce of
    the partial result -- every rank ends with the full (replicated) result.
    Returns (result, is_sharded).
    """
    r = mul_sum(x_local, w_local, dim)
    if dim == x_plan.shard_dim:
        allreduce_partial(data_of(r), group)
        return r, False
    return r, True


def chain_mul_sum(x_local, w_local, dim: int, x_plan: ShardPlan, fold: Callable, finish: Callable,
                  n_out: int, new_acc: Callable[[int], Any], chunks: int = 16, group=None):
    """Exact tt_sum(tt_mul(X, W), dim) for dim == shard_dim (see module doc).

    fold(x, w, dim, (lo, hi), init) -> accumulator tiles of output tiles
    [lo, hi) (init None on the first rank); finish(acc) -> the result from
    the accumulated tiles of all n_out outputs; new_acc(k) -> a buffer of k
    accumulator tiles to receive into.  On GPUs these are tt.mul_fold,
    tt_sum over fold_shape and Session.empty_tiles (`gpu_chain_ops`).
    Returns the result on the last rank, None on the others."""
    dist = _dist()
    world = dist.get_world_size(group) if dist is not None else 1
    rank = dist.get_rank(group) if dist is not None else 0
    if dim != x_plan.shard_dim or world == 1:
        acc = fold(x_local, w_local, dim, (0, n_out), None)
        return finish(acc)
    chunks = max(1, min(chunks, n_out))
    bounds = [(n_out * c // chunks, n_out * (c + 1) // chunks) for c in range(chunks)]
    parts = []
    for lo, hi in bounds:
        if hi <= lo:
            continue
        init = None
        if rank > 0:
            init = new_acc(hi - lo)
            _recv_into(dist, init, rank - 1, group)
        acc = fold(x_local, w_local, dim, (lo, hi), init)
        if rank < world - 1:
            _send(dist, acc, rank + 1, group)
        else:
            parts.append(acc)
    result = finish(parts) if rank == world - 1 else None
    return result


def gpu_chain_ops(tt, x_local, w_local, dim: int):
    """The (fold, finish, n_out, new_acc) of chain_mul_sum on this package's
    CUDA path: tt.mul_fold over a tile range, and tt_sum of the concatenated
    accumulators viewed with fold_shape (one external tile along dim)."""
    import torch
    s = x_local.session()
    fshape = tt.fold_shape(x_local.shape(), w_local.shape() if w_local is not None else None, dim)

    def fold(x, w, d, rng, init):
        return tt.mul_fold(x, w, d, out_range=rng, init=init)[0]

    def finish(parts):
        acc = parts if isinstance(parts, torch.Tensor) else torch.cat(parts, dim=0)
        return tt.tt_sum(tt.TileTensor(fshape, acc, s), dim)

    return fold, finish, fshape.tile_count(), s.empty_tiles


def local_result_tile_range(x_plan: ShardPlan, result_shape: TileTensorShape):
    """Tile rows [lo, hi) of the GLOBAL result that this rank's sharded result
    holds (row-major external order, shard_dim outermost-relative slab)."""
    ext = result_shape.external_extents()
    k = x_plan.shard_dim - 1
    inner = 1
    for e in ext[k + 1:]:
        inner *= e
    outer = 1
    for e in ext[:k]:
        outer *= e
    if outer != 1:
        raise ValueError("contiguous tile range only when shard_dim is the outermost non-unit dim")
    return x_plan.begin * inner, x_plan.end * inner


__all__ = ["ShardPlan", "plan", "operand_plan", "allreduce_partial", "broadcast_operand",
           "sharded_mul_sum", "chain_mul_sum", "gpu_chain_ops", "local_result_tile_range"]
