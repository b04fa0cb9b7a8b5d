"""Multi-GPU plumbing around the C ABI (host logic only; all arithmetic stays in
the library's kernels and its NCCL calls).

One process per GPU.  The long dimension of X is split in contiguous blocks
(`shard_range`); the library's `cpa_svt_apply` with SHARD_COLS / SHARD_ROWS
sums the partial Grams with one NCCL all-reduce (G = sum_p X_p X_p^T,
PAPER.md:278-307) and broadcasts Lambda from rank 0, after which every rank
runs the recurrence on its own block.  Sparse X (config 4) is row-sharded with
X replicated, batched problems are split by matrix: neither has a collective.
"""

from __future__ import annotations


def shard_range(n: int, world: int, rank: int) -> tuple[int, int]:
    """Balanced contiguous block [begin, end) of range(n) owned by `rank`."""
    if world < 1 or not 0 <= rank < world or n < 0:
        raise ValueError("bad shard request")
    base, rem = divmod(n, world)
    begin = rank * base + min(rank, rem)
    return begin, begin + base + (1 if rank < rem else 0)


def broadcast_nccl_id(make_id=None, group=None) -> bytes:
    """ncclUniqueId created on rank 0 (cpa_svt_nccl_unique_id) and broadcast over torch.distributed."""
    import torch.distributed as dist
    obj = [None]
    if dist.get_rank(group) == 0:
        if make_id is None:
            from . import nccl_unique_id
            make_id = nccl_unique_id
        obj[0] = make_id()
    dist.broadcast_object_list(obj, src=0, group=group)
    return obj[0]


def sharded_side(m_global: int, n_global: int) -> str:
    """Which dimension is sharded: the long one (reading R3: left iff m <= n -> columns)."""
    return "cols" if m_global <= n_global else "rows"


def local_block(X, world: int, rank: int):
    """This rank's block of a full (host or device) matrix, split along its long dimension."""
    m, n = X.shape
    if sharded_side(m, n) == "cols":
        b, e = shard_range(n, world, rank)
        return X[:, b:e]
    b, e = shard_range(m, world, rank)
    return X[b:e, :]


def make_handle(device: int, group=None, comm: bool = True):
    """A Handle whose library-side NCCL communicator spans the torch.distributed world.

    comm=True creates the communicator at any world size -- also a one-rank one, so the
    sharded path with its NCCL all-reduce / broadcast runs on a single GPU.  Without
    torch.distributed the id is made locally (world 1)."""
    import torch.distributed as dist
    from . import Handle, nccl_unique_id
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    if world > 1:
        nid = broadcast_nccl_id(group=group)
    else:
        nid = nccl_unique_id() if comm else None
    return Handle(device, nccl_id=nid, rank=rank, world=world)


def shard_args(m_global: int, n_global: int, has_comm: bool) -> dict:
    """shard / long_global arguments of cpa_svt_apply for a block of the (m_global x n_global) X."""
    if not has_comm:
        return {"shard": "none", "long_global": 0}
    shard = sharded_side(m_global, n_global)
    return {"shard": shard, "long_global": n_global if shard == "cols" else m_global}


def apply_sharded(h, X_local, m_global: int, n_global: int, kernel, K: int, **kw):
    """cpa_svt_apply on this rank's block; returns this rank's block of Y.  With a communicator
    (any world size) the library runs the exchange: all-reduce of the partial Grams, broadcast
    of the series parameters."""
    return h.apply(X_local, kernel, K, **shard_args(m_global, n_global, getattr(h, "has_comm", h.world > 1)),
                   **kw)


def panel_ranges(s: int, world: int) -> list[tuple[int, int]]:
    """Tile ranges of the multi-GPU s x s recurrence (the library's partition, dense_f64.cu
    dense_sym_panel_tile0): the T(T+1)/2 lower 64 x 64 tiles of an s x s matrix in column-major
    order, T = ceil(s / 64), split in `world` contiguous ranges [ntri p / P, ntri (p+1) / P)."""
    T = (s + 63) // 64
    ntri = T * (T + 1) // 2
    return [(ntri * p // world, ntri * (p + 1) // world) for p in range(world)]
