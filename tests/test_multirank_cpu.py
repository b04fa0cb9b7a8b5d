"""N > 1 host logic on CPU: world_size-2 gloo process groups (no GPU).

Covers the sharding helpers of paper_1705_07112_b200.dist, the NCCL-id
broadcast, bench.py's max-over-ranks timing reduction, and -- with the oracle
standing in for each rank's kernels -- that the decomposition the library uses
(column shards + one all-reduce of the partial Grams + Lambda from rank 0;
sparse row shards with X replicated) reproduces the single-process result.
"""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
import workloads as W


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(fn, world=2):
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_entry, args=(fn, r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    errs = [o for o in out if isinstance(o, str)]
    assert not errs, errs
    return {o[0]: o[1] for o in out}


def _entry(fn, rank, world, port, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        res = fn(rank, world)
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, res))
    except Exception as e:  # pragma: no cover - reported to the parent
        import traceback
        q.put(f"rank {rank}: {e}\n{traceback.format_exc()}")


# ---------------------------------------------------------------- helpers (import-free of the CUDA lib)
def _load_dist():
    import importlib.util
    here = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    spec = importlib.util.spec_from_file_location("cpa_dist", os.path.join(here, "paper_1705_07112_b200", "dist.py"))
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    return m


def test_shard_range_partitions():
    D = _load_dist()
    for n in (0, 1, 7, 64, 65537):
        for world in (1, 2, 3, 8):
            spans = [D.shard_range(n, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [e - b for b, e in spans]
            assert max(sizes) - min(sizes) <= 1
    assert D.sharded_side(16384, 65536) == "cols" and D.sharded_side(300, 20) == "rows"


def _nccl_id_bcast(rank, world):
    D = _load_dist()
    nid = D.broadcast_nccl_id(make_id=lambda: bytes(range(128)))
    return nid


def test_nccl_id_broadcast_gloo():
    res = _run(_nccl_id_bcast)
    assert res[0] == res[1] == bytes(range(128))


def _max_over_ranks(rank, world):
    import torch
    import bench
    return bench.max_over_ranks(1.5 + rank, torch.device("cpu"))


def test_bench_max_over_ranks_gloo():
    res = _run(_max_over_ranks)
    assert res[0] == res[1] == 2.5


def _dense_sharded(rank, world):
    import torch
    D = _load_dist()
    X = W.gen_c2(m=64, n=301, seed=3)             # wide: left side, columns sharded
    kern = O.Kernel("soft", tau=0.1, tau_relative=True)
    Xp = D.local_block(X, world, rank)
    # partial Gram on this rank, one all-reduce (the library's NCCL step)
    G = torch.from_numpy(Xp @ Xp.T)
    dist.all_reduce(G)
    G = G.numpy()
    # Lambda on rank 0, broadcast (the library broadcasts its series parameters)
    lam = torch.zeros(1, dtype=torch.float64)
    if rank == 0:
        lam[0] = 1.01 * O.power_iteration(lambda v: G @ v, G.shape[0], 60)[0]
    dist.broadcast(lam, 0)
    lam = float(lam[0])
    c = O.kernel_coefficients(kern, 12, lam, (lam / 1.01) ** 0.5)
    Yp = O.cpa_apply_vectors(lambda V: G @ V, Xp, c, lam)
    parts = [None] * world
    dist.all_gather_object(parts, Yp)
    return np.concatenate(parts, axis=1)


def test_dense_column_sharding_matches_single_process():
    res = _run(_dense_sharded)
    X = W.gen_c2(m=64, n=301, seed=3)
    Y = O.cpa_shrink(X, O.Kernel("soft", tau=0.1, tau_relative=True), 12, T=60)
    assert np.array_equal(res[0], res[1])
    assert O.rel_fro(res[0], Y) <= 1e-12


def _sparse_rows(rank, world):
    import scipy.sparse as sp
    D = _load_dist()
    m, n = 60, 700
    rp, col, val = W.gen_c4(seed=2, m=m, n=n, nnz=1400)
    Xs = sp.csr_matrix((val, col, rp), shape=(m, n))
    b, e = D.shard_range(m, world, rank)
    Yp, _ = O.cpa_shrink_sparse_rows(Xs, list(range(b, e)), O.Kernel("hard", tau=0.5, tau_relative=True), 10, T=80)
    parts = [None] * world
    dist.all_gather_object(parts, Yp)
    return np.concatenate(parts, axis=0)


def test_sparse_row_sharding_matches_single_process():
    import scipy.sparse as sp
    res = _run(_sparse_rows)
    m, n = 60, 700
    rp, col, val = W.gen_c4(seed=2, m=m, n=n, nnz=1400)
    Xs = sp.csr_matrix((val, col, rp), shape=(m, n))
    Y, _ = O.cpa_shrink_sparse_rows(Xs, list(range(m)), O.Kernel("hard", tau=0.5, tau_relative=True), 10, T=80)
    assert np.array_equal(res[0], Y)


def _batched_split(rank, world):
    D = _load_dist()
    Xb = W.gen_c3(batch=9, seed=4)
    b, e = D.shard_range(Xb.shape[0], world, rank)
    Y, _ = O.cpa_shrink_batched(Xb[b:e], O.Kernel(**W.CONFIGS["c3"]["kernel"]), 8, T=20)
    parts = [None] * world
    dist.all_gather_object(parts, Y)
    return np.concatenate(parts, axis=0)


def test_batched_split_matches_single_process():
    res = _run(_batched_split)
    Xb = W.gen_c3(batch=9, seed=4)
    Y, _ = O.cpa_shrink_batched(Xb, O.Kernel(**W.CONFIGS["c3"]["kernel"]), 8, T=20)
    assert np.array_equal(res[0], Y)


def test_panel_partition_host_logic():
    """Tile ranges of the multi-GPU s x s recurrence: contiguous, covering all T(T+1)/2 lower
    tiles, balanced to one tile."""
    D = _load_dist()
    for s in (1, 64, 65, 1024, 16384):
        T = (s + 63) // 64
        ntri = T * (T + 1) // 2
        for P_ in (1, 2, 3, 8):
            r = D.panel_ranges(s, P_)
            assert r[0][0] == 0 and r[-1][1] == ntri and all(a[1] == b[0] for a, b in zip(r, r[1:]))
            sizes = [b - a for a, b in r]
            assert max(sizes) - min(sizes) <= 1


class _RecordingHandle:
    """Stands in for the library Handle: records what dist.apply_sharded passes to cpa_svt_apply."""

    def __init__(self, world, has_comm=True):
        self.world, self.has_comm, self.calls = world, has_comm, []

    def apply(self, X, kernel, K, **kw):
        self.calls.append(kw)
        return X


def _sharded_args(rank, world):
    D = _load_dist()
    out = []
    for (m, n) in ((64, 301), (301, 64)):
        h = _RecordingHandle(world)
        X = np.zeros((m, n))
        D.apply_sharded(h, D.local_block(X, world, rank), m, n, {"kind": "soft"}, 5, T=3)
        out.append((h.calls[0]["shard"], h.calls[0]["long_global"], D.local_block(X, world, rank).shape))
    return out


def test_apply_sharded_arguments_gloo():
    """dist.apply_sharded passes the library the shard mode and the GLOBAL long extent on every
    rank, each rank's block being its contiguous share of the long dimension."""
    res = _run(_sharded_args)
    for r in (0, 1):
        (s1, l1, sh1), (s2, l2, sh2) = res[r]
        assert (s1, l1) == ("cols", 301) and (s2, l2) == ("rows", 301)
    assert res[0][0][2][1] + res[1][0][2][1] == 301 and res[0][1][2][0] + res[1][1][2][0] == 301
    D = _load_dist()
    h = _RecordingHandle(1, has_comm=False)
    D.apply_sharded(h, np.zeros((4, 9)), 4, 9, {"kind": "soft"}, 5)
    assert h.calls[0]["shard"] == "none"


def _empty_block_args(rank, world):
    D = _load_dist()
    out = []
    for (m, n) in ((3, 3), (5, 4)):     # long extent 3 / 5 < 2 ranks x 2: ... and a tall one
        X = np.zeros((m, n))
        h = _RecordingHandle(world)
        blk = D.local_block(X, 4 * world, rank)   # 4 * world "ranks" of which this is one: empty blocks
        D.apply_sharded(h, blk, m, n, {"kind": "soft"}, 5, T=3)
        out.append((h.calls[0]["shard"], h.calls[0]["long_global"], blk.shape))
    return out


def test_empty_blocks_make_the_same_call_gloo():
    """A long extent below the number of ranks leaves some ranks an empty block; those ranks make
    the SAME library call (shard mode, global long extent) as their peers, only with a zero-width
    block -- the library then joins every collective with a zero partial Gram (empty
    inputs) instead of returning early."""
    res = _run(_empty_block_args)
    for r in (0, 1):
        (s1, l1, sh1), (s2, l2, sh2) = res[r]
        assert (s1, l1) == ("cols", 3) and (s2, l2) == ("rows", 5)
    D = _load_dist()
    shapes = [D.local_block(np.zeros((3, 3)), 8, r).shape for r in range(8)]
    assert sum(sh[1] for sh in shapes) == 3 and shapes[-1] == (3, 0)
