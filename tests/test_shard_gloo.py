"""Multi-process (gloo, CPU) tests of the doc-ID sharded rerank merge
(paper_2504_02921_b200/shard.py): partition, local top-k, one all-gather,
merge — the merged top-k must equal the single-process selection of the
reference's _select (pipeline.py:285-287) on the same scores.

The per-segment top-k here is the oracle's ordering (a CPU checker); on the
GPU box the same host logic runs with the CUDA kernel (tests/test_gpu_*).
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2504_02921_b200 import shard


def cpu_topk(scores, ids, n_seg, seg_len, k):
    s = scores.view(n_seg, seg_len).numpy()
    i = ids.view(n_seg, seg_len).numpy()
    idx = np.full((n_seg, k), -1, np.int32)
    out = np.full((n_seg, k), -np.inf, np.float32)
    for r in range(n_seg):
        order = sorted(range(seg_len), key=lambda j: (-s[r, j], i[r, j], j))[:k]
        idx[r, :len(order)] = order
        out[r, :len(order)] = s[r, order]
    return torch.from_numpy(idx), torch.from_numpy(out)


def workload(n_q=6, n_c=37, corpus=200, seed=0):
    rng = np.random.default_rng(seed)
    cand = np.stack([rng.choice(corpus, n_c, replace=False) for _ in range(n_q)])
    # scores with deliberate exact ties across shards
    table = np.round(rng.standard_normal((n_q, corpus)), 1).astype(np.float32)
    return cand, table


def expected(cand, table, k):
    out = []
    for q in range(cand.shape[0]):
        ids = [f"doc-{d:05d}" for d in cand[q]]
        sc = [float(table[q, d]) for d in cand[q]]
        out.append([int(cand[q][j]) for j in oracle.select_topk(sc, ids, k)])
    return out


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, k, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cand, table = workload()
        work = shard.local_work(cand, rank, world)
        doc = cand[work.pair_query, work.pair_cand]
        scores = torch.from_numpy(table[work.pair_query, doc])
        ids = torch.from_numpy(doc.astype(np.int32))   # doc index == chunk-id rank
        mi, ms = shard.sharded_select(scores, ids, work, cand.shape[0], k, cpu_topk)
        q.put((rank, mi.numpy().tolist(), ms.numpy().tolist()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,k", [(2, 20), (3, 5), (2, 40)])
def test_sharded_merge_equals_single_process(world, k):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, k, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    cand, table = workload()
    want = expected(cand, table, k)
    for _, ids, sc in res:
        assert ids == res[0][1]                     # every rank holds the same merge
        for qi in range(cand.shape[0]):
            real = [d for d in ids[qi] if d != shard.PAD_ID]
            assert real == want[qi]
            assert sc[qi][:len(real)] == [float(table[qi, d]) for d in real]


def test_local_work_partition_covers_every_pair_once():
    cand, _ = workload(n_q=5, n_c=30)
    seen = np.zeros(cand.shape, int)
    for r in range(4):
        w = shard.local_work(cand, r, 4)
        seen[w.pair_query, w.pair_cand] += 1
        assert (shard.owner_of(cand[w.pair_query, w.pair_cand], 4) == r).all()
        # segment positions are dense per query
        for qi in range(5):
            pos = np.sort(w.seg_pos[w.pair_query == qi])
            assert pos.tolist() == list(range(pos.size)) and pos.size <= w.seg_len
    assert (seen == 1).all()


def _bcast_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        toks = np.arange(3 * 7, dtype=np.int64).reshape(3, 7) + 100 if rank == 0 else None
        t = shard.broadcast_queries(toks, 3, 7)
        q.put((rank, t.dtype == torch.int32, t.numpy().tolist()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_broadcast_queries(world):
    """Rank 0's query tokens reach every rank unchanged (north_star (d))."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_bcast_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = (np.arange(21).reshape(3, 7) + 100).tolist()
    assert sorted(r for r, _, _ in res) == list(range(world))
    assert all(ok and got == want for _, ok, got in res)
