"""Document-ID sharding across the GPUs of one box.

One process per GPU.  The corpus KV is partitioned by document index
(``owner = doc_index % world``) into each rank's HBM pool; queries are
broadcast; every rank scores only the (query, candidate) pairs whose
candidate it owns, keeps a local top-k per query, and ONE all-gather of
``[n_queries, k] x (f32 score, i32 doc rank)`` merges the results.  KV never
crosses GPUs.  The merge uses the same (score desc, chunk-id asc) order as
the reference's ``_select`` (pipeline.py:285-287) with doc ranks taken in
sorted chunk-id order, and every kernel is batch-invariant, so the merged
top-k is bit-identical to the 1-GPU result.

The collective goes through ``torch.distributed`` (NCCL on the GPU box;
gloo in the CPU tests).  ``topk_fn`` is the per-segment top-k: the CUDA
kernel (``engine.segmented_topk``) in the product path.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

PAD_ID = np.iinfo(np.int32).max


def broadcast_queries(q_tokens, n_q: int, query_len: int, device=None, src: int = 0,
                      group=None):
    """Queries are broadcast (north_star (d)): rank ``src`` holds the host
    token matrix ``[n_q, query_len]``; every rank returns it as an int32 tensor
    on ``device`` (its GPU for NCCL; the CPU for gloo).  Ids are range-checked
    as int64 on the source before the int32 cast."""
    import torch
    import torch.distributed as dist
    if device is None:
        device = torch.device("cpu")
    rank = dist.get_rank(group) if dist.is_initialized() else src
    if rank == src:
        q = np.asarray(q_tokens, dtype=np.int64)
        if q.shape != (n_q, query_len):
            raise ValueError(f"query tokens must be [{n_q}, {query_len}], got {q.shape}")
        if q.size and (q.min() < 0 or q.max() > np.iinfo(np.int32).max):
            raise ValueError("query token ids outside int32")
        t = torch.as_tensor(q.astype(np.int32)).to(device)
    else:
        t = torch.empty((n_q, query_len), dtype=torch.int32, device=device)
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.broadcast(t, src=src, group=group)
    return t


def owner_of(doc_index, world: int):
    """Rank that holds a document's KV (contiguous-free, load-balanced)."""
    return np.asarray(doc_index) % world


@dataclass
class LocalWork:
    """This rank's slice of a query batch."""

    pair_query: np.ndarray      # [n_local] query index of each local pair
    pair_cand: np.ndarray       # [n_local] candidate position within its query's list
    seg_len: int                # padded per-query segment length (max local count)
    seg_pos: np.ndarray         # [n_local] slot of each pair inside its query segment


def local_work(cand_doc_index: np.ndarray, rank: int, world: int) -> LocalWork:
    """Pairs owned by ``rank`` from a [n_q, n_c] matrix of candidate doc indices."""
    own = owner_of(cand_doc_index, world) == rank
    qi, ci = np.nonzero(own)
    counts = own.sum(axis=1)
    seg_len = int(counts.max()) if counts.size else 0
    starts = np.concatenate([[0], np.cumsum(counts)[:-1]])
    pos = np.arange(qi.size) - np.repeat(starts, counts)
    return LocalWork(qi.astype(np.int64), ci.astype(np.int64), seg_len, pos.astype(np.int64))


def pad_segments(scores, ids, work: LocalWork, n_q: int):
    """Scatter local pair scores/ids into [n_q, seg_len] segments; empty slots
    get score -inf and id PAD_ID so they sort last."""
    import torch
    dev = scores.device
    L = max(work.seg_len, 1)
    s = torch.full((n_q, L), float("-inf"), dtype=torch.float32, device=dev)
    i = torch.full((n_q, L), PAD_ID, dtype=torch.int32, device=dev)
    if work.pair_query.size:
        # pinned, non-blocking copies: a pageable host->device copy would make the
        # host wait for the stream (serialising it with the scoring kernels)
        from .kvpool import to_device
        q = to_device(work.pair_query, dev)
        p = to_device(work.seg_pos, dev)
        s[q, p] = scores.to(torch.float32)
        i[q, p] = ids.to(torch.int32)
    return s, i


def merge_topk(local_scores, local_ids, k: int, topk_fn, group=None):
    """All-gather per-rank top-k ``[n_q, k]`` (score, doc rank) and merge.

    ``local_scores``/``local_ids`` are already each rank's top-k (padded with
    -inf / PAD_ID).  Returns merged ``(ids [n_q, k], scores [n_q, k])`` on every
    rank; positions beyond the number of real candidates hold PAD_ID / -inf."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    n_q = local_scores.shape[0]
    if world == 1:
        return local_ids, local_scores
    gs = [torch.empty_like(local_scores) for _ in range(world)]
    gi = [torch.empty_like(local_ids) for _ in range(world)]
    dist.all_gather(gs, local_scores.contiguous(), group=group)
    dist.all_gather(gi, local_ids.contiguous(), group=group)
    cs = torch.cat(gs, dim=1).contiguous()          # [n_q, world*k]
    ci = torch.cat(gi, dim=1).contiguous()
    idx, sc = topk_fn(cs.view(-1), ci.view(-1), n_q, world * k, k)
    return ci.gather(1, idx.long().clamp_min(0)), sc


def local_topk(scores, ids, work: LocalWork, n_q: int, k: int, topk_fn):
    """Per-query top-k over this rank's pairs -> ([n_q, k] scores, [n_q, k] ids)."""
    import torch
    s, i = pad_segments(scores, ids, work, n_q)
    idx, sc = topk_fn(s.view(-1), i.view(-1), n_q, s.shape[1], k)
    good = idx >= 0
    out_i = torch.where(good, i.gather(1, idx.long().clamp_min(0)),
                        torch.full_like(idx, PAD_ID))
    out_s = torch.where(good, sc, torch.full_like(sc, float("-inf")))
    return out_s, out_i


def sharded_select(scores, ids, work: LocalWork, n_q: int, k: int, topk_fn, group=None):
    """Local top-k then the one all-gather merge: the whole (e) row."""
    s, i = local_topk(scores, ids, work, n_q, k, topk_fn)
    return merge_topk(s, i, k, topk_fn, group)
