"""Rerank + select stage of the reference pipeline on the device.

Restates the scoring and selection stages of handle_query
(pipeline.py:274-287, 297-326) for many queries at once:

  candidates (chunk ids) --page-table lookup--> pool slots      (_fetch_items, :251-271)
  every (query, candidate) pair scored in one batch             (_score_item, :274-282)
  per-query top-keep_m by (-score, chunk_id) on the device      (_select, :285-287)

A candidate whose KV is not resident (cache miss) falls back to full
recompute for that pair, exactly like the reference (:258-265); misses are
counted.  Doc ids passed to the top-k kernel are ranks in sorted chunk-id
order, so the integer tie-break equals the reference's string tie-break.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import engine
from .errors import ConfigError, ShapeError
from .kvpool import KVPool, to_device
from .model import RerankModel
from .reranker import ScoredPair, _check_vocab, _doc_valid


@dataclass
class RerankResult:
    query_ids: list
    selected: list          # per query: list[ScoredPair] (best first)
    cache_misses: int
    pairs: int


PAD_RANK = np.iinfo(np.int32).max

# Latency-sized calls (all candidates cached, equal-length lists, at most this
# many suffix rows = pairs x query_len) replay a CUDA graph of the whole scoring
# pass once the same shape has been seen before: the per-layer launches and
# their host-side setup cost ~1 ms per call at the Gemma shape (C2 p50: 10.1 ms
# eager vs 9.0 ms replayed).  Two graphs per pool are kept, each owning a
# workspace for its rows (<= ~0.6 GB at the 7B shape).
GRAPH_MAX_ROWS = 8192
GRAPH_CACHE = 2


def _graph_for(pool: KVPool, w, n_q: int, n_c: int, Q: int, k: int):
    """The pool's GraphedScorer for this shape, captured on the second call with
    it (a one-off shape is scored eagerly), or None."""
    from collections import OrderedDict
    graphs = pool.__dict__.setdefault("_rerank_graphs", OrderedDict())
    seen = pool.__dict__.setdefault("_rerank_shapes", set())
    key = (id(w), n_q, n_c, Q, k)
    gs = graphs.get(key)
    if gs is not None:
        graphs.move_to_end(key)
        return gs
    if key not in seen:
        seen.add(key)
        return None
    gs = engine.GraphedScorer(w, pool, n_q, n_c, Q, k)
    graphs[key] = gs
    while len(graphs) > GRAPH_CACHE:
        graphs.popitem(last=False)
    return gs


def _id_ranks(chunk_ids_2d) -> np.ndarray:
    """Rank of every candidate in sorted chunk-id order, [n_q, max_len] int32;
    ragged rows are padded with PAD_RANK."""
    flat = sorted(set(c for row in chunk_ids_2d for c in row))
    rank = {c: i for i, c in enumerate(flat)}
    n_c = max((len(r) for r in chunk_ids_2d), default=0)
    out = np.full((len(chunk_ids_2d), n_c), PAD_RANK, dtype=np.int32)
    for i, row in enumerate(chunk_ids_2d):
        out[i, :len(row)] = [rank[c] for c in row]
    return out


def rerank(model: RerankModel, pool: KVPool, query_ids, query_tokens, candidates, keep_m: int,
           doc_tokens: dict | None = None, path: str = "fast") -> RerankResult:
    """Score every candidate of every query against its cached document KV
    and keep the best ``keep_m`` per query.

    query_tokens: int [n_q, Q] host array; candidates: n_q lists of chunk ids
    (any lengths); doc_tokens: chunk_id -> tokens for miss fallback."""
    import torch
    if keep_m < 1:
        raise ConfigError("keep_m must be >= 1")
    w = model.weights_for(path)
    q = np.asarray(query_tokens)
    n_q = len(query_ids)
    if q.shape != (n_q, model.layout.query_len):
        raise ShapeError(f"query tokens must be [{n_q}, {model.layout.query_len}]")
    if any((row != 0).sum() == 0 for row in q):
        from .errors import DegenerateInputError
        raise DegenerateInputError("query is entirely padding")
    # the reference's _check_call rejects ids outside [0, vocab) (model.py:203-204);
    # checked before the int32 cast so int64 ids cannot wrap into range
    _check_vocab(model, q)
    if len(candidates) != n_q:
        raise ShapeError("one candidate list per query")
    lens = np.array([len(c) for c in candidates], dtype=np.int64)
    n_c = int(lens.max()) if n_q else 0
    flat = [c for row in candidates for c in row]
    pair_q = np.repeat(np.arange(n_q), lens)
    slots = pool.lookup(flat)
    miss = np.nonzero(slots < 0)[0]
    if (n_c and len(miss) == 0 and (lens == n_c).all() and
            len(flat) * q.shape[1] <= GRAPH_MAX_ROWS):
        k = min(keep_m, n_c)
        gs = _graph_for(pool, w, n_q, n_c, q.shape[1], k)
        if gs is not None:
            idx_h, sc_h = gs(slots, q, _id_ranks(candidates).reshape(-1))
            selected = [[ScoredPair(chunk_id=candidates[i][int(j)], query_id=query_ids[i],
                                    score=float(s)) for j, s in zip(idx_h[i], sc_h[i])]
                        for i in range(n_q)]
            return RerankResult(list(query_ids), selected, 0, len(flat))
    dev = w.device
    scores = torch.empty(len(flat), dtype=torch.float32, device=dev)
    hit = np.nonzero(slots >= 0)[0]
    q_dev = to_device(q.astype(np.int32), dev)
    if len(hit):
        qi = to_device(pair_q[hit], dev)
        sc = engine.score_slots(w, pool, to_device(slots[hit], dev), q_dev.index_select(0, qi))
        scores[to_device(hit, dev)] = sc
    if len(miss):
        if doc_tokens is None:
            raise ShapeError("cache miss without doc_tokens for full-recompute fallback")
        docs = np.stack([np.asarray(doc_tokens[flat[i]]) for i in miss])
        for dd in docs:
            _doc_valid(model, dd)
        stage = KVPool(model.config, model.layout.document_len, len(miss), w.dtype, dev)
        st_slots = stage.allocate_owned(len(miss))
        engine.prefill_slots(w, stage, st_slots, docs, (docs != 0).sum(axis=1))
        qi = to_device(pair_q[miss], dev)
        scores[to_device(miss, dev)] = engine.score_slots(
            w, stage, st_slots, q_dev.index_select(0, qi))
    if n_c == 0:
        return RerankResult(list(query_ids), [[] for _ in range(n_q)], 0, 0)
    ids = _id_ranks(candidates)
    if not (lens == n_c).all():          # ragged: pad segments (-inf sorts last)
        seg = torch.full((n_q, n_c), float("-inf"), dtype=torch.float32, device=dev)
        pos = np.arange(len(flat)) - np.repeat(np.cumsum(lens) - lens, lens)
        seg[to_device(pair_q, dev), to_device(pos, dev)] = scores
        scores = seg.view(-1)
    k = min(keep_m, n_c)
    idx, sc = engine.segmented_topk(scores, ids.reshape(-1), n_q, n_c, k)
    idx_h, sc_h = idx.cpu().numpy(), sc.cpu().numpy()
    selected = [[ScoredPair(chunk_id=candidates[i][int(j)], query_id=query_ids[i],
                            score=float(s)) for j, s in zip(idx_h[i], sc_h[i])
                 if 0 <= j < lens[i]]
                for i in range(n_q)]
    return RerankResult(list(query_ids), selected, int(len(miss)), int(lens.sum()))


def populate_store(model: RerankModel, docs, index, store, scheme=None, path: str = "fast",
                   on_entry=None, batch: int = 64) -> int:
    """Prefill, encode and place every doc's cache entry; returns total bytes
    (pipeline.py:156-171).

    ``docs`` are objects with ``.id`` / ``.text`` (the reference's CorpusDoc),
    ``index`` anything with ``centroid_of(doc_id)`` (IvfIndex), ``store`` a
    ShardedStore.  Prefill runs batched on the GPU straight into pool pages.
    A shard backed by a DevicePagedKVStore keeps the page where the prefill
    wrote it when the scheme is F32 or F16 (no bytes cross PCIe; the count is the
    entry size the reference would have written); other backends, and
    quantised schemes, receive HRKV bytes."""
    from .codec import HEADER, QuantScheme, encode_entry, payload_nbytes
    from .reranker import doc_prefill_batch, tokenize
    from .store import DevicePagedKVStore
    scheme = scheme or QuantScheme.F32
    cfg, lay = model.config, model.layout
    total = 0
    for i in range(0, len(docs), batch):
        chunk = docs[i:i + batch]
        toks = np.stack([tokenize(d.text, lay.document_len, vocab_size=cfg.vocab_size)
                         for d in chunk])
        targets = [store.backends[store.shard_for(index.centroid_of(d.id))] for d in chunk]
        # docs bound for a device shard prefill into that shard's pool
        by_pool: dict[int, list[int]] = {}
        for j, b in enumerate(targets):
            # quantised schemes go through the bytes (the page must hold the
            # dequantised values the reference would score with)
            device = isinstance(b, DevicePagedKVStore) and not scheme.quantised
            key = id(b.pool) if device else 0
            by_pool.setdefault(key, []).append(j)
        for key, js in by_pool.items():
            pool = targets[js[0]].pool if key else None
            # device shards: pages registered under the doc id in the shard's
            # pool (the store owns them); bytes shards: a temporary owned page
            kvs = doc_prefill_batch(model, toks[js], [chunk[j].id for j in js], path=path,
                                    pool=pool, register=bool(key))
            for j, kv in zip(js, kvs):
                d, b = chunk[j], targets[j]
                if key:
                    b.put_from_device([d.id], [kv.kv.slot])
                    n = HEADER.size + len(d.id.encode()) + payload_nbytes(
                        cfg.layers, cfg.kv_heads, lay.document_len, cfg.head_dim, scheme)
                else:
                    data = encode_entry(kv, scheme)
                    store.put_entry(d.id, index.centroid_of(d.id), data)
                    kv.kv.lease.release()
                    n = len(data)
                total += n
                if on_entry is not None:
                    on_entry(d.id, n)
    return total


def select(scored: list[ScoredPair], keep_m: int) -> list[ScoredPair]:
    """Host form of _select (pipeline.py:285-287)."""
    return sorted(scored, key=lambda p: (-p.score, p.chunk_id))[:keep_m]
