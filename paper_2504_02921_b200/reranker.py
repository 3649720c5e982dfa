"""Two-phase relevance scoring — the reference's public API (reranker.py:1-300)
on the B200 engine.

Same names, signatures, validation and errors as the reference:
``tokenize``, ``doc_prefill``, ``score_full``, ``score_reuse``,
``score_batch``, ``DocKV``, ``CounterReport``, ``ScoredPair``.  Differences
are in where things live and how they run:

* a DocKV produced here is a handle to a page in an HBM ``KVPool``
  (``DeviceKV``); ``.kv.keys``/``.kv.values`` materialise host f32 copies on
  demand, so reference-style code that inspects them keeps working;
* ``score_batch`` really batches: all pairs' query suffixes run through the
  layer stack together (one krr_forward per workspace-sized chunk), instead
  of one forward per pair (reranker.py:280-289).  Results are independent of
  grouping because every kernel is batch-invariant.
* ``path``: "fast" = the model's precision on tensor cores (f16 default);
  "reference" = the f32 CUDA-core debug build.  Unknown -> ConfigError.
"""

from __future__ import annotations

import weakref
from dataclasses import dataclass, field

import numpy as np

from . import engine
from .config import PAD_ID, LayoutConfig, ModelConfig
from .errors import ConfigError, DegenerateInputError, ShapeError
from .hashing import fnv1a64
from .kvpool import KVPool
from .model import KVTensorSet, RerankModel

__all__ = ["DocKV", "DeviceKV", "SlotLease", "CounterReport", "ScoredPair", "RerankModel", "LayoutConfig",
           "tokenize", "doc_prefill", "doc_prefill_batch", "score_full", "score_reuse",
           "score_batch", "pool_for"]


class SlotLease:
    """Ownership of one caller-owned KVPool slot: the slot returns to the pool
    when the last reference to the lease (held by a DeviceKV) goes away, so a
    reference-style ``doc_prefill`` loop does not grow the pool without bound."""

    __slots__ = ("pool", "slot", "_fin", "__weakref__")

    def __init__(self, pool: KVPool, slot: int):
        self.pool, self.slot = pool, slot
        self._fin = weakref.finalize(self, pool.free_owned, [slot])

    def release(self) -> None:
        self._fin()


@dataclass(frozen=True)
class DeviceKV:
    """KVTensorSet look-alike for a cache resident in a KVPool slot.

    ``lease`` is set when the DocKV owns its slot (``doc_prefill``); handles
    onto page-table entries (a device store's pages) carry none."""

    pool: KVPool
    slot: int
    position_offset: int = 0
    lease: SlotLease | None = field(default=None, compare=False, repr=False)

    @property
    def token_count(self) -> int:
        return self.pool.document_len

    @property
    def shape(self):
        L, _, KVH, D, HD = self.pool.page_shape
        return (L, KVH, D, HD)

    @property
    def keys(self) -> np.ndarray:
        return self.pool.read_host_kv(self.slot)[0]

    @property
    def values(self) -> np.ndarray:
        return self.pool.read_host_kv(self.slot)[1]

    def to_host(self) -> KVTensorSet:
        k, v = self.pool.read_host_kv(self.slot)
        return KVTensorSet(k, v, 0)

    @property
    def payload_nbytes(self) -> int:
        # the reference's f32 payload size (model.py:93-95), counter parity
        return int(np.prod(self.shape)) * 4 * 2


@dataclass(frozen=True)
class DocKV:
    """A document's fixed-length KV cache plus its non-pad prefix length (reranker.py:49-63)."""

    chunk_id: str
    kv: object  # KVTensorSet (host) or DeviceKV (pool page)
    valid_len: int

    @property
    def document_len(self) -> int:
        return self.kv.token_count

    @property
    def payload_nbytes(self) -> int:
        return self.kv.payload_nbytes


@dataclass
class CounterReport:
    """Work counters (reranker.py:66-86)."""

    linear_token_count: int = 0
    attn_mac_pairs: int = 0
    peak_activation_tokens: int = 0
    kv_bytes_loaded: int = 0

    def merge(self, other: "CounterReport") -> None:
        self.linear_token_count += other.linear_token_count
        self.attn_mac_pairs += other.attn_mac_pairs
        self.peak_activation_tokens = max(self.peak_activation_tokens,
                                          other.peak_activation_tokens)
        self.kv_bytes_loaded += other.kv_bytes_loaded

    def as_dict(self) -> dict:
        return {
            "linear_token_count": self.linear_token_count,
            "attn_mac_pairs": self.attn_mac_pairs,
            "peak_activation_tokens": self.peak_activation_tokens,
            "kv_bytes_loaded": self.kv_bytes_loaded,
        }


@dataclass(frozen=True)
class ScoredPair:
    chunk_id: str
    query_id: str
    score: float


def tokenize(text: str, max_len: int, pad_id: int = PAD_ID,
             vocab_size: int = ModelConfig.vocab_size) -> np.ndarray:
    """Hash words to ids in [1, vocab), truncate, right-pad (reranker.py:132-143)."""
    if max_len < 1:
        raise ConfigError("max_len must be >= 1")
    out = np.full(max_len, pad_id, dtype=np.int64)
    for i, word in enumerate(text.split()[:max_len]):
        out[i] = 1 + fnv1a64(word) % (vocab_size - 1)
    return out


# ------------------------------------------------------------ validation
def _check_vocab(model: RerankModel, tokens: np.ndarray) -> None:
    if tokens.size and (tokens.min() < 0 or tokens.max() >= model.config.vocab_size):
        raise ShapeError("token id out of vocabulary range")


def _doc_valid(model: RerankModel, doc_tokens) -> tuple[np.ndarray, int]:
    """reranker.py:154-167"""
    layout = model.layout
    doc_tokens = np.asarray(doc_tokens)
    if doc_tokens.shape != (layout.document_len,):
        raise ShapeError(
            f"document tokens must have length {layout.document_len}, got {doc_tokens.shape}")
    valid = doc_tokens != layout.pad_id
    valid_len = int(valid.sum())
    if valid_len == 0:
        raise DegenerateInputError("document is entirely padding")
    if not valid[:valid_len].all():
        raise ShapeError("document pads must be trailing (non-pad prefix only)")
    _check_vocab(model, doc_tokens)
    return valid, valid_len


def _query_valid(model: RerankModel, query_tokens) -> np.ndarray:
    """reranker.py:170-179"""
    layout = model.layout
    query_tokens = np.asarray(query_tokens)
    if query_tokens.shape != (layout.query_len,):
        raise ShapeError(
            f"query tokens must have length {layout.query_len}, got {query_tokens.shape}")
    valid = query_tokens != layout.pad_id
    if not valid.any():
        raise DegenerateInputError("query is entirely padding")
    _check_vocab(model, query_tokens)
    return valid


def pair_count(valid: np.ndarray, row_start: int) -> np.ndarray:
    """Unmasked causal pairs among valid positions for rows >= row_start
    (reranker.py:293-300), vectorised over a leading batch axis."""
    valid = np.atleast_2d(np.asarray(valid, dtype=bool))
    csum = np.cumsum(valid, axis=1, dtype=np.int64)
    return (csum[:, row_start:] * valid[:, row_start:]).sum(axis=1)


def _check_path(path: str) -> None:
    if path not in ("fast", "reference"):
        raise ConfigError(f"unknown scoring path {path!r} (use 'fast' or 'reference')")


# ------------------------------------------------------------ pools
def pool_for(model: RerankModel, path: str = "fast", min_free: int = 1) -> KVPool:
    """The model's default HBM pool for a path's precision (grows on demand,
    within the device's free memory)."""
    w = model.weights_for(path)
    pools = model.__dict__.setdefault("_pools", {})
    pool = pools.get(w.dtype)
    if pool is None:
        pool = KVPool(model.config, model.layout.document_len, max(64, min_free), w.dtype,
                      w.device)
        pools[w.dtype] = pool
    short = min_free - pool.free_slots
    if short > 0:
        pool.grow(max(pool.capacity * 2, pool.capacity + short),
                  min_capacity=pool.capacity + short)
    return pool


def _staging_pool(model: RerankModel, path: str, n: int) -> KVPool:
    """Per-model pool for host DocKVs staged into HBM for one scoring call
    (used under the device lock; slots are owned by that call)."""
    w = model.weights_for(path)
    st = model.__dict__.setdefault("_staging", {})
    pool = st.get(w.dtype)
    if pool is None or pool.capacity < n:
        pool = KVPool(model.config, model.layout.document_len, max(n, 16), w.dtype, w.device)
        st[w.dtype] = pool
    return pool


# ------------------------------------------------------------ prefill
def doc_prefill_batch(model: RerankModel, docs_tokens, chunk_ids=None, path: str = "fast",
                      pool: KVPool | None = None, counters: CounterReport | None = None,
                      register: bool = False) -> list[DocKV]:
    """Batched doc_prefill: n documents through one device forward into pool pages.

    By default every DocKV owns a fresh slot (released when the DocKV is
    dropped), so prefilling the same chunk id twice yields two independent
    caches, as in the reference.  ``register=True`` instead writes the pages
    under their chunk ids in the pool's page table (a device store's entries,
    ``populate_store``); ids must then be non-empty and distinct."""
    _check_path(path)
    docs = np.asarray(docs_tokens)
    if docs.ndim != 2:
        raise ShapeError("docs_tokens must be [n, document_len]")
    n = docs.shape[0]
    chunk_ids = list(chunk_ids) if chunk_ids is not None else [""] * n
    if len(chunk_ids) != n:
        raise ShapeError("one chunk id per document")
    if register and (any(not c for c in chunk_ids) or len(set(chunk_ids)) != n):
        raise ConfigError("registered prefill needs distinct, non-empty chunk ids")
    valid_lens = np.empty(n, dtype=np.int64)
    for i in range(n):
        _, valid_lens[i] = _doc_valid(model, docs[i])
    w = model.weights_for(path)
    pool = pool if pool is not None else pool_for(model, path, n)
    if register:
        slots = pool.allocate(chunk_ids)
        leases = [None] * n
    else:
        slots = pool.allocate_owned(n)
        leases = [SlotLease(pool, int(s)) for s in slots]
    try:
        engine.prefill_slots(w, pool, slots, docs, valid_lens)
    except BaseException:
        for le in leases:
            if le is not None:
                le.release()
        raise
    if counters is not None:
        valid = docs != model.layout.pad_id
        counters.merge(CounterReport(
            linear_token_count=int(valid_lens.sum()),
            attn_mac_pairs=int(pair_count(valid, 0).sum()),
            peak_activation_tokens=int(valid_lens.max()) if n else 0))
    return [DocKV(chunk_id=c, kv=DeviceKV(pool, int(s), lease=le), valid_len=int(v))
            for c, s, v, le in zip(chunk_ids, slots, valid_lens, leases)]


def doc_prefill(model: RerankModel, doc_tokens, chunk_id: str = "", path: str = "fast",
                counters: CounterReport | None = None, pool: KVPool | None = None) -> DocKV:
    """Run the document segment alone and keep its fixed-length KV
    (reranker.py:182-201); the cache lands in an HBM pool page."""
    _doc_valid(model, doc_tokens)
    return doc_prefill_batch(model, np.asarray(doc_tokens)[None], [chunk_id], path, pool,
                             counters)[0]


# ------------------------------------------------------------ scoring
def _reuse_counters(model: RerankModel, dvalid_len: np.ndarray, qvalid: np.ndarray,
                    payload: int) -> list[CounterReport]:
    D = model.layout.document_len
    n = qvalid.shape[0]
    dvalid = np.arange(D)[None, :] < dvalid_len[:, None]
    full = np.concatenate([dvalid, qvalid], axis=1)
    macs = pair_count(full, D)
    ql = qvalid.sum(axis=1)
    return [CounterReport(int(ql[i]), int(macs[i]), int(ql[i]), payload) for i in range(n)]


def _full_counters(model: RerankModel, doc_tokens: np.ndarray,
                   qvalid: np.ndarray) -> list[CounterReport]:
    dvalid = doc_tokens != model.layout.pad_id
    full = np.concatenate([dvalid, qvalid], axis=1)
    macs = pair_count(full, 0)
    tot = dvalid.sum(axis=1) + qvalid.sum(axis=1)
    return [CounterReport(int(tot[i]), int(macs[i]), int(tot[i]), 0)
            for i in range(len(tot))]


def _resolve_kv(model: RerankModel, kvs: list[DocKV], path: str):
    """Group DocKVs by the pool that can serve ``path``; host caches or pools
    of another precision are staged into slots of the staging pool owned by
    this call.  Returns (pool, slots) per group, the group index of each pair,
    and the staging slots to free.  Caller holds the device lock."""
    w = model.weights_for(path)
    cfg, layout = model.config, model.layout
    expected = (cfg.layers, cfg.kv_heads, layout.document_len, cfg.head_dim)
    groups: dict[int, tuple[KVPool, list]] = {}
    order = []
    stage = [i for i, d in enumerate(kvs)
             if not (isinstance(d.kv, DeviceKV) and d.kv.pool.code == w.code)]
    staging = _staging_pool(model, path, len(stage)) if stage else None
    st_slots = {}
    taken = np.zeros(0, np.int64)
    if stage:
        taken = staging.allocate_owned(len(stage))
        try:
            for j, i in enumerate(stage):
                d = kvs[i]
                host = d.kv.to_host() if isinstance(d.kv, DeviceKV) else d.kv
                if tuple(host.keys.shape) != expected:
                    raise ShapeError(f"cached KV shape {tuple(host.keys.shape)} does not match "
                                     f"layout/model {expected}")
                staging.write_host_kv(int(taken[j]), host.keys, host.values, d.valid_len)
                st_slots[i] = int(taken[j])
        except BaseException:
            staging.free_owned(taken)
            raise
    for i, d in enumerate(kvs):
        if i in st_slots:
            pool, slot = staging, st_slots[i]
        else:
            pool, slot = d.kv.pool, d.kv.slot
            if pool.host_valid_len(slot) != d.valid_len:
                pool.set_valid_len([slot], [d.valid_len])
        g = groups.setdefault(id(pool), (pool, []))
        order.append((id(pool), len(g[1])))
        g[1].append(slot)
    return groups, order, (staging, taken)


def _validate_kv(model: RerankModel, doc_kv: DocKV) -> None:
    """reranker.py:240-249"""
    layout, cfg = model.layout, model.config
    expected = (cfg.layers, cfg.kv_heads, layout.document_len, cfg.head_dim)
    shape = doc_kv.kv.shape if isinstance(doc_kv.kv, DeviceKV) else doc_kv.kv.keys.shape
    if tuple(shape) != expected:
        raise ShapeError(f"cached KV shape {tuple(shape)} does not match layout/model {expected}")
    if doc_kv.kv.position_offset != 0:
        raise ShapeError("document KV must start at position 0")
    if not (0 < doc_kv.valid_len <= layout.document_len):
        raise ShapeError(f"valid_len {doc_kv.valid_len} out of range")


def score_reuse_many(model: RerankModel, kvs: list[DocKV], queries, path: str = "fast"):
    """Scores of n (DocKV, query) pairs in one batched device run -> (np f32 [n], counters)."""
    _check_path(path)
    q = np.asarray(queries, dtype=np.int64).reshape(len(kvs), -1) if len(kvs) else \
        np.zeros((0, model.layout.query_len), np.int64)
    for d in kvs:
        _validate_kv(model, d)
    qvalid = np.stack([_query_valid(model, row) for row in q]) if len(kvs) else \
        np.zeros((0, model.layout.query_len), bool)
    if not kvs:
        return np.zeros(0, np.float32), []
    w = model.weights_for(path)
    out = np.empty(len(kvs), dtype=np.float32)
    # staging + scoring under one device lock: concurrent callers (the
    # reference's threaded rerank workers) never see each other's staged pages
    with engine.device_lock(w.device):
        groups, order, (staging, taken) = _resolve_kv(model, kvs, path)
        try:
            for key, (pool, slots) in groups.items():
                idx = [i for i, (k, _) in enumerate(order) if k == key]
                sc = engine.score_slots(w, pool, np.asarray(slots), q[idx].astype(np.int32))
                out[idx] = sc.cpu().numpy()
        finally:
            if staging is not None:
                staging.free_owned(taken)
    dvl = np.array([d.valid_len for d in kvs], dtype=np.int64)
    payload = kvs[0].payload_nbytes
    return out, _reuse_counters(model, dvl, qvalid, payload)


def score_reuse(model: RerankModel, doc_kv: DocKV, query_tokens,
                path: str = "fast") -> tuple[float, CounterReport]:
    """Score one pair on top of a cached document KV (reranker.py:236-262)."""
    s, c = score_reuse_many(model, [doc_kv], np.asarray(query_tokens)[None], path)
    return float(s[0]), c[0]


def score_full_many(model: RerankModel, docs, queries, path: str = "fast"):
    """Full recompute for n pairs: batched prefill into a staging pool, then the suffix."""
    _check_path(path)
    docs = np.asarray(docs, dtype=np.int64)
    q = np.asarray(queries, dtype=np.int64)
    n = docs.shape[0]
    if n == 0:
        return np.zeros(0, np.float32), []
    for i in range(n):
        _doc_valid(model, docs[i])
    qvalid = np.stack([_query_valid(model, row) for row in q])
    w = model.weights_for(path)
    staging = KVPool(model.config, model.layout.document_len, n, w.dtype, w.device)
    slots = staging.allocate_owned(n)
    vl = (docs != model.layout.pad_id).sum(axis=1)
    engine.prefill_slots(w, staging, slots, docs, vl)
    sc = engine.score_slots(w, staging, slots, q.astype(np.int32)).cpu().numpy()
    return sc, _full_counters(model, docs, qvalid)


def score_full(model: RerankModel, doc_tokens, query_tokens,
               path: str = "fast") -> tuple[float, CounterReport]:
    """Score a pair from raw tokens, computing the document side in place (reranker.py:215-233)."""
    s, c = score_full_many(model, np.asarray(doc_tokens)[None], np.asarray(query_tokens)[None],
                           path)
    return float(s[0]), c[0]


def score_batch(model: RerankModel, pairs, mode: str, max_batch: int = 8,
                path: str = "fast") -> tuple[list[ScoredPair], CounterReport]:
    """Score (query_id, chunk_id, doc, query_tokens) pairs (reranker.py:265-290).

    ``doc`` is a DocKV in reuse mode and a token array in full mode.  All
    pairs run as one device batch; ``max_batch`` is validated for API parity
    but grouping cannot change results (batch-invariant kernels)."""
    if mode not in ("full", "reuse"):
        raise ConfigError(f"unknown rerank mode {mode!r}")
    if max_batch < 1:
        raise ConfigError("max_batch must be >= 1")
    _check_path(path)
    totals = CounterReport()
    if not pairs:
        return [], totals
    qids = [p[0] for p in pairs]
    cids = [p[1] for p in pairs]
    docs = [p[2] for p in pairs]
    queries = np.stack([np.asarray(p[3]) for p in pairs]) if all(
        np.asarray(p[3]).shape == np.asarray(pairs[0][3]).shape for p in pairs) else None
    if mode == "reuse":
        for d in docs:
            if not isinstance(d, DocKV):
                raise ShapeError("reuse mode requires DocKV entries")
        if queries is None:
            raise ShapeError(f"query tokens must have length {model.layout.query_len}")
        scores, counters = score_reuse_many(model, docs, queries, path)
    else:
        if queries is None:
            raise ShapeError(f"query tokens must have length {model.layout.query_len}")
        try:
            dt = np.stack([np.asarray(d) for d in docs])
        except ValueError:
            raise ShapeError(f"document tokens must have length {model.layout.document_len}")
        scores, counters = score_full_many(model, dt, queries, path)
    results = []
    for i in range(len(pairs)):
        totals.merge(counters[i])
        results.append(ScoredPair(chunk_id=cids[i], query_id=qids[i], score=float(scores[i])))
    return results, totals
