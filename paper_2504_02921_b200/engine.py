"""Batched device execution of the rerank hot path through the C ABI.

The reference scores one pair per forward call (reranker.py:280-289) and
re-streams every weight per pair.  Here every candidate pair's query suffix
is stacked into one M dimension (rows = pairs x query_len) and the whole
layer stack runs once per batch inside krr_forward (C++), with per-pair
prefix KV read straight from pool slots.
"""

from __future__ import annotations

import ctypes as C
import threading

import numpy as np

from . import _lib
from .errors import ConfigError
from .kvpool import CodePages, KVPool, to_device
from .model import DeviceWeights

DEFAULT_WORKSPACE_BUDGET = 32 << 30  # bytes of activations per krr_forward call
# Suffix rows per scoring pass.  Large batches are scored in passes of about
# this many rows: measured on the C3 step, passes of 32k rows run 1.5% faster
# than one 307k-row pass (the power-capped clock is higher; the extra weight
# streaming is ~7 ms per pass-boundary against a 3.1 s step;
# profiles/r02_chunk_ab.txt).
SCORE_ROWS_PER_PASS = 32768   # cap; passes are balanced (_balanced_step)
# Document rows per prefill pass (same reasoning; 64 documents of 512 tokens)
PREFILL_ROWS_PER_PASS = 32768

# The reference calls score_* from several rerank worker threads at once
# (pipeline.py:375-379, 488-504).  Device scratch (workspace,
# suffix KV) is shared per device, so device passes are serialised per device;
# the GPU executes them back to back anyway.
_DEVICE_LOCKS: dict = {}
_LOCKS_GUARD = threading.Lock()


def device_lock(device) -> threading.RLock:
    with _LOCKS_GUARD:
        return _DEVICE_LOCKS.setdefault(str(device), threading.RLock())


class _Workspace:
    def __init__(self):
        self.buf = None

    def get(self, nbytes: int, device):
        import torch
        if self.buf is None or self.buf.numel() < nbytes or self.buf.device != device:
            grow = self.buf is not None
            self.buf = None
            if grow:
                # hand the old block back to the driver first: with a pool filling
                # most of HBM (C4) the cached block cannot be split to fit the
                # larger request, and both do not fit at once
                torch.cuda.empty_cache()
            self.buf = torch.empty(max(nbytes, 1 << 20), dtype=torch.uint8, device=device)
        return self.buf


_WS: dict = {}


def _workspace(device):
    return _WS.setdefault(str(device), _Workspace())


def workspace_bytes(w: DeviceWeights, rows: int) -> int:
    out = C.c_size_t()
    _lib.check(_lib.lib().krr_workspace_bytes(C.byref(w.struct()), rows, C.byref(out)))
    return out.value


def rows_budget(w: DeviceWeights, budget: int | None = None) -> int:
    """Rows per krr_forward call: at most DEFAULT_WORKSPACE_BUDGET of
    activations, and no more than ~80% of what is free on the device (plus the
    workspace already held), so a pool that fills most of the 180 GB HBM
    (C4: 2,500 x 67 MB pages per GPU) still runs in smaller chunks."""
    import torch
    if budget is None:
        free, _ = torch.cuda.mem_get_info(w.device)
        held = _workspace(w.device).buf
        held = held.numel() if held is not None else 0
        budget = min(DEFAULT_WORKSPACE_BUDGET, int(0.8 * (free + held)))
    per_row = workspace_bytes(w, 1 << 16) / float(1 << 16)
    return max(1, int(budget // per_row))


def _ptr(t):
    return 0 if t is None else t.data_ptr()


def _extent(t):
    """(base pointer, bytes) of the allocation a KV pointer table points into."""
    if t is None:
        return 0, 0
    return t.data_ptr(), t.numel() * t.element_size()


def run_forward(w: DeviceWeights, tokens, tok_valid, pos0: int, prefix_len: int,
                prefix_valid, prefix_ptrs, cur_ptrs, cur_kv_layers: int, last_index=None,
                scores=None, stream=None, prefix_pool=None, cur_pool=None, x_in=None,
                x_out=None, ws: "_Workspace | None" = None, positions=None,
                prefix_bits: int = 0, prefix_scales=None) -> None:
    """One krr_forward call over n sequences (all device tensors, contiguous):
    tokens int32 [n, T], tok_valid uint8 [n, T], prefix_valid int32 [n],
    prefix_ptrs / cur_ptrs int64 [n], last_index int32 [n], scores f32 [n].
    ``prefix_pool`` / ``cur_pool`` are the tensors those pointers point into
    (pool slab, suffix scratch); they let attention address pages via TMA.
    ``prefix_bits`` 8 / 4: the prefix pages are HRKV INT8 / INT4 codes with f32
    ``prefix_scales`` (kvpool.CodePages), dequantised inside attention."""
    import torch
    n, T = tokens.shape
    if n == 0:
        return
    rows = n * T
    need = workspace_bytes(w, rows)
    ws = (ws or _workspace(w.device)).get(need, w.device)
    pp, pb = _extent(prefix_pool)
    cp, cb = _extent(cur_pool)
    b = _lib.Batch(n, T, pos0, prefix_len, cur_kv_layers, _ptr(tokens), _ptr(tok_valid),
                   _ptr(prefix_valid), _ptr(prefix_ptrs), _ptr(cur_ptrs), _ptr(last_index),
                   _ptr(scores), pp, pb, cp, cb, _ptr(x_in), _ptr(x_out), _ptr(positions),
                   prefix_bits, _ptr(prefix_scales))
    if stream is None:
        stream = torch.cuda.current_stream(w.device).cuda_stream
    _lib.check(_lib.lib().krr_forward(C.byref(w.struct()), C.byref(b), ws.data_ptr(),
                                      ws.numel(), stream))


def prefill_slots(w: DeviceWeights, pool: KVPool, slots, doc_tokens, valid_len,
                  max_rows: int | None = None) -> None:
    """Document prefill (reranker.py:182-201) of n docs straight into pool
    slots: positions [0, D), pad rows computed and kept, K/V written by the
    QKV epilogue into the slot pages."""
    with device_lock(w.device):
        _prefill_slots(w, pool, slots, doc_tokens, valid_len, max_rows)


def _balanced_step(n: int, cap: int) -> int:
    """Pass size for n units with at most cap per pass, spread evenly over the
    minimum number of passes (C3: 10 passes of 640 pairs rather than 9 of 682 plus
    a 262-pair tail that would fall below the CTA-pair GEMM geometry's 16k rows)."""
    passes = -(-n // cap) if n > 0 else 1
    return max(1, -(-n // passes))


def _prefill_slots(w, pool, slots, doc_tokens, valid_len, max_rows):
    import torch
    if pool.code != w.code:
        raise ConfigError(f"pool dtype {pool.dtype} != weights dtype {w.dtype}")
    dev = w.device
    D = pool.document_len
    tok = to_device(np.asarray(doc_tokens), dev).to(torch.int32).reshape(-1, D)
    n = tok.shape[0]
    valid = (tok != 0).to(torch.uint8)
    slots_t = (slots if isinstance(slots, torch.Tensor) else
               to_device(np.asarray(slots, dtype=np.int64), dev)).to(dev).to(torch.int64)
    ptrs = pool.slot_ptrs(slots_t)
    step = _balanced_step(n, max(1, (max_rows or min(rows_budget(w), PREFILL_ROWS_PER_PASS)) // D))
    for i in range(0, n, step):
        j = min(n, i + step)
        run_forward(w, tok[i:j].contiguous(), valid[i:j].contiguous(), 0, 0, None, None,
                    ptrs[i:j].contiguous(), w.config.layers, cur_pool=pool.slab)
    pool.set_valid_len(np.asarray(slots), np.asarray(valid_len))


class SuffixScratch:
    """Per-layer suffix K/V scratch ([n][1][2][KVH][Q][HD]), reused across layers."""

    def __init__(self):
        self.buf = None

    def ptrs(self, w: DeviceWeights, n: int, Q: int):
        import torch
        cfg = w.config
        shape = (n, 1, 2, cfg.kv_heads, Q, cfg.head_dim)
        need = int(np.prod(shape))
        tdt = w.wqkv[0].dtype
        if self.buf is None or self.buf.numel() < need or self.buf.dtype != tdt:
            self.buf = torch.empty(need, dtype=tdt, device=w.device)
        per = need // n * self.buf.element_size()
        return torch.arange(n, device=w.device, dtype=torch.int64) * per + self.buf.data_ptr()

    def extent(self):
        return self.buf


_SCRATCH: dict = {}


def score_slots(w: DeviceWeights, pool: KVPool, slots, q_tokens, q_valid=None, last_index=None,
                max_rows: int | None = None, out=None, ws=None, scratch=None):
    """Score pairs (pool slot, query tokens) on the device; returns f32 [n] on device.

    slots int [n] (host or device), q_tokens int [n, Q] (host or device).
    ``ws`` / ``scratch``: private workspace / suffix scratch (a CUDA graph's);
    default the per-device shared ones."""
    with device_lock(w.device):
        return _score_slots(w, pool, slots, q_tokens, q_valid, last_index, max_rows, out, ws,
                            scratch)


def _score_slots(w, pool, slots, q_tokens, q_valid, last_index, max_rows, out, ws=None,
                 scratch=None):
    import torch
    if pool.code != w.code:
        raise ConfigError(f"pool dtype {pool.dtype} != weights dtype {w.dtype}")
    dev = w.device
    q = q_tokens if isinstance(q_tokens, torch.Tensor) else to_device(
        np.asarray(q_tokens), dev)
    q = q.to(dev)
    if q.dtype != torch.int32:
        q = q.to(torch.int32)
    n, Q = q.shape
    if q_valid is None:
        q_valid = (q != 0).to(torch.uint8)
    if last_index is None:
        ar = torch.arange(Q, device=dev, dtype=torch.int32)
        last_index = torch.where(q_valid.bool(), ar, torch.full_like(ar, -1)).max(dim=1).values
        last_index = last_index.to(torch.int32)
    slots_t = (slots if isinstance(slots, torch.Tensor) else to_device(
        np.asarray(slots, dtype=np.int64), dev)).to(dev).to(torch.int64)
    scores = out if out is not None else torch.empty(n, dtype=torch.float32, device=dev)
    # Pairs that share a document are made adjacent (stable sort by slot) so the
    # attention kernel attends all of a document's queries as one row group and
    # streams its K/V once (krr_forward's item table); scores are scattered
    # back to pair order.  Per-pair results do not depend on the grouping.
    order = None
    if n > 1:
        if isinstance(slots, torch.Tensor):
            slots_t, order = torch.sort(slots_t, stable=True)
        else:
            o = np.argsort(np.asarray(slots), kind="stable")
            if (o != np.arange(n)).any():
                order = to_device(o, dev)
                slots_t = slots_t.index_select(0, order)
    if order is not None:
        q, q_valid, last_index = (t.index_select(0, order) for t in (q, q_valid, last_index))
        final, scores = scores, torch.empty(n, dtype=torch.float32, device=dev)
    prefix_ptrs = pool.slot_ptrs(slots_t)
    prefix_valid = pool.valid_len[slots_t]
    step = _balanced_step(n, max(1, (max_rows or min(rows_budget(w), SCORE_ROWS_PER_PASS)) // Q))
    scratch = scratch or _SCRATCH.setdefault(str(dev), SuffixScratch())
    D = pool.document_len
    for i in range(0, n, step):
        j = min(n, i + step)
        cur = scratch.ptrs(w, j - i, Q)
        run_forward(w, q[i:j].contiguous(), q_valid[i:j].contiguous(), D, D,
                    prefix_valid[i:j].contiguous(), prefix_ptrs[i:j].contiguous(), cur, 1,
                    last_index[i:j].contiguous(), scores[i:j], prefix_pool=pool.slab,
                    cur_pool=scratch.extent(), ws=ws, prefix_bits=getattr(pool, "bits", 0),
                    prefix_scales=getattr(pool, "scales", None))
    if order is not None:
        final.index_copy_(0, order, scores)
        return final
    return scores


def segmented_topk(scores, doc_ids, n_seg: int, seg_len: int, k: int):
    """Per-segment top-k by (score desc, doc id asc) on the device.
    Returns (idx int32 [n_seg, k], score f32 [n_seg, k]) device tensors."""
    import torch
    dev = scores.device
    idx = torch.empty((n_seg, k), dtype=torch.int32, device=dev)
    sc = torch.empty((n_seg, k), dtype=torch.float32, device=dev)
    ids = doc_ids if isinstance(doc_ids, torch.Tensor) else to_device(
        np.asarray(doc_ids), dev)
    ids = ids.to(torch.int32).contiguous()
    stream = torch.cuda.current_stream(dev).cuda_stream
    _lib.check(_lib.lib().krr_segmented_topk(scores.contiguous().data_ptr(), ids.data_ptr(),
                                             n_seg, seg_len, k, idx.data_ptr(), sc.data_ptr(),
                                             stream))
    return idx, sc


def fused_dequant_supported(w: DeviceWeights) -> bool:
    """INT8/INT4 prefix pages can be dequantised inside attention (the tcgen05
    TMEM-P kernel: head_dim 64|128, 16-bit activations)."""
    return (w.code in (_lib.F16, _lib.BF16) and w.config.head_dim in (64, 128) and
            w.attn_backend in (_lib.ATTN_AUTO, _lib.ATTN_TCGEN05))


def score_host_tier(w: DeviceWeights, tier, staging: KVPool, host_slots, q_tokens,
                    copy_stream=None, max_rows: int | None = None):
    """Score pairs whose document KV lives in the pinned host tier (the paper's
    SSD/DRAM tier).

    Distinct documents are streamed H2D (cudaMemcpyAsync on ``copy_stream``)
    into one half of a double-buffered HBM staging pool while the main stream
    scores every pair of the previously landed half; events order the reuse of
    each half.  A quantised tier lands HRKV codes + scales and the attention
    kernel dequantises them in shared memory (no expand pass, the
    staging pool's 16-bit slots stay unused) where it can (head_dim 64|128,
    16-bit activations), else they are expanded into the staging slots first.
    Each document crosses PCIe once per call however many pairs reference it.
    Returns f32 [n] scores on the device (pair order)."""
    import torch
    if staging.code != w.code:
        raise ConfigError(f"staging dtype {staging.dtype} != weights dtype {w.dtype}")
    dev = w.device
    hs = np.asarray(host_slots, dtype=np.int64)
    q = to_device(np.asarray(q_tokens), dev).to(torch.int32)
    n = hs.size
    scores = torch.empty(n, dtype=torch.float32, device=dev)
    if n == 0:
        return scores
    half = staging.capacity // 2
    if half < 1:
        raise ConfigError("host-tier staging pool needs >= 2 slots")
    if len(staging):
        raise ConfigError("host-tier staging pool must be dedicated (empty)")
    st_slots = np.arange(staging.capacity, dtype=np.int64)
    fused = tier.quant is not None and fused_dequant_supported(w)
    pages = CodePages(tier, staging) if fused else staging
    docs = np.unique(hs)
    groups = [docs[i:i + half] for i in range(0, docs.size, half)]
    main = torch.cuda.current_stream(dev)
    cs = copy_stream or torch.cuda.Stream(device=dev)
    ready = [torch.cuda.Event() for _ in range(2)]
    free = [torch.cuda.Event() for _ in range(2)]

    def slots_of(gi):
        b = gi & 1
        return st_slots[b * half:b * half + groups[gi].size]

    def issue_copy(gi):
        b = gi & 1
        with torch.cuda.stream(cs):
            if gi >= 2:
                cs.wait_event(free[b])
            for h, s in zip(groups[gi], slots_of(gi)):
                tier.h2d(int(h), staging, int(s), int(s))
            ready[b].record(cs)

    # both halves' transfers are queued before any scoring is, so the host
    # thread enqueueing a group's layers never delays the next transfer
    for gi in range(min(2, len(groups))):
        issue_copy(gi)
    for gi, grp in enumerate(groups):
        b = gi & 1
        slots = slots_of(gi)
        main.wait_event(ready[b])
        # a quantised tier expands on the main stream, keeping the copy stream
        # (and the PCIe link) busy with the next group's transfers
        if not fused:
            for s in slots:
                tier.expand(staging, int(s), int(s))
        staging.set_valid_len(slots, tier.valid_len[grp])
        slot_of = dict(zip(grp.tolist(), slots.tolist()))
        sel = np.nonzero(np.isin(hs, grp))[0]
        sel_t = to_device(sel, dev)
        sc = score_slots(w, pages, np.array([slot_of[h] for h in hs[sel]]),
                         q.index_select(0, sel_t), max_rows=max_rows)
        scores[sel_t] = sc
        free[b].record(main)
        if gi + 2 < len(groups):
            issue_copy(gi + 2)
    return scores


def layer_slice(w: DeviceWeights, l0: int, l1: int):
    """krr_model_t covering layers [l0, l1) only (layer-split execution with
    krr_batch_t.x_in / x_out).  KV pointers passed with it must be advanced to
    layer l0 (``layer_offset_bytes``)."""
    base = w.struct()
    cfg = w.config
    if not (0 <= l0 < l1 <= cfg.layers):
        raise ConfigError(f"bad layer range [{l0}, {l1})")
    arr = lambda ts: (C.c_void_p * (l1 - l0))(*[t.data_ptr() for t in ts[l0:l1]])
    keep = [arr(w.attn_gain), arr(w.mlp_gain), arr(w.wqkv), arr(w.wo), arr(w.w_up),
            arr(w.w_down)]
    m = _lib.Model(l1 - l0, cfg.model_dim, cfg.heads, cfg.kv_heads, cfg.head_dim,
                   cfg.vocab_size, cfg.max_position, w.code, w.gemm_backend, w.attn_backend,
                   base.token_embedding, base.rope_cos, base.rope_sin, base.final_gain,
                   base.score_head, *[C.cast(a, C.c_void_p) for a in keep], *w.variant_fields())
    m._keep = keep
    return m


def layer_offset_bytes(w: DeviceWeights, kv_len: int, layers: int) -> int:
    """Byte offset of layer ``layers`` inside a [L][2][KVH][kv_len][HD] KV slab."""
    cfg = w.config
    es = 4 if w.code == _lib.F32 else 2
    return layers * 2 * cfg.kv_heads * kv_len * cfg.head_dim * es


def run_layers(w: DeviceWeights, l0: int, l1: int, tokens, tok_valid, pos0: int,
               prefix_len: int, prefix_valid, prefix_ptrs, cur_ptrs, cur_kv_layers: int,
               x_in=None, x_out=None, prefix_pool=None, cur_pool=None) -> None:
    """krr_forward over layers [l0, l1) with the residual stream taken from
    ``x_in`` (or the embedding when None) and written to ``x_out``.  Pointer
    tables address layer 0 of each slab; they are advanced to l0 here."""
    import torch
    n, T = tokens.shape
    m = layer_slice(w, l0, l1)
    off_p = layer_offset_bytes(w, prefix_len, l0) if prefix_len else 0
    off_c = layer_offset_bytes(w, T, l0) if cur_kv_layers > 1 else 0
    pre = (prefix_ptrs + off_p).contiguous() if prefix_ptrs is not None else None
    cur = (cur_ptrs + off_c).contiguous()
    ckl = (l1 - l0) if cur_kv_layers > 1 else 1
    rows = n * T
    out = C.c_size_t()
    _lib.check(_lib.lib().krr_workspace_bytes(C.byref(m), rows, C.byref(out)))
    ws = _workspace(w.device).get(out.value, w.device)
    pp, pb = _extent(prefix_pool)
    cp, cb = _extent(cur_pool)
    b = _lib.Batch(n, T, pos0, prefix_len, ckl, _ptr(tokens), _ptr(tok_valid),
                   _ptr(prefix_valid), _ptr(pre), _ptr(cur), 0, 0, pp, pb, cp, cb,
                   _ptr(x_in), _ptr(x_out))
    stream = torch.cuda.current_stream(w.device).cuda_stream
    _lib.check(_lib.lib().krr_forward(C.byref(m), C.byref(b), ws.data_ptr(), ws.numel(), stream))


class GraphedScorer:
    """CUDA-graph replay of one scoring pass (krr_forward over n pairs of query
    length Q + per-query top-k) for a fixed batch shape, for latency-critical
    serving: the ~7 launches per layer and the host-side argument marshalling
    are recorded once; a call is two small H2D copies, one graph launch and a
    D2H of the top-k.  Inputs are copied into static device buffers.

    The graph owns its workspace and suffix scratch (eager calls cannot
    reallocate memory it replays into), replays under the device lock, and is
    re-captured when the pool's slab was re-homed (``KVPool.grow``)."""

    def __init__(self, w: DeviceWeights, pool: KVPool, n_q: int, n_c: int, Q: int, k: int):
        import torch
        self.w, self.pool, self.n_q, self.n_c, self.Q, self.k = w, pool, n_q, n_c, Q, k
        dev = w.device
        n = n_q * n_c
        self.slots = torch.zeros(n, dtype=torch.int64, device=dev)
        self.q = torch.ones((n_q, Q), dtype=torch.int32, device=dev)
        self.ids = torch.arange(n, dtype=torch.int32, device=dev)
        self.qidx = torch.arange(n_q, device=dev).repeat_interleave(n_c)
        self.scores = torch.empty(n, dtype=torch.float32, device=dev)
        self._ws = _Workspace()
        self._scratch = SuffixScratch()
        self.stream = torch.cuda.Stream(device=dev)
        with device_lock(dev):
            self._capture()

    def _capture(self):
        import torch
        dev = self.w.device
        self.stream.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.stream(self.stream):
            for _ in range(2):                    # warm-up: workspace, descriptors, attributes
                self._body()
        torch.cuda.current_stream(dev).wait_stream(self.stream)
        torch.cuda.synchronize(dev)
        self.graph = torch.cuda.CUDAGraph()
        n0 = _lib.launch_count()
        with torch.cuda.graph(self.graph, stream=self.stream):
            self.out_idx, self.out_sc = self._body()
        self.launches = _lib.launch_count() - n0      # this library's kernels per replay
        self._generation = self.pool.generation
        self._slab_ptr = self.pool.slab.data_ptr()

    def _body(self):
        score_slots(self.w, self.pool, self.slots, self.q.index_select(0, self.qidx),
                    out=self.scores, max_rows=self.n_q * self.n_c * self.Q, ws=self._ws,
                    scratch=self._scratch)
        return segmented_topk(self.scores, self.ids, self.n_q, self.n_c, self.k)

    def replay_device(self, slots, q_tokens, doc_ids):
        """Device-resident variant of ``__call__``: slots int64 [n_q*n_c], q_tokens
        int32 [n_q, Q], doc_ids int32 [n_q*n_c] already on the device are copied
        into the static buffers on the current stream; returns the device
        (idx, scores) [n_q, k] the replay writes (valid until the next replay)."""
        import torch
        with device_lock(self.w.device):
            if (self.pool.generation != self._generation or
                    self.pool.slab.data_ptr() != self._slab_ptr):
                self._capture()
            self.slots.copy_(slots)
            self.q.copy_(q_tokens)
            self.ids.copy_(doc_ids)
            self.graph.replay()
            return self.out_idx, self.out_sc

    def __call__(self, slots, q_tokens, doc_ids):
        """slots int [n_q*n_c], q_tokens int [n_q, Q], doc_ids int [n_q*n_c] (host);
        returns (idx, scores) host arrays [n_q, k] (idx = position within the query's
        candidates)."""
        import torch
        with device_lock(self.w.device):
            if (self.pool.generation != self._generation or
                    self.pool.slab.data_ptr() != self._slab_ptr):
                self._capture()
            self.slots.copy_(torch.as_tensor(np.asarray(slots, np.int64)), non_blocking=True)
            self.q.copy_(torch.as_tensor(np.asarray(q_tokens, np.int32)), non_blocking=True)
            self.ids.copy_(torch.as_tensor(np.asarray(doc_ids, np.int32)), non_blocking=True)
            self.graph.replay()
            return self.out_idx.cpu().numpy(), self.out_sc.cpu().numpy()
