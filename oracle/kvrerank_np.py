"""numpy restatement of the reference's rerank hot path (TEST INFRASTRUCTURE).

Every function cites the reference code it restates
(paths relative to ``/root/reference/pkg/src/kvrerank/``).  The restatement
is written independently: attention is computed over the concatenated
``[past | current]`` key set instead of the reference's two pieces, which
changes only float32 summation order (<=1e-6 relative, pinned by
``tests/test_oracle.py`` against vectors produced by the reference itself).

Never imported by the product package; see ``oracle/__init__.py``.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

_M64 = (1 << 64) - 1
_EPS = np.float32(1e-6)                      # model.py:33
_GELU_A = np.float32(math.sqrt(2.0 / math.pi))  # model.py:34
_GELU_B = np.float32(0.044715)               # model.py:35


# --------------------------------------------------------------------------
# a1: deterministic weights  (hashing.py:23-31, 58-80; model.py:123-183)

def fnv1a64(data) -> int:
    """FNV-1a 64 over UTF-8 bytes (hashing.py:23-31)."""
    if isinstance(data, str):
        data = data.encode("utf-8")
    h = 0xCBF29CE484222325
    for byte in data:
        h = ((h ^ byte) * 0x100000001B3) & _M64
    return h


def splitmix64_array(seed: int, count: int) -> np.ndarray:
    """Outputs 1..count of the counter-based SplitMix64 stream (hashing.py:58-69)."""
    state = np.uint64(seed & _M64) + np.arange(1, count + 1, dtype=np.uint64) \
        * np.uint64(0x9E3779B97F4A7C15)
    state ^= state >> np.uint64(30)
    state *= np.uint64(0xBF58476D1CE4E5B9)
    state ^= state >> np.uint64(27)
    state *= np.uint64(0x94D049BB133111EB)
    state ^= state >> np.uint64(31)
    return state


def uniform_signed(seed: int, count: int, bound: float) -> np.ndarray:
    """Top 24 bits -> [0,1] in float64 -> [-b, b] -> float32 (hashing.py:72-80)."""
    top = (splitmix64_array(seed, count) >> np.uint64(40)).astype(np.float64)
    unit = top / float((1 << 24) - 1)
    return ((2.0 * unit - 1.0) * bound).astype(np.float32)


def init_tensor(seed: int, name: str, shape) -> np.ndarray:
    """Per-tensor stream seed ^ FNV(name), Xavier bound (model.py:123-129)."""
    fan_in, fan_out = shape[0], shape[-1]
    bound = math.sqrt(6.0 / (fan_in + fan_out))
    n = int(np.prod(shape))
    return uniform_signed(seed ^ fnv1a64(name), n, bound).reshape(shape)


def init_rows(seed: int, name: str, shape, rows) -> np.ndarray:
    """Selected rows of ``init_tensor(seed, name, shape)`` without generating the
    whole stream: SplitMix64 here is counter-based (hashing.py:58-69), so
    element ``i`` is output ``i + 1`` of the stream."""
    fan_in, fan_out = shape[0], shape[-1]
    bound = math.sqrt(6.0 / (fan_in + fan_out))
    rows = np.asarray(rows, np.int64).reshape(-1)
    cols = int(np.prod(shape[1:]))
    s0 = np.uint64((seed ^ fnv1a64(name)) & _M64)
    idx = (rows[:, None] * cols + np.arange(cols)[None, :]).astype(np.uint64) + np.uint64(1)
    with np.errstate(over="ignore"):
        state = s0 + idx * np.uint64(0x9E3779B97F4A7C15)
        state ^= state >> np.uint64(30)
        state *= np.uint64(0xBF58476D1CE4E5B9)
        state ^= state >> np.uint64(27)
        state *= np.uint64(0x94D049BB133111EB)
        state ^= state >> np.uint64(31)
    unit = (state >> np.uint64(40)).astype(np.float64) / float((1 << 24) - 1)
    return ((2.0 * unit - 1.0) * bound).astype(np.float32)


class LazyEmbedding:
    """``token_embedding`` (model.py:169) generated row by row on lookup, so
    wide-vocab configs (C2: 256000 x 2048) need not materialise 2 GB."""

    def __init__(self, seed: int, vocab_size: int, model_dim: int):
        self.seed, self.shape = seed, (vocab_size, model_dim)

    def __getitem__(self, tokens) -> np.ndarray:
        t = np.asarray(tokens, np.int64)
        return init_rows(self.seed, "token_embedding", self.shape, t).reshape(*t.shape, -1)


def score_head(cfg: "OracleConfig") -> np.ndarray:
    """d-vector score head, bound sqrt(6/(d+1)) (reranker.py:121-129)."""
    bound = math.sqrt(6.0 / (cfg.model_dim + 1))
    return uniform_signed(cfg.seed ^ fnv1a64("score_head"), cfg.model_dim, bound)


def rope_tables(base: float, head_dim: int, max_position: int):
    """float64 angle table cast to f32 cos/sin (model.py:138-147)."""
    half = np.arange(0, head_dim, 2, dtype=np.float64) / head_dim
    inv = base ** (-half)
    ang = np.outer(np.arange(max_position, dtype=np.float64), inv)
    return np.cos(ang).astype(np.float32), np.sin(ang).astype(np.float32)


@dataclass(frozen=True)
class OracleConfig:
    """Mirror of ModelConfig (model.py:38-67) plus the layout (reranker.py:32-46)."""
    layers: int = 4
    model_dim: int = 128
    heads: int = 8
    kv_heads: int = 2
    head_dim: int = 16
    vocab_size: int = 32768
    rope_base: float = 10000.0
    max_position: int = 1024
    seed: int = 0
    document_len: int = 256
    query_len: int = 48
    # architecture variants (not in the reference -- defaults
    # are the reference model): gated MLP kind and width, Gemma embedding
    # scale, softmax scale on q.k
    mlp: str = "gelu"
    ffn_dim: int = 0
    embed_scale: float = 1.0
    attn_scale: float = 1.0

    @property
    def group(self) -> int:
        return self.heads // self.kv_heads

    @property
    def ffn(self) -> int:
        return self.ffn_dim or 4 * self.model_dim


@dataclass
class OracleWeights:
    cfg: OracleConfig
    emb: np.ndarray                 # [V, d] f32
    wqkv: list                      # per layer [d, (H+2KVH)HD]   (x @ W orientation)
    wo: list                        # per layer [H*HD, d]
    w_up: list                      # per layer [d, F]   (F = 4d for the reference)
    w_down: list                    # per layer [F, d]
    attn_gain: list
    mlp_gain: list
    final_gain: np.ndarray
    cos: np.ndarray                 # [max_position, HD/2]
    sin: np.ndarray
    head: np.ndarray                # [d] score head
    w_gate: list | None = None      # per layer [d, F] (gated-MLP variants only)


def init_weights(cfg: OracleConfig, layers=None, with_embedding=True,
                 lazy_embedding=False) -> OracleWeights:
    """Same tensors, names and order as init_weights (model.py:150-183).

    ``layers`` restricts generation to a subset of layer indices (others are
    None) so per-layer CPU timing does not have to build a whole 7B model.
    """
    d, h, kvh, hd = cfg.model_dim, cfg.heads, cfg.kv_heads, cfg.head_dim
    idx = range(cfg.layers) if layers is None else layers
    wqkv, wo, up, down, gate = ([None] * cfg.layers for _ in range(5))
    F = cfg.ffn
    for i in idx:
        p = f"layers.{i}"
        wqkv[i] = np.concatenate([init_tensor(cfg.seed, f"{p}.attn.wq", (d, h * hd)),
                                  init_tensor(cfg.seed, f"{p}.attn.wk", (d, kvh * hd)),
                                  init_tensor(cfg.seed, f"{p}.attn.wv", (d, kvh * hd))],
                                 axis=1)
        wo[i] = init_tensor(cfg.seed, f"{p}.attn.wo", (h * hd, d))
        up[i] = init_tensor(cfg.seed, f"{p}.mlp.w_up", (d, F))
        down[i] = init_tensor(cfg.seed, f"{p}.mlp.w_down", (F, d))
        if cfg.mlp != "gelu":
            gate[i] = init_tensor(cfg.seed, f"{p}.mlp.w_gate", (d, F))
    ones = [np.ones(d, np.float32) for _ in range(cfg.layers)]
    if lazy_embedding:
        emb = LazyEmbedding(cfg.seed, cfg.vocab_size, d)
    else:
        emb = (init_tensor(cfg.seed, "token_embedding", (cfg.vocab_size, d))
               if with_embedding else None)
    cos, sin = rope_tables(cfg.rope_base, hd, cfg.max_position)
    return OracleWeights(cfg, emb, wqkv, wo, up, down, ones, list(ones),
                         np.ones(d, np.float32), cos, sin, score_head(cfg),
                         gate if cfg.mlp != "gelu" else None)


def round_weights(w: OracleWeights, dtype=np.float16) -> OracleWeights:
    """Round the GEMM operands through a 16-bit type (what the f16 device path
    multiplies with) so 16-bit parity compares activation rounding only."""
    r = lambda ms: [None if m is None else m.astype(dtype).astype(np.float32) for m in ms]
    return OracleWeights(w.cfg, w.emb, r(w.wqkv), r(w.wo), r(w.w_up), r(w.w_down),
                         w.attn_gain, w.mlp_gain, w.final_gain, w.cos, w.sin, w.head,
                         None if w.w_gate is None else r(w.w_gate))


# --------------------------------------------------------------------------
# a5-a10: forward  (model.py:332-446)

def _rms(x: np.ndarray, gain: np.ndarray) -> np.ndarray:
    """x * 1/sqrt(mean(x^2)+eps) * gain, f32 (model.py:439-441)."""
    ms = (x * x).mean(axis=-1, keepdims=True, dtype=np.float32)
    return x * (np.float32(1.0) / np.sqrt(ms + _EPS)) * gain


def _gelu(x: np.ndarray) -> np.ndarray:
    """tanh GELU (model.py:444-446)."""
    return np.float32(0.5) * x * (np.float32(1.0) + np.tanh(_GELU_A * (x + _GELU_B * x * x * x)))


def _mlp(w: OracleWeights, li: int, xn: np.ndarray) -> np.ndarray:
    """Reference MLP gelu(xn W_up) W_down (model.py:399-400); the gated
    variants (f4) use act(xn W_gate) * (xn W_up) with act = gelu (GeGLU) or
    silu (SwiGLU), as in Gemma / Mistral."""
    kind = w.cfg.mlp
    if kind == "gelu":
        return _gelu(xn @ w.w_up[li]) @ w.w_down[li]
    g = xn @ w.w_gate[li]
    act = _gelu(g) if kind == "geglu" else g / (np.float32(1.0) + np.exp(-g))
    return (act * (xn @ w.w_up[li])) @ w.w_down[li]


def _rotate(x: np.ndarray, cos: np.ndarray, sin: np.ndarray) -> np.ndarray:
    """Interleaved (GPT-J) rotary: pair (2i, 2i+1) times cos+i*sin (model.py:144,370-371).

    x: [T, heads, HD]; cos/sin: [T, HD/2]."""
    a, b = x[..., 0::2], x[..., 1::2]
    c, s = cos[:, None, :], sin[:, None, :]
    out = np.empty_like(x)
    out[..., 0::2] = a * c - b * s
    out[..., 1::2] = a * s + b * c
    return out


def forward(w: OracleWeights, tokens, positions, past_k=None, past_v=None, valid=None,
            layer_range=None, x_in=None, capture=None, return_residual=False):
    """Restates ``forward`` (model.py:332-403).

    past_k/past_v: [L, KVH, P, HD] f32 (RoPE already applied) or None.
    valid: bool[P+T] or None.  Returns (hidden [T,d] final-normed, new_k, new_v).
    ``layer_range``/``x_in``/``capture`` expose the residual stream for
    teacher-forced per-layer checks (capture[li] = layer input);
    ``return_residual`` returns the raw residual instead of the final norm.
    """
    cfg = w.cfg
    tokens = np.asarray(tokens, np.int64)
    positions = np.asarray(positions, np.int64)
    T = tokens.size
    P = 0 if past_k is None else past_k.shape[2]
    valid = np.ones(P + T, bool) if valid is None else np.asarray(valid, bool)
    H, KVH, HD, d, G = cfg.heads, cfg.kv_heads, cfg.head_dim, cfg.model_dim, cfg.group
    L = cfg.layers
    if not valid.any():                                   # model.py:339-340 / 226-232
        z = np.zeros((L, KVH, T, HD), np.float32)
        return np.zeros((T, d), np.float32), z, z.copy()

    cos, sin = w.cos[positions], w.sin[positions]
    # key visibility [T, P+T]: key valid, and for the current block j <= i (model.py:346-387)
    vis = np.broadcast_to(valid[None, :], (T, P + T)).copy()
    vis[:, P:] &= np.tri(T, dtype=bool)
    bias = np.where(vis, np.float32(0.0), np.float32(-np.inf))

    x = np.asarray(w.emb[tokens], np.float32) if x_in is None else x_in.astype(np.float32)
    if x_in is None and cfg.embed_scale != 1.0:
        x = x * np.float32(cfg.embed_scale)
    new_k = np.zeros((L, KVH, T, HD), np.float32)
    new_v = np.zeros_like(new_k)
    layers = range(L) if layer_range is None else layer_range
    for li in layers:
        if capture is not None:
            capture[li] = x.copy()
        xn = _rms(x, w.attn_gain[li])
        qkv = xn @ w.wqkv[li]
        qp = qkv[:, :H * HD]
        if cfg.attn_scale != 1.0:                        # variant: scaled q.k
            qp = qp * np.float32(cfg.attn_scale)
        q = _rotate(qp.reshape(T, H, HD), cos, sin)
        k = _rotate(qkv[:, H * HD:(H + KVH) * HD].reshape(T, KVH, HD), cos, sin)
        v = qkv[:, (H + KVH) * HD:].reshape(T, KVH, HD)
        new_k[li] = k.transpose(1, 0, 2)
        new_v[li] = v.transpose(1, 0, 2)
        out = np.empty((T, H, HD), np.float32)
        for kh in range(KVH):
            keys, vals = new_k[li, kh], new_v[li, kh]
            if P:
                keys = np.concatenate([past_k[li, kh], keys], axis=0)
                vals = np.concatenate([past_v[li, kh], vals], axis=0)
            # query head h -> kv head h // G (model.py:377); no 1/sqrt(HD) (model.py:380,383)
            qh = q[:, kh * G:(kh + 1) * G, :]                     # [T, G, HD]
            logits = np.einsum("tgc,jc->gtj", qh, keys) + bias[None]
            m = logits.max(axis=-1, keepdims=True)
            m = np.where(np.isfinite(m), m, np.float32(0.0))      # model.py:425-426
            e = np.exp(logits - m)
            z = e.sum(axis=-1, keepdims=True)
            z = np.where(z == 0.0, np.float32(1.0), z)            # model.py:434-435
            o = np.einsum("gtj,jc->gtc", e, vals) / z              # (P V)/z, model.py:391-394
            out[:, kh * G:(kh + 1) * G, :] = o.transpose(1, 0, 2)
        x = x + out.reshape(T, H * HD) @ w.wo[li]                  # model.py:395-397
        x = x + _mlp(w, li, _rms(x, w.mlp_gain[li]))                # model.py:399-400
    return (x if return_residual else _rms(x, w.final_gain)), new_k, new_v


# --------------------------------------------------------------------------
# a4, a10, a11: reranker entry points  (reranker.py:154-300)

def doc_prefill(w: OracleWeights, doc_tokens):
    """(keys, values, valid_len) for one document (reranker.py:182-201)."""
    doc_tokens = np.asarray(doc_tokens, np.int64)
    valid = doc_tokens != 0
    _, k, v = forward(w, doc_tokens, np.arange(doc_tokens.size), valid=valid)
    return k, v, int(valid.sum())


def score_reuse(w: OracleWeights, keys, values, valid_len: int, query_tokens) -> float:
    """Suffix on top of cached doc KV; last valid row . score_head (reranker.py:204-212, 236-262)."""
    D = keys.shape[2]
    q = np.asarray(query_tokens, np.int64)
    qvalid = q != 0
    valid = np.concatenate([np.arange(D) < valid_len, qvalid])
    hidden, _, _ = forward(w, q, np.arange(D, D + q.size), keys, values, valid)
    last = int(np.nonzero(qvalid)[0][-1])
    return float(np.dot(hidden[last], w.head))


def score_full(w: OracleWeights, doc_tokens, query_tokens) -> float:
    """Full recompute = prefill + suffix (reranker.py:215-233)."""
    k, v, vl = doc_prefill(w, doc_tokens)
    return score_reuse(w, k, v, vl, query_tokens)


def pair_count(valid: np.ndarray, row_start: int) -> int:
    """Unmasked causal pairs among valid positions for rows >= row_start (reranker.py:293-300)."""
    valid = np.asarray(valid, bool)
    csum = np.cumsum(valid, dtype=np.int64)
    return int(csum[row_start:][valid[row_start:]].sum())


def select_topk(scores, chunk_ids, keep: int):
    """Sort by (-score, chunk_id) and keep the first ``keep`` (pipeline.py:285-287)."""
    order = sorted(range(len(scores)), key=lambda i: (-scores[i], chunk_ids[i]))
    return [order[i] for i in range(min(keep, len(order)))]
