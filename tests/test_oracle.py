"""Pin the CPU oracle (oracle/kvrerank_np.py) to the reference's own outputs.

tests/golden/*.npz were produced by running the reference package
``kvrerank`` 0.1.0 itself (tests/golden/make_golden.py).  These CPU tests
check the numpy restatement against them, so the GPU parity tests that use
the oracle are anchored on the reference, not on a re-derivation:

* weight streams: bit-exact (sha256 of every C1 tensor, SPEC.md:65 value);
* scores: <= 5e-5 of the reference's fast path (f32 summation order only;
  the reference's own fast and reference paths differ by ~1e-5);
* DocKV (keys post-RoPE, values): <= 1e-5 relative;
* counters: exact (closed forms of SPEC.md:159,169,577).
"""

import hashlib
import os

import numpy as np
import pytest

import oracle

C1 = oracle.OracleConfig(layers=2, model_dim=256, heads=4, kv_heads=2, head_dim=64,
                         vocab_size=32768, document_len=128, query_len=48)
TOL = 5e-5


def rel_err(s, r):
    s, r = np.asarray(s, np.float64), np.asarray(r, np.float64)
    rms = np.sqrt((r ** 2).mean())
    return float(np.max(np.abs(s - r) / np.maximum(np.abs(r), rms)))


@pytest.fixture(scope="module")
def w_c1():
    return oracle.init_weights(C1)


@pytest.fixture(scope="module")
def g_c1(golden_dir):
    return np.load(os.path.join(golden_dir, "c1_scores.npz"))


def test_weights_bit_exact(golden_dir, w_c1):
    g = np.load(os.path.join(golden_dir, "weights_c1.npz"))
    H, KVH, HD = C1.heads, C1.kv_heads, C1.head_dim
    t = {"token_embedding": w_c1.emb}
    for i in range(C1.layers):
        wqkv = w_c1.wqkv[i]
        t[f"layers.{i}.attn.wq"] = wqkv[:, :H * HD]
        t[f"layers.{i}.attn.wk"] = wqkv[:, H * HD:(H + KVH) * HD]
        t[f"layers.{i}.attn.wv"] = wqkv[:, (H + KVH) * HD:]
        t[f"layers.{i}.attn.wo"] = w_c1.wo[i]
        t[f"layers.{i}.mlp.w_up"] = w_c1.w_up[i]
        t[f"layers.{i}.mlp.w_down"] = w_c1.w_down[i]
    for name, a in t.items():
        a = np.ascontiguousarray(a)
        assert hashlib.sha256(a.tobytes()).digest() == g[f"{name}|sha256"].tobytes(), name
        assert np.array_equal(a.reshape(-1)[:64], g[f"{name}|head"]), name
    assert np.array_equal(w_c1.cos, g["rope_cos"]) and np.array_equal(w_c1.sin, g["rope_sin"])
    # SPEC.md:65 golden: default config, seed 42, embedding[0][0]
    e = oracle.init_rows(42, "token_embedding", (32768, 128), [0])[0, 0]
    assert e == g["default_seed42_emb00"] == np.float32(0.001367543125525117)


def test_lazy_embedding_rows_match_full_stream(w_c1):
    lazy = oracle.LazyEmbedding(0, C1.vocab_size, C1.model_dim)
    toks = np.array([[0, 1, 32767], [17, 17, 4096]])
    assert np.array_equal(lazy[toks], w_c1.emb[toks])


def test_c1_dockv_vs_reference(g_c1, w_c1):
    for i in (0, 1):
        k, v, vl = oracle.doc_prefill(w_c1, g_c1["doc_tokens"][i])
        assert vl == 128
        for got, want in ((k, g_c1[f"doc{i}_keys"]), (v, g_c1[f"doc{i}_values"])):
            assert np.abs(got - want).max() / np.abs(want).max() <= TOL


def test_c1_scores_vs_reference(g_c1, w_c1):
    docs, q = g_c1["doc_tokens"], g_c1["query_tokens"]
    s = []
    for i in range(16):
        k, v, vl = oracle.doc_prefill(w_c1, docs[i])
        s.append(oracle.score_reuse(w_c1, k, v, vl, q))
    assert rel_err(s, g_c1["scores_fast"][:16]) <= TOL
    # the reference's own "reference" path and full recompute agree with it too
    assert rel_err(s[:4], g_c1["scores_reference_path"]) <= 1e-4
    full = [oracle.score_full(w_c1, docs[i], q) for i in range(4)]
    assert rel_err(full, g_c1["scores_full_fast"]) <= TOL


def test_c1_padded_vs_reference(golden_dir, w_c1):
    g = np.load(os.path.join(golden_dir, "c1_padded.npz"))
    kv = [oracle.doc_prefill(w_c1, d) for d in g["doc_tokens"]]
    assert [x[2] for x in kv] == list(g["valid_len"])
    s = np.array([[oracle.score_reuse(w_c1, *kv[i], g["query_tokens"][j]) for j in range(4)]
                  for i in range(4)])
    assert rel_err(s, g["scores"]) <= TOL
    k1, v1, _ = kv[1]
    assert np.abs(k1 - g["doc1_keys"]).max() / np.abs(g["doc1_keys"]).max() <= TOL
    full = [oracle.score_full(w_c1, g["doc_tokens"][i], g["query_tokens"][i]) for i in range(4)]
    assert rel_err(full, g["full_scores"]) <= TOL


def test_closed_form_counters(golden_dir):
    g = np.load(os.path.join(golden_dir, "counters.npz"))
    valid = np.ones(256 + 48, bool)
    assert oracle.pair_count(valid, 0) == int(g["full_pairs"]) == 46360
    assert oracle.pair_count(valid, 256) == int(g["reuse_pairs"]) == 13464


def test_padded_counters(golden_dir):
    g = np.load(os.path.join(golden_dir, "c1_padded.npz"))
    D = 128
    for i in range(4):
        for j in range(4):
            qv = g["query_tokens"][j] != 0
            valid = np.concatenate([np.arange(D) < g["valid_len"][i], qv])
            lin, macs, peak, kvb = g["counters"][i, j]
            assert lin == qv.sum() == peak
            assert macs == oracle.pair_count(valid, D)
            assert kvb == 2 * 2 * 2 * 128 * 64 * 4   # f32 payload, model.py:93-95


def test_select_topk_tie_break():
    scores = [0.5, 0.9, 0.5, 0.1, 0.9]
    ids = ["doc-3", "doc-2", "doc-1", "doc-0", "doc-9"]
    assert oracle.select_topk(scores, ids, 4) == [1, 4, 2, 0]
    assert oracle.select_topk(scores, ids, 10) == [1, 4, 2, 0, 3]


@pytest.mark.parametrize("name", ["c3w_l2", "c2w_l1"])
def test_wide_shapes_vs_reference(golden_dir, name):
    """Full-width shallow gates: 7B width at 2 layers, Gemma
    width at 1 layer; two pairs each (one with a padded document)."""
    g = np.load(os.path.join(golden_dir, f"{name}.npz"))
    L, d, H, KVH, HD, V, MP = [int(x) for x in g["cfg"]]
    D, Q = g["doc_tokens"].shape[1], g["query_tokens"].shape[1]
    cfg = oracle.OracleConfig(layers=L, model_dim=d, heads=H, kv_heads=KVH, head_dim=HD,
                              vocab_size=V, max_position=MP, document_len=D, query_len=Q)
    w = oracle.init_weights(cfg, lazy_embedding=True)
    s = [oracle.score_full(w, g["doc_tokens"][i], g["query_tokens"][i]) for i in (0, 1)]
    assert rel_err(s, g["scores"][:2]) <= 1e-4


@pytest.mark.parametrize("variant", [dict(mlp="geglu", ffn_dim=96, embed_scale=8.0, attn_scale=0.25),
                                     dict(mlp="swiglu", ffn_dim=160, attn_scale=0.25)])
def test_variant_oracle_is_self_consistent(variant):
    """Architecture variants (outside the reference): defaults
    reproduce the reference model exactly, a gated MLP is act(x Wg) * (x Wu),
    the w_gate stream has its own name, and KV reuse == full recompute."""
    geo = dict(layers=2, model_dim=64, heads=4, kv_heads=2, head_dim=16, vocab_size=4096,
               document_len=24, query_len=8)
    base = oracle.init_weights(oracle.OracleConfig(**geo))
    w = oracle.init_weights(oracle.OracleConfig(**geo, **variant))
    F = variant["ffn_dim"]
    assert w.w_up[0].shape == (64, F) and w.w_gate[0].shape == (64, F)
    assert np.array_equal(w.wqkv[1], base.wqkv[1])            # attention weights unchanged
    assert not np.array_equal(w.w_gate[0][:, :8], w.w_up[0][:, :8])
    x = np.random.default_rng(0).standard_normal((3, 64)).astype(np.float32)
    g, u = x @ w.w_gate[0], x @ w.w_up[0]
    act = oracle.kvrerank_np._gelu(g) if variant["mlp"] == "geglu" else g / (1 + np.exp(-g))
    assert np.allclose(oracle.kvrerank_np._mlp(w, 0, x), (act * u) @ w.w_down[0], rtol=1e-6)
    rng = np.random.default_rng(1)
    doc, q = rng.integers(1, 4096, 24), rng.integers(1, 4096, 8)
    k, v, vl = oracle.doc_prefill(w, doc)
    assert oracle.score_reuse(w, k, v, vl, q) == pytest.approx(oracle.score_full(w, doc, q),
                                                              rel=1e-5, abs=1e-6)


def test_c5_geometry_oracle_vs_reference(golden_dir):
    """C5 geometry (7B width, L=2, D=2048, RoPE positions past 1,024, Q=16 with
    padded doc and query): the oracle reproduces the reference's score."""
    g = np.load(os.path.join(golden_dir, "c5w_l2.npz"))
    L, d, H, KVH, HD, V, MP = [int(x) for x in g["cfg"]]
    cfg = oracle.OracleConfig(layers=L, model_dim=d, heads=H, kv_heads=KVH, head_dim=HD,
                              vocab_size=V, max_position=MP, document_len=2048, query_len=16)
    w = oracle.init_weights(cfg, lazy_embedding=True)
    k, v, vl = oracle.doc_prefill(w, g["doc_tokens"][1])            # 300 trailing pads
    assert vl == g["valid_len"][1]
    s = oracle.score_reuse(w, k, v, vl, g["q16_tokens"][1])          # padded query
    r = g["q16_scores"]
    assert abs(s - r[4 + 1]) <= 1e-4 * max(abs(r[5]), np.sqrt(np.mean(r ** 2)))


@pytest.mark.parametrize("name", ["topk_c3w_l2", "topk_c2w_l1"])
def test_topk_goldens_follow_select_order(golden_dir, name):
    """The reference's _select output (pipeline.py:285-287) is the oracle's
    (score desc, chunk id asc) order over the 100 golden scores."""
    g = np.load(os.path.join(golden_dir, f"{name}.npz"))
    ids = [f"doc-{i:05d}" for i in range(len(g["scores"]))]
    order = oracle.select_topk(list(g["scores"]), ids, 20)
    assert [ids[i] for i in order] == list(g["top_ids"])
    assert np.array_equal(g["scores"][order], g["top_scores"])


def test_topk_c2w_oracle_scores(golden_dir):
    """Two of the 100 Gemma-width candidates (one padded) re-scored by the oracle."""
    g = np.load(os.path.join(golden_dir, "topk_c2w_l1.npz"))
    L, d, H, KVH, HD, V, MP = [int(x) for x in g["cfg"]]
    cfg = oracle.OracleConfig(layers=L, model_dim=d, heads=H, kv_heads=KVH, head_dim=HD,
                              vocab_size=V, max_position=MP, document_len=512, query_len=48)
    w = oracle.init_weights(cfg, lazy_embedding=True)
    r = g["scores"]
    s = np.array([oracle.score_full(w, g["doc_tokens"][i], g["query_tokens"]) for i in (0, 5)])
    rms = np.sqrt(np.mean(r ** 2))
    assert np.all(np.abs(s - r[[0, 5]]) <= 1e-4 * np.maximum(np.abs(r[[0, 5]]), rms))
