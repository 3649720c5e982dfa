"""Generate golden vectors by running the REFERENCE package itself.

Run in the build container only (it needs /root/reference, which does not
exist on the GPU box):

    python tests/golden/make_golden.py [--skip-wide]

Writes small .npz fixtures next to this file.  They pin the CPU oracle
(oracle/kvrerank_np.py) and, through it, the GPU path.  Every array here is
produced by ``kvrerank`` 0.1.0 calls (reranker.score_batch / doc_prefill /
score_full, model.init_weights); nothing is computed by this repo's code.
"""

from __future__ import annotations

import argparse
import hashlib
import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def _ref():
    sys.path.insert(0, REF)
    import kvrerank  # noqa: F401
    from kvrerank import model, reranker
    return model, reranker


def _tokens(rng, n, length, vocab):
    return rng.integers(1, vocab, size=(n, length), dtype=np.int64)


def weights_fixture(model):
    """Weight stream pins: head values and f64 sums of every C1 tensor, plus
    SPEC.md:65's embedding[0][0] at the default config with seed 42."""
    cfg = model.ModelConfig(layers=2, model_dim=256, heads=4, kv_heads=2, head_dim=64,
                            vocab_size=32768, seed=0)
    w = model.init_weights(cfg)
    out = {}
    tensors = {"token_embedding": w.token_embedding}
    for i, lw in enumerate(w.layers):
        tensors[f"layers.{i}.attn.wq"] = lw.wq
        tensors[f"layers.{i}.attn.wk"] = lw.wk
        tensors[f"layers.{i}.attn.wv"] = lw.wv
        tensors[f"layers.{i}.attn.wo"] = lw.wo
        tensors[f"layers.{i}.mlp.w_up"] = lw.w_up
        tensors[f"layers.{i}.mlp.w_down"] = lw.w_down
    for name, t in tensors.items():
        out[f"{name}|head"] = np.ascontiguousarray(t).reshape(-1)[:64].copy()
        out[f"{name}|tail"] = np.ascontiguousarray(t).reshape(-1)[-64:].copy()
        out[f"{name}|sha256"] = np.frombuffer(
            hashlib.sha256(np.ascontiguousarray(t).tobytes()).digest(), np.uint8)
    out["rope_cos"] = w.rope_cos
    out["rope_sin"] = w.rope_sin
    w42 = model.init_weights(model.ModelConfig(seed=42))
    out["default_seed42_emb00"] = np.float32(w42.token_embedding[0][0])
    np.savez_compressed(os.path.join(HERE, "weights_c1.npz"), **out)


def c1_fixture(model, reranker):
    """C1 (BASELINE configs[0]): 1 query x 64 cached docs x 128 tok, Q=48."""
    cfg = model.ModelConfig(layers=2, model_dim=256, heads=4, kv_heads=2, head_dim=64,
                            vocab_size=32768, seed=0)
    layout = reranker.LayoutConfig(document_len=128, query_len=48)
    rm = reranker.RerankModel.build(cfg, layout)
    rng = np.random.default_rng(1234)
    docs = _tokens(rng, 64, 128, cfg.vocab_size)
    query = _tokens(rng, 1, 48, cfg.vocab_size)[0]
    kvs = [reranker.doc_prefill(rm, d, chunk_id=f"doc-{i:05d}") for i, d in enumerate(docs)]
    pairs = [("q0", kv.chunk_id, kv, query) for kv in kvs]
    t0 = time.time()
    scored, counters = reranker.score_batch(rm, pairs, mode="reuse", path="fast")
    t_fast = time.time() - t0
    ref_scored, _ = reranker.score_batch(rm, pairs[:4], mode="reuse", path="reference")
    full = [reranker.score_full(rm, docs[i], query, path="fast")[0] for i in range(4)]
    np.savez_compressed(
        os.path.join(HERE, "c1_scores.npz"),
        doc_tokens=docs, query_tokens=query,
        scores_fast=np.array([s.score for s in scored], np.float64),
        scores_reference_path=np.array([s.score for s in ref_scored], np.float64),
        scores_full_fast=np.array(full, np.float64),
        counters=np.array([counters.linear_token_count, counters.attn_mac_pairs,
                           counters.peak_activation_tokens, counters.kv_bytes_loaded]),
        doc0_keys=kvs[0].kv.keys, doc0_values=kvs[0].kv.values,
        doc1_keys=kvs[1].kv.keys, doc1_values=kvs[1].kv.values,
        cpu_seconds_fast_64=np.float64(t_fast),
    )


def padded_fixture(model, reranker):
    """Pads: doc valid_len < D (trailing), trailing and interior query pads."""
    cfg = model.ModelConfig(layers=2, model_dim=256, heads=4, kv_heads=2, head_dim=64,
                            vocab_size=32768, seed=0)
    layout = reranker.LayoutConfig(document_len=128, query_len=48)
    rm = reranker.RerankModel.build(cfg, layout)
    rng = np.random.default_rng(99)
    docs = _tokens(rng, 4, 128, cfg.vocab_size)
    for i, vl in enumerate([128, 100, 1, 64]):
        docs[i, vl:] = 0
    queries = _tokens(rng, 4, 48, cfg.vocab_size)
    queries[1, 30:] = 0                      # trailing pads
    queries[2, [3, 7, 20, 21]] = 0           # interior pads
    queries[3, 0:10] = 0                     # leading pads
    queries[3, 40:] = 0
    scores, counters, full_scores, full_counters = [], [], [], []
    kvs = [reranker.doc_prefill(rm, d, chunk_id=f"pad-{i}") for i, d in enumerate(docs)]
    for i in range(4):
        for j in range(4):
            s, c = reranker.score_reuse(rm, kvs[i], queries[j], path="fast")
            scores.append(s)
            counters.append([c.linear_token_count, c.attn_mac_pairs,
                             c.peak_activation_tokens, c.kv_bytes_loaded])
        s, c = reranker.score_full(rm, docs[i], queries[i], path="fast")
        full_scores.append(s)
        full_counters.append([c.linear_token_count, c.attn_mac_pairs,
                              c.peak_activation_tokens, c.kv_bytes_loaded])
    np.savez_compressed(
        os.path.join(HERE, "c1_padded.npz"),
        doc_tokens=docs, query_tokens=queries,
        valid_len=np.array([kv.valid_len for kv in kvs]),
        scores=np.array(scores, np.float64).reshape(4, 4),
        counters=np.array(counters).reshape(4, 4, 4),
        full_scores=np.array(full_scores, np.float64),
        full_counters=np.array(full_counters),
        doc1_keys=kvs[1].kv.keys, doc1_values=kvs[1].kv.values,
    )


def counters_fixture(reranker):
    """SPEC.md:577 closed-form counters at D=256, Q=48 (no model needed)."""
    D, Q = 256, 48
    valid = np.ones(D + Q, bool)
    np.savez_compressed(
        os.path.join(HERE, "counters.npz"),
        full_pairs=np.int64(reranker._pair_count(valid, 0)),
        reuse_pairs=np.int64(reranker._pair_count(valid, D)),
    )


def wide_fixture(model, reranker, name, cfg_kw, D, Q, n_pairs, seed):
    """Full-width shallow models (SURVEY Appendix A gates): scores only."""
    cfg = model.ModelConfig(**cfg_kw)
    layout = reranker.LayoutConfig(document_len=D, query_len=Q)
    t0 = time.time()
    rm = reranker.RerankModel.build(cfg, layout)
    t_init = time.time() - t0
    rng = np.random.default_rng(seed)
    docs = _tokens(rng, n_pairs, D, cfg.vocab_size)
    queries = _tokens(rng, n_pairs, Q, cfg.vocab_size)
    docs[1, D - 37:] = 0
    queries[2, Q - 5:] = 0
    scores = []
    t0 = time.time()
    for i in range(n_pairs):
        kv = reranker.doc_prefill(rm, docs[i], chunk_id=f"w{i}")
        scores.append(reranker.score_reuse(rm, kv, queries[i], path="fast")[0])
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), doc_tokens=docs,
                        query_tokens=queries, scores=np.array(scores, np.float64),
                        cfg=np.array([cfg.layers, cfg.model_dim, cfg.heads, cfg.kv_heads,
                                      cfg.head_dim, cfg.vocab_size, cfg.max_position]),
                        cpu_seconds=np.float64(time.time() - t0),
                        init_seconds=np.float64(t_init))
    print(name, "init", round(t_init, 1), "s; scored in", round(time.time() - t0, 1), "s")


def codec_fixture(model, reranker):
    """HRKV bytes written by the reference codec (codec.py:128-157) for one C1
    document (F32 / INT8 / INT4), plus its decode of the quantised entries and a
    hand-made tensor with zero channels and exact .5 ties."""
    from kvrerank import codec
    cfg = model.ModelConfig(layers=2, model_dim=256, heads=4, kv_heads=2, head_dim=64,
                            vocab_size=32768, seed=0)
    layout = reranker.LayoutConfig(document_len=128, query_len=48)
    rm = reranker.RerankModel.build(cfg, layout)
    rng = np.random.default_rng(5)
    doc = _tokens(rng, 1, 128, cfg.vocab_size)[0]
    doc[90:] = 0
    kv = reranker.doc_prefill(rm, doc, chunk_id="doc-00042")
    out = {"doc_tokens": doc}
    for sch in (codec.QuantScheme.F32, codec.QuantScheme.INT8_PER_CHANNEL,
                codec.QuantScheme.INT4_PER_CHANNEL):
        data = codec.encode_entry(kv, sch)
        out[f"entry_{sch.short_name}"] = np.frombuffer(data, np.uint8)
        dec = codec.decode_entry(data)
        out[f"decoded_keys_{sch.short_name}"] = np.asarray(dec.kv.keys)
        out[f"decoded_values_{sch.short_name}"] = np.asarray(dec.kv.values)
    t = np.array([[[0.0, 1.0, -2.5], [0.0, -0.5, 1.25], [0.0, 0.25, 2.5]]], np.float32)
    for sch in (codec.QuantScheme.INT8_PER_CHANNEL, codec.QuantScheme.INT4_PER_CHANNEL):
        q, sc = codec.quantize_tensor(t, sch)
        out[f"edge_codes_{sch.short_name}"] = np.frombuffer(q, np.uint8)
        out[f"edge_scales_{sch.short_name}"] = sc
    out["edge_tensor"] = t
    np.savez_compressed(os.path.join(HERE, "codec_c1.npz"), **out)


def c5_fixture(model, reranker, L=2):
    """C5 geometry at 7B width, L layers: D=2048 docs
    (positions up to 2047+Q, max_position 4096), Q in {16, 48, 256}, padded
    docs and queries.  One prefill per doc (the DocKV depends on D only), then
    every doc x query pair through the reference's score_batch per Q."""
    cfg = model.ModelConfig(layers=L, model_dim=4096, heads=32, kv_heads=8, head_dim=128,
                            vocab_size=32000, max_position=4096, seed=0)
    t0 = time.time()
    w = model.init_weights(cfg)
    head = reranker._score_head(cfg)
    t_init = time.time() - t0
    D = 2048
    rng = np.random.default_rng(2048)
    docs = _tokens(rng, 4, D, cfg.vocab_size)
    docs[1, D - 300:] = 0
    docs[2, 1000:] = 0
    rm = reranker.RerankModel(config=cfg, weights=w, score_head=head,
                              layout=reranker.LayoutConfig(document_len=D, query_len=48))
    t0 = time.time()
    kvs = [reranker.doc_prefill(rm, d, chunk_id=f"c5-{i}") for i, d in enumerate(docs)]
    t_pre = time.time() - t0
    out = {"doc_tokens": docs, "valid_len": np.array([k.valid_len for k in kvs]),
           "cfg": np.array([cfg.layers, cfg.model_dim, cfg.heads, cfg.kv_heads, cfg.head_dim,
                            cfg.vocab_size, cfg.max_position]),
           # K/V of doc 0 at positions 1500..1563 (RoPE beyond 1024), both layers
           "doc0_keys_1500": np.ascontiguousarray(kvs[0].kv.keys[:, :, 1500:1564]),
           "doc0_values_1500": np.ascontiguousarray(kvs[0].kv.values[:, :, 1500:1564]),
           "init_seconds": np.float64(t_init), "prefill_seconds": np.float64(t_pre)}
    for Q in (16, 48, 256):
        rmq = reranker.RerankModel(config=cfg, weights=w, score_head=head,
                                   layout=reranker.LayoutConfig(document_len=D, query_len=Q))
        qs = _tokens(rng, 2, Q, cfg.vocab_size)
        qs[1, Q - Q // 4:] = 0                       # trailing pads
        qs[1, 1] = 0                                 # interior pad
        pairs = [(f"q{j}", kv.chunk_id, kv, qs[j]) for j in range(2) for kv in kvs]
        t0 = time.time()
        scored, counters = reranker.score_batch(rmq, pairs, mode="reuse", path="fast")
        out[f"q{Q}_tokens"] = qs
        out[f"q{Q}_scores"] = np.array([p.score for p in scored], np.float64)
        out[f"q{Q}_seconds"] = np.float64(time.time() - t0)
        out[f"q{Q}_counters"] = np.array([counters.linear_token_count, counters.attn_mac_pairs,
                                          counters.peak_activation_tokens,
                                          counters.kv_bytes_loaded])
    np.savez_compressed(os.path.join(HERE, f"c5w_l{L}.npz"), **out)
    print("c5", "init", round(t_init, 1), "prefill", round(t_pre, 1))


def topk_fixture(model, reranker, pipeline, name, cfg_kw, D, n_docs, keep, seed):
    """1 query x n_docs candidates at full width (shallow): the reference's
    scores and its own _select top-keep (pipeline.py:285-287)."""
    from types import SimpleNamespace
    cfg = model.ModelConfig(**cfg_kw)
    rm = reranker.RerankModel.build(cfg, reranker.LayoutConfig(document_len=D, query_len=48))
    rng = np.random.default_rng(seed)
    docs = _tokens(rng, n_docs, D, cfg.vocab_size)
    docs[5, D - 100:] = 0
    query = _tokens(rng, 1, 48, cfg.vocab_size)[0]
    query[44:] = 0
    t0 = time.time()
    kvs = [reranker.doc_prefill(rm, d, chunk_id=f"doc-{i:05d}") for i, d in enumerate(docs)]
    scored, _ = reranker.score_batch(rm, [("q0", kv.chunk_id, kv, query) for kv in kvs],
                                     mode="reuse", path="fast")
    sel = pipeline._select(SimpleNamespace(config=SimpleNamespace(keep_m=keep)), scored)
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), doc_tokens=docs, query_tokens=query,
                        scores=np.array([p.score for p in scored], np.float64),
                        top_ids=np.array([p.chunk_id for p in sel]),
                        top_scores=np.array([p.score for p in sel], np.float64),
                        cfg=np.array([cfg.layers, cfg.model_dim, cfg.heads, cfg.kv_heads,
                                      cfg.head_dim, cfg.vocab_size, cfg.max_position]),
                        cpu_seconds=np.float64(time.time() - t0))
    print(name, "scored in", round(time.time() - t0, 1), "s")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--skip-wide", action="store_true")
    ap.add_argument("--only", default="")
    args = ap.parse_args()
    model, reranker = _ref()
    from kvrerank import pipeline
    only = {
        "codec": lambda: codec_fixture(model, reranker),
        "c5": lambda: c5_fixture(model, reranker),
        "topk_c3w": lambda: topk_fixture(
            model, reranker, pipeline, "topk_c3w_l2",
            dict(layers=2, model_dim=4096, heads=32, kv_heads=8, head_dim=128,
                 vocab_size=32000, max_position=1024, seed=0), D=512, n_docs=100, keep=20,
            seed=21),
        "topk_c2w": lambda: topk_fixture(
            model, reranker, pipeline, "topk_c2w_l1",
            dict(layers=1, model_dim=2048, heads=8, kv_heads=1, head_dim=256,
                 vocab_size=256000, max_position=1024, seed=0), D=512, n_docs=100, keep=20,
            seed=22),
    }
    if args.only:
        for k in args.only.split(","):
            only[k]()
        return
    codec_fixture(model, reranker)
    weights_fixture(model)
    c1_fixture(model, reranker)
    padded_fixture(model, reranker)
    counters_fixture(reranker)
    if not args.skip_wide:
        wide_fixture(model, reranker, "c3w_l2",
                     dict(layers=2, model_dim=4096, heads=32, kv_heads=8, head_dim=128,
                          vocab_size=32000, max_position=1024, seed=0),
                     D=512, Q=48, n_pairs=4, seed=7)
        wide_fixture(model, reranker, "c2w_l1",
                     dict(layers=1, model_dim=2048, heads=8, kv_heads=1, head_dim=256,
                          vocab_size=256000, max_position=1024, seed=0),
                     D=512, Q=48, n_pairs=4, seed=8)
        for k in ("c5", "topk_c3w", "topk_c2w"):
            only[k]()


if __name__ == "__main__":
    main()
