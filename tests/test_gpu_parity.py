"""End-to-end parity of the device path against the reference's own golden
vectors (tests/golden, produced by kvrerank itself) and the CPU oracle.

Gates:
  * f32 debug build  : max|d|/max(|r|, rms(r)) <= 1e-4
  * f16 fast path    : norm-wise ||s-r||/||r|| <= 2e-2, top-k equal modulo
                       reference ties within tolerance
"""

import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2504_02921_b200 as krr  # noqa: E402
from paper_2504_02921_b200 import ModelConfig, LayoutConfig  # noqa: E402

F32_TOL = 1e-4
F16_NORMWISE = 2e-2


def rel_err(s, r):
    s, r = np.asarray(s, np.float64), np.asarray(r, np.float64)
    rms = np.sqrt((r ** 2).mean())
    return float(np.max(np.abs(s - r) / np.maximum(np.abs(r), rms)))


def normwise(s, r):
    s, r = np.asarray(s, np.float64), np.asarray(r, np.float64)
    return float(np.linalg.norm(s - r) / np.linalg.norm(r))


def topk_equal_modulo_ties(s, r, k, tol):
    """Top-k by the reference must match, except where reference scores tie
    within tol (then either order is accepted)."""
    r = np.asarray(r)
    s = np.asarray(s)
    want = list(np.argsort(-r, kind="stable")[:k])
    got = list(np.argsort(-s, kind="stable")[:k])
    for a, b in zip(want, got):
        if a != b and abs(r[a] - r[b]) > tol * max(1.0, abs(r[a])):
            return False
    return True


C1 = (ModelConfig(layers=2, model_dim=256, heads=4, kv_heads=2, head_dim=64, vocab_size=32768),
      LayoutConfig(document_len=128, query_len=48))


@pytest.fixture(scope="module")
def c1_golden(golden_dir):
    return np.load(os.path.join(golden_dir, "c1_scores.npz"))


@pytest.fixture(scope="module")
def model_f32():
    return krr.RerankModel.build(*C1, precision="f32")


@pytest.fixture(scope="module")
def model_f16():
    return krr.RerankModel.build(*C1, precision="f16")


def test_weights_bit_exact(golden_dir, model_f32):
    import hashlib
    g = np.load(os.path.join(golden_dir, "weights_c1.npz"))
    w = model_f32.weights
    emb = w.token_embedding.cpu().numpy()
    assert hashlib.sha256(emb.tobytes()).digest() == g["token_embedding|sha256"].tobytes()
    H, KVH, HD = 4, 2, 64
    for i in range(2):
        wqkv = w.wqkv[i].cpu().numpy().T   # back to reference [in, out]
        wq, wk, wv = wqkv[:, :H * HD], wqkv[:, H * HD:(H + KVH) * HD], wqkv[:, (H + KVH) * HD:]
        for name, t in (("attn.wq", wq), ("attn.wk", wk), ("attn.wv", wv),
                        ("attn.wo", w.wo[i].cpu().numpy().T),
                        ("mlp.w_up", w.w_up[i].cpu().numpy().T),
                        ("mlp.w_down", w.w_down[i].cpu().numpy().T)):
            digest = hashlib.sha256(np.ascontiguousarray(t).tobytes()).digest()
            assert digest == g[f"layers.{i}.{name}|sha256"].tobytes(), name


def _c1_scores(model, g, path="fast"):
    docs, q = g["doc_tokens"], g["query_tokens"]
    kvs = krr.doc_prefill_batch(model, docs, [f"doc-{i:05d}" for i in range(len(docs))],
                                path=path)
    pairs = [("q0", kv.chunk_id, kv, q) for kv in kvs]
    res, counters = krr.score_batch(model, pairs, mode="reuse", path=path)
    return np.array([r.score for r in res]), counters, kvs


def test_c1_f32_scores_vs_reference(c1_golden, model_f32):
    s, counters, _ = _c1_scores(model_f32, c1_golden)
    r = c1_golden["scores_fast"]
    assert rel_err(s, r) <= F32_TOL, rel_err(s, r)
    assert [counters.linear_token_count, counters.attn_mac_pairs,
            counters.peak_activation_tokens, counters.kv_bytes_loaded] == \
        list(c1_golden["counters"])


def test_c1_f32_dockv_vs_reference(c1_golden, model_f32):
    kv = krr.doc_prefill(model_f32, c1_golden["doc_tokens"][0], chunk_id="d0")
    k, v = kv.kv.keys, kv.kv.values
    for got, want in ((k, c1_golden["doc0_keys"]), (v, c1_golden["doc0_values"])):
        err = np.abs(got - want).max() / np.abs(want).max()
        assert err <= F32_TOL, err


def test_c1_f16_scores_vs_reference(c1_golden, model_f16):
    s, _, _ = _c1_scores(model_f16, c1_golden)
    r = c1_golden["scores_fast"]
    nw = normwise(s, r)
    assert nw <= F16_NORMWISE, nw
    assert topk_equal_modulo_ties(s, r, 20, F16_NORMWISE)


def test_reference_path_is_f32(c1_golden, model_f16):
    """path='reference' runs the f32 debug build even on an f16 model."""
    s, _, _ = _c1_scores(model_f16, c1_golden, path="reference")
    assert rel_err(s, c1_golden["scores_fast"]) <= F32_TOL


def test_full_equals_reuse_bit_exact(c1_golden, model_f16):
    docs, q = c1_golden["doc_tokens"][:8], c1_golden["query_tokens"]
    kvs = krr.doc_prefill_batch(model_f16, docs, [f"fe{i}" for i in range(8)])
    reuse, _ = krr.score_batch(model_f16, [("q", k.chunk_id, k, q) for k in kvs], "reuse")
    full, _ = krr.score_batch(model_f16, [("q", f"fe{i}", docs[i], q) for i in range(8)], "full")
    assert [r.score for r in reuse] == [f.score for f in full]


def test_batch_invariance(c1_golden, model_f16):
    s_all, _, kvs = _c1_scores(model_f16, c1_golden)
    q = c1_golden["query_tokens"]
    sub = [("q", kvs[i].chunk_id, kvs[i], q) for i in (5, 17, 40)]
    res, _ = krr.score_batch(model_f16, sub, "reuse")
    assert [r.score for r in res] == [float(s_all[i]) for i in (5, 17, 40)]


@pytest.mark.parametrize("precision,gate", [("f32", "f32"), ("f16", "f16")])
def test_padded_cases(golden_dir, precision, gate):
    g = np.load(os.path.join(golden_dir, "c1_padded.npz"))
    model = krr.RerankModel.build(*C1, precision=precision)
    kvs = krr.doc_prefill_batch(model, g["doc_tokens"], [f"pad-{i}" for i in range(4)])
    assert [k.valid_len for k in kvs] == list(g["valid_len"])
    pairs = [("q", kvs[i].chunk_id, kvs[i], g["query_tokens"][j])
             for i in range(4) for j in range(4)]
    res, _ = krr.score_batch(model, pairs, "reuse")
    s = np.array([r.score for r in res]).reshape(4, 4)
    for i in range(4):
        for j in range(4):
            _, c = krr.score_reuse(model, kvs[i], g["query_tokens"][j])
            assert [c.linear_token_count, c.attn_mac_pairs, c.peak_activation_tokens,
                    c.kv_bytes_loaded] == list(g["counters"][i, j])
    if gate == "f32":
        assert rel_err(s, g["scores"]) <= F32_TOL
    else:
        assert normwise(s, g["scores"]) <= F16_NORMWISE
    full = [krr.score_full(model, g["doc_tokens"][i], g["query_tokens"][i]) for i in range(4)]
    for i in range(4):
        assert [full[i][1].linear_token_count, full[i][1].attn_mac_pairs] == \
            list(g["full_counters"][i][:2])
    if gate == "f32":
        assert rel_err([f[0] for f in full], g["full_scores"]) <= F32_TOL


def _wide(golden_dir, name, precision):
    g = np.load(os.path.join(golden_dir, f"{name}.npz"))
    L, d, H, KVH, HD, V, MP = [int(x) for x in g["cfg"]]
    cfg = ModelConfig(layers=L, model_dim=d, heads=H, kv_heads=KVH, head_dim=HD, vocab_size=V,
                      max_position=MP)
    lay = LayoutConfig(document_len=g["doc_tokens"].shape[1], query_len=g["query_tokens"].shape[1])
    model = krr.RerankModel.build(cfg, lay, precision=precision)
    kvs = krr.doc_prefill_batch(model, g["doc_tokens"], [f"w{i}" for i in range(len(g["scores"]))])
    res, _ = krr.score_batch(model, [("q", k.chunk_id, k, q) for k, q in
                                     zip(kvs, g["query_tokens"])], "reuse")
    return np.array([r.score for r in res]), g["scores"]


@pytest.mark.parametrize("name", ["c3w_l2", "c2w_l1"])
def test_wide_shapes_f32(golden_dir, name):
    s, r = _wide(golden_dir, name, "f32")
    assert rel_err(s, r) <= F32_TOL, rel_err(s, r)


@pytest.mark.parametrize("name", ["c3w_l2", "c2w_l1"])
def test_wide_shapes_f16(golden_dir, name):
    s, r = _wide(golden_dir, name, "f16")
    assert normwise(s, r) <= F16_NORMWISE, normwise(s, r)


def test_yes_no_head_is_two_row_logit_difference(c1_golden):
    """head='yes_no': score == logit(yes) - logit(no) of a tied lm_head on the
    last valid token, computed from the final-normed hidden state that the
    default head dots with score_head (self-consistency; outside reference parity)."""
    m = krr.RerankModel.build(*C1, precision="f32", head="yes_no", yes_no_ids=(11, 7))
    docs, q = c1_golden["doc_tokens"][:3], c1_golden["query_tokens"]
    kvs = krr.doc_prefill_batch(m, docs, [f"yn{i}" for i in range(3)])
    res, _ = krr.score_batch(m, [("q", k.chunk_id, k, q) for k in kvs], "reuse")
    import oracle
    ow = oracle.init_weights(oracle.OracleConfig(layers=2, model_dim=256, heads=4, kv_heads=2,
                                                 head_dim=64, vocab_size=32768,
                                                 document_len=128, query_len=48))
    emb = m.weights.token_embedding.cpu().numpy()
    v = emb[11] - emb[7]
    for r, d in zip(res, docs):
        kk, vv, vl = oracle.doc_prefill(ow, d)
        D = kk.shape[2]
        hidden, _, _ = oracle.forward(ow, q, np.arange(D, D + q.size), kk, vv,
                                      np.concatenate([np.arange(D) < vl, q != 0]))
        want = float(hidden[int(np.nonzero(q != 0)[0][-1])] @ v)
        assert abs(r.score - want) <= 1e-4 * max(1.0, abs(want))


@pytest.mark.parametrize("cfg,lay", [
    (ModelConfig(), LayoutConfig()),                       # reference default desk config (HD=16)
    (ModelConfig(layers=2, model_dim=96, heads=3, kv_heads=3, head_dim=32),
     LayoutConfig(document_len=70, query_len=20)),         # MHA, odd widths -> CUDA-core paths
    (ModelConfig(layers=2, model_dim=192, heads=3, kv_heads=1, head_dim=64),
     LayoutConfig(document_len=100, query_len=33)),        # G=3, ragged tiles
])
@pytest.mark.parametrize("precision", ["f32", "f16"])
def test_other_configs_vs_oracle(cfg, lay, precision):
    """Any ModelConfig the reference accepts runs (tensor-core kernels where the
    shape allows, CUDA-core kernels otherwise) and matches the oracle."""
    import oracle
    rng = np.random.default_rng(3)
    D, Q = lay.document_len, lay.query_len
    docs = rng.integers(1, cfg.vocab_size, (4, D))
    docs[1, D - 9:] = 0
    qs = rng.integers(1, cfg.vocab_size, (4, Q))
    qs[2, Q - 4:] = 0
    model = krr.RerankModel.build(cfg, lay, precision=precision)
    kvs = krr.doc_prefill_batch(model, docs, [f"o{i}" for i in range(4)])
    res, _ = krr.score_batch(model, [("q", k.chunk_id, k, q) for k, q in zip(kvs, qs)], "reuse")
    s = np.array([r.score for r in res])
    ow = oracle.init_weights(oracle.OracleConfig(
        layers=cfg.layers, model_dim=cfg.model_dim, heads=cfg.heads, kv_heads=cfg.kv_heads,
        head_dim=cfg.head_dim, vocab_size=cfg.vocab_size, max_position=cfg.max_position,
        document_len=D, query_len=Q))
    if precision == "f16":
        ow = oracle.round_weights(ow)
    ref = np.array([oracle.score_full(ow, docs[i], qs[i]) for i in range(4)])
    if precision == "f32":
        assert rel_err(s, ref) <= F32_TOL, rel_err(s, ref)
    else:
        assert normwise(s, ref) <= F16_NORMWISE, normwise(s, ref)


@pytest.mark.parametrize("variant", [
    dict(mlp="geglu", ffn_dim=768, embed_scale=16.0, attn_scale=0.125),      # Gemma-style
    dict(mlp="swiglu", ffn_dim=704, attn_scale=0.125),                       # Mistral-style
    dict(mlp="gelu", ffn_dim=512, attn_scale=0.125),                         # plain, other F
])
@pytest.mark.parametrize("dims", ["c1", "odd"])
@pytest.mark.parametrize("precision", ["f32", "f16"])
def test_architecture_variants_vs_oracle(variant, dims, precision):
    """SURVEY §8 f4 (outside reference parity): gated GeGLU / SwiGLU MLPs of
    width F, Gemma's embedding scale and a softmax scale, against the oracle's
    restatement of the same architecture, on the tensor-core kernels (c1) and
    the CUDA-core kernels (odd widths)."""
    import oracle
    if dims == "c1":
        geo = dict(layers=2, model_dim=256, heads=4, kv_heads=2, head_dim=64)
        D, Q = 128, 48
    else:
        geo = dict(layers=2, model_dim=96, heads=3, kv_heads=1, head_dim=32)
        D, Q = 70, 20
        variant = dict(variant, ffn_dim=320)
    cfg = ModelConfig(vocab_size=32768, **geo, **variant)
    lay = LayoutConfig(document_len=D, query_len=Q)
    rng = np.random.default_rng(11)
    docs = rng.integers(1, cfg.vocab_size, (4, D))
    docs[1, D - 9:] = 0
    qs = rng.integers(1, cfg.vocab_size, (4, Q))
    qs[2, Q - 4:] = 0
    model = krr.RerankModel.build(cfg, lay, precision=precision)
    kvs = krr.doc_prefill_batch(model, docs, [f"v{i}" for i in range(4)])
    res, _ = krr.score_batch(model, [("q", k.chunk_id, k, q) for k, q in zip(kvs, qs)], "reuse")
    s = np.array([r.score for r in res])
    full, _ = krr.score_batch(model, [("q", f"f{i}", docs[i], qs[i]) for i in range(4)], "full")
    assert np.array_equal(s, np.array([r.score for r in full]))     # reuse == full, bit-exact
    ow = oracle.init_weights(oracle.OracleConfig(vocab_size=cfg.vocab_size, document_len=D,
                                                 query_len=Q, **geo, **variant))
    if precision == "f16":
        ow = oracle.round_weights(ow)
    ref = np.array([oracle.score_full(ow, docs[i], qs[i]) for i in range(4)])
    if precision == "f32":
        assert rel_err(s, ref) <= F32_TOL, rel_err(s, ref)
    else:
        assert normwise(s, ref) <= F16_NORMWISE, normwise(s, ref)


def test_concurrent_score_batch_threads(c1_golden, model_f16):
    """score_batch from several threads at once (the reference's rerank
    workers) gives the same scores as one call."""
    import threading
    docs, q = c1_golden["doc_tokens"][:12], c1_golden["query_tokens"]
    kvs = krr.doc_prefill_batch(model_f16, docs, [f"t{i}" for i in range(12)])
    want, _ = krr.score_batch(model_f16, [("q", k.chunk_id, k, q) for k in kvs], "reuse")
    got = [None] * 4

    def work(i):
        got[i], _ = krr.score_batch(model_f16, [("q", k.chunk_id, k, q) for k in kvs], "reuse")
    th = [threading.Thread(target=work, args=(i,)) for i in range(4)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for g in got:
        assert [r.score for r in g] == [r.score for r in want]


def test_entry_point_errors(c1_golden, model_f16):
    """The public entry points raise the reference's error classes
    (reranker.py:146-151, 154-179, 241-249, 265-290)."""
    from paper_2504_02921_b200.errors import ConfigError, DegenerateInputError, ShapeError
    docs, q = c1_golden["doc_tokens"][:1], c1_golden["query_tokens"]
    kv = krr.doc_prefill_batch(model_f16, docs, ["e0"])[0]
    with pytest.raises(ShapeError):
        krr.score_reuse(model_f16, kv, q[:-1])
    with pytest.raises(DegenerateInputError):
        krr.score_reuse(model_f16, kv, np.zeros_like(q))
    with pytest.raises(ConfigError):
        krr.score_reuse(model_f16, kv, q, path="fused")
    with pytest.raises(ShapeError):
        krr.score_full(model_f16, docs[0][:-1], q)
    with pytest.raises(DegenerateInputError):
        krr.score_full(model_f16, np.zeros_like(docs[0]), q)
    with pytest.raises(ConfigError):
        krr.score_batch(model_f16, [("q", "e0", kv, q)], mode="bogus")
    with pytest.raises(ShapeError):
        krr.score_batch(model_f16, [("q", "e0", docs[0], q)], mode="reuse")
