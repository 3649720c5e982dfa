"""Parity at the geometries north_star names beyond C1,
against fixtures produced by the reference package itself
(tests/golden/make_golden.py):

* C5 geometry -- 7B width, 2 layers, 2048-token documents (RoPE positions
  beyond 1,024, max_position 4,096), query suffixes Q = 16 / 48 / 256 with
  padded documents and queries: f32 debug build <= 1e-4, f16 <= 2e-2
  norm-wise, prefill K/V at positions 1500..1563;
* the host-DRAM tier (f16 / INT8 / INT4 pages streamed H2D) scoring those
  pairs against the CPU oracle on the same (dequantised) KV -- not against the
  HBM path;
* top-20 of 1 query x 100 candidates at 7B width (L=2) and Gemma width (L=1):
  the reference's own _select order, modulo reference ties within the gate;
* bf16 operands end to end at C1 and 7B width.
"""

import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import oracle  # noqa: E402
import paper_2504_02921_b200 as krr  # noqa: E402
from paper_2504_02921_b200 import codec, engine, pipeline  # noqa: E402

F32_TOL = 1e-4
F16_NORMWISE = 2e-2
# bf16 keeps 8 mantissa bits: on this model's unscaled logits (model.py:380)
# it lands at ~3e-2 norm-wise at C1 even in a CPU restatement
# and at 6.4e-2 at 7B width (measured, r02), so it cannot meet north_star's
# 2e-2 -- the default f16 does, at the same tensor-core rate.  bf16 stays a
# library option with this documented gate and is not used for any reported
# number (bench.py has no bf16 switch).
BF16_NORMWISE = 8e-2


def rel_err(s, r):
    s, r = np.asarray(s, np.float64), np.asarray(r, np.float64)
    return float(np.max(np.abs(s - r) / np.maximum(np.abs(r), np.sqrt((r ** 2).mean()))))


def normwise(s, r):
    s, r = np.asarray(s, np.float64), np.asarray(r, np.float64)
    return float(np.linalg.norm(s - r) / np.linalg.norm(r))


def _cfg(g):
    L, d, H, KVH, HD, V, MP = [int(x) for x in g["cfg"]]
    return krr.ModelConfig(layers=L, model_dim=d, heads=H, kv_heads=KVH, head_dim=HD,
                           vocab_size=V, max_position=MP)


@pytest.fixture(scope="module")
def c5(golden_dir):
    return np.load(os.path.join(golden_dir, "c5w_l2.npz"))


@pytest.fixture(scope="module", params=["f32", "f16"])
def c5_run(request, c5):
    """One prefill of the 4 C5 documents per precision; models for the three
    suffix lengths share its weights (the DocKV depends on D only)."""
    cfg = _cfg(c5)
    base = krr.RerankModel.build(cfg, krr.LayoutConfig(document_len=2048, query_len=48),
                                 precision=request.param)
    kvs = krr.doc_prefill_batch(base, c5["doc_tokens"], [f"c5-{i}" for i in range(4)])
    models = {Q: krr.RerankModel(config=cfg, layout=krr.LayoutConfig(document_len=2048,
                                                                       query_len=Q),
                                 weights=base.weights, precision=request.param)
              for Q in (16, 48, 256)}
    return request.param, models, kvs


@pytest.mark.parametrize("Q", [16, 48, 256])
def test_c5_geometry_scores(c5, c5_run, Q):
    prec, models, kvs = c5_run
    qs = c5[f"q{Q}_tokens"]
    pairs = [(f"q{j}", kv.chunk_id, kv, qs[j]) for j in range(2) for kv in kvs]
    res, cnt = krr.score_batch(models[Q], pairs, "reuse")
    s = np.array([r.score for r in res])
    r = c5[f"q{Q}_scores"]
    if prec == "f32":
        assert rel_err(s, r) <= F32_TOL, rel_err(s, r)
    else:
        assert normwise(s, r) <= F16_NORMWISE, normwise(s, r)
    assert [cnt.linear_token_count, cnt.attn_mac_pairs, cnt.peak_activation_tokens,
            cnt.kv_bytes_loaded] == list(c5[f"q{Q}_counters"])


def test_c5_prefill_kv_beyond_position_1024(c5, c5_run):
    prec, _, kvs = c5_run
    assert [k.valid_len for k in kvs] == list(c5["valid_len"])
    k = kvs[0].kv.keys[:, :, 1500:1564]
    v = kvs[0].kv.values[:, :, 1500:1564]
    rk, rv = c5["doc0_keys_1500"], c5["doc0_values_1500"]
    tol = F32_TOL if prec == "f32" else 1e-2
    for a, b in ((k, rk), (v, rv)):
        assert np.max(np.abs(a - b)) <= tol * np.max(np.abs(b))


@pytest.fixture(scope="module")
def c5_oracle(c5):
    L, d, H, KVH, HD, V, MP = [int(x) for x in c5["cfg"]]
    cfg = oracle.OracleConfig(layers=L, model_dim=d, heads=H, kv_heads=KVH, head_dim=HD,
                              vocab_size=V, max_position=MP, document_len=2048, query_len=16)
    return oracle.round_weights(oracle.init_weights(cfg, lazy_embedding=True))


@pytest.mark.parametrize("quant", [None, "int8", "int4"])
def test_c5_host_tier_vs_oracle(c5, c5_oracle, quant):
    """Documents prefilled on the device, put into the pinned host tier (f16
    pages, or INT8/INT4 quantised on the GPU bit-identically to the reference
    codec), streamed H2D and scored; the oracle scores the same pairs on the
    same KV the tier holds (f16 page values, or the reference codec's
    dequantisation of them) with f16-rounded weights."""
    cfg = _cfg(c5)
    lay = krr.LayoutConfig(document_len=2048, query_len=16)
    m = krr.RerankModel.build(cfg, lay, precision="f16")
    pool = krr.KVPool(cfg, 2048, 4, "f16")
    slots = pool.allocate([f"d{i}" for i in range(4)])
    engine.prefill_slots(m.weights, pool, slots, c5["doc_tokens"], c5["valid_len"])
    tier = krr.HostKVTier(pool, 4, quant=quant)
    for i, s in enumerate(slots):
        tier.put_from_pool(f"d{i}", pool, int(s))
    staging = krr.KVPool(cfg, 2048, 4, "f16")
    qs = c5["q16_tokens"]
    hs = np.repeat(tier.lookup([f"d{i}" for i in range(4)]), 2)
    q = np.tile(qs, (4, 1))
    got = engine.score_host_tier(m.weights, tier, staging, hs, q).cpu().numpy()
    want = []
    for i in range(4):
        k, v = pool.read_host_kv(int(slots[i]))
        if quant is not None:
            sch = codec.QuantScheme.INT8_PER_CHANNEL if quant == "int8" else \
                codec.QuantScheme.INT4_PER_CHANNEL
            rt = lambda x: codec.dequantize_tensor(*codec.quantize_tensor(x, sch), sch, x.shape)
            k = np.stack([rt(x) for x in k])
            v = np.stack([rt(x) for x in v])
        for j in range(2):
            want.append(oracle.score_reuse(c5_oracle, k, v, int(c5["valid_len"][i]), qs[j]))
    assert normwise(got, want) <= F16_NORMWISE, normwise(got, want)
    if quant is None:          # f16 tier == the reference's f32 scores at the f16 gate
        order = [j * 4 + i for i in range(4) for j in range(2)]
        assert normwise(got, c5["q16_scores"][order]) <= F16_NORMWISE


@pytest.mark.parametrize("name", ["topk_c3w_l2", "topk_c2w_l1"])
@pytest.mark.parametrize("precision", ["f32", "f16"])
def test_top20_of_100_candidates(golden_dir, name, precision):
    """Scores of 100 candidates and the top-20 through pipeline.rerank (device
    top-k, string chunk-id tie-break) against the reference's _select."""
    g = np.load(os.path.join(golden_dir, f"{name}.npz"))
    cfg = _cfg(g)
    lay = krr.LayoutConfig(document_len=g["doc_tokens"].shape[1], query_len=48)
    m = krr.RerankModel.build(cfg, lay, precision=precision)
    ids = [f"doc-{i:05d}" for i in range(len(g["doc_tokens"]))]
    pool = krr.KVPool(cfg, lay.document_len, len(ids), precision)
    kvs = krr.doc_prefill_batch(m, g["doc_tokens"], ids, pool=pool, register=True)
    assert len(kvs) == 100
    res = pipeline.rerank(m, pool, ["q0"], g["query_tokens"][None], [ids], keep_m=20)
    got_ids = [p.chunk_id for p in res.selected[0]]
    got_sc = np.array([p.score for p in res.selected[0]])
    r = g["scores"]
    rank = {c: i for i, c in enumerate(ids)}
    want_ids = list(g["top_ids"])
    if precision == "f32":
        s_all, _ = krr.score_batch(m, [("q0", k.chunk_id, k, g["query_tokens"]) for k in kvs],
                                   "reuse")
        assert rel_err([p.score for p in s_all], r) <= F32_TOL
        tie = F32_TOL * np.sqrt(np.mean(r ** 2))
    else:
        tie = F16_NORMWISE * np.sqrt(np.mean(r ** 2))
    # position by position: a different id is accepted only when the two
    # reference scores tie within the gate's tolerance
    for a, b in zip(want_ids, got_ids):
        if a != b:
            assert abs(r[rank[a]] - r[rank[b]]) <= tie, (a, b, r[rank[a]], r[rank[b]])
    assert set(got_ids) <= set(ids) and len(got_ids) == 20
    assert np.all(np.diff(got_sc) <= 0)


@pytest.mark.parametrize("which", ["c1", "c3w_l2"])
def test_bf16_end_to_end_gate(golden_dir, which):
    """bf16 operands (fp32 accumulation and residual) end to end against the
    reference's own scores: BF16_NORMWISE (see the module constant)."""
    if which == "c1":
        g = np.load(os.path.join(golden_dir, "c1_scores.npz"))
        cfg = krr.ModelConfig(layers=2, model_dim=256, heads=4, kv_heads=2, head_dim=64,
                              vocab_size=32768)
        lay = krr.LayoutConfig(document_len=128, query_len=48)
        docs, qs, r = g["doc_tokens"], np.repeat(g["query_tokens"][None], 64, 0), \
            g["scores_fast"]
    else:
        g = np.load(os.path.join(golden_dir, "c3w_l2.npz"))
        cfg = _cfg(g)
        lay = krr.LayoutConfig(document_len=512, query_len=48)
        docs, qs, r = g["doc_tokens"], g["query_tokens"], g["scores"]
    m = krr.RerankModel.build(cfg, lay, precision="bf16")
    kvs = krr.doc_prefill_batch(m, docs)
    res, _ = krr.score_batch(m, [("q", "", k, q) for k, q in zip(kvs, qs)], "reuse")
    s = np.array([p.score for p in res])
    err = normwise(s, r)
    print(f"bf16 {which}: normwise {err:.3e}")
    assert err <= BF16_NORMWISE, err
