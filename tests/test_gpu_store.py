"""Device side of the KV-store interface: HRKV entries written by the
reference (tests/golden/codec_c1.npz) decoded into HBM pool pages (F32 cast,
INT8/INT4 dequant kernel), DevicePagedKVStore, populate_store, the rerank
stage with cache misses, and the sharded top-k merge on the CUDA kernel."""

import os
from dataclasses import dataclass

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import oracle  # noqa: E402
import paper_2504_02921_b200 as krr  # noqa: E402
from paper_2504_02921_b200 import codec, engine, pipeline, shard, store  # noqa: E402

C1 = (krr.ModelConfig(layers=2, model_dim=256, heads=4, kv_heads=2, head_dim=64,
                      vocab_size=32768),
      krr.LayoutConfig(document_len=128, query_len=48))


@pytest.fixture(scope="module")
def g(golden_dir):
    return np.load(os.path.join(golden_dir, "codec_c1.npz"))


@pytest.fixture(scope="module")
def model32():
    return krr.RerankModel.build(*C1, precision="f32")


@pytest.fixture(scope="module")
def model16():
    return krr.RerankModel.build(*C1, precision="f16")


@pytest.mark.parametrize("name", ["f32", "int8", "int4"])
def test_entry_to_pool_matches_reference_decode(g, model32, name):
    pool = krr.KVPool(C1[0], 128, 4, "f32")
    kv = codec.decode_entry_to_pool(g[f"entry_{name}"].tobytes(), pool)
    torch.cuda.synchronize()
    assert kv.chunk_id == "doc-00042" and kv.valid_len == 90
    k, v = pool.read_host_kv(kv.kv.slot)
    assert np.array_equal(k, g[f"decoded_keys_{name}"])
    assert np.array_equal(v, g[f"decoded_values_{name}"])


def test_entry_to_f16_pool(g):
    pool = krr.KVPool(C1[0], 128, 2, "f16")
    kv = codec.decode_entry_to_pool(g["entry_int8"].tobytes(), pool)
    k, _ = pool.read_host_kv(kv.kv.slot)
    want = g["decoded_keys_int8"].astype(np.float16).astype(np.float32)
    assert np.array_equal(k, want)


def test_f16_entries_through_device_store(g, model16):
    """Scheme code 1 (F16): put lands the exact f16 values in an f16 pool page,
    get with export_scheme=F16 returns the same bytes (the page itself), and
    an F32 export of that page decodes to the same values."""
    cid, k, v, vl = codec.decode_arrays(g["entry_f32"].tobytes())
    data = codec.encode_arrays(cid, np.array(k), np.array(v), vl, codec.QuantScheme.F16)
    pool = krr.KVPool(C1[0], 128, 2, "f16")
    dev = store.DevicePagedKVStore(pool, export_scheme=codec.QuantScheme.F16)
    dev.put(cid, data)
    slot = int(pool.lookup([cid])[0])
    kk, vv = pool.read_host_kv(slot)
    assert np.array_equal(kk, np.asarray(k).astype(np.float16).astype(np.float32))
    assert np.array_equal(vv, np.asarray(v).astype(np.float16).astype(np.float32))
    assert dev.get(cid) == data
    f32 = codec.encode_pool_page(cid, pool, slot, codec.QuantScheme.F32)
    _, k3, v3, vl3 = codec.decode_arrays(f32)
    assert vl3 == vl and np.array_equal(k3, kk) and np.array_equal(v3, vv)


def test_device_store_scores_like_reference_entry(g, model32):
    """An F32 entry written by the reference, put into a device shard, scores
    like the oracle on the same KV (f32 debug build, 1e-4 gate)."""
    pool = krr.pool_for(model32, "fast")
    st = krr.ShardedStore([store.MemoryBackend(), store.DevicePagedKVStore(pool)])
    st.put_entry("doc-00042", 1, g["entry_f32"].tobytes())
    assert st.exists_entry("doc-00042", 1) and not st.exists_entry("doc-00042", 0)
    dkv = st.backends[1].doc_kv("doc-00042")
    q = np.random.default_rng(3).integers(1, 32768, 48)
    s, c = krr.score_reuse(model32, dkv, q)
    w = oracle.init_weights(oracle.OracleConfig(layers=2, model_dim=256, heads=4, kv_heads=2,
                                                head_dim=64, vocab_size=32768,
                                                document_len=128, query_len=48))
    _, k, v, vl = codec.decode_arrays(g["entry_f32"].tobytes())
    ref = oracle.score_reuse(w, k, v, vl, q)
    assert abs(s - ref) <= 1e-4 * max(1.0, abs(ref))
    assert c.kv_bytes_loaded == 262144
    back = st.get_entry("doc-00042", 1)           # re-encoded F32 bytes
    assert back == g["entry_f32"].tobytes()        # f32 pool: exact round trip


@dataclass
class Doc:
    id: str
    text: str


class CentroidIndex:
    def centroid_of(self, doc_id):
        return int(doc_id.split("-")[1]) % 5


def _docs(n):
    rng = np.random.default_rng(11)
    words = [f"w{i}" for i in range(5000)]
    return [Doc(f"doc-{i:05d}", " ".join(rng.choice(words, rng.integers(60, 200))))
            for i in range(n)]


def test_populate_store_device_and_bytes_backends(model16):
    docs = _docs(12)
    pool = krr.KVPool(C1[0], 128, 16, "f16")
    st = krr.ShardedStore([store.MemoryBackend(), store.DevicePagedKVStore(pool),
                           store.MemoryBackend()])
    seen = []
    total = krr.populate_store(model16, docs, CentroidIndex(), st,
                               on_entry=lambda i, n: seen.append((i, n)))
    assert len(seen) == 12 and total == sum(n for _, n in seen)
    per = codec.HEADER.size + len("doc-00000") + codec.payload_nbytes(2, 2, 128, 64,
                                                                      codec.QuantScheme.F32)
    assert all(n == per for _, n in seen)
    for d in docs:
        sh = st.shard_for(CentroidIndex().centroid_of(d.id))
        assert st.exists_entry(d.id, CentroidIndex().centroid_of(d.id))
        if sh == 1:
            assert d.id in pool
    # bytes shards hold reference-format entries that decode to the same KV
    d0 = [d for d in docs if st.shard_for(CentroidIndex().centroid_of(d.id)) == 0][0]
    cid, k, _, vl = codec.decode_arrays(st.get_entry(d0.id, CentroidIndex().centroid_of(d0.id)))
    toks = krr.tokenize(d0.text, 128)
    again = krr.doc_prefill(model16, toks, "again")
    assert cid == d0.id and vl == again.valid_len
    assert np.array_equal(k, again.kv.keys)


def test_rerank_with_cache_misses_equals_full(model16):
    rng = np.random.default_rng(5)
    docs = rng.integers(1, 32768, (10, 128))
    ids = [f"doc-{i:05d}" for i in range(10)]
    pool = krr.KVPool(C1[0], 128, 10, "f16")
    slots = pool.allocate(ids[:6])
    engine.prefill_slots(model16.weights, pool, slots, docs[:6], np.full(6, 128))
    q = rng.integers(1, 32768, (2, 48))
    cands = [ids[:5] + ids[8:], ids[3:8]]
    res = pipeline.rerank(model16, pool, ["qa", "qb"], q, cands, keep_m=3,
                          doc_tokens=dict(zip(ids, docs)))
    assert res.cache_misses == 4 and res.pairs == 12
    for qi in range(2):
        full, _ = krr.score_batch(model16, [("q", c, docs[ids.index(c)], q[qi])
                                            for c in cands[qi]], "full")
        want = krr.select(full, 3)
        assert [p.chunk_id for p in res.selected[qi]] == [p.chunk_id for p in want]
        assert [p.score for p in res.selected[qi]] == [p.score for p in want]


def test_rerank_graph_replay_matches_eager(model16, monkeypatch):
    """A repeated latency-sized rerank shape replays a captured CUDA graph
    (pipeline._graph_for): selections and scores equal the eager path bit for
    bit, new queries / candidate orders are picked up on every replay, and
    ragged or missing candidates keep the eager path."""
    rng = np.random.default_rng(11)
    docs = rng.integers(1, 32768, (8, 128))
    ids = [f"doc-{i:05d}" for i in range(8)]
    pool = krr.KVPool(C1[0], 128, 8, "f16")
    slots = pool.allocate(ids)
    engine.prefill_slots(model16.weights, pool, slots, docs, np.full(8, 128))

    def eager(q, cands, k):
        monkeypatch.setattr(pipeline, "GRAPH_MAX_ROWS", 0)
        try:
            return pipeline.rerank(model16, pool, ["qa", "qb"], q, cands, keep_m=k)
        finally:
            monkeypatch.undo()

    for trial in range(4):                 # 1st call eager, 2nd captures, then replays
        q = rng.integers(1, 32768, (2, 48))
        cands = [list(rng.permutation(ids)[:6]) for _ in range(2)]
        got = pipeline.rerank(model16, pool, ["qa", "qb"], q, cands, keep_m=3)
        want = eager(q, cands, 3)
        for a, b in zip(got.selected, want.selected):
            assert [p.chunk_id for p in a] == [p.chunk_id for p in b]
            assert [p.score for p in a] == [p.score for p in b]
    assert len(pool._rerank_graphs) == 1
    q = rng.integers(1, 32768, (2, 48))
    ragged = [ids[:6], ids[2:5]]
    res = pipeline.rerank(model16, pool, ["qa", "qb"], q, ragged, keep_m=3)
    want = eager(q, ragged, 3)
    assert [[p.score for p in r] for r in res.selected] == \
        [[p.score for p in r] for r in want.selected]
    assert len(pool._rerank_graphs) == 1


def test_sharded_select_on_device_matches_single():
    """shard.sharded_select host logic with the CUDA top-k kernel, world=1 and
    a simulated 4-way split merged by the same kernel."""
    rng = np.random.default_rng(0)
    n_q, n_c, k = 8, 100, 20
    cand = np.stack([rng.choice(1000, n_c, replace=False) for _ in range(n_q)])
    table = np.round(rng.standard_normal((n_q, 1000)), 2).astype(np.float32)
    want = []
    for qi in range(n_q):
        sc = [float(table[qi, d]) for d in cand[qi]]
        want.append([int(cand[qi][j]) for j in
                     oracle.select_topk(sc, [f"doc-{d:05d}" for d in cand[qi]], k)])
    parts = []
    for r in range(4):
        w = shard.local_work(cand, r, 4)
        doc = cand[w.pair_query, w.pair_cand]
        s = torch.as_tensor(table[w.pair_query, doc], device="cuda")
        i = torch.as_tensor(doc.astype(np.int32), device="cuda")
        parts.append(shard.local_topk(s, i, w, n_q, k, engine.segmented_topk))
    cs = torch.cat([p[0] for p in parts], 1).contiguous()
    ci = torch.cat([p[1] for p in parts], 1).contiguous()
    idx, _ = engine.segmented_topk(cs.view(-1), ci.view(-1), n_q, 4 * k, k)
    got = ci.gather(1, idx.long()).cpu().numpy().tolist()
    assert got == want


def test_host_tier_streaming_matches_device_pool(model16):
    """Docs in the pinned host tier, streamed H2D through a 2x2-slot staging
    pool on a side stream, score bit-identically to the same docs resident in
    HBM (batch-invariant kernels; PCIe only moves bytes)."""
    rng = np.random.default_rng(21)
    n_docs = 7
    docs = rng.integers(1, 32768, (n_docs, 128))
    docs[2, 90:] = 0
    pool = krr.KVPool(C1[0], 128, n_docs, "f16")
    slots = pool.allocate([f"d{i}" for i in range(n_docs)])
    engine.prefill_slots(model16.weights, pool, slots, docs, (docs != 0).sum(axis=1))
    tier = krr.HostKVTier(pool, n_docs)
    hslots = [tier.put_from_pool(f"d{i}", pool, int(s)) for i, s in enumerate(slots)]
    pair_doc = rng.integers(0, n_docs, 20)
    q = rng.integers(1, 32768, (20, 48))
    staging = krr.KVPool(C1[0], 128, 4, "f16")
    got = engine.score_host_tier(model16.weights, tier, staging, np.asarray(hslots)[pair_doc], q)
    want = engine.score_slots(model16.weights, pool, slots[pair_doc], q)
    torch.cuda.synchronize()
    assert torch.equal(got, want)


@pytest.mark.parametrize("bits,scheme", [(8, codec.QuantScheme.INT8_PER_CHANNEL),
                                         (4, codec.QuantScheme.INT4_PER_CHANNEL)])
@pytest.mark.parametrize("src", ["f32", "f16"])
@pytest.mark.parametrize("HD", [64, 40])               # 40: the scalar (non-vector) dequant
def test_quant_pages_bit_exact_vs_host_codec(bits, scheme, src, HD):
    """krr_quant_pages / krr_dequant_pages == codec.quantize_tensor /
    dequantize_tensor (the reference's codec.py:58-95 semantics), tensor by tensor."""
    from paper_2504_02921_b200 import _lib
    rng = np.random.default_rng(bits)
    n, KVH, D = 4, 2, 37                                # odd D*... exercises int4 packing
    x = (rng.standard_normal((n, KVH, D, HD)) * 3).astype(np.float32)
    x[1, 0, :, 5] = 0.0                                 # all-zero channel -> scale 1
    x[2, 1, 3, 7] = 2.5                                 # exact .5 tie after scaling is likely
    if src == "f16":
        x = x.astype(np.float16).astype(np.float32)
    xt = torch.as_tensor(x, device="cuda").to(torch.float16 if src == "f16" else torch.float32)
    te = KVH * D * HD
    tb = te if bits == 8 else (te + 1) // 2
    codes = torch.empty(n * tb, dtype=torch.uint8, device="cuda")
    scales = torch.empty(n * KVH * HD, dtype=torch.float32, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    _lib.check(_lib.lib().krr_quant_pages(xt.data_ptr(), _lib.F16 if src == "f16" else _lib.F32,
                                          n, KVH, D, HD, bits, codes.data_ptr(),
                                          scales.data_ptr(), s))
    out = torch.empty(n, KVH, D, HD, dtype=torch.float32, device="cuda")
    _lib.check(_lib.lib().krr_dequant_pages(codes.data_ptr(), scales.data_ptr(), bits, n, KVH, D,
                                            HD, _lib.F32, out.data_ptr(), s))
    torch.cuda.synchronize()
    c_h, s_h, o_h = codes.cpu().numpy(), scales.cpu().numpy(), out.cpu().numpy()
    for t in range(n):
        q, sc = codec.quantize_tensor(x[t], scheme)
        assert c_h[t * tb:(t + 1) * tb].tobytes() == q, t
        assert np.array_equal(s_h[t * KVH * HD:(t + 1) * KVH * HD].reshape(KVH, HD), sc), t
        assert np.array_equal(o_h[t], codec.dequantize_tensor(q, sc, scheme, (KVH, D, HD))), t
    # 16-bit landing (the staging-pool path): the f32 product rounded once
    o16 = torch.empty(n, KVH, D, HD, dtype=torch.float16, device="cuda")
    _lib.check(_lib.lib().krr_dequant_pages(codes.data_ptr(), scales.data_ptr(), bits, n, KVH, D,
                                            HD, _lib.F16, o16.data_ptr(), s))
    torch.cuda.synchronize()
    assert np.array_equal(o16.cpu().numpy(), o_h.astype(np.float16))


@pytest.mark.parametrize("fused", [True, False])
@pytest.mark.parametrize("quant,scheme", [("int8", codec.QuantScheme.INT8_PER_CHANNEL),
                                          ("int4", codec.QuantScheme.INT4_PER_CHANNEL)])
def test_quantised_host_tier_matches_hrkv_entries(model16, quant, scheme, fused, monkeypatch):
    """A quantised host tier scores like the same docs stored as HRKV INT8/INT4
    entries (reference codec) and decoded into HBM: exactly with the separate
    expand pass into the staging pool, and within the f16 rounding of the
    scales (2^-11 per K/V element) with the codes dequantised inside attention
    (the default)."""
    assert engine.fused_dequant_supported(model16.weights)
    if not fused:
        monkeypatch.setattr(engine, "fused_dequant_supported", lambda w: False)
    calls = []
    orig_expand = krr.HostKVTier.expand
    monkeypatch.setattr(krr.HostKVTier, "expand",
                        lambda self, *a, **k: (calls.append(1), orig_expand(self, *a, **k)))
    rng = np.random.default_rng(31)
    n_docs = 5
    docs = rng.integers(1, 32768, (n_docs, 128))
    pool = krr.KVPool(C1[0], 128, n_docs, "f16")
    slots = pool.allocate([f"d{i}" for i in range(n_docs)])
    engine.prefill_slots(model16.weights, pool, slots, docs, np.full(n_docs, 128))
    tier = krr.HostKVTier(pool, n_docs, quant=quant)
    hs = np.array([tier.put_from_pool(f"d{i}", pool, int(s)) for i, s in enumerate(slots)])
    assert tier.slot_bytes < pool.slot_bytes
    ref_pool = krr.KVPool(C1[0], 128, n_docs, "f16")
    ref_slots = []
    for i, s in enumerate(slots):
        kv = krr.DocKV(f"e{i}", krr.DeviceKV(pool, int(s)), 128)
        entry = codec.encode_entry(kv, scheme)
        ref_slots.append(codec.decode_entry_to_pool(entry, ref_pool).kv.slot)
    pair_doc = rng.integers(0, n_docs, 12)
    q = rng.integers(1, 32768, (12, 48))
    staging = krr.KVPool(C1[0], 128, 2, "f16")
    got = engine.score_host_tier(model16.weights, tier, staging, hs[pair_doc], q)
    want = engine.score_slots(model16.weights, ref_pool, np.array(ref_slots)[pair_doc], q)
    torch.cuda.synchronize()
    if fused:
        normwise = ((got - want).norm() / want.norm()).item()
        assert normwise <= 5e-3, normwise
    else:
        assert torch.equal(got, want)
    assert (len(calls) == 0) == fused


def test_host_dockv_from_reference_entry_scores(g, model32, model16):
    """Reference-style usage: decode_entry() gives a host f32 DocKV (zero-copy
    view over the HRKV bytes) and score_reuse / score_batch stage it into HBM;
    f32 debug build matches the oracle, f16 path within the 16-bit gate, and a
    mixed batch (host + device DocKVs) scores each pair like its single call."""
    data = g["entry_f32"].tobytes()
    dkv = codec.decode_entry(data)
    assert isinstance(dkv.kv, krr.KVTensorSet) and dkv.valid_len == 90
    q = np.random.default_rng(8).integers(1, 32768, 48)
    w = oracle.init_weights(oracle.OracleConfig(layers=2, model_dim=256, heads=4, kv_heads=2,
                                                head_dim=64, vocab_size=32768,
                                                document_len=128, query_len=48))
    ref = oracle.score_reuse(w, dkv.kv.keys, dkv.kv.values, dkv.valid_len, q)
    s32, c = krr.score_reuse(model32, dkv, q)
    assert abs(s32 - ref) <= 1e-4 * max(1.0, abs(ref))
    assert c.kv_bytes_loaded == 262144 and c.linear_token_count == 48
    s16, _ = krr.score_reuse(model16, dkv, q)
    assert abs(s16 - ref) <= 2e-2 * max(1.0, abs(ref))
    dev = krr.doc_prefill(model16, g["doc_tokens"], "dev")
    res, _ = krr.score_batch(model16, [("q", "h", dkv, q), ("q", "dev", dev, q)], "reuse")
    assert res[0].score == s16
    assert res[1].score == krr.score_reuse(model16, dev, q)[0]


def test_graphed_scorer_matches_eager(model16):
    """CUDA-graph replay of the scoring pass gives the eager scores and top-k,
    and picks up new inputs on every replay."""
    rng = np.random.default_rng(9)
    docs = rng.integers(1, 32768, (6, 128))
    pool = krr.KVPool(C1[0], 128, 6, "f16")
    slots = pool.allocate([f"g{i}" for i in range(6)])
    engine.prefill_slots(model16.weights, pool, slots, docs, np.full(6, 128))
    gs = engine.GraphedScorer(model16.weights, pool, 2, 6, 48, 3)
    for trial in range(2):
        q = rng.integers(1, 32768, (2, 48))
        perm = np.stack([rng.permutation(6) for _ in range(2)])
        sl = slots[perm].reshape(-1)
        idx, sc = gs(sl, q, perm.reshape(-1))
        want = engine.score_slots(model16.weights, pool, sl, np.repeat(q, 6, axis=0)).cpu().numpy()
        for qi in range(2):
            seg = want[qi * 6:(qi + 1) * 6]
            order = sorted(range(6), key=lambda j: (-seg[j], perm[qi, j]))[:3]
            assert idx[qi].tolist() == order
            assert np.array_equal(sc[qi], seg[order])


def test_graphed_scorer_replay_device_matches_host_call(model16):
    """replay_device (device-resident inputs, bench's latency-sized timed step)
    returns the same top-k as the host-buffer call and counts its launches."""
    import torch
    rng = np.random.default_rng(11)
    docs = rng.integers(1, 32768, (6, 128))
    pool = krr.KVPool(C1[0], 128, 6, "f16")
    slots = pool.allocate([f"d{i}" for i in range(6)])
    engine.prefill_slots(model16.weights, pool, slots, docs, np.full(6, 128))
    gs = engine.GraphedScorer(model16.weights, pool, 2, 6, 48, 3)
    assert gs.launches > 0
    q = rng.integers(1, 32768, (2, 48))
    perm = np.stack([rng.permutation(6) for _ in range(2)])
    sl = slots[perm].reshape(-1)
    idx_h, sc_h = gs(sl, q, perm.reshape(-1))
    dev = model16.weights.device
    idx_d, sc_d = gs.replay_device(torch.as_tensor(sl, device=dev),
                                   torch.as_tensor(q.astype(np.int32), device=dev),
                                   torch.as_tensor(perm.reshape(-1).astype(np.int32), device=dev))
    assert np.array_equal(idx_d.cpu().numpy(), idx_h)
    assert np.array_equal(sc_d.cpu().numpy(), sc_h)
