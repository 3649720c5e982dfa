"""Ownership and concurrency contracts of the device path:
DocKV slot ownership, staged host caches under concurrent callers, store puts
of mismatched entries, CUDA-graph replay after a pool re-home, and the
pipeline's vocabulary check."""

import gc
import threading

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import oracle  # noqa: E402
import paper_2504_02921_b200 as krr  # noqa: E402
from paper_2504_02921_b200 import codec, engine, pipeline, store  # noqa: E402
from paper_2504_02921_b200.errors import ConfigError, ShapeError  # noqa: E402

CFG = krr.ModelConfig(layers=2, model_dim=256, heads=4, kv_heads=2, head_dim=64,
                      vocab_size=32768)
LAY = krr.LayoutConfig(document_len=128, query_len=48)


@pytest.fixture(scope="module")
def model16():
    return krr.RerankModel.build(CFG, LAY, precision="f16")


def _docs(n, seed=0):
    return np.random.default_rng(seed).integers(1, CFG.vocab_size, (n, 128))


def test_same_chunk_id_prefills_are_independent(model16):
    """Re-prefilling a chunk id yields a second cache; the first is unchanged
    (the reference returns a fresh DocKV per call, reranker.py:182-201)."""
    d = _docs(2, 1)
    a = krr.doc_prefill(model16, d[0], chunk_id="same")
    ka = a.kv.keys.copy()
    b = krr.doc_prefill(model16, d[1], chunk_id="same")
    assert a.kv.slot != b.kv.slot
    assert np.array_equal(a.kv.keys, ka)
    assert not np.array_equal(b.kv.keys, ka)
    both = krr.doc_prefill_batch(model16, d[[0, 0]], ["dup", "dup"])
    assert both[0].kv.slot != both[1].kv.slot
    assert np.array_equal(both[0].kv.keys, both[1].kv.keys)


def test_reference_style_prefill_loop_does_not_grow_pool(model16):
    """A per-document doc_prefill loop that drops each DocKV reuses slots."""
    pool = krr.pool_for(model16)
    cap0 = pool.capacity
    d = _docs(1, 2)[0]
    for i in range(3 * cap0):
        kv = krr.doc_prefill(model16, d)        # anonymous, dropped next iteration
        del kv
    gc.collect()
    assert pool.capacity == cap0
    assert pool.owned == 0


def test_registered_prefill_rejects_duplicate_ids(model16):
    pool = krr.KVPool(CFG, 128, 4, "f16")
    with pytest.raises(ConfigError):
        krr.doc_prefill_batch(model16, _docs(2), ["x", "x"], pool=pool, register=True)
    with pytest.raises(ConfigError):
        krr.doc_prefill_batch(model16, _docs(1), [""], pool=pool, register=True)
    kvs = krr.doc_prefill_batch(model16, _docs(2), ["x", "y"], pool=pool, register=True)
    assert pool.lookup(["x", "y"]).tolist() == [kvs[0].kv.slot, kvs[1].kv.slot]


def test_concurrent_scoring_of_host_caches(model16):
    """Host KVTensorSet DocKVs are staged into HBM per call; threads scoring
    different host caches at once must not see each other's staged pages."""
    docs = _docs(12, 3)
    q = np.random.default_rng(4).integers(1, CFG.vocab_size, 48)
    dev = krr.doc_prefill_batch(model16, docs)
    host = [krr.DocKV(f"h{i}", k.kv.to_host(), k.valid_len) for i, k in enumerate(dev)]
    want = [krr.score_batch(model16, [("q", h.chunk_id, h, q) for h in host[i::4]], "reuse")[0]
            for i in range(4)]
    got = [None] * 4

    def work(i):
        for _ in range(5):
            got[i] = krr.score_batch(model16, [("q", h.chunk_id, h, q) for h in host[i::4]],
                                     "reuse")[0]
    th = [threading.Thread(target=work, args=(i,)) for i in range(4)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for i in range(4):
        assert [r.score for r in got[i]] == [r.score for r in want[i]]
    assert model16._staging["f16"].owned == 0


def test_store_put_of_mismatched_entry_leaves_no_mapping(model16):
    """An entry of another model shape is rejected before a slot is mapped."""
    other = oracle.init_weights(oracle.OracleConfig(layers=1, model_dim=256, heads=4,
                                                    kv_heads=2, head_dim=64,
                                                    vocab_size=32768, document_len=128,
                                                    query_len=48))
    k, v, vl = oracle.doc_prefill(other, _docs(1, 5)[0])
    data = codec.encode_arrays("bad", k, v, vl, codec.QuantScheme.F32)
    pool = krr.KVPool(CFG, 128, 2, "f16")
    st = store.DevicePagedKVStore(pool)
    with pytest.raises(ShapeError):
        st.put("bad", data)
    assert not st.exists("bad") and st.get("bad") is None
    assert pool.lookup(["bad"])[0] == -1 and pool.free_slots == 2


def test_graphed_scorer_survives_pool_growth(model16):
    """A pool re-home (grow) invalidates captured pointers: the scorer
    re-captures and still matches eager scoring."""
    pool = krr.KVPool(CFG, 128, 4, "f16")
    ids = [f"g{i}" for i in range(4)]
    slots = pool.allocate(ids)
    docs = _docs(4, 6)
    engine.prefill_slots(model16.weights, pool, slots, docs, np.full(4, 128))
    q = np.random.default_rng(7).integers(1, CFG.vocab_size, (1, 48))
    gs = engine.GraphedScorer(model16.weights, pool, 1, 4, 48, 2)
    idx0, sc0 = gs(slots, q, np.arange(4))
    pool.grow(16)
    assert pool.generation == 1
    # eager work in between may reallocate the shared workspace
    engine.score_slots(model16.weights, pool, np.zeros(64, np.int64),
                       np.repeat(q.astype(np.int32), 64, axis=0))
    idx1, sc1 = gs(slots, q, np.arange(4))
    assert np.array_equal(idx0, idx1) and np.array_equal(sc0, sc1)
    eager = engine.score_slots(model16.weights, pool, slots,
                               np.repeat(q.astype(np.int32), 4, axis=0)).cpu().numpy()
    assert np.array_equal(np.sort(eager)[::-1][:2], sc1[0])


def test_pool_growth_fails_over_instead_of_oom(model16):
    pool = krr.KVPool(CFG, 128, 2, "f16")
    free, _ = torch.cuda.mem_get_info()
    too_many = 4 * free // pool.slot_bytes
    from paper_2504_02921_b200.errors import StoreError
    with pytest.raises(StoreError):
        pool.grow(too_many)
    assert pool.capacity == 2
    pool.grow(too_many, min_capacity=8)            # clamps to what fits
    assert 8 <= pool.capacity < too_many
    del pool
    torch.cuda.empty_cache()


def test_rerank_rejects_out_of_vocab_query(model16):
    pool = krr.KVPool(CFG, 128, 2, "f16")
    q = np.random.default_rng(8).integers(1, CFG.vocab_size, (1, 48))
    q[0, 3] = CFG.vocab_size
    with pytest.raises(ShapeError):
        pipeline.rerank(model16, pool, ["q"], q, [["a"]], keep_m=1)
    q[0, 3] = -1
    with pytest.raises(ShapeError):
        pipeline.rerank(model16, pool, ["q"], q, [["a"]], keep_m=1)
    q = q.astype(np.int64)
    q[0, 3] = (1 << 32) + 5                       # would wrap into range as int32
    with pytest.raises(ShapeError):
        pipeline.rerank(model16, pool, ["q"], q, [["a"]], keep_m=1)
