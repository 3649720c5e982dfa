"""The drop-in boundary: the reference package's OWN entry points
(kvrerank.reranker.doc_prefill / score_reuse / score_batch / score_full) run
with its operator switch ``_forward_fn`` pointed at this build's
``forward`` -- exactly the binding INTEGRATION.md shows -- and reproduce the
reference's fast-path goldens.

The reference is imported from ``baseline/_ref`` (installed unmodified from
/root/reference with pip, git-ignored, shipped to the GPU box by gpurun)."""

import os
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import oracle  # noqa: E402
import paper_2504_02921_b200 as krr  # noqa: E402
from paper_2504_02921_b200 import forward as b200_forward  # noqa: E402
from paper_2504_02921_b200.errors import PositionError, ShapeError  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")


@pytest.fixture(scope="module")
def ref():
    if not os.path.isdir(os.path.join(REF, "kvrerank")):
        pytest.fail("baseline/_ref/kvrerank is not staged (see DESIGN.md §5: "
                    "pip install --target baseline/_ref /root/reference/pkg)")
    sys.path.insert(0, REF)
    try:
        import kvrerank
        from kvrerank import model, reranker
    finally:
        sys.path.remove(REF)
    assert os.path.realpath(kvrerank.__file__).startswith(os.path.realpath(REF))
    return model, reranker


@pytest.fixture(scope="module")
def c1(golden_dir):
    return np.load(os.path.join(golden_dir, "c1_scores.npz"))


@pytest.fixture(scope="module")
def ref_model(ref):
    model, reranker = ref
    cfg = model.ModelConfig(layers=2, model_dim=256, heads=4, kv_heads=2, head_dim=64,
                            vocab_size=32768, seed=0)
    return reranker.RerankModel.build(cfg, reranker.LayoutConfig(document_len=128, query_len=48))


@pytest.fixture
def patched(ref, monkeypatch):
    """The reference's operator switch with the two paths INTEGRATION.md §2 adds."""
    _, reranker = ref
    orig = reranker._forward_fn

    def _forward_fn(path):
        if path in ("b200", "b200_f16"):
            return krr.forward_fn("f32" if path == "b200" else "f16")
        return orig(path)
    monkeypatch.setattr(reranker, "_forward_fn", _forward_fn)
    return reranker


def _err(s, r):
    s, r = np.asarray(s, np.float64), np.asarray(r, np.float64)
    return float(np.max(np.abs(s - r)) / max(np.max(np.abs(r)), np.sqrt(np.mean(r * r))))


def test_reference_entry_points_through_b200_forward(patched, ref_model, c1):
    """doc_prefill + score_batch(reuse) of the reference, computed by the B200
    forward (f32 debug build): scores within 1e-4 of the reference's own fast
    path, DocKVs within 1e-4, counters identical."""
    R = patched
    docs, q = c1["doc_tokens"][:16], c1["query_tokens"]
    kvs = [R.doc_prefill(ref_model, d, chunk_id=f"doc-{i:05d}", path="b200")
           for i, d in enumerate(docs)]
    k0 = np.asarray(kvs[0].kv.keys)
    assert k0.shape == c1["doc0_keys"].shape
    assert np.max(np.abs(k0 - c1["doc0_keys"])) <= 1e-4 * np.max(np.abs(c1["doc0_keys"]))
    assert np.max(np.abs(np.asarray(kvs[1].kv.values) - c1["doc1_values"])) <= \
        1e-4 * np.max(np.abs(c1["doc1_values"]))
    scored, counters = R.score_batch(ref_model, [("q0", kv.chunk_id, kv, q) for kv in kvs],
                                     mode="reuse", path="b200")
    assert _err([p.score for p in scored], c1["scores_fast"][:16]) <= 1e-4
    # counters are closed-form (reranker.py:293-300): the first 16 of 64 pairs
    want = c1["counters"]
    assert counters.linear_token_count == want[0] // 4
    assert counters.kv_bytes_loaded == want[3] // 4
    s, _ = R.score_reuse(ref_model, kvs[2], q, path="b200")
    assert abs(s - c1["scores_fast"][2]) <= 1e-4 * max(1.0, abs(c1["scores_fast"][2]))
    full = [R.score_full(ref_model, docs[i], q, path="b200")[0] for i in range(2)]
    assert _err(full, c1["scores_full_fast"][:2]) <= 1e-4


def test_reference_entry_points_f16(patched, ref_model, c1):
    """Same entry points on the tensor-core build (f16 operands): 2e-2 norm-wise."""
    R = patched
    docs, q = c1["doc_tokens"][:8], c1["query_tokens"]
    kvs = [R.doc_prefill(ref_model, d, path="b200_f16") for d in docs]
    scored, _ = R.score_batch(ref_model, [("q0", f"d{i}", kv, q) for i, kv in enumerate(kvs)],
                              mode="reuse", path="b200_f16")
    s = np.array([p.score for p in scored])
    r = c1["scores_fast"][:8]
    assert np.linalg.norm(s - r) / np.linalg.norm(r) <= 2e-2


def test_forward_matches_reference_forward(ref, ref_model, c1):
    """forward() itself against the reference's forward on the same call,
    including padded past / current masks."""
    model, _ = ref
    w = ref_model.weights
    d, q = c1["doc_tokens"][3].copy(), c1["query_tokens"].copy()
    d[100:] = 0
    q[[5, 6]] = 0
    dv = d != 0
    h_ref, kv_ref = model.forward(w, d, np.arange(128), None, dv)
    h, kv = b200_forward(w, d, np.arange(128), None, dv)
    assert _err(h, h_ref) <= 1e-4 and _err(kv.keys, kv_ref.keys) <= 1e-4
    assert kv.position_offset == 0
    valid = np.concatenate([dv, q != 0])
    h_ref, kv2_ref = model.forward(w, q, np.arange(128, 176), kv_ref, valid)
    h, kv2 = b200_forward(w, q, np.arange(128, 176), kv_ref, valid)
    assert _err(h, h_ref) <= 1e-4
    assert _err(kv2.values, kv2_ref.values) <= 1e-4 and kv2.position_offset == 128


def test_forward_arbitrary_positions(ref, ref_model):
    """Strictly increasing positions with gaps (model.py:358 takes any): RoPE
    uses the given positions (krr_batch_t.positions)."""
    model, _ = ref
    w = ref_model.weights
    toks = np.random.default_rng(3).integers(1, 32768, 40)
    pos = np.cumsum(np.random.default_rng(4).integers(1, 7, 40)) + 11
    h_ref, kv_ref = model.forward(w, toks, pos)
    h, kv = b200_forward(w, toks, pos)
    assert _err(h, h_ref) <= 1e-4 and _err(kv.keys, kv_ref.keys) <= 1e-4
    assert kv.position_offset == pos[0]


def test_forward_errors_match_reference(ref, ref_model):
    model, _ = ref
    w = ref_model.weights
    toks = np.arange(1, 11)
    for args, exc in [((toks, np.arange(10)[::-1]), ShapeError),
                      ((toks, np.arange(1020, 1030)), PositionError),
                      ((toks, np.arange(9)), ShapeError),
                      ((np.array([], np.int64), np.array([], np.int64)), ShapeError),
                      ((np.array([1, 40000]), np.arange(2)), ShapeError)]:
        with pytest.raises(Exception) as e_ref:
            model.forward(w, *args)
        with pytest.raises(exc):
            b200_forward(w, *args)
        assert type(e_ref.value).__name__ == exc.__name__
    # all keys masked -> zeros (model.py:225-230)
    h, kv = b200_forward(w, toks, np.arange(10), None, np.zeros(10, bool))
    assert not h.any() and not kv.keys.any()


def test_forward_accepts_device_kv_past(ref_model, c1):
    """A DeviceKV page from this build's doc_prefill is a valid ``past``."""
    m = krr.RerankModel.build(krr.ModelConfig(layers=2, model_dim=256, heads=4, kv_heads=2,
                                              head_dim=64, vocab_size=32768),
                              krr.LayoutConfig(document_len=128, query_len=48),
                              precision="f32")
    d, q = c1["doc_tokens"][0], c1["query_tokens"]
    kv = krr.doc_prefill(m, d).kv
    valid = np.concatenate([d != 0, q != 0])
    h_dev, _ = b200_forward(m, q, np.arange(128, 176), kv, valid)
    h_host, _ = b200_forward(m, q, np.arange(128, 176), kv.to_host(), valid)
    assert np.array_equal(h_dev, h_host)
    s = float(np.dot(h_dev[47], m.weights.score_head[0].cpu().numpy()))
    assert abs(s - c1["scores_fast"][0]) <= 1e-4 * max(1.0, abs(c1["scores_fast"][0]))
