"""Cross-query KV reuse inside attention: pairs that share a cached document are
scored as one row group (krr_forward builds the item table; engine.score_slots
sorts pairs by slot).  Every pair's score must be bit-identical to scoring it
alone -- rows of other sequences in a shared item only ever see fully masked
suffix blocks (P = 0) -- across GQA packings where one 256-row item (128 rows at head_dim 256) spans
1-4 sequences and where R is not a multiple of 64 (padded group rows)."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2504_02921_b200 as krr  # noqa: E402
from paper_2504_02921_b200 import engine  # noqa: E402

# (heads, kv_heads, head_dim, query_len): R = heads/kv_heads * query_len rows per sequence
SHAPES = [(4, 2, 64, 48),      # C1 packing: R = 96 -> 128 group rows (padded)
          (8, 2, 128, 48),     # 7B packing: R = 192
          (8, 2, 128, 16),     # R = 64: one item spans 4 sequences
          (4, 1, 128, 100),    # R = 400 -> 448: items straddle sequences unevenly
          (8, 1, 256, 48),     # Gemma packing (head_dim 256, 128-row items): R = 384
          (2, 1, 256, 16)]     # R = 32 -> 64: one 128-row item spans 2 sequences


@pytest.mark.parametrize("H,KVH,HD,Q", SHAPES)
@pytest.mark.parametrize("precision", ["f16", "bf16"])
def test_grouped_scores_equal_single_pair_scores(H, KVH, HD, Q, precision):
    D, n_docs, n_pairs = 128, 5, 29
    cfg = krr.ModelConfig(layers=2, model_dim=H * HD, heads=H, kv_heads=KVH, head_dim=HD,
                          vocab_size=4096)
    model = krr.RerankModel.build(cfg, krr.LayoutConfig(document_len=D, query_len=Q),
                                  precision=precision)
    w = model.weights
    rng = np.random.default_rng(H * 1000 + Q)
    docs = rng.integers(1, cfg.vocab_size, (n_docs, D))
    valid = np.array([D, 77, D, 5, 120])
    for i, v in enumerate(valid):
        docs[i, v:] = 0
    pool = krr.KVPool(cfg, D, n_docs, w.dtype)
    slots = pool.allocate([f"g{i}" for i in range(n_docs)])
    engine.prefill_slots(w, pool, slots, docs, valid)
    pair_doc = rng.integers(0, n_docs, n_pairs)
    pair_doc[:6] = 2                                   # one popular document
    q = rng.integers(1, cfg.vocab_size, (n_pairs, Q))
    q[3, Q - 4:] = 0                                   # padded queries
    q[10, Q // 2:] = 0
    got = engine.score_slots(w, pool, slots[pair_doc], q)
    dev = engine.score_slots(w, pool, torch.as_tensor(slots[pair_doc], device="cuda"), q)
    single = torch.cat([engine.score_slots(w, pool, slots[pair_doc[i:i + 1]], q[i:i + 1])
                        for i in range(n_pairs)])
    torch.cuda.synchronize()
    assert torch.isfinite(got).all()
    assert torch.equal(got, single)
    assert torch.equal(dev, single)

