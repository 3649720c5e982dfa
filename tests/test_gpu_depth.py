"""Full-depth parity, gated per layer with teacher forcing (SURVEY §8(c),
Appendix A): the random-init model amplifies rounding ~1.2x per layer, so
end-to-end 32-layer scores cannot meet 2e-2 for ANY re-implementation (two
fp32 CPU implementations differ by 2.9e-2).  Instead, at layers {0, L/2, L-1}
of the full C3 (7B) and C2 (Gemma) shapes, the GPU's own layer-l input is fed
to the oracle's layer l (weights rounded to the same 16-bit values) and both
layer outputs are compared:

  * doc prefill: layer-l K/V written into the pool page vs the oracle's K/V;
  * query suffix: the residual update x_{l+1} - x_l on top of the GPU's cached
    doc KV (all layers) vs the oracle's.

Gate (f16 operands): relative error <= 2e-2 (norm-wise).
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import oracle  # noqa: E402
import paper_2504_02921_b200 as krr  # noqa: E402
from paper_2504_02921_b200 import engine  # noqa: E402
from paper_2504_02921_b200.config import PRESETS  # noqa: E402

GATE = 2e-2


def rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.mark.parametrize("preset", ["c3_mistral7b", "c2_gemma2b"])
def test_teacher_forced_layers_full_depth(preset):
    cfg, lay = PRESETS[preset]
    L, D, Q, d = cfg.layers, lay.document_len, lay.query_len, cfg.model_dim
    KVH, HD = cfg.kv_heads, cfg.head_dim
    model = krr.RerankModel.build(cfg, lay, precision="f16")
    w = model.weights
    dev = w.device
    rng = np.random.default_rng(17)
    doc = rng.integers(1, cfg.vocab_size, (1, D))
    doc[0, D - 40:] = 0                                   # padded tail
    q = rng.integers(1, cfg.vocab_size, (1, Q))
    pool = krr.KVPool(cfg, D, 1, "f16", dev)
    slot = pool.allocate(["d"])
    engine.prefill_slots(w, pool, slot, doc, [D - 40])
    ptr = pool.slot_ptrs(slot)
    dtok = torch.as_tensor(doc, device=dev, dtype=torch.int32)
    dval = (dtok != 0).to(torch.uint8)
    qtok = torch.as_tensor(q, device=dev, dtype=torch.int32)
    qval = torch.ones_like(qtok, dtype=torch.uint8)
    pvl = torch.tensor([D - 40], dtype=torch.int32, device=dev)
    page = pool.slab[int(slot[0])].float().cpu().numpy()     # [L, 2, KVH, D, HD]
    ocfg = oracle.OracleConfig(layers=L, model_dim=d, heads=cfg.heads, kv_heads=KVH,
                               head_dim=HD, vocab_size=cfg.vocab_size,
                               max_position=cfg.max_position, document_len=D, query_len=Q)
    scratch = torch.empty((1, 1, 2, KVH, Q, HD), dtype=torch.float16, device=dev)
    sptr = torch.tensor([scratch.data_ptr()], dtype=torch.int64, device=dev)
    dscr = torch.empty((1, L, 2, KVH, D, HD), dtype=torch.float16, device=dev)
    dptr = torch.tensor([dscr.data_ptr()], dtype=torch.int64, device=dev)
    for l in sorted({0, L // 2, L - 1}):
        ow = oracle.round_weights(oracle.init_weights(ocfg, layers=[l], with_embedding=False))
        # ---- doc prefill, layer l, teacher-forced on the GPU's layer input
        xd = torch.empty((D, d), dtype=torch.float32, device=dev)
        if l == 0:
            xd = w.token_embedding[dtok[0].long()].clone()
        else:
            engine.run_layers(w, 0, l, dtok, dval, 0, 0, None, None, dptr, L, x_out=xd,
                              cur_pool=dscr)
        torch.cuda.synchronize()
        _, k, v = oracle.forward(ow, doc[0], np.arange(D), valid=doc[0] != 0,
                                 layer_range=[l], x_in=xd.cpu().numpy())
        ek, ev = rel(page[l, 0], k[l]), rel(page[l, 1], v[l])
        print(f"{preset} layer {l}: prefill K {ek:.2e} V {ev:.2e}", end="")
        assert ek <= GATE and ev <= GATE, ("KV", l, ek, ev)
        # ---- query suffix on the cached doc KV, layer l
        xq = torch.empty((Q, d), dtype=torch.float32, device=dev)
        if l == 0:
            xq = w.token_embedding[qtok[0].long()].clone()
        else:
            engine.run_layers(w, 0, l, qtok, qval, D, D, pvl, ptr, sptr, 1, x_out=xq,
                              prefix_pool=pool.slab, cur_pool=scratch)
        xo = torch.empty_like(xq)
        engine.run_layers(w, l, l + 1, qtok, qval, D, D, pvl, ptr, sptr, 1, x_in=xq, x_out=xo,
                          prefix_pool=pool.slab, cur_pool=scratch)
        torch.cuda.synchronize()
        x_in = xq.cpu().numpy()
        valid = np.concatenate([np.arange(D) < D - 40, np.ones(Q, bool)])
        ref, _, _ = oracle.forward(ow, q[0], np.arange(D, D + Q),
                                   past_k=page[:, 0], past_v=page[:, 1], valid=valid,
                                   layer_range=[l], x_in=x_in, return_residual=True)
        err = rel(xo.cpu().numpy() - x_in, ref - x_in)
        print(f"  suffix residual update {err:.2e}")
        assert err <= GATE, ("suffix", l, err)
