"""Max |x| of the residual stream per layer (C3 / C2 shapes, a few pairs) -- is an
unnormalised f16 copy of x safe (f16 max 65504)?"""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_02921_b200 as krr
from paper_2504_02921_b200 import engine
from paper_2504_02921_b200.config import PRESETS
for preset in ("c3_mistral7b", "c2_gemma2b"):
    cfg, lay = PRESETS[preset]
    m = krr.RerankModel.build(cfg, lay, precision="f16")
    w = m.weights
    D, Q, L = lay.document_len, lay.query_len, cfg.layers
    rng = np.random.default_rng(0)
    n = 4
    doc = rng.integers(1, cfg.vocab_size, (n, D))
    pool = krr.KVPool(cfg, D, n, "f16")
    sl = pool.allocate([f"d{i}" for i in range(n)])
    engine.prefill_slots(w, pool, sl, doc, np.full(n, D))
    q = torch.as_tensor(rng.integers(1, cfg.vocab_size, (n, Q)), device="cuda", dtype=torch.int32)
    qv = torch.ones_like(q, dtype=torch.uint8)
    scr = torch.empty((n, 1, 2, cfg.kv_heads, Q, cfg.head_dim), dtype=torch.float16, device="cuda")
    sp = torch.arange(n, device="cuda", dtype=torch.int64) * (scr[0].numel() * 2) + scr.data_ptr()
    out = []
    x = torch.empty((n * Q, cfg.model_dim), dtype=torch.float32, device="cuda")
    for l in range(1, L + 1):
        engine.run_layers(w, 0, l, q, qv, D, D, pool.valid_len[torch.as_tensor(sl, device="cuda")],
                          pool.slot_ptrs(sl), sp, 1, x_out=x, prefix_pool=pool.slab, cur_pool=scr)
        torch.cuda.synchronize()
        rms = x.pow(2).mean(-1).sqrt()
        out.append((l, float(x.abs().max()), float(rms.max())))
    print(preset, "layer, max|x|, max row rms:", [(a, round(b, 1), round(c, 2)) for a, b, c in out[::4] + [out[-1]]])
