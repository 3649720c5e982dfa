"""C5 host tier: engine.score_host_tier with the in-attention dequant (fused) vs
the expand pass, per page format and query length; per-class device time
(krr_profile: gemm / attention / misc) to see where a step goes."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2504_02921_b200 as krr  # noqa: E402
from paper_2504_02921_b200 import _lib, engine  # noqa: E402
from paper_2504_02921_b200.config import PRESETS  # noqa: E402

cfg, lay = PRESETS["c5_mistral7b_d2048"]
D, N = lay.document_len, 48
dev = torch.device("cuda", 0)
model = krr.RerankModel.build(cfg, lay, precision="f16", device=dev)
w = model.weights
tmp = krr.KVPool(cfg, D, 8, w.dtype, dev)
docs = np.random.default_rng(0).integers(1, cfg.vocab_size, (8, D))
sl = tmp.allocate([f"d{i}" for i in range(8)])
engine.prefill_slots(w, tmp, sl, docs, np.full(8, D))
staging = krr.KVPool(cfg, D, 16, w.dtype, dev)
cs = torch.cuda.Stream(device=dev)
orig = engine.fused_dequant_supported
for quant in ("int8", "int4"):
    tier = krr.HostKVTier(tmp, N, quant=quant)
    for i in range(N):
        tier.put_from_pool(f"h{i}", tmp, int(sl[i % 8]))
    hs = np.arange(N)
    for Q in (16, 256):
        q = np.random.default_rng(1).integers(1, cfg.vocab_size, (N, Q))
        for fused in (True, False):
            engine.fused_dequant_supported = orig if fused else (lambda w: False)
            for _ in range(2):
                engine.score_host_tier(w, tier, staging, hs, q, copy_stream=cs)
            torch.cuda.synchronize()
            _lib.profile_enable(True)
            t0 = time.perf_counter()
            for _ in range(3):
                engine.score_host_tier(w, tier, staging, hs, q, copy_stream=cs)
            torch.cuda.synchronize()
            dt = (time.perf_counter() - t0) / 3 * 1e3
            p = _lib.profile_read()
            _lib.profile_enable(False)
            print(f"{quant} Q={Q:3d} fused={fused!s:5}: {dt:7.1f} ms/step = {N / dt * 1e3:6.1f} "
                  f"pairs/s | per step gemm {p['gemm_ms'] / 3:6.1f} attn {p['attn_ms'] / 3:6.1f} "
                  f"misc {p['misc_ms'] / 3:5.1f} ms ({p['attn_launches'] // 3} attn launches)",
                  flush=True)
    engine.fused_dequant_supported = orig
    del tier
