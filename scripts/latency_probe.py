"""Per-query latency path (1 query x 100 cached docs, engine.score_slots + top-k):
one pass between cudaProfilerStart/Stop for an ncu launch list, plus the eager
wall time and the krr_profile class split.

    python scripts/latency_probe.py [c3_mistral7b|c2_gemma2b] [n_docs]
    ncu --profile-from-start off --metrics gpu__time_duration.sum --csv ... python scripts/latency_probe.py
"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2504_02921_b200 as krr  # noqa: E402
from paper_2504_02921_b200 import _lib, engine  # noqa: E402
from paper_2504_02921_b200.config import PRESETS  # noqa: E402

preset = sys.argv[1] if len(sys.argv) > 1 else "c3_mistral7b"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 100
cfg, lay = PRESETS[preset]
D, Q = lay.document_len, lay.query_len
dev = torch.device("cuda", 0)
model = krr.RerankModel.build(cfg, lay, precision="f16", device=dev)
w = model.weights
pool = krr.KVPool(cfg, D, n, w.dtype, dev)
slots = pool.allocate([f"d{i}" for i in range(n)])
rng = np.random.default_rng(0)
engine.prefill_slots(w, pool, slots, rng.integers(1, cfg.vocab_size, (n, D)), np.full(n, D))
q = torch.as_tensor(rng.integers(1, cfg.vocab_size, (1, Q)), device=dev).to(torch.int32)
qq = q.expand(n, Q).contiguous()
ids = np.arange(n, dtype=np.int32)


def one():
    sc = engine.score_slots(w, pool, slots, qq)
    return engine.segmented_topk(sc, ids, 1, n, 20)


for _ in range(3):
    one()
torch.cuda.synchronize()
ts = []
for _ in range(10):
    t0 = time.perf_counter()
    one()
    torch.cuda.synchronize()
    ts.append((time.perf_counter() - t0) * 1e3)
_lib.profile_enable(True)
one()
torch.cuda.synchronize()
p = _lib.profile_read()
_lib.profile_enable(False)
print(f"{preset} 1 q x {n} docs: p50 {np.median(ts):.2f} ms; classes gemm {p['gemm_ms']:.2f} "
      f"attn {p['attn_ms']:.2f} misc {p['misc_ms']:.2f} ms; gemm {p['gemm_flops'] / p['gemm_ms'] / 1e9:.0f} TF/s",
      flush=True)
torch.cuda.cudart().cudaProfilerStart()
one()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
