"""Compare the fused-RMSNorm and unfused layer loops layer by layer (x_out)."""
import os, subprocess, sys, json
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_02921_b200 as krr
from paper_2504_02921_b200 import engine
from paper_2504_02921_b200.config import PRESETS
preset = sys.argv[1] if len(sys.argv) > 1 else "c3_mistral7b"
cfg, lay = PRESETS[preset]
m = krr.RerankModel.build(cfg, lay, precision="f16")
w = m.weights
D, L = lay.document_len, cfg.layers
rng = np.random.default_rng(17)
doc = torch.as_tensor(rng.integers(1, cfg.vocab_size, (1, D)), device="cuda", dtype=torch.int32)
dv = torch.ones_like(doc, dtype=torch.uint8)
dscr = torch.empty((1, L, 2, cfg.kv_heads, D, cfg.head_dim), dtype=torch.float16, device="cuda")
dptr = torch.tensor([dscr.data_ptr()], dtype=torch.int64, device="cuda")
res = {}
for l in [1, 2, 3, 8, 16]:
    x = torch.empty((D, cfg.model_dim), dtype=torch.float32, device="cuda")
    engine.run_layers(w, 0, l, doc, dv, 0, 0, None, None, dptr, L, x_out=x, cur_pool=dscr)
    torch.cuda.synchronize()
    res[l] = x.cpu().numpy()
np.save(f"/tmp/fused_{os.environ.get('KRR_FUSED_NORM','1')}.npy", np.stack([res[k] for k in sorted(res)]))
print(os.environ.get('KRR_FUSED_NORM','1'), {k: float(np.abs(v).max()) for k, v in res.items()})
