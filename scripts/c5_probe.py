"""C5 host-tier probe: per-document H2D and dequant times (CUDA events) for the
16-bit / int8 / int4 tiers at the C5 page shape (no model needed)."""
import sys, torch
sys.path.insert(0, ".")
import paper_2504_02921_b200 as krr
from paper_2504_02921_b200.config import PRESETS
cfg, lay = PRESETS["c5_mistral7b_d2048"]
D = lay.document_len
pool = krr.KVPool(cfg, D, 4, "f16", "cuda")
ev = lambda: torch.cuda.Event(enable_timing=True)
for q in (None, "int8", "int4"):
    tier = krr.HostKVTier(pool, 4, quant=q)
    if q:
        tier.codes.random_(0, 255); tier.scales.uniform_(0.01, 1.0)
    for rep in range(2):
        a, b, c = ev(), ev(), ev()
        a.record()
        for h in range(4):
            tier.h2d(h, pool, h, h)
        b.record()
        for h in range(4):
            tier.expand(pool, h, h)
        c.record()
        torch.cuda.synchronize()
    t_h2d, t_dq = a.elapsed_time(b) / 4, b.elapsed_time(c) / 4
    print(f"{q or 'f16'}: {tier.slot_bytes/1e6:.0f} MB/doc  h2d {t_h2d:.2f} ms/doc "
          f"({tier.slot_bytes/t_h2d/1e6:.1f} GB/s)  dequant {t_dq:.3f} ms/doc "
          f"({2*tier.tensor_elems*tier.n_tensors/t_dq/1e6:.0f} GB/s written)")
