"""Host-tier H2D bandwidth vs tier size: 48 random documents' pages copied from
a pinned tier of N documents (f16 / int4), CUDA events on a side stream."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2504_02921_b200 as krr  # noqa: E402
from paper_2504_02921_b200.config import PRESETS  # noqa: E402

cfg, lay = PRESETS["c5_mistral7b_d2048"]
D = lay.document_len
staging = krr.KVPool(cfg, D, 16, "f16", "cuda")
cs = torch.cuda.Stream()
for quant, sizes in ((None, (48, 460)), ("int4", (48, 1860))):
    for n in sizes:
        tier = krr.HostKVTier(staging, n, quant=quant)
        rng = np.random.default_rng(0)
        for rep in range(3):
            docs = rng.choice(n, 48, replace=False)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(cs):
                a.record(cs)
                for i, h in enumerate(docs):
                    tier.h2d(int(h), staging, i % 16, i % 16)
                b.record(cs)
            torch.cuda.synchronize()
            ms = a.elapsed_time(b)
            print(f"{quant or 'f16'} tier {n:5d} docs ({n * tier.slot_bytes / 1e9:6.1f} GB): 48 docs "
                  f"{ms:7.1f} ms = {48 * tier.slot_bytes / ms / 1e6:5.1f} GB/s", flush=True)
        del tier
