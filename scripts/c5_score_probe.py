"""Why is the first group's scoring slow in score_host_tier? Time score_slots on
8 staged docs (Q=48) alone, after a fresh H2D burst on a side stream, and with
max_rows given (no mem_get_info)."""
import sys, time, numpy as np, torch
sys.path.insert(0, ".")
import paper_2504_02921_b200 as krr
from paper_2504_02921_b200 import engine
from paper_2504_02921_b200.config import PRESETS
cfg, lay = PRESETS["c5_mistral7b_d2048"]
D, Q = lay.document_len, int(sys.argv[1]) if len(sys.argv) > 1 else 48
dev = torch.device("cuda", 0)
model = krr.RerankModel.build(cfg, lay, precision="f16", device=dev)
w = model.weights
staging = krr.KVPool(cfg, D, 16, w.dtype, dev)
sl = staging.allocate([f"d{i}" for i in range(16)])
engine.prefill_slots(w, staging, sl[:8], np.random.default_rng(0).integers(1, 32000, (8, D)),
                     np.full(8, D))
q = torch.as_tensor(np.random.default_rng(1).integers(1, 32000, (8, Q)), device=dev)
host = torch.empty(8 * staging.slot_bytes // 2, dtype=torch.float16, pin_memory=True)
cs = torch.cuda.Stream()
ev = lambda: torch.cuda.Event(enable_timing=True)
def timed(label, fn, reps=3):
    for r in range(reps):
        torch.cuda.synchronize()
        a, b = ev(), ev()
        t0 = time.perf_counter()
        a.record(); fn(); b.record()
        t1 = time.perf_counter()
        torch.cuda.synchronize()
        print(f"{label} rep{r}: gpu {a.elapsed_time(b):7.2f} ms  host-enqueue {1e3*(t1-t0):7.2f} ms")
timed("score alone", lambda: engine.score_slots(w, staging, sl[:8], q))
timed("score alone max_rows", lambda: engine.score_slots(w, staging, sl[:8], q, max_rows=8 * Q))
def with_copy(mr):
    with torch.cuda.stream(cs):
        staging.slab[8:16].view(-1).copy_(host, non_blocking=True)
    engine.score_slots(w, staging, sl[:8], q, max_rows=mr)
timed("score + concurrent H2D", lambda: with_copy(None))
timed("score + concurrent H2D max_rows", lambda: with_copy(8 * Q))
