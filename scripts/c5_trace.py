"""Timeline of engine.score_host_tier at C5 (events per group on the copy and
main streams) for the 16-bit / int8 / int4 tiers: where does a step go?"""
import sys, time, numpy as np, torch
sys.path.insert(0, ".")
import paper_2504_02921_b200 as krr
from paper_2504_02921_b200 import engine
from paper_2504_02921_b200.config import PRESETS

cfg, lay = PRESETS["c5_mistral7b_d2048"]
D, N, Q = lay.document_len, 48, int(sys.argv[1]) if len(sys.argv) > 1 else 16
dev = torch.device("cuda", 0)
model = krr.RerankModel.build(cfg, lay, precision="f16", device=dev)
w = model.weights
tmp = krr.KVPool(cfg, D, 8, w.dtype, dev)
docs = np.random.default_rng(0).integers(1, cfg.vocab_size, (8, D))
sl = tmp.allocate([f"d{i}" for i in range(8)])
engine.prefill_slots(w, tmp, sl, docs, np.full(8, D))
staging = krr.KVPool(cfg, D, int(sys.argv[2]) if len(sys.argv) > 2 else 16, w.dtype, dev)
q = np.random.default_rng(1).integers(1, cfg.vocab_size, (N, Q))
ev = lambda: torch.cuda.Event(enable_timing=True)
for quant in (None, "int8", "int4"):
    tier = krr.HostKVTier(tmp, N, quant=quant)
    for i in range(N):
        tier.put_from_pool(f"h{i}", tmp, int(sl[i % 8]))
    torch.cuda.synchronize()
    hs = np.arange(N)
    cs = torch.cuda.Stream(device=dev)
    for rep in range(3):
        t0 = ev(); t0.record()
        # mirror of score_host_tier with events
        half = staging.capacity // 2
        st = np.arange(staging.capacity)
        groups = [hs[i:i + half] for i in range(0, N, half)]
        main = torch.cuda.current_stream(dev)
        ready = [torch.cuda.Event() for _ in range(2)]
        free = [torch.cuda.Event() for _ in range(2)]
        marks = [[ev() for _ in range(5)] for _ in groups]
        slots_of = lambda gi: st[(gi & 1) * half:(gi & 1) * half + groups[gi].size]

        def issue(gi):
            c0, c1 = marks[gi][:2]
            with torch.cuda.stream(cs):
                if gi >= 2:
                    cs.wait_event(free[gi & 1])
                c0.record(cs)
                for h, s in zip(groups[gi], slots_of(gi)):
                    tier.h2d(int(h), staging, int(s), int(s))
                c1.record(cs)
                ready[gi & 1].record(cs)
        for gi in range(min(2, len(groups))):
            issue(gi)
        for gi, grp in enumerate(groups):
            b = gi & 1
            slots = slots_of(gi)
            _, _, m0, m1, m2 = marks[gi]
            main.wait_event(ready[b])
            m0.record(main)
            for s in slots:
                tier.expand(staging, int(s), int(s))
            m1.record(main)
            staging.set_valid_len(slots, tier.valid_len[grp])
            engine.score_slots(w, staging, slots, q[grp])
            m2.record(main)
            free[b].record(main)
            if gi + 2 < len(groups):
                issue(gi + 2)
        t1 = ev(); t1.record()
        torch.cuda.synchronize()
        print(f"  rep{rep}: step {t0.elapsed_time(t1):.1f} ms; score per group " +
              " ".join(f"{m[3].elapsed_time(m[4]):.1f}" for m in marks), flush=True)
    tot = t0.elapsed_time(t1)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    for _ in range(3):
        engine.score_host_tier(w, tier, staging, hs, q, copy_stream=cs)
    torch.cuda.synchronize()
    api = (time.perf_counter() - t2) / 3 * 1e3
    print(f"{quant or 'f16'} Q={Q} staging={staging.capacity}: engine.score_host_tier {api:.1f} ms "
          f"= {N / api * 1e3:.0f} pairs/s (wall)")
    print(f"{quant or 'f16'} Q={Q}: step {tot:.1f} ms = {N / tot * 1e3:.0f} pairs/s")
    for gi, (c0, c1, m0, m1, m2) in enumerate(marks):
        print(f"  g{gi}: copy [{t0.elapsed_time(c0):7.1f},{t0.elapsed_time(c1):7.1f}] "
              f"expand [{t0.elapsed_time(m0):7.1f},{t0.elapsed_time(m1):7.1f}] "
              f"score ->{t0.elapsed_time(m2):7.1f}")
    del tier
