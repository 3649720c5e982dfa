import sys, json
for l in open(sys.argv[1]) if len(sys.argv) > 1 else sys.stdin:
    l = l.strip()
    if not l.startswith('{'):
        print(l); continue
    d = json.loads(l)
    if 'metric' in d:
        r = d.get('roofline') or {}
        print(f"BENCH value={d['value']:.1f} e2e={d['e2e']['value']:.1f} ms/step={d['ms_per_step']:.0f} "
              f"clk={d['clocks']['sm_mhz']} gemmTF={r.get('achieved',0):.0f} frac={r.get('frac',0):.3f} "
              f"gemm%={r.get('gemm_share_of_step',0):.3f} attn%={r.get('attn_share_of_step',0):.3f} "
              f"misc%={r.get('misc_share_of_step',0):.3f} pairs_frac={r.get('pairs_frac',0):.3f} "
              f"p50={d.get("p50_query_latency_ms")} p50g={d.get("p50_query_latency_graph_ms")} full={d.get('full_recompute_pairs_per_s')}")
    else:
        print('GEMM CTA', d.get('cta'))
        for k, v in d.items():
            if isinstance(v, dict): print('  ', k, v)
