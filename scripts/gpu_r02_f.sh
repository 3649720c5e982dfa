#!/bin/bash
# Round 2, call F: GPU suite after the GEMM cleanup, smoke, and C5 (host-DRAM tier)
# sized from the box's free RAM, per page format.
mkdir -p gpurun_out
(free -g; nproc; nvidia-smi --query-gpu=name,memory.total,pcie.link.gen.current,pcie.link.width.current --format=csv) > gpurun_out/f_box.txt 2>&1
cat gpurun_out/f_box.txt
timeout 1800 python -m pytest tests -q -m gpu -p no:cacheprovider -rf > gpurun_out/f_tests.log 2>&1
tail -5 gpurun_out/f_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f_smoke.log 2>&1; tail -2 gpurun_out/f_smoke.log
for qt in "" int8 int4; do
  tag=${qt:-f16}
  timeout 1500 python bench.py --config c5 --corpus -1 --steps 3 --warmup 2 --query-lens 16,48,256 ${qt:+--host-quant $qt} > gpurun_out/f_c5_$tag.log 2>&1
  tail -1 gpurun_out/f_c5_$tag.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); c=d['config']; print('$tag', c['host_docs'], round(c['host_tier_gb'],1), {q: round(v['pairs_per_s'],1) for q,v in d['query_len_sweep'].items()}, round(d['h2d_peak_gbs'],1))"
done
