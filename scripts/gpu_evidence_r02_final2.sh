#!/bin/bash
# Last-session evidence on the committed tree: GPU suite, smoke, default C3 bench (staged
# reference as cpu_baseline), reference arm, C3 launch list, ncu --set full of the MLP-up
# GEMM and the attention kernel, C2 line.  (C4 / C5 unchanged since gpu_evidence_final.sh.)
TAG=${1:-r02f}
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv,noheader
timeout -s KILL 1500 python -m pytest tests -q -m gpu --timeout 1200 -p no:cacheprovider > gpurun_out/${TAG}_pytest.log 2>&1
echo "pytest rc=$?"; grep -E "passed|failed|^FAILED|^ERROR" gpurun_out/${TAG}_pytest.log | tail -8
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/${TAG}_smoke.log
timeout -s KILL 1500 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
echo -n "bench rc=$? "; python scripts/show.py gpurun_out/${TAG}_bench.json
timeout -s KILL 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${TAG}_ref.json 2> gpurun_out/${TAG}_ref.err
echo "ref rc=$? $(tail -c 300 gpurun_out/${TAG}_ref.json)"
timeout -s KILL 900 python bench.py --config c2 --steps 20 --warmup 3 --latency-reps 15 > gpurun_out/${TAG}_c2.json 2> gpurun_out/${TAG}_c2.err
echo -n "c2 rc=$? "; python scripts/show.py gpurun_out/${TAG}_c2.json
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --latency-reps 0 --full-pairs 4"
timeout -s KILL 1200 ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv $CMD > /dev/null 2>&1
echo "ncu list rc=$?"; python scripts/ncu_list_summary.py gpurun_out/${TAG}_launches.csv > gpurun_out/${TAG}_launches.txt; head -6 gpurun_out/${TAG}_launches.txt
timeout -s KILL 1200 ncu --nvtx --nvtx-include "timed/" --set full --clock-control none --import-source on -k regex:"gemm_tcgen05" -s 2 -c 1 -o gpurun_out/${TAG}_gemm_full $CMD > /dev/null 2>&1
echo "ncu gemm rc=$?"
timeout -s KILL 900 ncu --nvtx --nvtx-include "timed/" --set full --clock-control none --import-source on -k regex:"attn_fa" -c 1 -o gpurun_out/${TAG}_attn_full $CMD > /dev/null 2>&1
echo "ncu attn rc=$?"
