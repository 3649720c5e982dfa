#!/bin/bash
# Round-2 evidence, part 2: drop-in tests (staged reference), C2 launch list,
# C4 capacity, C5 host tier at the RAM cap (f16 / int8 / int4), C2 bench line.
TAG=${1:-r02b}
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv,noheader
free -g | head -2
timeout -s KILL 600 python -m pytest tests/test_gpu_dropin.py -q -m gpu -p no:cacheprovider > gpurun_out/${TAG}_dropin.log 2>&1
echo "dropin rc=$?"; tail -2 gpurun_out/${TAG}_dropin.log
CMD="python bench.py --config c2 --steps 2 --warmup 1 --no-cpu-baseline --latency-reps 0 --full-pairs 4"
timeout -s KILL 900 ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_c2_launches.csv $CMD > gpurun_out/${TAG}_c2_launches.log 2>&1
echo "ncu c2 list rc=$?"; python scripts/ncu_list_summary.py gpurun_out/${TAG}_c2_launches.csv > gpurun_out/${TAG}_c2_launches.txt; head -14 gpurun_out/${TAG}_c2_launches.txt
timeout -s KILL 900 python bench.py --config c2 --steps 20 --warmup 3 --latency-reps 15 > gpurun_out/${TAG}_c2.json 2> gpurun_out/${TAG}_c2.err
echo -n "c2 rc=$? "; python scripts/show.py gpurun_out/${TAG}_c2.json
timeout -s KILL 1500 python bench.py --config c4 --steps 3 --warmup 3 --latency-reps 5 --no-cpu-baseline > gpurun_out/${TAG}_c4.json 2> gpurun_out/${TAG}_c4.err
echo -n "c4 rc=$? "; python scripts/show.py gpurun_out/${TAG}_c4.json
for qz in "" int8 int4; do
  timeout -s KILL 1800 python bench.py --config c5 --corpus -1 --steps 5 --warmup 3 --query-lens 16,48,256 --no-cpu-baseline ${qz:+--host-quant $qz} > gpurun_out/${TAG}_c5_${qz:-f16}.json 2> gpurun_out/${TAG}_c5_${qz:-f16}.err
  echo "c5 ${qz:-f16} rc=$?"; tail -1 gpurun_out/${TAG}_c5_${qz:-f16}.err; tail -c 600 gpurun_out/${TAG}_c5_${qz:-f16}.json
done
