#!/bin/bash
# head_dim 256 through the persistent TMEM-P attention: GPU tests, C2 launch list,
# C2 bench (x2), C3 bench.
TAG=${1:-a256}
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout -s KILL 1200 python -m pytest tests -q -m gpu --timeout 900 -p no:cacheprovider > gpurun_out/${TAG}_pytest.log 2>&1
echo "pytest rc=$?"; grep -E "passed|failed|^FAILED|^ERROR" gpurun_out/${TAG}_pytest.log | tail -12
CMD="python bench.py --config c2 --steps 2 --warmup 1 --no-cpu-baseline --latency-reps 0 --full-pairs 4"
timeout -s KILL 900 ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_c2_launches.csv $CMD > /dev/null 2>&1
python scripts/ncu_list_summary.py gpurun_out/${TAG}_c2_launches.csv > gpurun_out/${TAG}_c2_launches.txt; head -6 gpurun_out/${TAG}_c2_launches.txt
for r in 1 2; do
  timeout -s KILL 600 python bench.py --config c2 --steps 20 --warmup 3 --latency-reps 15 --no-cpu-baseline --full-pairs 4 > gpurun_out/${TAG}_c2_$r.json 2>/dev/null
  echo -n "c2 r$r: "; python scripts/show.py gpurun_out/${TAG}_c2_$r.json
done
timeout -s KILL 900 python bench.py --steps 3 --warmup 3 --latency-reps 10 --no-cpu-baseline --full-pairs 4 > gpurun_out/${TAG}_c3.json 2>/dev/null
echo -n "c3: "; python scripts/show.py gpurun_out/${TAG}_c3.json
