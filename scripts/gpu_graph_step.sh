#!/bin/bash
# C2 / C1 bench lines with the timed step as one CUDA-graph replay (auto) vs eager launches,
# alternating; a short C3 line (eager, unchanged path).
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
for i in 1 2; do
  for g in off auto; do
    timeout -s KILL 600 python bench.py --config c2 --graph $g --steps 20 --warmup 3 --latency-reps 15 > gpurun_out/gs_c2_${g}_$i.json 2> gpurun_out/gs_c2_${g}_$i.err
    echo -n "c2 graph=$g $i rc=$? "; python scripts/show.py gpurun_out/gs_c2_${g}_$i.json | cut -c1-200; tail -2 gpurun_out/gs_c2_${g}_$i.err | grep -i error
  done
done
timeout -s KILL 600 python bench.py --config c1 --steps 20 --warmup 3 --latency-reps 5 > gpurun_out/gs_c1.json 2> gpurun_out/gs_c1.err
echo -n "c1 auto rc=$? "; python scripts/show.py gpurun_out/gs_c1.json | cut -c1-200; tail -2 gpurun_out/gs_c1.err | grep -i error
timeout -s KILL 900 python bench.py --steps 3 --warmup 3 --latency-reps 3 --no-cpu-baseline --full-pairs 4 > gpurun_out/gs_c3.json 2> gpurun_out/gs_c3.err
echo -n "c3 rc=$? "; python scripts/show.py gpurun_out/gs_c3.json | cut -c1-200
grep -o '"timed_step": "[^"]*"\|"gpu_launches": [0-9]*' gpurun_out/gs_c2_auto_1.json gpurun_out/gs_c3.json
