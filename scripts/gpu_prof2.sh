CMD="python bench.py --config c3 --queries 8 --cands 100 --corpus 100 --steps 1 --warmup 1 --no-cpu-baseline --latency-reps 0 --full-pairs 4"
timeout -s KILL 900 ncu --nvtx --nvtx-include "timed/" --set full --clock-control none --import-source on -k regex:"attn_prefix_mma" -c 1 -o gpurun_out/r01_prof_attn $CMD > gpurun_out/r01_prof_attn.log 2>&1
tail -2 gpurun_out/r01_prof_attn.log
