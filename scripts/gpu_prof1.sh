# launch list of the timed region (small C3-shaped run) + full capture of top kernels
CMD="python bench.py --config c3 --queries 8 --cands 100 --corpus 100 --steps 1 --warmup 1 --no-cpu-baseline --latency-reps 0 --full-pairs 4"
timeout -s KILL 900 ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01_launches_c3.csv $CMD > gpurun_out/r01_launches.log 2>&1
tail -3 gpurun_out/r01_launches.log
timeout -s KILL 900 ncu --nvtx --nvtx-include "timed/" --set full --clock-control none --import-source on -k regex:"attn_mma|gemm_kernel" -c 6 -o gpurun_out/r01_prof_c3 $CMD > gpurun_out/r01_prof.log 2>&1
tail -3 gpurun_out/r01_prof.log
ls -la gpurun_out
