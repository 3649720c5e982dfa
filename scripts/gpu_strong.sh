#!/bin/bash
# strong-scaling mode: N=1 (C1, C3) and a 2-rank run on one GPU (gloo) for C1/C2
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
for cfg in c1 c2; do for mode in weak strong; do
  timeout -s KILL 600 python bench.py --config $cfg --scaling $mode --steps 3 --warmup 3 --latency-reps 3 --no-cpu-baseline > gpurun_out/st_${cfg}_${mode}_1.json 2> gpurun_out/st_${cfg}_${mode}_1.err
  echo -n "$cfg $mode N=1 rc=$? "; tail -1 gpurun_out/st_${cfg}_${mode}_1.json | cut -c1-200
  KRR_BENCH_ONE_DEVICE=1 KRR_BENCH_DIST_BACKEND=gloo timeout -s KILL 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 2 --config $cfg --scaling $mode --steps 3 --warmup 3 --latency-reps 3 --no-cpu-baseline > gpurun_out/st_${cfg}_${mode}_2.json 2> gpurun_out/st_${cfg}_${mode}_2.err
  echo -n "$cfg $mode N=2 rc=$? "; grep '^{' gpurun_out/st_${cfg}_${mode}_2.json | tail -1 | cut -c1-200; tail -2 gpurun_out/st_${cfg}_${mode}_2.err
done; done
# bench.py re-launching itself under torch.distributed.run (no WORLD_SIZE in the env)
KRR_BENCH_ONE_DEVICE=1 KRR_BENCH_DIST_BACKEND=gloo timeout -s KILL 900 python bench.py --gpus 2 --config c2 --steps 3 --warmup 3 --latency-reps 3 --no-cpu-baseline > gpurun_out/st_self_2.json 2> gpurun_out/st_self_2.err
echo -n "c2 self-launched N=2 rc=$? "; grep '^{' gpurun_out/st_self_2.json | tail -1 | cut -c1-200
