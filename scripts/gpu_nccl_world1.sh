#!/bin/bash
# The driver's torchrun launch with the NCCL backend, at the one GPU a box has (world 1):
# communicator init, query broadcast, local top-k and the all-gather merge all run on NCCL.
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
for cfg in c2 c3; do
  NCCL_DEBUG=INFO timeout -s KILL 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29633 bench.py --gpus 1 --config $cfg --steps 5 --warmup 3 --latency-reps 5 --no-cpu-baseline > gpurun_out/nccl1_$cfg.json 2> gpurun_out/nccl1_$cfg.err
  echo -n "$cfg torchrun nccl N=1 rc=$? "; grep '^{' gpurun_out/nccl1_$cfg.json | tail -1 | cut -c1-220; echo
  grep -E "NCCL INFO (comm|Init|NCCL version)" gpurun_out/nccl1_$cfg.err | head -4
done
