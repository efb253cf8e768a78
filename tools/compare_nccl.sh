#!/bin/bash
# One-rank-per-GPU comparison of the fused WAGMA kernel with the NCCL
# sub-communicator baseline (blocking semantics) on N GPUs, for S in a list
# and model sizes from the 1 MB - 1 GB sweep (BASELINE.json configs[4]).
# usage: tools/compare_nccl.sh N "S list" "n list"
N=${1:-2}; SL=${2:-"2"}; NL=${3:-"25559081"}
mkdir -p gpurun_out
for n in $NL; do for S in $SL; do
  [ $S -gt $N ] && continue
  for impl in ours nccl; do
    timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
      --master-port 29561 bench.py --gpus $N --P $N --S $S --nparams $n --impl $impl --steps 100 --warmup 10 \
      --no-cpu --no-e2e > gpurun_out/cmp_${impl}_N${N}_S${S}_n${n}.log 2>&1
    echo "$impl N=$N S=$S n=$n $(tail -1 gpurun_out/cmp_${impl}_N${N}_S${S}_n${n}.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],4), "ms", round(d["value"],1), "it/s")' 2>/dev/null)"
  done
done; done
