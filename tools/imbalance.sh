#!/bin/bash
# Wait-avoiding (alpha) vs blocking (beta) group averaging under injected stragglers.
# usage: tools/imbalance.sh N P S base_ms victims extra_ms [nparams]
N=$1; P=$2; S=$3; B=$4; V=$5; X=$6; NP=${7:-25559081}
mkdir -p gpurun_out
for mode in "" "--blocking"; do
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29571 \
    bench.py --gpus $N --P $P --S $S --nparams $NP --base-ms $B --victims $V --extra-ms $X $mode --steps 100 --warmup 10 \
    --no-cpu --no-e2e > gpurun_out/imb.log 2>&1
  echo "${mode:-alpha} N=$N P=$P S=$S base=$B victims=$V extra=$X: $(tail -1 gpurun_out/imb.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); i=d["imbalance"]; print(round(d["value"],1), "it/s", round(d["ms_per_step"],3), "ms/step stale_frac", i["stale_contribution_fraction"])' 2>/dev/null)"
done
