#!/bin/bash
# C3-style imbalance: per-(rank, t) compute time from length buckets; alpha vs beta.
# usage: tools/imbalance_lengths.sh N P S base_ms [nparams]
N=$1; P=$2; S=$3; B=$4; NP=${5:-25559081}
for mode in "" "--blocking"; do
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29573 \
    bench.py --gpus $N --P $P --S $S --nparams $NP --base-ms $B --length-buckets --tau 8 $mode --steps 100 --warmup 10 \
    --no-cpu --no-e2e > gpurun_out/imbl.log 2>&1
  echo "${mode:-alpha} lengths N=$N P=$P S=$S base=$B: $(tail -1 gpurun_out/imbl.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); i=d["imbalance"]; print(round(d["value"],1), "it/s", round(d["ms_per_step"],3), "ms/step stale_frac", i["stale_contribution_fraction"])' 2>/dev/null)"
done
