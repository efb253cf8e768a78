#!/bin/bash
# A/B of libwagma builds on N GPUs: tools/ab_multi2.sh N "lib1 lib2" [bench args]
N=$1; LIBS=$2; shift 2
for L in $LIBS; do
  WAGMA_B200_LIB=$PWD/$L timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29613 bench.py --gpus $N --steps 200 --warmup 10 --no-e2e "$@" > gpurun_out/ab_m.log 2>&1
  echo "$L N=$N $* $(tail -1 gpurun_out/ab_m.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print(round(d["value"]), round(r["kernel_ms"],4), r["bound"], round(r["frac"],3), d.get("protocol_last_versions"))' 2>&1 | tail -1)"
done
