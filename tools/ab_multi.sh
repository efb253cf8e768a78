#!/bin/bash
# A/B of alternative libwagma builds on N GPUs: tools/ab_multi.sh N "lib1 lib2 ..." "S list" [P]
N=$1; LIBS=$2; SL=$3; P=${4:-8}
for L in $LIBS; do for S in $SL; do
  WAGMA_B200_LIB=$PWD/$L timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29555 bench.py --gpus $N --P $P --no-cpu --no-e2e --S $S --steps 200 > gpurun_out/ab_m.log 2>&1
  echo "$L P=$P S=$S $(tail -1 gpurun_out/ab_m.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print(round(d["value"]), round(r["kernel_ms"],4), r["bound"], round(r["frac"],3))' 2>/dev/null)"
done; done
