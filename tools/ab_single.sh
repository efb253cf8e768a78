#!/bin/bash
# A/B of alternative libwagma builds on 1 GPU: tools/ab_single.sh "lib1 lib2 ..." [bench args]
LIBS=$1; shift
for L in $LIBS; do
  WAGMA_B200_LIB=$PWD/$L timeout 300 python bench.py --no-cpu --no-e2e --steps 200 "$@" > gpurun_out/ab_s.log 2>&1
  echo "$L $* $(tail -1 gpurun_out/ab_s.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print(round(d["value"]), round(r["kernel_ms"],4), r["bound"], round(r["frac"],3))' 2>/dev/null)"
done
