#!/bin/bash
# A/B of environment knobs on N GPUs: tools/ab_env.sh N "K1=V1 K2=V2|K3=V3|-" [bench args]
# ("-" = defaults). Prints one line per variant: it/s, kernel ms, bound, frac, stale contributions.
N=$1; VARS=$2; shift 2
IFS='|' read -ra VS <<< "$VARS"
for V in "${VS[@]}"; do
  E=""; [ "$V" != "-" ] && E="$V"
  if [ "$N" = 1 ]; then
    env $E timeout 300 python bench.py --steps 200 --warmup 10 --no-e2e --no-cpu "$@" > gpurun_out/ab_e.log 2>&1
  else
    env $E timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
      --master-port 29613 bench.py --gpus $N --steps 200 --warmup 10 --no-e2e "$@" > gpurun_out/ab_e.log 2>&1
  fi
  echo "N=$N [$V] $* :: $(tail -1 gpurun_out/ab_e.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print(round(d["value"]), round(r["kernel_ms"],4), r["bound"], round(r["frac"],3), r.get("nvlink_frac"), d.get("protocol_last_versions"))' 2>&1 | tail -1)"
done
