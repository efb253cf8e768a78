for n in 262144 1048576 4194304; do for sp in 1 0; do
  WG_SPLIT=$sp timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29581 bench.py --gpus 4 --P 4 --S 4 --nparams $n --steps 100 --warmup 10 --no-cpu --no-e2e > gpurun_out/sm.log 2>&1
  echo "split=$sp n=$n $(tail -1 gpurun_out/sm.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],4), "ms")' 2>/dev/null)"
done; done
