# 2-GPU: multi parity (3 kernel families), benches; then 1-GPU tests
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests/test_gpu_multi.py -q -x > gpurun_out/r2e_multi.log 2>&1; echo "rc=$?" >> gpurun_out/r2e_multi.log
for S in 8 4; do for V in "1 1" "1 0" "0 1"; do set -- $V
WG_HIER=$1 WG_MG=$2 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 2 --steps 200 --warmup 10 --no-e2e --S $S > gpurun_out/r2e_b2.log 2>&1
echo "S=$S hier=$1 mg=$2 $(tail -1 gpurun_out/r2e_b2.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print(round(d["value"]), round(r["kernel_ms"],4), r["bound"], round(r["frac"],3), r.get("t_star_frac"))' 2>&1 | tail -1)" >> gpurun_out/r2e_bench2.txt
done; done
timeout 900 python -m pytest tests -m gpu -q --deselect tests/test_gpu_multi.py > gpurun_out/r2e_gpu1.log 2>&1; echo "rc=$?" >> gpurun_out/r2e_gpu1.log
tail -4 gpurun_out/r2e_multi.log; cat gpurun_out/r2e_bench2.txt; tail -2 gpurun_out/r2e_gpu1.log
