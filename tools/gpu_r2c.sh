# 2-GPU box: single-GPU A/B + tests, then multi-GPU parity (hier on/off) and benches
cd $GRAFT_REPO_ROOT
bash tools/ab_single.sh "ab/lib_default.so ab/lib_w16.so ab/lib_noef.so ab/lib_default.so" > gpurun_out/r2c_ab.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py tests/test_gpu_api.py -x -q > gpurun_out/r2c_gpu1.log 2>&1; echo "rc=$?" >> gpurun_out/r2c_gpu1.log
timeout 1500 python -m pytest tests/test_gpu_multi.py -q -x > gpurun_out/r2c_multi.log 2>&1; echo "rc=$?" >> gpurun_out/r2c_multi.log
for S in 8 4; do for H in 1 0; do
WG_HIER=$H timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 2 --steps 200 --warmup 10 --no-e2e --S $S > gpurun_out/r2c_b2_S${S}_h$H.log 2>&1
echo "S=$S hier=$H $(tail -1 gpurun_out/r2c_b2_S${S}_h$H.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print(round(d["value"]), round(r["kernel_ms"],4), r["bound"], round(r["frac"],3), r.get("nvlink_frac"), r["algorithmic_bytes_per_launch"])' 2>&1 | tail -1)" >> gpurun_out/r2c_bench2.txt
done; done
cat gpurun_out/r2c_ab.txt; tail -2 gpurun_out/r2c_gpu1.log; tail -4 gpurun_out/r2c_multi.log; cat gpurun_out/r2c_bench2.txt
