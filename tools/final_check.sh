#!/bin/bash
# Round-end verification on a 4-GPU box: GPU test suite, smoke(), default bench lines at N=1, 2, 4.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/final_gpu_tests.log 2>&1; tail -1 gpurun_out/final_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/final_smoke.log 2>&1; tail -1 gpurun_out/final_smoke.log
timeout 600 python bench.py > gpurun_out/final_bench_n1.json 2> gpurun_out/final_bench_n1.err
for N in 2 4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29571 \
    bench.py --gpus $N > gpurun_out/final_bench_n$N.log 2>&1
  tail -1 gpurun_out/final_bench_n$N.log > gpurun_out/final_bench_n$N.json
done
for N in 1 2 4; do python -c "import json; d=json.load(open('gpurun_out/final_bench_n$N.json')); print($N, round(d['value'],1), d['unit'], round(d['ms_per_step'],4), d['roofline']['bound'], round(d['roofline']['frac'],3), 'e2e', d['e2e']['value'] if d.get('e2e') else None)"; done
