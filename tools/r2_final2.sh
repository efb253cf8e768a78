#!/bin/bash
# Final validation of the last build on 4 GPUs: multi-GPU parity (default + leaf-level families), smoke, bench lines.
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_multi.py -q -rA -k "not mg" > gpurun_out/rf3_multi.log 2>&1; echo "multi rc=$?"; tail -1 gpurun_out/rf3_multi.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/rf3_smoke.log 2>&1; tail -1 gpurun_out/rf3_smoke.log
timeout 600 python bench.py > gpurun_out/rf3_bench_n1.json 2> gpurun_out/rf3_bench_n1.err
for N in 2 4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29571 \
    bench.py --gpus $N > gpurun_out/rf3_bench_n$N.log 2>&1
  tail -1 gpurun_out/rf3_bench_n$N.log > gpurun_out/rf3_bench_n$N.json
done
for N in 1 2 4; do python -c "import json; d=json.load(open('gpurun_out/rf3_bench_n$N.json')); print($N, round(d['value'],1), d['unit'], round(d['ms_per_step'],4), d['roofline']['bound'], round(d['roofline']['frac'],3), 'e2e', d['e2e']['value'] if d.get('e2e') else None, d['clocks'])"; done
