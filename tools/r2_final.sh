#!/bin/bash
# Round-2 evidence on a 4-GPU box: whole GPU suite, smoke(), default bench lines at N=1/2/4, reference arm.
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
nvidia-smi -L > gpurun_out/rf_gpus.txt
timeout 2400 python -m pytest tests -m gpu -q -rA > gpurun_out/rf_gpu_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/rf_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/rf_smoke.log 2>&1; tail -1 gpurun_out/rf_smoke.log
timeout 600 python bench.py > gpurun_out/rf_bench_n1.json 2> gpurun_out/rf_bench_n1.err
for N in 2 4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29571 \
    bench.py --gpus $N > gpurun_out/rf_bench_n$N.log 2>&1
  tail -1 gpurun_out/rf_bench_n$N.log > gpurun_out/rf_bench_n$N.json
done
timeout 600 python bench.py --impl reference > gpurun_out/rf_ref_n1.json 2> gpurun_out/rf_ref_n1.err
for N in 1 2 4; do python -c "import json; d=json.load(open('gpurun_out/rf_bench_n$N.json')); print($N, round(d['value'],1), d['unit'], round(d['ms_per_step'],4), d['roofline']['bound'], round(d['roofline']['frac'],3), 'e2e', d['e2e']['value'] if d.get('e2e') else None, d['clocks'])"; done
python -c "import json; d=json.load(open('gpurun_out/rf_ref_n1.json')); print('reference', d['value'], d['cpu_baseline']['cores'])"
{
bash tools/ab_env.sh 2 "-|WG_HIER=0" --P 2 --S 2
bash tools/ab_env.sh 4 "-" --S 4
} > gpurun_out/rf_extra.txt 2>&1; cat gpurun_out/rf_extra.txt
