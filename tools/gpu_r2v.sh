#!/bin/bash
# Round-2 multi-GPU evidence on 4 GPUs: fence scope, C3/C4 configs, grace-window cost, C4 fixed victim.
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
{
echo "## fence scope (default kernels)"
bash tools/ab_env.sh 2 "-|WG_FENCE_SCOPE=sys" --S 8
bash tools/ab_env.sh 4 "-|WG_FENCE_SCOPE=sys" --S 8
bash tools/ab_env.sh 4 "-|WG_FENCE_SCOPE=sys" --S 4
bash tools/ab_env.sh 4 "-|WG_FENCE_SCOPE=sys" --P 4 --S 4
echo "## C4 n=8,476,421 tau=8"
for N in 1 2 4; do bash tools/ab_env.sh $N "-" --nparams 8476421 --tau 8; done
echo "## C3 n=213,000,000 tau=8"
for N in 1 2 4; do bash tools/ab_env.sh $N "-" --nparams 213000000 --tau 8 --steps 30; done
echo "## grace window: P=4 S=4 on 4 GPUs, base 1.0 ms/step on every GPU, one StragglerPolicy victim +3.2 ms"
bash tools/ab_env.sh 4 "-|WG_ADAPTIVE_GRACE=0" --P 4 --S 4 --base-ms 1.0 --victims 1 --extra-ms 3.2
bash tools/ab_env.sh 4 "-" --P 4 --S 4 --base-ms 1.0 --victims 1 --extra-ms 3.2 --grace-us 0
bash tools/ab_env.sh 4 "-" --P 4 --S 4 --base-ms 1.0 --victims 1 --extra-ms 3.2 --blocking
bash tools/ab_env.sh 4 "-" --P 4 --S 4 --base-ms 1.0
bash tools/ab_env.sh 4 "-" --P 4 --S 4 --base-ms 1.0 --grace-us 0
echo "## C4 fixed victim (rank 1), P=2 S=2 on 2 GPUs, base 1.0 ms, +3.2 ms"
bash tools/ab_env.sh 2 "-" --P 2 --S 2 --nparams 8476421 --tau 8 --base-ms 1.0 --fixed-victim 1 --extra-ms 3.2
bash tools/ab_env.sh 2 "-" --P 2 --S 2 --nparams 8476421 --tau 8 --base-ms 1.0 --fixed-victim 1 --extra-ms 3.2 --blocking
} > gpurun_out/r2v.txt 2>&1
cat gpurun_out/r2v.txt
