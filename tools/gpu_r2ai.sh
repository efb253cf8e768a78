#!/bin/bash
# Final-kernel refresh of the other BASELINE configs and the imbalance runs on 4 GPUs.
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
{
echo "## C4 n=8,476,421 tau=8, P=8 S=8"
for N in 1 2 4; do bash tools/ab_env.sh $N "-" --nparams 8476421 --tau 8; done
echo "## C3 n=213,000,000 tau=8, P=8 S=8"
for N in 1 2 4; do bash tools/ab_env.sh $N "-" --nparams 213000000 --tau 8 --steps 30; done
echo "## rotating straggler: P=4 S=4 on 4 GPUs, base 1.0 ms/step on every GPU, one StragglerPolicy victim +3.2 ms"
bash tools/ab_env.sh 4 "-" --P 4 --S 4 --base-ms 1.0 --victims 1 --extra-ms 3.2
bash tools/ab_env.sh 4 "-" --P 4 --S 4 --base-ms 1.0 --victims 1 --extra-ms 3.2 --grace-us 0
bash tools/ab_env.sh 4 "-" --P 4 --S 4 --base-ms 1.0 --victims 1 --extra-ms 3.2 --blocking
echo "## C3-style bucketed sequence lengths, P=8 S=8 on 4 GPUs, base 2.0 ms"
bash tools/ab_env.sh 4 "-" --S 8 --tau 8 --base-ms 2.0 --length-buckets
bash tools/ab_env.sh 4 "-" --S 8 --tau 8 --base-ms 2.0 --length-buckets --blocking
} > gpurun_out/r2ai.txt 2>&1
cat gpurun_out/r2ai.txt
