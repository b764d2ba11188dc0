#!/bin/bash
# Launch list + ncu --set full captures of the two trailing-update GEMMs of the
# config-3 bench (run on the GPU box from the repo root; outputs in gpurun_out/).
set -u
OUT=gpurun_out
TAG=${1:-head}
CMD="python bench.py --steps 1 --warmup 1 --cfg5-slices 0 --e2e-steps 0"
ncu --metrics gpu__time_duration.sum --clock-control none -c ${NLAUNCH:-1200} --csv \
    --log-file $OUT/launches_$TAG.csv $CMD > $OUT/ncu_list_$TAG.log 2>&1
echo "launch list rc=$?"
NN_SKIP=$(python tools/ncu_pick.py $OUT/launches_$TAG.csv 'gemm_nn_sub_asyncepi$' 148 longest)
TN_SKIP=$(python tools/ncu_pick.py $OUT/launches_$TAG.csv 'gemm_dmma_kernel' 1000 longest)
echo "nn skip $NN_SKIP tn skip $TN_SKIP"
ncu --set full --clock-control none --import-source on -k regex:gemm_nn_sub_asyncepi \
    --launch-skip $NN_SKIP --launch-count 1 -o $OUT/ncu_nn_$TAG -f $CMD > $OUT/ncu_nn_$TAG.log 2>&1
echo "nn full rc=$?"
ncu --set full --clock-control none --import-source on -k regex:gemm_dmma_kernel \
    --launch-skip $TN_SKIP --launch-count 1 -o $OUT/ncu_tn_$TAG -f $CMD > $OUT/ncu_tn_$TAG.log 2>&1
echo "tn full rc=$?"
