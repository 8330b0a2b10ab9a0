#!/bin/bash
# A/B of one knob on the captured step (exp_overlap.py), then quick tests + bench.
# usage: KNOBS="MSPIPE_SPLIT_COMMIT=0,1" CONFIGS="wiki gdelt" bash scripts/gpu_ab.sh
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
for c in ${CONFIGS:-wiki}; do
  EXP_EVENTS=$([ $c = gdelt ] && echo 2000000) EXP_KNOBS="$KNOBS" timeout 600 python scripts/exp_overlap.py $c >> gpurun_out/ab.txt 2>&1
done
cat gpurun_out/ab.txt
bash scripts/gpu_quick.sh
