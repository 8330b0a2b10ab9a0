#!/bin/bash
# GEMM phase anatomy (per-CTA globaltimer marks, -DMSPIPE_PHASES debug build) at GDELT and wiki, warm and cold
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
for c in gdelt wiki; do
  echo "== $c warm" >> gpurun_out/phases.txt
  timeout 600 python scripts/exp_gru_phases.py $c >> gpurun_out/phases.txt 2>&1
  echo "== $c cold" >> gpurun_out/phases.txt
  EXP_COLD=1 timeout 600 python scripts/exp_gru_phases.py $c >> gpurun_out/phases.txt 2>&1
done
cat gpurun_out/phases.txt
