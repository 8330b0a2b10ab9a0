#!/bin/bash
# phase marks of the 20-unit GEMM tile (GDELT S = 2, wiki S = 4), in-step and alone
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
for cfg in gdelt wiki; do
  echo "== $cfg in-step"; timeout 600 python scripts/exp_gru_phases.py $cfg 2>&1 | tail -16
  echo "== $cfg alone"; EXP_COLD=1 timeout 600 python scripts/exp_gru_phases.py $cfg 2>&1 | tail -16
done > gpurun_out/phases_v.txt
cat gpurun_out/phases_v.txt
