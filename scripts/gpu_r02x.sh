#!/bin/bash
# what the GEMM's gate phase waits on: phase marks without the stores / without the math (timing only)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
for v in "" "-DMSPIPE_DBG_NOSTORE" "-DMSPIPE_DBG_NOMATH"; do
  for cfg in gdelt wiki; do
    echo "== $cfg [$v] in-step"; EXP_FLAGS="$v" timeout 600 python scripts/exp_gru_phases.py $cfg 2>&1 | tail -13 | grep -v "^entry\|^acc_full\|^sync\|dead"
    echo "== $cfg [$v] alone"; EXP_COLD=1 EXP_FLAGS="$v" timeout 600 python scripts/exp_gru_phases.py $cfg 2>&1 | tail -13 | grep -v "^entry\|^acc_full\|^sync\|dead"
  done
done > gpurun_out/phases_x.txt
cat gpurun_out/phases_x.txt
