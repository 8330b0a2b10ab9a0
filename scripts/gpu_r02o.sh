#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
EXP_FULL=1 timeout 600 python scripts/exp_prep_phases.py gdelt > gpurun_out/prep_phases.txt 2>&1
timeout 600 python scripts/exp_prep_phases.py wiki >> gpurun_out/prep_phases.txt 2>&1
cat gpurun_out/prep_phases.txt
