#!/bin/bash
# ncu --set full of named kernels inside a short bench run (1 GPU).
# usage: [BENCH_ARGS="..."] bash scripts/gpu_prof.sh kernel_regex...
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
ARGS="${BENCH_ARGS:---profile --steps 12 --warmup 3}"
TAG="${PROF_TAG:-}"
for k in "$@"; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 4 -c 1 -o gpurun_out/prof_${k}${TAG} python bench.py $ARGS > gpurun_out/ncu_full_${k}${TAG}.log 2>&1
done
ls -la gpurun_out
