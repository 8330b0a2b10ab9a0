#!/bin/bash
# One gpurun call: GPU tests, smoke, bench, ncu launch list + full capture.
set -x
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
nvidia-smi -L > gpurun_out/gpu.txt 2>&1
lscpu | grep -E "Model name|^CPU\(s\)" >> gpurun_out/gpu.txt
timeout 900 python -m pytest tests -m gpu -x -q -s > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --profile --steps 20 --warmup 3 > gpurun_out/ncu_launch_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gru_simt -s 30 -c 2 -o gpurun_out/prof_gru python bench.py --profile --steps 20 --warmup 3 > gpurun_out/ncu_full_gru.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fetch_gather -s 30 -c 2 -o gpurun_out/prof_fetch python bench.py --profile --steps 20 --warmup 3 > gpurun_out/ncu_full_fetch.log 2>&1
ls -la gpurun_out
