#!/bin/bash
# GPU tests (shard loopback first: the new window transport), bench GDELT / wiki / GDELT bf16
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_shard.py -q -x -s > gpurun_out/pytest_shard.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_shard.log
timeout 2400 python -m pytest tests -m gpu -q -s > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 1500 python bench.py > gpurun_out/bench_gdelt.json 2> gpurun_out/bench_gdelt.err; echo "rc=$?" >> gpurun_out/bench_gdelt.err
timeout 600 python bench.py --config wiki --no-probe > gpurun_out/bench_wiki.json 2> gpurun_out/bench_wiki.err; echo "rc=$?" >> gpurun_out/bench_wiki.err
timeout 900 python bench.py --gru bf16 --no-probe --no-cpu > gpurun_out/bench_gdelt_bf16.json 2> gpurun_out/bench_gdelt_bf16.err; echo "rc=$?" >> gpurun_out/bench_gdelt_bf16.err
ls -la gpurun_out
