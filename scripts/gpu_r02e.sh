#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "graph or staged" > gpurun_out/pytest_graph.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_graph.log
timeout 600 python bench.py --config wiki --no-probe --no-cpu --steps 40 > gpurun_out/bench_wiki.json 2> gpurun_out/bench_wiki.err; echo "rc=$?" >> gpurun_out/bench_wiki.err
timeout 2400 python -m pytest tests -m gpu -q -s > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
bash scripts/gpu_r02d.sh
