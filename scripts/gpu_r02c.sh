#!/bin/bash
# full GPU test suite, smoke, bench (GDELT headline + wiki), one ncu --set full capture per kernel at GDELT
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -s -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1500 python bench.py > gpurun_out/bench_gdelt.json 2> gpurun_out/bench_gdelt.err; echo "rc=$?" >> gpurun_out/bench_gdelt.err
timeout 600 python bench.py --config wiki --no-probe > gpurun_out/bench_wiki.json 2> gpurun_out/bench_wiki.err; echo "rc=$?" >> gpurun_out/bench_wiki.err
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:'k_prep|k_build_x|k_gru_tc|k_writeback' -s 40 -c 4 -o gpurun_out/prof_gdelt_multi python bench.py --profile --steps 20 --warmup 3 > gpurun_out/ncu_full_gdelt.log 2>&1
ls -la gpurun_out
