#!/bin/bash
# One gpurun call: GPU tests, smoke, bench, ncu launch list + full captures.
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
nvidia-smi -L > gpurun_out/gpu.txt 2>&1
lscpu | grep -E "Model name|^CPU\(s\)" >> gpurun_out/gpu.txt
timeout 180 python -m pytest tests/test_gpu_parity.py -q -x -k "update_teacher_forced and tiny" > gpurun_out/pytest_tc_first.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_tc_first.log
timeout 900 python -m pytest tests -m gpu -q -s > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
bash scripts/bench_sweep.sh > gpurun_out/sweep_summary.txt 2>&1
timeout 900 python bench.py --gru simt --no-cpu > gpurun_out/bench_simt.json 2> gpurun_out/bench_simt.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --profile --steps 20 --warmup 3 > gpurun_out/ncu_launch_bench.log 2>&1
for k in k_gru_tc k_build_x k_prep; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 4 -c 1 -o gpurun_out/prof_$k python bench.py --profile --steps 20 --warmup 3 > gpurun_out/ncu_full_$k.log 2>&1
done
ls -la gpurun_out
