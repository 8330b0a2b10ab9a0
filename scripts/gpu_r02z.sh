#!/bin/bash
# Round-2 evidence refresh on the current kernels: smoke, the whole GPU suite, the default bench
# (GDELT headline with probe + oracle), wiki, launch lists and one ncu --set full capture per kernel and config
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_z.log 2>&1; echo "rc=$?" >> gpurun_out/smoke_z.log
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/pytest_z.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_z.log
tail -3 gpurun_out/pytest_z.log
timeout 900 python bench.py > gpurun_out/z_bench_gdelt.json 2> gpurun_out/z_bench_gdelt.err
timeout 600 python bench.py --config wiki --no-probe > gpurun_out/z_bench_wiki.json 2> gpurun_out/z_bench_wiki.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/z_bench_reference.json 2> gpurun_out/z_bench_reference.err
for c in gdelt wiki; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$c.csv python bench.py --config $c --profile --steps 20 --warmup 3 > gpurun_out/ncu_launch_$c.log 2>&1
  for k in k_prep k_gru_tc k_build_x k_writeback; do
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 10 -c 1 -o gpurun_out/prof_${c}_$k python bench.py --config $c --profile --steps 20 --warmup 3 > gpurun_out/ncu_full_${c}_$k.log 2>&1
  done
done
ls gpurun_out
