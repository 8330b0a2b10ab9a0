#!/bin/bash
# bench (GDELT headline, wiki), ncu launch lists and one multi-kernel --set full capture per config
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 1500 python bench.py > gpurun_out/bench_gdelt.json 2> gpurun_out/bench_gdelt.err; echo "rc=$?" >> gpurun_out/bench_gdelt.err
timeout 600 python bench.py --config wiki --no-probe > gpurun_out/bench_wiki.json 2> gpurun_out/bench_wiki.err; echo "rc=$?" >> gpurun_out/bench_wiki.err
for c in gdelt wiki; do
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$c.csv python bench.py --config $c --profile --steps 20 --warmup 3 > gpurun_out/ncu_launch_$c.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:'k_prep|k_build_x|k_gru_tc|k_writeback' -s 40 -c 4 -o gpurun_out/prof_${c}_multi python bench.py --config $c --profile --steps 20 --warmup 3 > gpurun_out/ncu_full_$c.log 2>&1
done
ls -la gpurun_out
