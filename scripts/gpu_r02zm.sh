#!/bin/bash
# Round-2 final evidence after the cache-policy changes: smoke, the whole GPU suite, the default bench
# line, wiki, the reference arm, launch lists and ncu --set full of the step's kernels per config
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_zm.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/zm_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/zm_smoke.log
cat gpurun_out/zm_smoke.log
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/zm_pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/zm_pytest_gpu.log
tail -3 gpurun_out/zm_pytest_gpu.log
timeout 1200 python bench.py > gpurun_out/zm_bench_gdelt.json 2> gpurun_out/zm_bench_gdelt.err
timeout 900 python bench.py --config wiki --no-probe > gpurun_out/zm_bench_wiki.json 2> gpurun_out/zm_bench_wiki.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/zm_bench_reference.json 2> gpurun_out/zm_bench_reference.err
for c in gdelt wiki; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$c.csv python bench.py --config $c --profile --steps 20 --warmup 3 > gpurun_out/ncu_launch_$c.log 2>&1
  for k in k_prep k_gru_tc k_build_x k_writeback; do
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 10 -c 1 -o gpurun_out/prof_${c}_$k python bench.py --config $c --profile --steps 20 --warmup 3 > gpurun_out/ncu_full_${c}_$k.log 2>&1
  done
done
python - <<'PY'
import json
for f in ("gpurun_out/zm_bench_gdelt.json", "gpurun_out/zm_bench_wiki.json", "gpurun_out/zm_bench_reference.json"):
    try:
        d = json.load(open(f))
    except Exception as e:
        print(f, "FAILED", e); continue
    print(f, "%.3f Mev/s" % (d["value"] / 1e6), "ms/step", d.get("ms_per_step"), "e2e", (d.get("e2e") or {}).get("value"))
    for k in ("roofline", "roofline_gemm", "train", "apan", "clocks"):
        print("  ", k, json.dumps(d.get(k))[:200])
PY
