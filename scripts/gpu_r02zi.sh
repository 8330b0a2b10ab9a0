#!/bin/bash
# Round-2 final state: smoke, the whole GPU suite, the default bench line, wiki, the reference arm, F4 launch list
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_zi.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/zi_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/zi_smoke.log
cat gpurun_out/zi_smoke.log
timeout 1200 python -m pytest tests/test_gpu_train.py -q -s > gpurun_out/zi_pytest_train.log 2>&1; echo "rc=$?" >> gpurun_out/zi_pytest_train.log
grep -E "gdelt i=|passed|failed" gpurun_out/zi_pytest_train.log | tail -4
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/zi_pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/zi_pytest_gpu.log
tail -3 gpurun_out/zi_pytest_gpu.log
timeout 1200 python bench.py > gpurun_out/zi_bench_gdelt.json 2> gpurun_out/zi_bench_gdelt.err
timeout 900 python bench.py --config wiki --no-probe > gpurun_out/zi_bench_wiki.json 2> gpurun_out/zi_bench_wiki.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/zi_bench_reference.json 2> gpurun_out/zi_bench_reference.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_train_gdelt_zi.csv python scripts/exp_train_stage.py gdelt 12000 0 train > gpurun_out/ncu_train_gdelt_zi.log 2>&1
python - <<'PY'
import json
for f in ("gpurun_out/zi_bench_gdelt.json", "gpurun_out/zi_bench_wiki.json", "gpurun_out/zi_bench_reference.json"):
    try:
        d = json.load(open(f))
    except Exception as e:
        print(f, "FAILED", e); continue
    print(f, "%.3f Mev/s" % (d["value"] / 1e6), "ms/step", d.get("ms_per_step"), "e2e", (d.get("e2e") or {}).get("value"))
    for k in ("roofline", "roofline_gemm", "train", "apan", "hbm_probe", "cpu_baseline", "clocks"):
        print("  ", k, json.dumps(d.get(k))[:260])
PY
