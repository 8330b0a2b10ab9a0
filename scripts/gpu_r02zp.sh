#!/bin/bash
# the final commit: smoke, the whole GPU suite, the default bench line (timed), F4 launch list
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_zp.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/zp_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/zp_smoke.log
cat gpurun_out/zp_smoke.log
timeout 1200 python -m pytest tests/test_gpu_train.py -q -s > gpurun_out/zp_pytest_train.log 2>&1; echo "rc=$?" >> gpurun_out/zp_pytest_train.log
grep -E "gdelt i=|passed|failed" gpurun_out/zp_pytest_train.log | tail -4
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/zp_pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/zp_pytest_gpu.log
tail -3 gpurun_out/zp_pytest_gpu.log
t0=$(date +%s)
timeout 1200 python bench.py > gpurun_out/zp_bench_gdelt.json 2> gpurun_out/zp_bench_gdelt.err
echo "default bench wall: $(( $(date +%s) - t0 )) s"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_train_gdelt_zp.csv python scripts/exp_train_stage.py gdelt 12000 0 train > gpurun_out/ncu_train_gdelt_zp.log 2>&1
python - <<'PY'
import json
d = json.load(open("gpurun_out/zp_bench_gdelt.json"))
print("%.3f Mev/s" % (d["value"] / 1e6), d["ms_per_step"], "e2e", d["e2e"]["value"], "frac", d["roofline"]["frac"], "gemm", d["roofline_gemm"]["frac"], "train", d["train"].get("value"), d["train"]["roofline"]["frac"], "apan", d["apan"].get("value"), "launches", d["gpu_launches"])
PY
