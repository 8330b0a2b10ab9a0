#!/bin/bash
# the exact final commit: smoke, the whole GPU suite, the default bench line
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_zo.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/zo_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/zo_smoke.log
cat gpurun_out/zo_smoke.log
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/zo_pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/zo_pytest_gpu.log
tail -3 gpurun_out/zo_pytest_gpu.log
/usr/bin/time -v timeout 1200 python bench.py > gpurun_out/zo_bench_gdelt.json 2> gpurun_out/zo_bench_gdelt.err
grep -E "Elapsed" gpurun_out/zo_bench_gdelt.err
python - <<'PY'
import json
d = json.load(open("gpurun_out/zo_bench_gdelt.json"))
print("%.3f Mev/s" % (d["value"] / 1e6), d["ms_per_step"], "e2e", d["e2e"]["value"], "frac", d["roofline"]["frac"], "gemm", d["roofline_gemm"]["frac"], "train", d["train"].get("value"), "apan", d["apan"].get("value"), "launches", d["gpu_launches"])
PY
