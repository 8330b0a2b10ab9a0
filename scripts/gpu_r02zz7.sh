#!/bin/bash
# final commit: smoke, the whole GPU suite (incl. F4 + MSPipe-S), the default bench line
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_zz7.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/zz7_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/zz7_smoke.log
cat gpurun_out/zz7_smoke.log
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/zz7_pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/zz7_pytest_gpu.log
tail -3 gpurun_out/zz7_pytest_gpu.log
t0=$(date +%s)
timeout 1200 python bench.py > gpurun_out/zz7_bench_gdelt.json 2> gpurun_out/zz7_bench_gdelt.err
echo "default bench wall: $(( $(date +%s) - t0 )) s"
timeout 900 python bench.py --config wiki --no-probe > gpurun_out/zz7_bench_wiki.json 2> gpurun_out/zz7_bench_wiki.err
python - <<'PY'
import json
for f in ("gpurun_out/zz7_bench_gdelt.json", "gpurun_out/zz7_bench_wiki.json"):
    d = json.load(open(f))
    print(f, "%.3f Mev/s" % (d["value"] / 1e6), d["ms_per_step"], "e2e", d["e2e"]["value"], "frac", d["roofline"]["frac"], "gemm", (d.get("roofline_gemm") or {}).get("frac"), "train", d["train"].get("value"), "apan", d["apan"].get("value"), "launches", d["gpu_launches"])
PY
