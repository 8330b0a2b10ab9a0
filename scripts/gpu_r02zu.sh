#!/bin/bash
# the final commit's bench lines (default + wiki)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_zu.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/zu_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/zu_smoke.log
cat gpurun_out/zu_smoke.log
timeout 1200 python bench.py > gpurun_out/zu_bench_gdelt.json 2> gpurun_out/zu_bench_gdelt.err
timeout 900 python bench.py --config wiki --no-probe > gpurun_out/zu_bench_wiki.json 2> gpurun_out/zu_bench_wiki.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/zu_bench_reference.json 2> gpurun_out/zu_bench_reference.err
python - <<'PY'
import json
for f in ("gpurun_out/zu_bench_gdelt.json", "gpurun_out/zu_bench_wiki.json", "gpurun_out/zu_bench_reference.json"):
    d = json.load(open(f))
    r = d.get("roofline") or {}
    print(f, "%.3f Mev/s" % (d["value"] / 1e6), d["ms_per_step"], "e2e", (d.get("e2e") or {}).get("value"), "roofline", r.get("kernel"), r.get("frac"), "gemm", (d.get("roofline_gemm") or {}).get("frac"), "train", (d.get("train") or {}).get("value"), "apan", (d.get("apan") or {}).get("value"))
PY
