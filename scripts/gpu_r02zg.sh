#!/bin/bash
# APAN under staleness k >= 1: parity + the bench key at the config's k
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_zg.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_apan.py -q -s > gpurun_out/zg_pytest_apan.log 2>&1; echo "rc=$?" >> gpurun_out/zg_pytest_apan.log
tail -12 gpurun_out/zg_pytest_apan.log
timeout 900 python bench.py --no-probe --no-cpu --no-train > gpurun_out/zg_bench_gdelt.json 2> gpurun_out/zg_bench_gdelt.err
timeout 900 python bench.py --config wiki --no-probe --no-cpu --no-train > gpurun_out/zg_bench_wiki.json 2> gpurun_out/zg_bench_wiki.err
python - <<'PY'
import json
for f in ("gpurun_out/zg_bench_gdelt.json", "gpurun_out/zg_bench_wiki.json"):
    try:
        d = json.load(open(f))
    except Exception as e:
        print(f, "FAILED", e); continue
    print(f, "%.2f Mev/s" % (d["value"] / 1e6), "apan", json.dumps(d.get("apan"))[:400])
PY
