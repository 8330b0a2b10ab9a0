#!/bin/bash
# F4 pipelined with the fetch: parity (trajectories at k = 1, 2), the bench train key
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_zv.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_train.py tests/test_gpu_apan.py -q -s > gpurun_out/zv_pytest_f34.log 2>&1; echo "rc=$?" >> gpurun_out/zv_pytest_f34.log
grep -E "k=|passed|failed|Error" gpurun_out/zv_pytest_f34.log | tail -8
timeout 900 python bench.py --no-probe --no-cpu --no-apan > gpurun_out/zv_bench_gdelt.json 2> gpurun_out/zv_bench_gdelt.err
timeout 900 python bench.py --config wiki --no-probe --no-cpu --no-apan > gpurun_out/zv_bench_wiki.json 2> gpurun_out/zv_bench_wiki.err
python - <<'PY'
import json
for f in ("gpurun_out/zv_bench_gdelt.json", "gpurun_out/zv_bench_wiki.json"):
    try:
        d = json.load(open(f))
    except Exception as e:
        print(f, "FAILED", e); continue
    t = d.get("train") or {}
    print(f, "%.2f Mev/s" % (d["value"] / 1e6), "train", t.get("value"), t.get("ms_per_step"), t.get("train_ms_in_step"), t.get("error"))
PY
