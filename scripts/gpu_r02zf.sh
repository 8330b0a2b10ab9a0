#!/bin/bash
# APAN key ring + the extended smoke + F4 edge cases; the APAN bench key
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_zf.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/zf_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/zf_smoke.log
cat gpurun_out/zf_smoke.log
timeout 1200 python -m pytest tests/test_gpu_apan.py tests/test_gpu_train.py -q -s > gpurun_out/zf_pytest_f34.log 2>&1; echo "rc=$?" >> gpurun_out/zf_pytest_f34.log
grep -E "memory|k=|passed|failed|Error" gpurun_out/zf_pytest_f34.log | tail -14
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_apan_gdelt_zf.csv python scripts/exp_train_stage.py gdelt 12000 0 apan > gpurun_out/ncu_apan_gdelt_zf.log 2>&1
timeout 900 python bench.py --no-probe --no-cpu --no-train > gpurun_out/zf_bench_gdelt.json 2> gpurun_out/zf_bench_gdelt.err
python - <<'PY'
import json, csv, collections
d = json.load(open("gpurun_out/zf_bench_gdelt.json"))
print("gdelt %.2f Mev/s" % (d["value"] / 1e6), "apan", json.dumps(d.get("apan"))[:300])
t = collections.defaultdict(list)
rows = list(csv.reader(open("gpurun_out/launches_apan_gdelt_zf.csv")))
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]; ki, vi = h.index("Kernel Name"), h.index("Metric Value")
for r in rows[hdr + 1:]:
    if len(r) > vi:
        t[r[ki][:70]].append(float(r[vi].replace(",", "")))
for k, v in sorted(t.items(), key=lambda kv: -sum(kv[1]))[:10]:
    print("  %-70s n=%4d mean %9.1f ns" % (k, len(v), sum(v) / len(v)))
PY
