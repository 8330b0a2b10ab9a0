#!/bin/bash
# F4 parallel segment bounds: parity + bench (train key) + launch list
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_zn.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_train.py tests/test_gpu_apan.py -q -s > gpurun_out/zn_pytest_f34.log 2>&1; echo "rc=$?" >> gpurun_out/zn_pytest_f34.log
grep -E "gdelt i=|passed|failed" gpurun_out/zn_pytest_f34.log | tail -4
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_train_gdelt_zn.csv python scripts/exp_train_stage.py gdelt 12000 0 train > gpurun_out/ncu_train_gdelt_zn.log 2>&1
timeout 900 python bench.py --no-probe --no-cpu --no-apan > gpurun_out/zn_bench_gdelt.json 2> gpurun_out/zn_bench_gdelt.err
python - <<'PY'
import json, csv, collections
d = json.load(open("gpurun_out/zn_bench_gdelt.json"))
print("gdelt %.2f Mev/s" % (d["value"] / 1e6), "train", json.dumps(d.get("train"))[:300])
t = collections.defaultdict(list)
rows = list(csv.reader(open("gpurun_out/launches_train_gdelt_zn.csv")))
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]; ki, vi = h.index("Kernel Name"), h.index("Metric Value")
for r in rows[hdr + 1:]:
    if len(r) > vi:
        t[r[ki][:70]].append(float(r[vi].replace(",", "")))
for k, v in sorted(t.items(), key=lambda kv: -sum(kv[1]))[:14]:
    print("  %-70s n=%4d mean %9.1f ns" % (k, len(v), sum(v) / len(v)))
PY
