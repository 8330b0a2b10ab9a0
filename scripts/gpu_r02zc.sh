#!/bin/bash
# F4 after the tanh decoder, the parallel scatter and gather: parity, the train step's kernel breakdown, benches
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_zc.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_train.py -q -s > gpurun_out/pytest_train_zc.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_train_zc.log
grep -E "i=|k=|passed|failed" gpurun_out/pytest_train_zc.log | tail -14
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_train_gdelt.csv python scripts/exp_train_stage.py gdelt 12000 0 > gpurun_out/ncu_train_gdelt.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_train_wiki.csv python scripts/exp_train_stage.py wiki 3000 0 > gpurun_out/ncu_train_wiki.log 2>&1
timeout 900 python bench.py --no-probe --no-cpu > gpurun_out/zc_bench_gdelt.json 2> gpurun_out/zc_bench_gdelt.err
timeout 600 python bench.py --config wiki --no-probe --no-cpu > gpurun_out/zc_bench_wiki.json 2> gpurun_out/zc_bench_wiki.err
python - <<'PY'
import json, glob, csv, collections
for f in sorted(glob.glob("gpurun_out/zc_bench_*.json")):
    try:
        d = json.load(open(f))
    except Exception as e:
        print(f, "FAILED", e); continue
    print(f, "%.2f Mev/s" % (d["value"] / 1e6), "%.2f us/step" % (d["ms_per_step"] * 1e3), "train:", json.dumps(d.get("train"))[:500])
for f in sorted(glob.glob("gpurun_out/launches_train_*.csv")):
    t = collections.defaultdict(list)
    try:
        rows = list(csv.reader(open(f)))
        hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
        h = rows[hdr]; ki, vi = h.index("Kernel Name"), h.index("Metric Value")
        for r in rows[hdr + 1:]:
            if len(r) > vi:
                t[r[ki][:70]].append(float(r[vi].replace(",", "")))
    except Exception as e:
        print(f, "parse", e); continue
    print(f)
    for k, v in sorted(t.items(), key=lambda kv: -sum(kv[1]))[:16]:
        print("  %-70s n=%4d mean %9.1f ns total %10.1f us" % (k, len(v), sum(v) / len(v), sum(v) / 1e3))
PY
