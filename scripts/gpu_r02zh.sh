#!/bin/bash
# F4 with 3xTF32 tensor-core projections: parity + bench + launch list; graph node-priority A/B
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_zh.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_train.py -q -s > gpurun_out/zh_pytest_train.log 2>&1; echo "rc=$?" >> gpurun_out/zh_pytest_train.log
grep -E "i=|k=|passed|failed|Error" gpurun_out/zh_pytest_train.log | tail -14
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_train_gdelt_zh.csv python scripts/exp_train_stage.py gdelt 12000 0 train > gpurun_out/ncu_train_gdelt_zh.log 2>&1
timeout 900 python bench.py --no-probe --no-cpu --no-apan > gpurun_out/zh_bench_gdelt.json 2> gpurun_out/zh_bench_gdelt.err
timeout 900 python bench.py --config wiki --no-probe --no-cpu --no-apan > gpurun_out/zh_bench_wiki.json 2> gpurun_out/zh_bench_wiki.err
for p in 0 1; do
  MSPIPE_GRAPH_PRIO=1 MSPIPE_SIDE_PRIO=-$p timeout 900 python bench.py --no-probe --no-cpu --no-apan --no-train > gpurun_out/ab_gdelt_prio$p.json 2> gpurun_out/ab_gdelt_prio$p.err
  MSPIPE_GRAPH_PRIO=1 MSPIPE_SIDE_PRIO=-$p timeout 900 python bench.py --config wiki --no-probe --no-cpu --no-apan --no-train > gpurun_out/ab_wiki_prio$p.json 2> gpurun_out/ab_wiki_prio$p.err
done
python - <<'PY'
import json, glob, csv, collections
for f in sorted(glob.glob("gpurun_out/zh_bench_*.json") + glob.glob("gpurun_out/ab_*_prio*.json")):
    try:
        d = json.load(open(f))
    except Exception as e:
        print(f, "FAILED", e); continue
    print(f, "%.2f Mev/s" % (d["value"] / 1e6), "%.2f us/step" % (d["ms_per_step"] * 1e3), "train", json.dumps(d.get("train"))[:330])
t = collections.defaultdict(list)
rows = list(csv.reader(open("gpurun_out/launches_train_gdelt_zh.csv")))
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]; ki, vi = h.index("Kernel Name"), h.index("Metric Value")
for r in rows[hdr + 1:]:
    if len(r) > vi:
        t[r[ki][:70]].append(float(r[vi].replace(",", "")))
for k, v in sorted(t.items(), key=lambda kv: -sum(kv[1]))[:12]:
    print("  %-70s n=%4d mean %9.1f ns" % (k, len(v), sum(v) / len(v)))
PY
