#!/bin/bash
# F4 two-pass scatter: parity + launch list; sanitizer on the F3/F4 kernels; benches with the F3 APAN and F4 keys
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_zd.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_train.py tests/test_gpu_apan.py -q -s > gpurun_out/pytest_f34_zd.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_f34_zd.log
grep -E "i=|k=|memory|passed|failed" gpurun_out/pytest_f34_zd.log | tail -20
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_train_gdelt_zd.csv python scripts/exp_train_stage.py gdelt 12000 0 > gpurun_out/ncu_train_gdelt_zd.log 2>&1
timeout 1500 compute-sanitizer --tool memcheck python -m pytest tests/test_gpu_train.py tests/test_gpu_apan.py -q -x -k "tiny" > gpurun_out/zd_memcheck_f34.log 2>&1; echo "rc=$?" >> gpurun_out/zd_memcheck_f34.log
tail -4 gpurun_out/zd_memcheck_f34.log
timeout 1500 compute-sanitizer --tool racecheck python -m pytest tests/test_gpu_train.py -q -x -k "tiny-1" > gpurun_out/zd_racecheck_f4.log 2>&1; echo "rc=$?" >> gpurun_out/zd_racecheck_f4.log
tail -4 gpurun_out/zd_racecheck_f4.log
timeout 900 python bench.py --no-probe --no-cpu > gpurun_out/zd_bench_gdelt.json 2> gpurun_out/zd_bench_gdelt.err
timeout 600 python bench.py --config wiki --no-probe --no-cpu > gpurun_out/zd_bench_wiki.json 2> gpurun_out/zd_bench_wiki.err
python - <<'PY'
import json, glob, csv, collections
for f in sorted(glob.glob("gpurun_out/zd_bench_*.json")):
    try:
        d = json.load(open(f))
    except Exception as e:
        print(f, "FAILED", e); continue
    print(f, "%.2f Mev/s" % (d["value"] / 1e6), "%.2f us/step" % (d["ms_per_step"] * 1e3))
    print("  train:", json.dumps(d.get("train"))[:400])
    print("  apan:", json.dumps(d.get("apan"))[:400])
for f in sorted(glob.glob("gpurun_out/launches_train_gdelt_zd.csv")):
    t = collections.defaultdict(list)
    rows = list(csv.reader(open(f)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]; ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    for r in rows[hdr + 1:]:
        if len(r) > vi:
            t[r[ki][:70]].append(float(r[vi].replace(",", "")))
    print(f)
    for k, v in sorted(t.items(), key=lambda kv: -sum(kv[1]))[:12]:
        print("  %-70s n=%4d mean %9.1f ns total %10.1f us" % (k, len(v), sum(v) / len(v), sum(v) / 1e3))
PY
