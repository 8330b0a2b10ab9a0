#!/bin/bash
# F4 fix check (ragged-loop shuffles), the GDELT-size train fault hunt, APAN, benches, WB_FIRST A/B
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_zb.log 2>&1
timeout 600 python scripts/exp_train_stage.py gdelt 40000 > gpurun_out/zb_train_gdelt.log 2>&1; echo "rc=$?" >> gpurun_out/zb_train_gdelt.log
tail -5 gpurun_out/zb_train_gdelt.log
if ! grep -q "rc=0" gpurun_out/zb_train_gdelt.log; then
  timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python scripts/exp_train_stage.py gdelt 12000 > gpurun_out/zb_memcheck_train.log 2>&1
  grep -m 30 -i "invalid\|error\|at 0x\|by thread\|k_" gpurun_out/zb_memcheck_train.log | head -40
fi
timeout 1200 python -m pytest tests/test_gpu_train.py -q -s > gpurun_out/pytest_train.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_train.log
tail -25 gpurun_out/pytest_train.log
timeout 900 python -m pytest tests/test_gpu_apan.py -q -s > gpurun_out/pytest_apan.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_apan.log
tail -4 gpurun_out/pytest_apan.log
timeout 900 python bench.py --no-probe --no-cpu > gpurun_out/zb_bench_gdelt.json 2> gpurun_out/zb_bench_gdelt.err
timeout 600 python bench.py --config wiki --no-probe --no-cpu > gpurun_out/zb_bench_wiki.json 2> gpurun_out/zb_bench_wiki.err
for v in 0 1; do
  MSPIPE_WB_FIRST=$v timeout 900 python bench.py --no-probe --no-cpu --no-train > gpurun_out/ab_gdelt_wb$v.json 2> gpurun_out/ab_gdelt_wb$v.err
  MSPIPE_WB_FIRST=$v timeout 600 python bench.py --config wiki --no-probe --no-cpu --no-train > gpurun_out/ab_wiki_wb$v.json 2> gpurun_out/ab_wiki_wb$v.err
done
python - <<'PY'
import json, glob
for f in sorted(glob.glob("gpurun_out/zb_bench_*.json") + glob.glob("gpurun_out/ab_*_wb*.json")):
    try:
        d = json.load(open(f))
    except Exception as e:
        print(f, "FAILED", e); continue
    r = d["roofline"]
    print(f, "%.2f Mev/s" % (d["value"] / 1e6), "%.2f us/step" % (d["ms_per_step"] * 1e3), "alone", {k: round(v * 1e3, 2) for k, v in r.get("dominant_of", {}).items()}, "in_step", {k: round(v * 1e3, 2) for k, v in r.get("in_step_ms", {}).items()}, "train:", json.dumps(d.get("train"))[:300])
PY
