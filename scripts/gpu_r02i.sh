#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -s > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -4 gpurun_out/pytest_gpu.log
for S in 1 2 4; do
  MSPIPE_TC_SPLITS=$S timeout 600 python bench.py --config wiki --no-probe --no-cpu > gpurun_out/ab_wiki_S$S.json 2> gpurun_out/ab_wiki_S$S.err
done
timeout 1500 python bench.py > gpurun_out/bench_gdelt.json 2> gpurun_out/bench_gdelt.err
python - <<'PY'
import json, glob
for f in sorted(glob.glob("gpurun_out/ab_*.json")) + ["gpurun_out/bench_gdelt.json"]:
    try:
        d = json.load(open(f))
    except Exception as e:
        print(f, "FAILED", e); continue
    r = d["roofline"]
    print(f, "%.2f Mev/s" % (d["value"] / 1e6), "%.2f us/step" % (d["ms_per_step"] * 1e3), "alone", {k: round(v * 1e3, 2) for k, v in r.get("dominant_of", {}).items()}, "in_step", {k: round(v * 1e3, 2) for k, v in r.get("in_step_ms", {}).items()})
PY
