#!/bin/bash
# 20-unit GEMM tile, S = 2 at GDELT size: the whole GPU suite, then GDELT and wiki benches
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_u.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_u.log
tail -3 gpurun_out/pytest_u.log
timeout 900 python bench.py --no-cpu > gpurun_out/ab_gdelt.json 2> gpurun_out/ab_gdelt.err
timeout 600 python bench.py --config wiki --no-probe --no-cpu > gpurun_out/ab_wiki.json 2> gpurun_out/ab_wiki.err
python - <<'PY'
import json, glob
for f in sorted(glob.glob("gpurun_out/ab_*.json")):
    try:
        d = json.load(open(f))
    except Exception as e:
        print(f, "FAILED", e); continue
    r = d["roofline"]
    print(f, "%.2f Mev/s" % (d["value"] / 1e6), "%.2f us/step" % (d["ms_per_step"] * 1e3), "e2e %.1f" % (d["e2e"]["value"] / 1e6), "alone", {k: round(v * 1e3, 2) for k, v in r.get("dominant_of", {}).items()}, "in_step", {k: round(v * 1e3, 2) for k, v in r.get("in_step_ms", {}).items()})
PY
