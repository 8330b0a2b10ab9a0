#!/bin/bash
# A/B after the cache-policy changes: GEMM K-split at GDELT (S = 1, 2, 4) and the split commit
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_zq.log 2>&1
for rep in 1 2; do
  for S in 1 2 4; do
    MSPIPE_TC_BIG_S=$S timeout 900 python bench.py --no-probe --no-cpu --no-train --no-apan > gpurun_out/ab_gdelt_S$S.$rep.json 2> gpurun_out/ab_gdelt_S$S.$rep.err
  done
  MSPIPE_SPLIT_COMMIT=0 timeout 900 python bench.py --no-probe --no-cpu --no-train --no-apan > gpurun_out/ab_gdelt_sc0.$rep.json 2> gpurun_out/ab_gdelt_sc0.$rep.err
done
python - <<'PY'
import json, glob
for f in sorted(glob.glob("gpurun_out/ab_gdelt_S*.json") + glob.glob("gpurun_out/ab_gdelt_sc0*.json")):
    try:
        d = json.load(open(f))
    except Exception as e:
        print(f, "FAILED", e); continue
    r = d["roofline"]
    print(f, "%.2f Mev/s" % (d["value"] / 1e6), "%.2f us/step" % (d["ms_per_step"] * 1e3), "alone", {k: round(v * 1e3, 2) for k, v in r.get("dominant_of", {}).items()}, "in_step", {k: round(v * 1e3, 2) for k, v in r.get("in_step_ms", {}).items()})
PY
