#!/bin/bash
# A/B: GEMM K-split at wiki size (S = 2 default, 4, 8)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_zz2.log 2>&1
for rep in 1 2; do
  for S in 2 4 8; do
    MSPIPE_TC_SPLITS=$S timeout 900 python bench.py --config wiki --no-probe --no-cpu --no-train --no-apan > gpurun_out/ab_wiki_S$S.$rep.json 2> gpurun_out/ab_wiki_S$S.$rep.err
  done
done
python - <<'PY'
import json, glob
for f in sorted(glob.glob("gpurun_out/ab_wiki_S*.json")):
    try:
        d = json.load(open(f))
    except Exception as e:
        print(f, "FAILED", e); continue
    r = d["roofline"]
    print(f, "%.2f Mev/s" % (d["value"] / 1e6), "%.2f us/step" % (d["ms_per_step"] * 1e3), "alone", {k: round(v * 1e3, 2) for k, v in r.get("dominant_of", {}).items()})
PY
