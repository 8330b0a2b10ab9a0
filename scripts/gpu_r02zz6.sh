#!/bin/bash
# A/B with the 167-register GEMM: launch order of the commit (GEMM first) and the build's blocks-per-SM cap
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_zz6.log 2>&1
for rep in 1 2; do
  timeout 900 python bench.py --no-probe --no-cpu --no-train --no-apan > gpurun_out/ab6_gdelt_base.$rep.json 2> /dev/null
  MSPIPE_WB_FIRST=0 timeout 900 python bench.py --no-probe --no-cpu --no-train --no-apan > gpurun_out/ab6_gdelt_wb0.$rep.json 2> /dev/null
  MSPIPE_BUILD_BPS=16 timeout 900 python bench.py --no-probe --no-cpu --no-train --no-apan > gpurun_out/ab6_gdelt_bps16.$rep.json 2> /dev/null
  MSPIPE_WB_FIRST=0 timeout 900 python bench.py --config wiki --no-probe --no-cpu --no-train --no-apan > gpurun_out/ab6_wiki_wb0.$rep.json 2> /dev/null
  timeout 900 python bench.py --config wiki --no-probe --no-cpu --no-train --no-apan > gpurun_out/ab6_wiki_base.$rep.json 2> /dev/null
done
python - <<'PY'
import json, glob
for f in sorted(glob.glob("gpurun_out/ab6_*.json")):
    try:
        d = json.load(open(f))
    except Exception as e:
        print(f, "FAILED", e); continue
    print(f, "%.2f Mev/s" % (d["value"] / 1e6), "%.2f us/step" % (d["ms_per_step"] * 1e3))
PY
