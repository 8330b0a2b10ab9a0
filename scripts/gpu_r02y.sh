#!/bin/bash
# A/B: the message build (A5) on the prep's side stream (after k_prep of t+k) or on the commit's stream (before GEMM t)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "switch" > gpurun_out/pytest_y.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_y.log
tail -2 gpurun_out/pytest_y.log
for rep in 1 2; do
for b in prep commit; do
  MSPIPE_BUILD_ON=$b timeout 900 python bench.py --no-probe --no-cpu > gpurun_out/ab_gdelt_$b$rep.json 2> gpurun_out/ab_gdelt_$b$rep.err
  MSPIPE_BUILD_ON=$b timeout 600 python bench.py --config wiki --no-probe --no-cpu > gpurun_out/ab_wiki_$b$rep.json 2> gpurun_out/ab_wiki_$b$rep.err
done
done
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
