#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
EXP_FULL=1 timeout 600 python scripts/exp_prep_phases.py gdelt > gpurun_out/prep_phases.txt 2>&1
MSPIPE_PREP_SMEM=0 EXP_FULL=1 timeout 600 python scripts/exp_prep_phases.py gdelt >> gpurun_out/prep_phases.txt 2>&1
cat gpurun_out/prep_phases.txt
timeout 900 python bench.py --no-probe --no-cpu > gpurun_out/ab_smem1.json 2> gpurun_out/ab_smem1.err
MSPIPE_PREP_SMEM=0 timeout 900 python bench.py --no-probe --no-cpu > gpurun_out/ab_smem0.json 2> gpurun_out/ab_smem0.err
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
