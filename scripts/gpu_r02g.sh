#!/bin/bash
# A/B: GEMM K-split at GDELT (prefix T-CSR), sampler hints at GDELT (full T-CSR); then the GPU tests
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -s -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -5 gpurun_out/pytest_gpu.log
for S in 1 2 4; do
  MSPIPE_TC_SPLITS=$S timeout 900 python bench.py --tcsr-events 4000000 --no-probe --no-cpu > gpurun_out/ab_splits_$S.json 2> gpurun_out/ab_splits_$S.err
done
MSPIPE_SAMPLE_HINT=0 timeout 900 python bench.py --no-probe --no-cpu > gpurun_out/ab_hint0.json 2> gpurun_out/ab_hint0.err
timeout 900 python bench.py --no-probe --no-cpu > gpurun_out/ab_hint1.json 2> gpurun_out/ab_hint1.err
python - <<'PY'
import json, glob
for f in sorted(glob.glob("gpurun_out/ab_*.json")):
    try:
        d = json.load(open(f))
    except Exception as e:
        print(f, "FAILED", e); continue
    r = d["roofline"]
    print(f, "%.2f Mev/s" % (d["value"] / 1e6), "%.2f us/step" % (d["ms_per_step"] * 1e3), "alone", {k: round(v * 1e3, 2) for k, v in r.get("dominant_of", {}).items()}, "in_step", {k: round(v * 1e3, 2) for k, v in r.get("in_step_ms", {}).items()})
PY
for c in gdelt wiki; do
  echo "== $c" >> gpurun_out/phases.txt
  timeout 600 python scripts/exp_gru_phases.py $c >> gpurun_out/phases.txt 2>&1
done
cat gpurun_out/phases.txt
