#!/bin/bash
# A/B: neighbour rows stored T-CSR probes loaded evict-first (MSPIPE_TCSR_LDCS=1); knob parity
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_zl.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "switch" > gpurun_out/zl_pytest_switch.log 2>&1; echo "rc=$?" >> gpurun_out/zl_pytest_switch.log
tail -3 gpurun_out/zl_pytest_switch.log
for rep in 1 2; do
for v in 0 1; do
  MSPIPE_TCSR_LDCS=$v timeout 900 python bench.py --no-probe --no-cpu --no-train --no-apan > gpurun_out/ab_gdelt_ldcs$v.$rep.json 2> gpurun_out/ab_gdelt_ldcs$v.$rep.err
  MSPIPE_TCSR_LDCS=$v timeout 900 python bench.py --config wiki --no-probe --no-cpu --no-train --no-apan > gpurun_out/ab_wiki_ldcs$v.$rep.json 2> gpurun_out/ab_wiki_ldcs$v.$rep.err
done
done
python - <<'PY'
import json, glob
for f in sorted(glob.glob("gpurun_out/ab_*_ldcs*.json")):
    try:
        d = json.load(open(f))
    except Exception as e:
        print(f, "FAILED", e); continue
    r = d["roofline"]
    print(f, "%.2f Mev/s" % (d["value"] / 1e6), "%.2f us/step" % (d["ms_per_step"] * 1e3), "alone", {k: round(v * 1e3, 2) for k, v in r.get("dominant_of", {}).items()}, "in_step", {k: round(v * 1e3, 2) for k, v in r.get("in_step_ms", {}).items()})
PY
