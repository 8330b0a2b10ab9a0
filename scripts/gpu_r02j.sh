#!/bin/bash
# GDELT full-T-CSR bench at K-split 1 and 2; wiki bench (default S now 2); ncu --set full per kernel at GDELT and wiki
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
for S in 1 2; do
  MSPIPE_TC_BIG_S=$S timeout 900 python bench.py --no-probe --no-cpu > gpurun_out/ab_bigS$S.json 2> gpurun_out/ab_bigS$S.err
done
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
for c in gdelt wiki; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$c.csv python bench.py --config $c --profile --steps 20 --warmup 3 > gpurun_out/ncu_launch_$c.log 2>&1
  for k in k_prep k_gru_tc k_build_x k_writeback; do
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 10 -c 1 -o gpurun_out/prof_${c}_$k python bench.py --config $c --profile --steps 20 --warmup 3 > gpurun_out/ncu_full_${c}_$k.log 2>&1
  done
done
ls gpurun_out
