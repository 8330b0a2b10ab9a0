#!/bin/bash
# GEMM epilogue: local K-split partials + MUFU gate math, phase marks per variant, parity, bench
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
for v in "" "-DMSPIPE_FAST_GATES=0"; do
  for cfg in gdelt wiki; do
    echo "== $cfg [$v] in-step"; EXP_FLAGS="$v" timeout 600 python scripts/exp_gru_phases.py $cfg 2>&1 | tail -13 | grep -v "^entry\|^acc_full\|^sync\|dead"
  done
done > gpurun_out/phases_w.txt
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -s -k "teacher_forced or switch or multi_step or bench_configuration or whole_stream or bf16 or rnn or deferred" > gpurun_out/pytest_w.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_w.log
grep -E "max err /|rel drift|passed|failed|rc=" gpurun_out/pytest_w.log | tail -40
timeout 900 python bench.py --no-cpu --no-probe > gpurun_out/ab_gdelt.json 2> gpurun_out/ab_gdelt.err
timeout 600 python bench.py --config wiki --no-probe --no-cpu > gpurun_out/ab_wiki.json 2> gpurun_out/ab_wiki.err
cat gpurun_out/phases_w.txt
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
