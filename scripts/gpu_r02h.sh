#!/bin/bash
# 8-warp GEMM epilogue: GEMM-heavy tests, K-split A/B at GDELT, phase marks, wiki bench
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shard.py -q -x -s -k "teacher_forced or multi_step or bench_configuration or switch or max_batch or degenerate or bf16 or sharded" > gpurun_out/pytest_gemm.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gemm.log
tail -3 gpurun_out/pytest_gemm.log
for S in 1 2 4; do
  MSPIPE_TC_SPLITS=$S timeout 900 python bench.py --tcsr-events 4000000 --no-probe --no-cpu > gpurun_out/ab_splits_$S.json 2> gpurun_out/ab_splits_$S.err
done
timeout 600 python bench.py --config wiki --no-probe --no-cpu > gpurun_out/bench_wiki.json 2> gpurun_out/bench_wiki.err
python - <<'PY'
import json, glob
for f in sorted(glob.glob("gpurun_out/ab_*.json")) + ["gpurun_out/bench_wiki.json"]:
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
