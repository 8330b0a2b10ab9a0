#!/bin/bash
# GEMM tile of 20 hidden units (N = 80): parity, then the K-split choice at GDELT and wiki
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -s -k "teacher_forced or switch or multi_step or bench_configuration or subgraph or whole_stream or bf16" > gpurun_out/pytest_t.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_t.log
tail -3 gpurun_out/pytest_t.log
for s in 1 2; do
  MSPIPE_TC_BIG_S=$s timeout 900 python bench.py --no-probe --no-cpu > gpurun_out/ab_gdelt_s$s.json 2> gpurun_out/ab_gdelt_s$s.err
done
timeout 600 python bench.py --config wiki --no-probe --no-cpu > gpurun_out/ab_wiki_auto.json 2> gpurun_out/ab_wiki_auto.err
for s in 2 4 8; do
  MSPIPE_TC_SPLITS=$s timeout 600 python bench.py --config wiki --no-probe --no-cpu > gpurun_out/ab_wiki_s$s.json 2> gpurun_out/ab_wiki_s$s.err
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
