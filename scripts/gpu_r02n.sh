#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
EXP_FULL=1 timeout 600 python scripts/exp_prep_phases.py gdelt > gpurun_out/prep_phases.txt 2>&1
timeout 600 python scripts/exp_prep_phases.py wiki >> gpurun_out/prep_phases.txt 2>&1
cat gpurun_out/prep_phases.txt
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -s -k "teacher_forced or degenerate or max_batch or switch or dedup" > gpurun_out/pytest_dedup.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_dedup.log
tail -3 gpurun_out/pytest_dedup.log
timeout 2400 python -m pytest tests -m gpu -q -s > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
timeout 1500 python bench.py --no-cpu > gpurun_out/bench_gdelt.json 2> gpurun_out/bench_gdelt.err
timeout 600 python bench.py --config wiki --no-probe --no-cpu > gpurun_out/bench_wiki.json 2> gpurun_out/bench_wiki.err
python scripts/summarize_bench.py gpurun_out/bench_gdelt.json gpurun_out/bench_wiki.json
python - <<'PY'
import json
for f in ["gpurun_out/bench_gdelt.json", "gpurun_out/bench_wiki.json"]:
    try:
        d = json.load(open(f))
    except Exception as e:
        print(f, "FAILED", e); continue
    r = d["roofline"]
    print(f, "alone", {k: round(v * 1e3, 2) for k, v in r.get("dominant_of", {}).items()}, "in_step", {k: round(v * 1e3, 2) for k, v in r.get("in_step_ms", {}).items()})
PY
