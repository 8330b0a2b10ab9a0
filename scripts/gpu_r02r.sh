#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -s -k "teacher_forced or switch or multi_step or bench_configuration or subgraph or whole_stream" > gpurun_out/pytest_pb.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_pb.log
tail -3 gpurun_out/pytest_pb.log
for pb in 1 0; do
  MSPIPE_PREP_BUILD=$pb timeout 900 python bench.py --no-probe --no-cpu > gpurun_out/ab_gdelt_pb$pb.json 2> gpurun_out/ab_gdelt_pb$pb.err
  MSPIPE_PREP_BUILD=$pb timeout 600 python bench.py --config wiki --no-probe --no-cpu > gpurun_out/ab_wiki_pb$pb.json 2> gpurun_out/ab_wiki_pb$pb.err
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
