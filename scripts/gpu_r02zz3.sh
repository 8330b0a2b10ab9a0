#!/bin/bash
# A/B: k_gru_tc at 167 registers (no min-blocks bound: a k_build_x block fits beside it) vs 213 (", 1")
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_zz3.log 2>&1
python -c "from paper_2402_15113_b200.build import build; print(build(force=True, extra_flags=['-DMSPIPE_GEMM_MINB1'], out='/tmp/libmspipe_minb1.so'))" >> gpurun_out/build_zz3.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -k "teacher_forced or bench_configuration or multi_step" > gpurun_out/zz3_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/zz3_pytest.log
tail -2 gpurun_out/zz3_pytest.log
for rep in 1 2; do
  timeout 900 python bench.py --no-probe --no-cpu --no-train --no-apan > gpurun_out/ab_gdelt_r167.$rep.json 2> /dev/null
  MSPIPE_LIB=/tmp/libmspipe_minb1.so timeout 900 python bench.py --no-probe --no-cpu --no-train --no-apan > gpurun_out/ab_gdelt_r213.$rep.json 2> /dev/null
  timeout 900 python bench.py --config wiki --no-probe --no-cpu --no-train --no-apan > gpurun_out/ab_wiki_r167.$rep.json 2> /dev/null
  MSPIPE_LIB=/tmp/libmspipe_minb1.so timeout 900 python bench.py --config wiki --no-probe --no-cpu --no-train --no-apan > gpurun_out/ab_wiki_r213.$rep.json 2> /dev/null
done
python - <<'PY'
import json, glob
for f in sorted(glob.glob("gpurun_out/ab_*_r*.json")):
    try:
        d = json.load(open(f))
    except Exception as e:
        print(f, "FAILED", e); continue
    r = d["roofline"]
    print(f, "%.2f Mev/s" % (d["value"] / 1e6), "%.2f us/step" % (d["ms_per_step"] * 1e3), "alone", {k: round(v * 1e3, 2) for k, v in r.get("dominant_of", {}).items()}, "in_step", {k: round(v * 1e3, 2) for k, v in r.get("in_step_ms", {}).items()})
PY
