#!/bin/bash
# A/B: k_gru_tc at 128 registers (min-blocks 2, small spills) alone and with the global-table dedup
# (k_prep without dynamic shared memory, so a k_prep block can share the SM with a GEMM CTA)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_zz5.log 2>&1
python -c "from paper_2402_15113_b200.build import build; print(build(force=True, extra_flags=['-DMSPIPE_GEMM_MINB=2'], out='/tmp/libmspipe_r128.so'))" >> gpurun_out/build_zz5.log 2>&1
MSPIPE_LIB=/tmp/libmspipe_r128.so timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -k "teacher_forced or bench_configuration" > gpurun_out/zz5_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/zz5_pytest.log
tail -2 gpurun_out/zz5_pytest.log
for rep in 1 2; do
  timeout 900 python bench.py --no-probe --no-cpu --no-train --no-apan > gpurun_out/ab_gdelt_base.$rep.json 2> /dev/null
  MSPIPE_LIB=/tmp/libmspipe_r128.so timeout 900 python bench.py --no-probe --no-cpu --no-train --no-apan > gpurun_out/ab_gdelt_r128.$rep.json 2> /dev/null
  MSPIPE_LIB=/tmp/libmspipe_r128.so MSPIPE_PREP_SMEM=0 timeout 900 python bench.py --no-probe --no-cpu --no-train --no-apan > gpurun_out/ab_gdelt_r128g.$rep.json 2> /dev/null
  MSPIPE_PREP_SMEM=0 timeout 900 python bench.py --no-probe --no-cpu --no-train --no-apan > gpurun_out/ab_gdelt_baseg.$rep.json 2> /dev/null
done
python - <<'PY'
import json, glob
for f in sorted(glob.glob("gpurun_out/ab_gdelt_base*.json") + glob.glob("gpurun_out/ab_gdelt_r128*.json")):
    try:
        d = json.load(open(f))
    except Exception as e:
        print(f, "FAILED", e); continue
    r = d["roofline"]
    print(f, "%.2f Mev/s" % (d["value"] / 1e6), "%.2f us/step" % (d["ms_per_step"] * 1e3), "alone", {k: round(v * 1e3, 2) for k, v in r.get("dominant_of", {}).items()}, "in_step", {k: round(v * 1e3, 2) for k, v in r.get("in_step_ms", {}).items()})
PY
