#!/bin/bash
# A/B: k_build_x items of 2 vs 4 K chunks, and its blocks-per-SM cap (4 / 8 / 16)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_zs.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "switch" > gpurun_out/zs_pytest_switch.log 2>&1; echo "rc=$?" >> gpurun_out/zs_pytest_switch.log
tail -2 gpurun_out/zs_pytest_switch.log
run() {  # tag, env...
  local tag=$1; shift
  env "$@" timeout 900 python bench.py --no-probe --no-cpu --no-train --no-apan > gpurun_out/ab_gdelt_$tag.json 2> gpurun_out/ab_gdelt_$tag.err
  env "$@" timeout 900 python bench.py --config wiki --no-probe --no-cpu --no-train --no-apan > gpurun_out/ab_wiki_$tag.json 2> gpurun_out/ab_wiki_$tag.err
}
run base MSPIPE_BUILD_CHUNKS=4
run c2 MSPIPE_BUILD_CHUNKS=2
run bps4 MSPIPE_BUILD_BPS=4
run bps16 MSPIPE_BUILD_BPS=16
run base2 MSPIPE_BUILD_CHUNKS=4
run c2b MSPIPE_BUILD_CHUNKS=2
python - <<'PY'
import json, glob
for f in sorted(glob.glob("gpurun_out/ab_*_base*.json") + glob.glob("gpurun_out/ab_*_c2*.json") + glob.glob("gpurun_out/ab_*_bps*.json")):
    try:
        d = json.load(open(f))
    except Exception as e:
        print(f, "FAILED", e); continue
    r = d["roofline"]
    print(f, "%.2f Mev/s" % (d["value"] / 1e6), "%.2f us/step" % (d["ms_per_step"] * 1e3), "alone", {k: round(v * 1e3, 2) for k, v in r.get("dominant_of", {}).items()})
PY
