#!/bin/bash
# Row F4 on the GPU: its parity tests, then the GDELT and wiki benches with the training measurement
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_za.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_train.py -q -x -s > gpurun_out/pytest_train.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_train.log
tail -30 gpurun_out/pytest_train.log
timeout 900 python -m pytest tests/test_gpu_apan.py -q -x -s > gpurun_out/pytest_apan.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_apan.log
tail -15 gpurun_out/pytest_apan.log
timeout 900 python bench.py --no-probe --no-cpu > gpurun_out/za_bench_gdelt.json 2> gpurun_out/za_bench_gdelt.err
timeout 600 python bench.py --config wiki --no-probe --no-cpu > gpurun_out/za_bench_wiki.json 2> gpurun_out/za_bench_wiki.err
python - <<'PY'
import json
for f in ("gpurun_out/za_bench_gdelt.json", "gpurun_out/za_bench_wiki.json"):
    try:
        d = json.load(open(f))
    except Exception as e:
        print(f, "FAILED", e); continue
    print(f, "%.2f Mev/s" % (d["value"] / 1e6), "%.2f us/step" % (d["ms_per_step"] * 1e3), "train:", json.dumps(d.get("train"))[:600])
PY
# GEMM phases: CTA entry spread vs the kernel duration (serialised step: EXP_COLD runs the commit alone)
for c in gdelt wiki; do
  EXP_COLD=1 timeout 600 python scripts/exp_gru_phases.py $c > gpurun_out/za_phases_$c.txt 2>&1
done
tail -20 gpurun_out/za_phases_gdelt.txt gpurun_out/za_phases_wiki.txt
