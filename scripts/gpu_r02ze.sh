#!/bin/bash
# Round-2 final evidence: smoke, the whole GPU suite (rows A-F), the default bench line (GDELT headline
# + HBM probe + oracle + F4 train + F3 APAN + GEMM-only timing), wiki, the reference arm,
# ncu --set full of the top hand-written F4 / F3 kernels at GDELT
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_ze.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ze_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/ze_smoke.log
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/ze_pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/ze_pytest_gpu.log
tail -3 gpurun_out/ze_pytest_gpu.log
timeout 1200 python bench.py > gpurun_out/ze_bench_gdelt.json 2> gpurun_out/ze_bench_gdelt.err
timeout 900 python bench.py --config wiki --no-probe > gpurun_out/ze_bench_wiki.json 2> gpurun_out/ze_bench_wiki.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/ze_bench_reference.json 2> gpurun_out/ze_bench_reference.err
for k in k_tr_gather k_tr_attn_bwd k_tr_seg_piece; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 -o gpurun_out/prof_gdelt_$k python scripts/exp_train_stage.py gdelt 16000 0 train > gpurun_out/ncu_full_gdelt_$k.log 2>&1
done
for k in k_apan_build k_apan_gather; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 -o gpurun_out/prof_gdelt_$k python scripts/exp_train_stage.py gdelt 16000 0 apan > gpurun_out/ncu_full_gdelt_$k.log 2>&1
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_apan_gdelt.csv python scripts/exp_train_stage.py gdelt 12000 0 apan > gpurun_out/ncu_apan_gdelt.log 2>&1
python - <<'PY'
import json
for f in ("gpurun_out/ze_bench_gdelt.json", "gpurun_out/ze_bench_wiki.json"):
    try:
        d = json.load(open(f))
    except Exception as e:
        print(f, "FAILED", e); continue
    print(f, "%.2f Mev/s" % (d["value"] / 1e6), "%.2f us/step" % (d["ms_per_step"] * 1e3), "e2e", d.get("e2e", {}).get("value"))
    print("  roofline", json.dumps({k: d["roofline"].get(k) for k in ("kernel", "achieved", "frac")}))
    print("  gemm", json.dumps({k: (d.get("roofline_gemm") or {}).get(k) for k in ("kernel", "achieved", "frac", "launch_ms_mean")}))
    print("  train", json.dumps(d.get("train"))[:300])
    print("  apan", json.dumps(d.get("apan"))[:200])
PY
ls gpurun_out | head -80
