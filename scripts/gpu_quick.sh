#!/bin/bash
# Quick GPU iteration: parity tests, a short bench, and the ncu launch list.
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -40 > gpurun_out/pytest_quick.log; cat gpurun_out/pytest_quick.log
timeout 600 python bench.py --no-cpu --steps 100 ${BENCH_EXTRA} > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err
python - <<'PY'
import json
d = json.load(open("gpurun_out/bench_quick.json"))
print("value", round(d["value"]), "ms/step", round(d["ms_per_step"], 4), "e2e", round(d["e2e"]["value"]))
print("op ms", {k: round(v, 4) for k, v in d["roofline"]["op_ms_mean"].items()})
PY
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --profile --steps 20 --warmup 3 ${BENCH_EXTRA} > /dev/null 2>&1
python - <<'PY'
import csv, collections
rows = list(csv.reader(open("gpurun_out/launches.csv")))
hdr = None
data = collections.defaultdict(list)
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d.get("Metric Name") == "gpu__time_duration.sum":
            data[d["Kernel Name"][:34]].append(float(d["Metric Value"]))
for k, v in data.items():
    print(f"{k:36s} n={len(v):4d} mean={sum(v)/len(v)/1000:7.2f}us")
PY
