#!/bin/bash
# Device bench on every config of BASELINE.json (no CPU baseline): gpurun_out/sweep_<cfg>.json
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
for c in tiny wiki reddit lastfm mooc; do
  timeout 600 python bench.py --config $c --no-cpu --steps 200 > gpurun_out/sweep_$c.json 2> gpurun_out/sweep_$c.err
done
timeout 900 python bench.py --config gdelt --events 4000000 --no-cpu --steps 200 > gpurun_out/sweep_gdelt.json 2> gpurun_out/sweep_gdelt.err
python - <<'PY'
import json
for c in ["tiny", "wiki", "reddit", "lastfm", "mooc", "gdelt"]:
    try:
        d = json.load(open(f"gpurun_out/sweep_{c}.json"))
    except Exception as e:
        print(c, "FAILED", e); continue
    r, g = d["roofline"], d.get("roofline_gather") or {}
    print(f"{c:7s} {d['value']/1e6:7.2f} Mev/s  {d['ms_per_step']*1e3:7.2f} us/step  e2e {d['e2e']['value']/1e6:6.2f} Mev/s"
          f"  dom {r['kernel'][:20]} frac {r['frac']:.3f}  gather {g.get('achieved', 0):7.0f} GB/s ({g.get('frac', 0):.2f})")
PY
