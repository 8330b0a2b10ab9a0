cd $GRAFT_REPO_ROOT
for pb in 1 0; do
MSPIPE_PREP_BUILD=$pb timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch_pb$pb.csv python bench.py --profile --steps 20 --warmup 3 > /dev/null 2>&1
python - <<PY
import csv, collections
rows = list(csv.reader(open("gpurun_out/launch_pb$pb.csv")))
hdr=None; data=collections.defaultdict(list)
for r in rows:
    if r and r[0]=="ID": hdr=r; continue
    if hdr and len(r)==len(hdr):
        d=dict(zip(hdr,r))
        if d.get("Metric Name")=="gpu__time_duration.sum": data[d["Kernel Name"][:30]].append(float(d["Metric Value"]))
print("prep_build=$pb")
for k,v in data.items(): print(f"  {k:32s} n={len(v):4d} mean={sum(v)/len(v)/1000:7.2f}us")
PY
done
