"""Summarise gpurun_out/ ncu artefacts into tracked files under profiles/.

  python scripts/make_profiles.py <round-tag> [config]

Writes profiles/<tag>_ncu_summary.md (key metrics of each --set full capture,
with units, plus the top stall-sampled SASS lines), profiles/<tag>_launches.csv
(the --metrics gpu__time_duration.sum launch list) and merges the per-op DRAM
traffic per launch into profiles/ncu_traffic.json (read by bench.py for
roofline.traffic).
"""
import collections
import csv
import io
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
        "launch__grid_size", "launch__block_size", "launch__registers_per_thread", "launch__cluster_dim_x",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_sector_hit_rate.pct", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum"]
# op (bench.py roofline key) -> kernels whose DRAM traffic makes up one launch of it
OPS = {"sample": ["k_sample_recent"], "dedup": ["k_dedup"], "fetch": ["k_fetch_gather"],
       "update": ["k_build_x", "k_gru_tc"], "writeback": ["k_writeback"]}
# fused step (StageConfig.use_fused): prep = k_prep, build = k_build_x, update = k_gru_tc with the commit
OPS_FUSED = {"prep": ["k_prep"], "build": ["k_build_x"], "update": ["k_gru_tc"]}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "B": 1, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def raw(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(txt)))
    return r[0], r[1], r[2:]


def top_sass(rep, n=12):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    if rows and rows[0] and rows[0][0] == "Kernel Name":
        rows = rows[1:]
    if not rows:
        return []
    h = rows[0]
    ci = next((i for i, x in enumerate(h) if x.startswith("Warp Stall Sampling (All")), None)
    si = next((i for i, x in enumerate(h) if x == "Source"), None)
    if ci is None or si is None:
        return []
    items = []
    for row in rows[1:]:
        try:
            items.append((float(row[ci] or 0), row[si].strip()))
        except (ValueError, IndexError):
            pass
    tot = sum(v for v, _ in items) or 1.0
    items.sort(reverse=True)
    return [(100 * v / tot, s) for v, s in items[:n]]


def main(tag, config="wiki"):
    os.makedirs(PROF, exist_ok=True)
    lines = [f"# ncu summary {tag} (config {config})", "",
             "Captured with `ncu --set full --clock-control none --import-source on` inside "
             "`python bench.py --profile --steps 20 --warmup 3` on one B200 (ncu flushes caches between "
             "replays: cold-cache, serialised).", ""]
    traffic = {}
    for f in sorted(os.listdir(OUT)):
        if not (f.startswith("prof_") and f.endswith(".ncu-rep")):
            continue
        h, units, rows = raw(os.path.join(OUT, f))
        for row in rows:
            d = dict(zip(h, row))
            u = dict(zip(h, units))
            name = d.get("Kernel Name", "?")
            lines.append(f"## {name[:100]}")
            lines.append("")
            lines.append("| metric | value | unit |")
            lines.append("|---|---|---|")
            for k in KEYS:
                if k in d:
                    lines.append(f"| {k} | {d[k]} | {u.get(k, '')} |")
            dram = 0.0
            for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                if k in d:
                    dram += float(d[k].replace(",", "")) * SCALE.get(u.get(k, "byte"), 1)
            short = name.split("(")[0].split("::")[-1].split("<")[0].replace("void ", "").strip()
            traffic[short] = traffic.get(short, 0.0) + dram
            lines.append("")
            sass = top_sass(os.path.join(OUT, f))
            if sass:
                lines.append("top stall-sampled SASS:")
                lines.append("")
                lines.append("```")
                for p, s in sass:
                    lines.append(f"{p:5.1f}%  {s[:110]}")
                lines.append("```")
                lines.append("")
    with open(os.path.join(PROF, f"{tag}_ncu_summary.md"), "w") as fh:
        fh.write("\n".join(lines) + "\n")
    # launch list
    lc = os.path.join(OUT, "launches.csv")
    if os.path.exists(lc):
        shutil.copy(lc, os.path.join(PROF, f"{tag}_launches.csv"))
        rows = list(csv.reader(open(lc)))
        hdr, data = None, collections.defaultdict(list)
        for r in rows:
            if r and r[0] == "ID":
                hdr = r
                continue
            if hdr and len(r) == len(hdr):
                d = dict(zip(hdr, r))
                if d.get("Metric Name") == "gpu__time_duration.sum":
                    data[d["Kernel Name"].split("(")[0]].append(float(d["Metric Value"]))
        tot = sum(sum(v) for k, v in data.items() if "mspipe" in k and "pack" not in k)
        with open(os.path.join(PROF, f"{tag}_launches_summary.md"), "w") as fh:
            fh.write(f"# ncu launch list {tag}: per-kernel device time (cold-cache, serialised)\n\n")
            fh.write("| kernel | launches | mean us | share of the library's per-step kernel time |\n|---|---|---|---|\n")
            for k, v in sorted(data.items(), key=lambda kv: -sum(kv[1])):
                share = sum(v) / tot if "mspipe" in k and "pack" not in k else float("nan")
                fh.write(f"| {k} | {len(v)} | {sum(v) / len(v) / 1000:.2f} | {share:.3f} |\n")
    tpath = os.path.join(PROF, "ncu_traffic.json")
    allt = json.load(open(tpath)) if os.path.exists(tpath) else {}
    ops = OPS_FUSED if "k_prep" in traffic else OPS
    allt[config] = {op: sum(traffic.get(k, 0.0) for k in ks) for op, ks in ops.items()
                    if all(k in traffic for k in ks)}
    allt[config]["_source"] = f"{tag}_ncu_summary.md (dram__bytes_read.sum + dram__bytes_write.sum per launch)"
    with open(tpath, "w") as fh:
        json.dump(allt, fh, indent=1)
    print(open(os.path.join(PROF, f"{tag}_launches_summary.md")).read() if os.path.exists(lc) else "")
    print(json.dumps(allt[config], indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "wiki")
