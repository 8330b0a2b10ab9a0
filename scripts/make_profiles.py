"""Summarise gpurun_out/ ncu artefacts into tracked files under profiles/.

  python scripts/make_profiles.py <round-tag>

Writes profiles/<tag>_ncu_summary.md (key metrics of each --set full capture,
with units, plus the top stall-sampled SASS lines), profiles/<tag>_launches*.csv
(the --metrics gpu__time_duration.sum launch lists) and, per config and per
kernel, ONE capture's DRAM bytes / L2 hit rate / duration per launch into
profiles/ncu_traffic.json (read by bench.py for roofline.traffic).
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
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "B": 1, "KB": 1e3, "MB": 1e6, "GB": 1e9,
         "nsecond": 1, "usecond": 1e3, "msecond": 1e6, "second": 1e9, "ns": 1, "us": 1e3, "ms": 1e6}


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


def _num(d, u, k):
    if k not in d or d[k] in ("", "n/a"):
        return None
    return float(d[k].replace(",", "")) * SCALE.get(u.get(k, ""), 1)


def main(tag):
    """Captures are gpurun_out/prof_<config>_<kernel>.ncu-rep, each ONE launch
    (`-k regex:<kernel> -s <skip> -c 1`).  ncu_traffic.json gets, per config and
    per kernel, that launch's DRAM bytes, L2 hit rate and duration — never a sum
    over captures or configs."""
    os.makedirs(PROF, exist_ok=True)
    lines = [f"# ncu summary {tag}", "",
             "Each section is ONE launch captured with `ncu --set full --clock-control none --import-source on "
             "-k regex:<kernel> -s <skip> -c 1` inside `python bench.py --profile --config <config>` on one B200 "
             "(ncu flushes caches between its replays: cold-cache, serialised).", ""]
    tpath = os.path.join(PROF, "ncu_traffic.json")
    allt = json.load(open(tpath)) if os.path.exists(tpath) else {}
    for f in sorted(os.listdir(OUT)):
        if not (f.startswith("prof_") and f.endswith(".ncu-rep")):
            continue
        parts = f[len("prof_"):-len(".ncu-rep")].split("_", 1)
        if len(parts) != 2:
            continue
        config, kern = parts
        h, units, rows = raw(os.path.join(OUT, f))
        seen = set()
        for li, row in enumerate(rows):  # a "multi" capture holds one launch of each of several kernels
            d, u = dict(zip(h, row)), dict(zip(h, units))
            name = d.get("Kernel Name", "?")
            short = name.split("(")[0].split("::")[-1].split("<")[0].replace("void ", "").strip()
            if short in seen:
                continue
            seen.add(short)
            lines += [f"## {config}: {name[:100]}", "", f"capture `{f}`, launch {li + 1} of {len(rows)}", "",
                      "| metric | value | unit |", "|---|---|---|"]
            lines += [f"| {k} | {d[k]} | {u.get(k, '')} |" for k in KEYS if k in d]
            dram = (_num(d, u, "dram__bytes_read.sum") or 0.0) + (_num(d, u, "dram__bytes_write.sum") or 0.0)
            rec = {"dram_bytes": dram, "dram_read_bytes": _num(d, u, "dram__bytes_read.sum"),
                   "dram_write_bytes": _num(d, u, "dram__bytes_write.sum"),
                   "l2_hit_pct": _num(d, u, "lts__t_sector_hit_rate.pct"),
                   "l2_bytes": _num(d, u, "lts__t_bytes.sum"),
                   "duration_ns": _num(d, u, "gpu__time_duration.sum"),
                   "dram_throughput_pct": _num(d, u, "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
                   "tensor_active_pct": _num(d, u,
                                             "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"),
                   "warps_active_pct": _num(d, u, "sm__warps_active.avg.pct_of_peak_sustained_active"),
                   "source": f"profiles/{tag}_ncu_summary.md ({f}, launch {li + 1}: one launch)"}
            allt.setdefault(config, {})[short] = rec
            lines.append("")
        sass = top_sass(os.path.join(OUT, f)) if len(rows) == 1 else []
        if sass:
            lines += ["top stall-sampled SASS:", "", "```"]
            lines += [f"{p_:5.1f}%  {s_[:110]}" for p_, s_ in sass]
            lines += ["```", ""]
    with open(os.path.join(PROF, f"{tag}_ncu_summary.md"), "w") as fh:
        fh.write("\n".join(lines) + "\n")
    # launch lists: gpurun_out/launches*.csv
    for f in sorted(os.listdir(OUT)):
        if not (f.startswith("launches") and f.endswith(".csv")):
            continue
        suffix = f[len("launches"):-len(".csv")]
        lc = os.path.join(OUT, f)
        shutil.copy(lc, os.path.join(PROF, f"{tag}_launches{suffix}.csv"))
        rows = list(csv.reader(open(lc)))
        hdr, data = None, collections.defaultdict(list)
        for r in rows:
            if r and r[0] == "ID":
                hdr = r
                continue
            if hdr and len(r) == len(hdr):
                d = dict(zip(hdr, r))
                if d.get("Metric Name") == "gpu__time_duration.sum":
                    data[d["Kernel Name"].split("(")[0]].append(float(d["Metric Value"].replace(",", "")))
        mine = {k: v for k, v in data.items() if "mspipe" in k and "pack" not in k}
        tot = sum(sum(v) for v in mine.values()) or 1.0
        out = os.path.join(PROF, f"{tag}_launches{suffix}_summary.md")
        with open(out, "w") as fh:
            fh.write(f"# ncu launch list {tag}{suffix}: per-kernel device time (cold-cache, serialised)\n\n")
            fh.write("| kernel | launches | mean us | share of the library's kernel time |\n|---|---|---|---|\n")
            for k, v in sorted(data.items(), key=lambda kv: -sum(kv[1])):
                share = sum(v) / tot if k in mine else float("nan")
                fh.write(f"| {k} | {len(v)} | {sum(v) / len(v) / 1000:.2f} | {share:.3f} |\n")
        print(open(out).read())
    with open(tpath, "w") as fh:
        json.dump(allt, fh, indent=1)
    print(json.dumps(allt, indent=1))


if __name__ == "__main__":
    main(sys.argv[1])
