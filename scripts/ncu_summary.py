"""Summarise an ncu report: key metrics + top stalled source lines."""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
        "launch__grid_size", "launch__block_size", "launch__registers_per_thread", "launch__cluster_dim_z",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__cycles_elapsed.avg", "smsp__cycles_active.avg", "launch__occupancy_limit_shared_mem",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__sass_inst_executed_op_local_ld.sum"]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    return r


def main(rep, nsrc=25):
    r = raw(rep)
    h = r[0]
    for row in r[2:]:
        d = dict(zip(h, row))
        print("kernel:", d.get("Kernel Name", "")[:80])
        for k in KEYS:
            for n in h:
                if n == k or (k.endswith("*") and n.startswith(k[:-1])):
                    print(f"  {n} = {d[n]}")
        tensor = [n for n in h if "tensor" in n and "pct" in n]
        for n in tensor[:6]:
            print(f"  {n} = {d[n]}")
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if not rows:
        return
    if rows[0] and rows[0][0] == "Kernel Name":
        rows = rows[1:]
    hh = rows[0]
    def col(name):
        for i, n in enumerate(hh):
            if n.startswith(name):
                return i
        return None
    ci = col("Warp Stall Sampling (All Samples)")
    si = col("Source")
    if ci is None:
        print("source columns:", hh[:12])
        return
    items = []
    for row in rows[1:]:
        try:
            items.append((float(row[ci] or 0), row[si]))
        except (ValueError, IndexError):
            pass
    tot = sum(v for v, _ in items) or 1
    items.sort(reverse=True)
    print(f"top stall-sampled SASS ({int(tot)} samples):")
    for v, s in items[:nsrc]:
        print(f"  {100 * v / tot:5.1f}%  {s[:110]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
