"""Summarise an ncu launch list (gpu__time_duration per launch) and a
--set full capture into profiles/ text: per-kernel share of device time,
DRAM traffic and throughput, FP64 / tensor pipe utilisation, occupancy."""
import collections
import csv
import subprocess
import sys


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    hdr = rows[hi]
    ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    agg = collections.defaultdict(lambda: collections.defaultdict(list))
    for r in rows[hi + 1:]:
        name = r[ki].split("(")[0].replace("void ", "").replace("hzg::<unnamed>::", "")
        agg[name][r[mi]].append(float(r[vi].replace(",", "")))
    T = "gpu__time_duration.sum"
    tot = sum(sum(d[T]) for d in agg.values())
    out = ["launch list: %s (--clock-control none; serialised, cold-cache)" % path,
           "%-36s %6s %12s %8s %12s %10s" % ("kernel", "n", "avg us", "share", "DRAM MB/l", "TB/s")]
    for k, d in sorted(agg.items(), key=lambda x: -sum(x[1][T])):
        t = d[T]
        b = [x + y for x, y in zip(d.get("dram__bytes_read.sum", []), d.get("dram__bytes_write.sum", []))]
        mb = sum(b) / len(b) / 1e6 if b else float("nan")
        out.append("%-36s %6d %12.2f %8.3f %12.1f %10.2f" % (k[:36], len(t), sum(t) / len(t) / 1e3, sum(t) / tot, mb,
                                                         (sum(b) / sum(t) / 1e3) if b else float("nan")))
    return out


WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "launch__grid_size", "launch__block_size",
        "smsp__inst_executed.sum"]


def full(path):
    txt = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    hdr, units = rows[0], rows[1]
    out = ["full capture: %s" % path]
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")].split("(")[0].replace("void ", "").replace("hzg::<unnamed>::", "")
        out.append(name)
        for w in WANT:
            if w in hdr:
                i = hdr.index(w)
                out.append("    %-66s %14s %s" % (w, r[i], units[i]))
    return out


if __name__ == "__main__":
    lines = []
    for p in sys.argv[1:]:
        lines += launches(p) if p.endswith(".csv") else full(p)
        lines.append("")
    print("\n".join(lines))
