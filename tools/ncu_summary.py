"""Summarise ncu reports into the tracked profiles/ directory.

    python tools/ncu_summary.py <report.ncu-rep> [...] > profiles/<name>.md
    python tools/ncu_summary.py --launches launches.csv       (launch-list shares)
"""
import collections
import csv
import io
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "duration_us", 1.0),
    ("dram__bytes_read.sum", "dram_read_MB", 1.0),
    ("dram__bytes_write.sum", "dram_write_MB", 1.0),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_pct", 1.0),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_pct", 1.0),
    ("sm__pipe_tensor_subpipe_imma_cycles_active_realtime.avg", "imma_active_cycles", 1.0),
    ("sm__cycles_elapsed.avg", "sm_cycles", 1.0),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "l2_pct", 1.0),
    ("smsp__inst_executed.sum", "warp_instr", 1.0),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue_active_pct", 1.0),
    ("launch__registers_per_thread", "regs", 1.0),
    ("launch__grid_size", "grid", 1.0),
    ("launch__block_size", "block", 1.0),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps_active_pct", 1.0),
]


def report(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    to_mb = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}
    res = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")][:90]}
        for m, k, _ in METRICS:
            if m in hdr:
                i = hdr.index(m)
                try:
                    v = float(r[i].replace(",", ""))
                    if k.endswith("_MB"):
                        v *= to_mb.get(units[i], 1.0)
                    d[k] = v
                except ValueError:
                    d[k] = r[i]
        res.append(d)
    return res


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    hdr = rows[hi]
    ik, iv = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[hi + 1:]:
        if len(r) > iv and r[iv]:
            name = r[ik].split("(")[0][:70]
            agg[name][0] += 1
            agg[name][1] += float(r[iv].replace(",", ""))
    tot = sum(v for _, v in agg.values())
    print("| kernel | launches | total us | share | avg us |")
    print("|---|---|---|---|---|")
    for k, (n, v) in sorted(agg.items(), key=lambda x: -x[1][1])[:20]:
        print(f"| `{k}` | {n} | {v / 1e3:.1f} | {100 * v / tot:.1f}% | {v / n / 1e3:.2f} |")


if __name__ == "__main__":
    if sys.argv[1] == "--launches":
        launches(sys.argv[2])
    else:
        for p in sys.argv[1:]:
            for d in report(p):
                print("- " + ", ".join(f"{k}={v:.4g}" if isinstance(v, float) else f"{k}={v}" for k, v in d.items()))
