"""Markdown table of an ncu --page raw --csv export: per kernel launch, duration
(us), DRAM bytes (MB), DRAM / L2 throughput, tcgen05 int8 / fp16 tensor-op
throughput as % of peak, issue activity.  python tools/ncu_raw_summary.py raw.csv"""
import csv
import sys

COLS = [("dur_us", "gpu__time_duration.sum", 1),
        ("dram_rd_MB", "dram__bytes_read.sum", 1),
        ("dram_wr_MB", "dram__bytes_write.sum", 1),
        ("dram_%", "dram__throughput.avg.pct_of_peak_sustained_elapsed", 1),
        ("int8_tc_%", "sm__ops_path_tensor_op_utcimma_src_int8_sparsity_off.sum.pct_of_peak_sustained_elapsed", 1),
        ("f16_tc_%", "sm__ops_path_tensor_op_utchmma_src_fp16_dst_fp32_sparsity_off.sum.pct_of_peak_sustained_elapsed", 1),
        ("l2_%", "lts__t_sectors.avg.pct_of_peak_sustained_elapsed", 1),
        ("issue_%", "sm__inst_issued.avg.pct_of_peak_sustained_active", 1)]


def main(path):
    rows = list(csv.reader(open(path)))
    h, units = rows[0], rows[1]
    idx = {}
    for name, key, _ in COLS:
        cand = [i for i, x in enumerate(h) if x == key or x.endswith("." + key) or x.endswith(key)]
        idx[name] = cand[0] if cand else None
    ki = h.index("Kernel Name")
    print("| kernel | " + " | ".join(n for n, _, _ in COLS) + " |")
    print("|---|" + "---|" * len(COLS))
    for r in rows[2:]:
        if len(r) <= ki:
            continue
        name = r[ki].split("(")[0][:60]
        vals = []
        for n, _, sc in COLS:
            i = idx[n]
            try:
                v = float(r[i].replace(",", "")) * sc if i is not None else None
                if v is not None and n == "dur_us" and units[i] == "ms":
                    v *= 1e3
                if v is not None and n.endswith("_MB") and units[i] == "Gbyte":
                    v *= 1e3
                if v is not None and n.endswith("_MB") and units[i] == "Kbyte":
                    v *= 1e-3
            except ValueError:
                v = None
            vals.append("" if v is None else f"{v:.2f}")
        print(f"| `{name}` | " + " | ".join(vals) + " |")


if __name__ == "__main__":
    main(sys.argv[1])
