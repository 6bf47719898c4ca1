"""Record per-launch DRAM traffic of a kernel family from an ncu --set full
report into profiles/traffic.json (read by bench.py's roofline `traffic`).

    python tools/traffic_from_ncu.py <report.ncu-rep> <key> <kernel-substring> <source-label>

traffic per launch = mean over the family's captured launches of
dram__bytes_read.sum + dram__bytes_write.sum."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from ncu_summary import report  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    rep, key, sub, label = sys.argv[1:5]
    rows = [r for r in report(rep) if sub in r["kernel"]]
    if not rows:
        raise SystemExit(f"no launches matching {sub!r} in {rep}")
    tot = [1e6 * (r["dram_read_MB"] + r["dram_write_MB"]) for r in rows]
    path = os.path.join(ROOT, "profiles", "traffic.json")
    d = json.load(open(path)) if os.path.exists(path) else {}
    d = {k: v for k, v in d.items() if isinstance(v, dict)}
    d[key] = {"bytes_per_launch": sum(tot) / len(tot), "launches": len(rows),
              "per_launch": [{"kernel": r["kernel"][:60], "dram_bytes": t, "us": r.get("duration_us")}
                             for r, t in zip(rows, tot)],
              "source": f"{label}: mean of dram__bytes_read.sum + dram__bytes_write.sum over {len(rows)} "
                        f"launches ({os.path.basename(rep)}); ncu replays each launch with a cold L2 and "
                        f"counts only what reaches DRAM during the launch, so outputs still resident in the "
                        f"126 MB L2 when it ends show up as near-zero writes"}
    json.dump(d, open(path, "w"), indent=1)
    print(json.dumps(d[key], indent=1))


if __name__ == "__main__":
    main()
