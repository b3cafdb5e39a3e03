"""Per-kernel totals and shares of an ncu launch list
(--metrics gpu__time_duration.sum --csv), e.g. profiles/r01/launches_cfg3.csv.

  python tools/launch_summary.py gpurun_out/prof/launches.csv "python bench.py ..."
"""
import csv
import re
import sys
from collections import defaultdict


def main():
    path = sys.argv[1]
    cmd = sys.argv[2] if len(sys.argv) > 2 else ""
    rows = [r for r in csv.reader(open(path)) if r]
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    tot, cnt = defaultdict(float), defaultdict(int)
    for r in rows[hdr + 1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        name = re.sub(r"\(.*", "", r[ki]).replace("(anonymous namespace)::", "")
        v = float(r[vi].replace(",", ""))
        unit = r[h.index("Metric Unit")] if "Metric Unit" in h else "nsecond"
        us = v / 1e3 if unit.startswith("n") else (v if unit.startswith("u") else v * 1e3)
        tot[name] += us
        cnt[name] += 1
    all_us = sum(tot.values())
    print(f"# ncu launch list (gpu__time_duration.sum, --clock-control none) {cmd}")
    print("# cold-cache, serialised per-launch times: compare SHARES, not absolutes.")
    print(f"{'launches':>8} {'total_us':>10} {'share':>6}  kernel")
    for name in sorted(tot, key=lambda n: -tot[n]):
        print(f"{cnt[name]:>8} {tot[name]:>10.1f} {100 * tot[name] / all_us:>5.1f}%  {name}")


if __name__ == "__main__":
    main()
