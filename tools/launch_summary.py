"""Per-kernel share of an ncu launch list (gpu__time_duration.sum, --csv).

    python tools/launch_summary.py gpurun_out/<tag>_launches.csv [top]

ncu serialises launches and runs them cold-cache, so absolute times are not
bench numbers; the SHARE of each kernel in the step is what this is for.
"""
import collections
import csv
import re
import sys


def main():
    path = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, mi = h.index("Kernel Name"), h.index("Metric Value")
    ui = h.index("Metric Unit") if "Metric Unit" in h else None
    scale = {"nsecond": 1.0, "usecond": 1e3, "msecond": 1e6, "second": 1e9}
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for r in rows[hi + 1:]:
        if len(r) <= mi:
            continue
        v = float(r[mi].replace(",", "")) * scale.get(r[ui] if ui is not None else "nsecond", 1.0)
        name = re.sub(r"\(.*", "", r[ki].replace("(anonymous namespace)::", ""))
        tot[name] += v
        cnt[name] += 1
    total = sum(tot.values())
    print(f"{path}: {sum(cnt.values())} launches, {total / 1e6:.2f} ms total (serialised, cold)")
    for k, v in sorted(tot.items(), key=lambda x: -x[1])[:top]:
        print(f"{v / 1e6:9.2f} ms {100 * v / total:5.1f}%  n={cnt[k]:6d}  avg={v / cnt[k] / 1e3:9.1f} us  {k[:100]}")


if __name__ == "__main__":
    main()
