"""Summarize an ncu launch list (--metrics gpu__time_duration.sum --csv) by
kernel: count, total and average time, share of the listed total."""
import collections
import csv
import sys

UNIT = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}


def summarize(path, steps=1, top=25):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr, rows = rows[0], rows[1:]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    total = 0.0
    for r in rows:
        v = float(r[vi].replace(",", "")) * UNIT[r[ui]]
        name = r[ki].split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "")
        name = name.replace("lr::", "")[:70]
        agg[name][0] += 1
        agg[name][1] += v
        total += v
    out = [f"{path}: {len(rows)} launches, {total:.1f} us total ({total / steps:.1f} us per step, "
           f"{steps} steps)"]
    out.append(f"{'kernel':70s} {'n':>5s} {'total us':>10s} {'avg us':>9s} {'share':>6s}")
    for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
        out.append(f"{k:70s} {c:5d} {t:10.1f} {t / c:9.2f} {100 * t / total:5.1f}%")
    return "\n".join(out)


if __name__ == "__main__":
    print(summarize(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 1))
