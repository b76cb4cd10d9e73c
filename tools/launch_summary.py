"""Summarise an ncu --metrics gpu__time_duration.sum launch list: per-kernel share and
average duration over the kernels in the file (torch's own kernels excluded)."""
import collections
import csv
import sys


def main(path, skip_prefix=("at::", "void at::")):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = collections.defaultdict(list)
    for r in rows[hdr + 1:]:
        if len(r) > vi and not r[ki].startswith(skip_prefix):
            agg[r[ki].split("(")[0][:70]].append(float(r[vi].replace(",", "")))
    tot = sum(sum(v) for v in agg.values())
    print(f"{'share':>6} {'n':>4} {'avg us':>9}  kernel")
    for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
        print(f"{sum(v) / tot * 100:5.1f}% {len(v):4d} {sum(v) / len(v) / 1e3:9.1f}  {k}")
    print(f"total {tot / 1e6:.3f} ms over {sum(len(v) for v in agg.values())} launches")


if __name__ == "__main__":
    main(sys.argv[1])
