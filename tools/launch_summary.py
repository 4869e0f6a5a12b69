"""Summarise an ncu launch list (``--metrics gpu__time_duration.sum --csv --log-file``):
total device time per kernel name, divided by the number of iterations the command ran.
Usage: python tools/launch_summary.py launches.csv [iterations]"""
import collections
import csv
import io
import sys


def main(path, iters=1):
    lines = [ln for ln in open(path) if ln.startswith('"')]
    rows = list(csv.DictReader(io.StringIO("".join(lines))))
    per = collections.OrderedDict()
    for r in rows:
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"].split("(")[0][:80]
        per.setdefault(name, []).append(float(r["Metric Value"].replace(",", "")) / 1e3)
    total = sum(sum(v) for v in per.values()) / iters
    print(f"{'us/iter':>10} {'share':>6} {'n/iter':>7}  kernel")
    for k, v in sorted(per.items(), key=lambda kv: -sum(kv[1])):
        print(f"{sum(v) / iters:10.1f} {sum(v) / iters / total:6.1%} {len(v) / iters:7.1f}  {k}")
    print(f"{total:10.1f}  total us per iteration")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 1)
