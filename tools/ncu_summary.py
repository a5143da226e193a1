"""Summarise an ncu --csv launch list: per-kernel time/DRAM bytes (last N launches)."""
import csv
import io
import sys


def load(path):
    text = open(path).read()
    i = text.index('"ID"')
    rows = list(csv.DictReader(io.StringIO(text[i:])))
    agg = {}
    for r in rows:
        key = (int(r["ID"]), r["Kernel Name"].split("(")[0].replace("r2::<unnamed>::", "").replace("r2::", ""))
        agg.setdefault(key, {})[r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
    return agg


def main():
    agg = load(sys.argv[1])
    first = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    items = [(k, v) for k, v in sorted(agg.items()) if k[0] >= first]
    tot = sum(v.get("gpu__time_duration.sum", 0) for _, v in items)
    print(f"{'id':>4} {'kernel':34s} {'us':>9} {'share':>6} {'rd MB':>9} {'wr MB':>9}")
    for (i, k), v in items:
        t = v.get("gpu__time_duration.sum", 0)
        print(f"{i:4d} {k[:34]:34s} {t / 1e3:9.1f} {100 * t / tot:5.1f}% "
              f"{v.get('dram__bytes_read.sum', 0) / 1e6:9.1f} {v.get('dram__bytes_write.sum', 0) / 1e6:9.1f}")
    print(f"total {tot / 1e6:.3f} ms over {len(items)} launches")


if __name__ == "__main__":
    main()
