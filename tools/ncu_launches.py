"""Summarise an ncu --csv launch list (gpu__time_duration per launch) by kernel and by position."""
import collections
import csv
import io
import sys


def load(path):
    lines = [ln for ln in open(path) if not ln.startswith("==")]
    rows = list(csv.DictReader(io.StringIO("".join(lines))))
    data = collections.OrderedDict()
    for r in rows:
        d = data.setdefault(int(r["ID"]), {"name": r["Kernel Name"].split("(")[0]})
        d[r["Metric Name"]] = r["Metric Value"]
    return data


def main(path, show=0):
    data = load(path)
    tot, cnt = collections.defaultdict(float), collections.Counter()
    seq = []
    for i, d in data.items():
        t = float(d["gpu__time_duration.sum"].replace(",", "")) / 1e3  # us
        tot[d["name"]] += t
        cnt[d["name"]] += 1
        seq.append((d["name"], d.get("launch__grid_size"), d.get("launch__cluster_dim_x"), t))
    T = sum(tot.values())
    print(f"{'kernel':34s} {'launches':>8s} {'ms':>9s} {'share':>6s}")
    for n in sorted(tot, key=lambda k: -tot[k]):
        print(f"{n:34s} {cnt[n]:8d} {tot[n] / 1e3:9.3f} {100 * tot[n] / T:5.1f}%")
    print(f"{'total':34s} {len(seq):8d} {T / 1e3:9.3f}")
    for s in seq[:show]:
        print(s)


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 0)
