"""Aggregate the per-launch `items tprof [tag] ...` lines (PT_INNER_TPROF=1) on stdin by stage tag."""
import re
import sys
from collections import defaultdict

agg = defaultdict(lambda: defaultdict(int))
cnt = defaultdict(int)
for line in sys.stdin:
    m = re.match(r"items tprof \[(\w+)\] \(cycles, CTA 0\): (.*)", line)
    if not m:
        continue
    tag, rest = m.groups()
    cnt[tag] += 1
    for k, v in re.findall(r"([a-z\-]+) (\d+)", rest):
        agg[tag][k] += int(v)
for tag in agg:
    n = cnt[tag]
    print(f"{tag:8s} launches {n:5d} | " + " ".join(f"{k} {v / n / 1965:.1f}us" if k not in ("phases", "tiles", "chunkn")
                                                  else f"{k} {v / n:.1f}" for k, v in agg[tag].items()))
