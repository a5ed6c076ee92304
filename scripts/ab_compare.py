"""Compare interleaved A/B sweep files: min us/step per (case, n) for each side."""
import json
import sys
from collections import defaultdict


def load(p):
    d = defaultdict(list)
    for line in open(p):
        try:
            r = json.loads(line)
        except ValueError:
            continue
        d[(r["case"], r["n"])].append(r["us_per_step"])
    return d


a, b = load(sys.argv[1]), load(sys.argv[2])
for k in a:
    x, y = min(a[k]), min(b.get(k, [float("nan")]))
    print(f"{k[0]:14s} {k[1]:>8d}  {x:9.2f}  {y:9.2f}  {100 * (x / y - 1):+6.1f}%  "
          f"spread {[round(v, 1) for v in a[k]]} {[round(v, 1) for v in b.get(k, [])]}")
