"""Compare interleaved A/B sweep outputs: python scripts/ab_compare.py new.jsonl old.jsonl"""
import json
import sys
from collections import defaultdict


def load(path):
    d = defaultdict(list)
    for line in open(path):
        try:
            r = json.loads(line)
        except ValueError:
            continue
        if "us_per_step" in r:
            d[(r["case"], r["n"])].append(r["us_per_step"])
    return d


a, b = load(sys.argv[1]), load(sys.argv[2])
for k in a:
    if k in b:
        x, y = min(a[k]), min(b[k])
        print(f"{k[0]:14s} {k[1]:>9d}  new {x:9.2f}  old {y:9.2f}  {100 * (x / y - 1):+6.1f}%")
