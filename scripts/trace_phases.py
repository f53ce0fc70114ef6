#!/usr/bin/env python3
"""Per-rank median phase times (ns) of the 256x256 cluster coding pass from a
DCSC_CL_TRACE build's printf lines (bench.py --config c3s stdout)."""
import collections
import re
import statistics
import sys

KEYS = ['start', 'dwait', 'gen1', 'ready_I', 'bf_I', 'recv_I', 'rif', 'rir', 'prox', 'ready_F', 'bi_F', 'recv_F',
        'cff', 'last']
lines = [ln for ln in open(sys.argv[1]) if ln.startswith('CLT')]
per = collections.defaultdict(lambda: collections.defaultdict(list))
tot = []
for ln in lines:
    d = dict(re.findall(r'(\w+)=(\d+)', ln))
    t = [int(d[k]) for k in KEYS]
    for a, b, k in zip(t, t[1:], KEYS[1:]):
        per[int(d['rank'])][k].append(b - a)
    tot.append(t[-1] - t[0])
print("phase    " + " ".join(f"rank{r:>5}" for r in range(4)))
for k in KEYS[1:]:
    print(f"{k:8s} " + " ".join(f"{statistics.median(per[r][k]):9.0f}" for r in range(4)))
print("start->last median", statistics.median(tot))
