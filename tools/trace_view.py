"""Summarise an SF_TRACE_FILE timeline: per-pulse intervals of each kind."""
import collections
import sys

NAMES = {0: "gemv", 1: "gram", 2: "loop", 3: "oper", 4: "lips", 5: "fista"}
rows = [l.split() for l in open(sys.argv[1]) if l.strip()]
ev = collections.defaultdict(list)
for k, i, a, b in rows:
    ev[int(k)].append((float(a), float(b)))
for k in sorted(ev):
    v = ev[k]
    print(NAMES[k], len(v), "mean dur %.1f us" % (1e3 * sum(b - a for a, b in v) / len(v)))
# timeline of the last few pulses
n = int(sys.argv[2]) if len(sys.argv) > 2 else 4
fi = ev[5][-n:]
t0 = fi[0][0] - 0.5
print("t(us) relative; fista calls:", [(round(1e3 * (a - t0)), round(1e3 * (b - t0))) for a, b in fi])
for k in (3, 1):
    sel = [(a, b) for a, b in ev[k] if b >= t0]
    print(NAMES[k], [(round(1e3 * (a - t0)), round(1e3 * (b - t0))) for a, b in sel])
