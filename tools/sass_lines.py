"""Aggregate ncu SASS stall samples per CUDA source line.

usage: sass_lines.py <ncu source csv> <nvdisasm --print-line-info dump> <mangled fn> [N]
"""
import collections
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
iss, iex = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
body = [r for r in rows[2:] if len(r) > iex and r[iss].isdigit()]
fn = sys.argv[3]
lines = open(sys.argv[2]).read().split("\n")
start = next(i for i, l in enumerate(lines) if l.startswith(".text." + fn + ":"))
cur = None
off2line = {}
for l in lines[start + 1:]:
    if l.startswith(".text.") or l.startswith("//----"):
        break
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        cur = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/", l)
    if m:
        off2line[int(m.group(1), 16)] = cur
agg = collections.Counter()
ex = collections.Counter()
for i, r in enumerate(body):
    key = off2line.get(i * 16, ("?", 0))
    agg[key] += int(r[iss])
    ex[key] += int(r[iex] or 0)
tot = sum(agg.values())
n = int(sys.argv[4]) if len(sys.argv) > 4 else 30
for k, v in agg.most_common(n):
    print(f"{k[0]}:{k[1]:<5d} {v:7d} {100 * v / tot:5.1f}%  exec {ex[k]}")
