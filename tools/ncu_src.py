"""Summarise an ncu --page source csv (cuda,sass): per-CUDA-line stall
samples and executed instructions (top N)."""
import csv
import sys
from collections import defaultdict

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
rows = list(csv.reader(open(path)))
hdr_i = next(i for i, r in enumerate(rows) if len(r) > 5 and r[0] == "Line No")
h = rows[hdr_i]
src_lines = {}
samp = defaultdict(float)
inst = defaultdict(float)
cur = None
for r in rows[hdr_i + 1:]:
    if len(r) < 8:
        continue
    if r[0] and r[0].isdigit():
        cur = int(r[0])
        src_lines[cur] = r[1]
    try:
        s = float(r[4] or 0)
        n = float(r[7] or 0)
    except ValueError:
        continue
    if cur is not None:
        samp[cur] += s
        inst[cur] += n
tot_s = sum(samp.values()) or 1
tot_i = sum(inst.values()) or 1
print("total samples %.0f  instructions %.3g" % (tot_s, tot_i))
for ln, s in sorted(samp.items(), key=lambda x: -x[1])[:top]:
    print("%5d  %5.1f%% samp  %5.1f%% inst  %s" % (ln, 100 * s / tot_s,
          100 * inst[ln] / tot_i, src_lines.get(ln, "")[:90]))
