"""Per-CUDA-line stall samples and executed warp instructions from
`ncu -i REP -k KERNEL --page source --csv --print-source cuda,sass`."""
import csv
import sys
from collections import defaultdict

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
rows = list(csv.reader(open(path)))
hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
h = rows[hdr_i]
i_samp = h.index("Warp Stall Sampling (All Samples)")
i_inst = h.index("Instructions Executed")
samp, inst, src = defaultdict(float), defaultdict(float), {}
cur = None
for r in rows[hdr_i + 1:]:
    if len(r) <= i_inst:
        continue
    if r[0] and r[0].isdigit() and r[2] == "-":      # CUDA line summary row
        cur = int(r[0])
        src[cur] = r[1]
        try:
            samp[cur] += float(r[i_samp] or 0)
            inst[cur] += float(r[i_inst] or 0)
        except ValueError:
            pass
ts, ti = sum(samp.values()) or 1, sum(inst.values()) or 1
print("total samples %.0f, warp instructions %.3e" % (ts, ti))
for ln in sorted(samp, key=lambda k: -samp[k])[:top]:
    print("%5d %5.1f%% samp %5.1f%% inst  %s" % (ln, 100 * samp[ln] / ts,
                                               100 * inst[ln] / ti, src[ln][:90]))
