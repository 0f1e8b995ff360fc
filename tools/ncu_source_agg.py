"""Aggregate an `ncu --page source --csv --print-source sass` export over all profiled launches
of one kernel: stall samples and executed instructions per SASS line, hottest lines and
100-instruction windows (the export of many launches is too large to keep)."""
import csv
import sys

lines = open(sys.argv[1]).read().splitlines()
blocks, cur = [], None
for ln in lines:
    if ln.startswith('"Kernel Name"'):
        cur = []
        blocks.append(cur)
        continue
    if cur is not None:
        cur.append(ln)
agg = {}
for b in blocks:
    rdr = csv.reader(b)
    hdr = next(rdr)
    i_s, i_e, i_src = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed"), hdr.index("Source")
    for idx, r in enumerate(rdr):
        if len(r) < len(hdr):
            continue
        a = agg.setdefault(idx, [0, 0, r[i_src].strip()])
        a[0] += int(r[i_s] or 0)
        a[1] += int(r[i_e] or 0)
tot = sum(v[0] for v in agg.values()) or 1
te = sum(v[1] for v in agg.values())
print("launches", len(blocks), "stall samples", tot, "instructions", te)
keys = sorted(agg)
for k0 in range(0, len(keys), 100):
    sm = sum(agg[k][0] for k in keys[k0:k0 + 100])
    ex = sum(agg[k][1] for k in keys[k0:k0 + 100])
    if sm > 0.02 * tot:
        print(f"{k0:5d} samples {sm:6d} ({100 * sm / tot:4.1f}%) inst {ex:9d}  {agg[keys[k0]][2][:60]}")
for k in sorted(sorted(keys, key=lambda k: -agg[k][0])[:40]):
    print(f"{k:5d} {agg[k][0]:6d} {agg[k][1]:8d} {agg[k][2][:100]}")
