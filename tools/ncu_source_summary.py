"""Summarise `ncu --page source --csv --print-source sass` output: warp-stall
samples by SASS opcode and by stall reason (first kernel in the file)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
data, seen = [], set()
for r in rows[2:]:
    if r and r[0] == "Address":
        break  # next kernel section
    if len(r) == len(hdr) and r[0].startswith("0x") and r[0] not in seen:
        seen.add(r[0])
        data.append(r)
i_s = hdr.index("Warp Stall Sampling (All Samples)")
i_src = hdr.index("Source")
i_ex = hdr.index("Instructions Executed")
agg, cnt = collections.Counter(), collections.Counter()
for r in data:
    op = [o for o in r[i_src].strip().split() if not o.startswith("@")]
    op = op[0] if op else "?"
    agg[op] += int(r[i_s] or 0)
    cnt[op] += int(r[i_ex] or 0)
tot = sum(agg.values()) or 1
print(f"{len(data)} SASS lines, {tot} stall samples")
for op, v in agg.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 25):
    print(f"{op:28s} {v:8d} {100 * v / tot:5.1f}%  executed {cnt[op]}")
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
sc = collections.Counter()
for r in data:
    for h in stalls:
        v = r[hdr.index(h)]
        if v.isdigit():
            sc[h] += int(v)
print("stall reasons:", ", ".join(f"{k}={100 * v / tot:.1f}%" for k, v in sc.most_common(8)))
