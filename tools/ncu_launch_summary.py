"""Summarise an `ncu --metrics gpu__time_duration.sum --csv --log-file X` launch
list: per-kernel launch count, total/avg device time and share of the step."""
import collections
import csv
import io
import sys

txt = open(sys.argv[1]).read()
rows = list(csv.reader(io.StringIO("\n".join(l for l in txt.splitlines() if l.startswith('"')))))
hdr, rows = rows[0], rows[1:]
ik, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
agg, cnt = collections.defaultdict(float), collections.Counter()
for r in rows:
    name = r[ik].split("(")[0].replace("void ", "").replace("b2s::<unnamed>::", "")
    if "onesweep_kernel<" in name:  # keep the mode (last template argument)
        mode = name.split("<", 1)[1].rstrip(">").split(",")[-1].strip().replace("(int)", "")
        name = name.split("<")[0] + f"[mode {mode}]"
    else:
        name = name.split("<")[0]
    agg[name] += float(r[iv].replace(",", "")) * scale.get(r[iu], 1e-3)
    cnt[name] += 1
tot = sum(agg.values())
print(f"{len(rows)} launches, {tot / 1e3:.3f} ms device time (cold-cache, serialised)")
for k, v in sorted(agg.items(), key=lambda x: -x[1]):
    print(f"{k:32s} n={cnt[k]:4d} total={v / 1e3:9.3f} ms avg={v / cnt[k]:9.1f} us share={100 * v / tot:5.1f}%")
