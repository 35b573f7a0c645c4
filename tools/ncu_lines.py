"""Per-CUDA-source-line warp-stall samples from
`ncu --page source --csv --print-source cuda,sass` (first function only)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[2]
i_s = hdr.index("Warp Stall Sampling (All Samples)")
stalls = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
lines = []
for r in rows[3:]:
    if r and r[0] == "File Path":
        break
    if len(r) >= len(hdr) and r[2] == "-" and r[0].isdigit():
        s = int(r[i_s] or 0)
        top = sorted(((int(r[i] or 0), hdr[i]) for i in stalls), reverse=True)[:2]
        lines.append((s, int(r[0]), r[1].strip()[:70], top))
tot = sum(l[0] for l in lines) or 1
for s, ln, src, top in sorted(lines, reverse=True)[: int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    print(f"{100 * s / tot:5.1f}% L{ln:<5d} {src:70s} {[(h[6:], v) for v, h in top]}")
