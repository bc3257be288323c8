"""Hot CUDA source lines of an `ncu --page source --csv --print-source cuda`
dump: lines by warp instructions executed and by stall samples."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if "Source" in r and any("Instructions Executed" in c for c in r))
h = rows[hi]
isrc = h.index("Source")
iln = h.index("#") if "#" in h else 0
iexe = next(i for i, c in enumerate(h) if c.startswith("Instructions Executed"))
isamp = next(i for i, c in enumerate(h) if c.startswith("Warp Stall Sampling (All"))
data = []
for r in rows[hi + 1:]:
    if len(r) <= max(iexe, isamp):
        continue
    try:
        data.append((int(r[iexe] or 0), int(r[isamp] or 0), r[iln], r[isrc].strip()[:110]))
    except ValueError:
        pass
te = sum(d[0] for d in data) or 1
ts = sum(d[1] for d in data) or 1
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
print(f"total warp instructions {te:,}, stall samples {ts:,}")
print("\nby instructions executed:")
for d in sorted(data, key=lambda d: -d[0])[:n]:
    print(f"{100 * d[0] / te:5.1f}% {100 * d[1] / ts:5.1f}%  L{d[2]:>5} {d[3]}")
print("\nby stall samples:")
for d in sorted(data, key=lambda d: -d[1])[:n]:
    print(f"{100 * d[0] / te:5.1f}% {100 * d[1] / ts:5.1f}%  L{d[2]:>5} {d[3]}")
