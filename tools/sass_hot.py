"""Hot SASS lines of an `ncu --page source --csv --print-source sass` dump:
instructions sorted by executed count and by stall samples, plus the total
instruction mix."""
import csv
import collections
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
ia, isrc, iexe, isamp = h.index("Address"), h.index("Source"), h.index("Instructions Executed"), h.index(
    "Warp Stall Sampling (All Samples)")
data = []
for r in rows[2:]:
    if len(r) <= iexe:
        continue
    try:
        data.append((int(r[iexe]), int(r[isamp] or 0), r[ia], r[isrc].strip()))
    except ValueError:
        pass
tot = sum(d[0] for d in data)
mix = collections.Counter()
for n, _, _, src in data:
    op = src.split()[0] if not src.startswith("@") else src.split()[1]
    mix[op.split(".")[0]] += n
print(f"total warp instructions {tot:,}")
for op, n in mix.most_common(25):
    print(f"  {op:10s} {n:>14,} {100 * n / tot:5.1f}%")
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
print("\nby stall samples:")
for d in sorted(data, key=lambda d: -d[1])[:n]:
    print(f"{d[1]:7d} {d[0]:>12,} {d[2][-5:]} {d[3]}")

if len(sys.argv) > 3:  # full per-instruction list: offset from the function start
    base = min(int(d[2], 16) for d in data)
    with open(sys.argv[3], "w") as f:
        f.write("offset,exec,samples,sass\n")
        for d in data:
            f.write(f"{int(d[2], 16) - base},{d[0]},{d[1]},\"{d[3]}\"\n")
