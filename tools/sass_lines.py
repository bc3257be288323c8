"""Map a profiled per-instruction SASS list (tools/sass_hot.py's CSV:
offset, exec, samples) to CUDA source lines with nvdisasm's line info of the
same kernel in the local build, and print the hot lines.

  python tools/sass_lines.py PROFILE.csv KERNEL_MANGLED_SUBSTR [N]
"""
import collections
import csv
import os
import re
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2205_04401_b200", "libvp_b200.so")


def main():
    prof, kname = sys.argv[1], sys.argv[2]
    n = int(sys.argv[3]) if len(sys.argv) > 3 else 30
    tmp = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", LIB], cwd=tmp, check=True, capture_output=True)
    cub = [os.path.join(tmp, f) for f in os.listdir(tmp) if f.endswith(".cubin")]
    fn = None
    for c in cub:
        syms = subprocess.run(["cuobjdump", "-symbols", c], capture_output=True, text=True).stdout
        m = [l.split()[-1] for l in syms.splitlines() if kname in l and "STT_FUNC" in l]
        if m:
            fn, cubin = m[0], c
            break
    if fn is None:
        sys.exit(f"kernel {kname} not found")
    dis = subprocess.run(["nvdisasm", "-g", cubin], capture_output=True, text=True).stdout
    line = None
    off2line = {}
    inside = False
    for l in dis.splitlines():
        if l.startswith(".text."):
            inside = l.startswith(".text." + fn + ":")
            continue
        if not inside:
            continue
        m = re.search(r'//## File "([^"]+)", line (\d+)', l)
        if m:
            line = (os.path.basename(m.group(1)), int(m.group(2)))
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", l)
        if m and line:
            off2line[int(m.group(1), 16)] = line
    agg = collections.defaultdict(lambda: [0, 0])
    tot = [0, 0]
    for r in csv.DictReader(open(prof)):
        o, e, s = int(r["offset"]), int(r["exec"]), int(r["samples"])
        ln = off2line.get(o, ("?", 0))
        agg[ln][0] += e
        agg[ln][1] += s
        tot[0] += e
        tot[1] += s
    files = {}

    def text(ln):
        f, k = ln
        if f not in files:
            p = os.path.join(ROOT, "paper_2205_04401_b200", "csrc", f)
            files[f] = open(p).read().splitlines() if os.path.exists(p) else []
        L = files[f]
        return L[k - 1].strip()[:100] if 0 < k <= len(L) else ""
    print(f"{fn}: {tot[0]:,} warp instructions, {tot[1]:,} stall samples")
    for title, key in (("by instructions", 0), ("by stall samples", 1)):
        print(f"\n{title}:")
        for ln, v in sorted(agg.items(), key=lambda kv: -kv[1][key])[:n]:
            print(f"{100 * v[0] / max(tot[0], 1):5.1f}% {100 * v[1] / max(tot[1], 1):5.1f}%  {ln[0]}:{ln[1]:<5d} {text(ln)}")


if __name__ == "__main__":
    main()
