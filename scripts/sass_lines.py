"""Attribute an ncu SASS source page (per-instruction metrics) to CUDA source lines.

    nvdisasm -g -c <cubin> > all.dis
    ncu -i <rep> --page source --csv --print-source sass > sass.csv
    python scripts/sass_lines.py all.dis <kernel-mangled-name> sass.csv [dets] [top]

Prints thread instructions per determinant and the share of warp-stall samples per
(file, line), innermost inlined location (development aid for the profiles/ summaries).
"""
import csv
import re
import sys
from collections import defaultdict


def line_map(dis, kern):
    m, cur, on = {}, None, False
    for ln in open(dis):
        if ln.startswith("//--------------------- .text."):
            on = kern in ln
            continue
        if not on:
            continue
        g = re.search(r'//## File "([^"]+)", line (\d+)', ln)
        if g:
            cur = (g.group(1).split("/")[-1], int(g.group(2)))
            continue
        a = re.search(r"/\*([0-9a-f]{4,})\*/", ln)
        if a and cur:
            m[int(a.group(1), 16)] = cur
    return m


def main():
    dis, kern, sass = sys.argv[1:4]
    dets = float(sys.argv[4]) if len(sys.argv) > 4 else 1.0
    top = int(sys.argv[5]) if len(sys.argv) > 5 else 40
    lm = line_map(dis, kern)
    rows = list(csv.reader(open(sass)))
    hdr = rows[1]
    ia, iex = hdr.index("Address"), hdr.index("Thread Instructions Executed")
    ist = hdr.index("Warp Stall Sampling (All Samples)")
    agg = defaultdict(lambda: [0.0, 0.0])
    addrs = []
    for r in rows[2:]:
        try:
            addrs.append(int(r[ia], 16))
        except (ValueError, IndexError):
            pass
    base = min(addrs)   # ncu prints absolute addresses; nvdisasm offsets from the entry
    for r in rows[2:]:
        try:
            a, n, s = int(r[ia], 16) - base, float(r[iex]), float(r[ist])
        except (ValueError, IndexError):
            continue
        k = lm.get(a, ("?", 0))
        agg[k][0] += n
        agg[k][1] += s
    tn = sum(v[0] for v in agg.values())
    ts = sum(v[1] for v in agg.values()) or 1.0
    print(f"total thread instructions per det: {tn / dets:.1f}")
    src = {}
    for (f, l), v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"{v[0] / dets:7.1f} /det {100 * v[1] / ts:5.1f}% stalls  {f}:{l}")


if __name__ == "__main__":
    main()


def by_opcode(dis, kern, sass, opcode, dets=1.0):
    """Source lines of one opcode (prefix match), per det."""
    lm = line_map(dis, kern)
    rows = list(csv.reader(open(sass)))
    hdr = rows[1]
    ia, iex, isrc = hdr.index("Address"), hdr.index("Thread Instructions Executed"), hdr.index("Source")
    base = min(int(r[ia], 16) for r in rows[2:] if r and r[ia].startswith("0x"))
    agg = defaultdict(float)
    for r in rows[2:]:
        try:
            a, n = int(r[ia], 16) - base, float(r[iex])
        except (ValueError, IndexError):
            continue
        src = r[isrc].strip()
        if src.startswith("@"):
            src = src.split(None, 1)[1]
        if src.startswith(opcode):
            agg[lm.get(a, ("?", 0))] += n
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:15]:
        print(f"{v / dets:7.1f} /det  {k[0]}:{k[1]}")
