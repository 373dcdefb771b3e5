"""Map an ncu SASS source-page CSV to CUDA source lines via nvdisasm line info.

    ncu -i rep --page source --csv --print-source sass > src.csv
    cuobjdump -xelf all lib.so; nvdisasm -g -c <cubin> > all.sass
    python tools/ncu_sass_lines.py src.csv all.sass <mangled kernel name> [top]
Prints stall samples (by reason) and executed instructions per source line.
"""
import collections
import csv
import re
import sys

src_csv, sass, kname = sys.argv[1:4]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
lines = open(sass).read().split('\n')
start = [i for i, l in enumerate(lines) if l.startswith('//----') and kname in l][0]
end = next((i for i in range(start + 1, len(lines)) if lines[i].startswith('//----')), len(lines))
cur = None
off2line = {}
for l in lines[start:end]:
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        cur = (m.group(1), int(m.group(2)))
        continue
    m = re.match(r'\s+/\*([0-9a-f]{4,})\*/\s+(.*)', l)
    if m:
        off2line[int(m.group(1), 16)] = cur
rows = list(csv.reader(open(src_csv)))
hdr = rows[1]
iA = hdr.index("Address")
iW = hdr.index("Warp Stall Sampling (All Samples)")
iE = hdr.index("Instructions Executed")
reasons = [h for h in hdr if h.startswith('stall_') and 'Not Issued' not in h]
base = int(rows[2][iA], 16)
agg = collections.defaultdict(lambda: collections.Counter())
tot = totE = 0
for r in rows[2:]:
    try:
        a = int(r[iA], 16) - base
        s = int(r[iW])
        e = int(r[iE])
    except (ValueError, IndexError):
        continue
    ln = off2line.get(a)
    c = agg[ln]
    c['_s'] += s
    c['_e'] += e
    for h in reasons:
        try:
            c[h] += int(r[hdr.index(h)] or 0)
        except ValueError:
            pass
    tot += s
    totE += e


def txt(ln):
    try:
        return open(ln[0]).read().split('\n')[ln[1] - 1].strip()[:70]
    except Exception:
        return ''


print("samples", tot, "instructions", totE)
for ln, c in sorted(agg.items(), key=lambda kv: -kv[1]['_s'])[:top]:
    rs = sorted(((v, k[6:]) for k, v in c.items() if k.startswith('stall_') and v), reverse=True)[:3]
    name = f"{ln[0].split('/')[-1]}:{ln[1]}" if ln else "?"
    print(f"{c['_s'] / tot * 100:5.1f}% st {c['_e'] / totE * 100:5.1f}% in {name:24s} "
          f"{' '.join(f'{k}={v}' for v, k in rs):40s} {txt(ln) if ln else ''}")
