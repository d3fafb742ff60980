"""Aggregate an ncu SASS source-page CSV (--page source --csv --print-source sass) by CUDA
source line, using nvdisasm -g line info of the kernel's cubin.
python scripts/ncu_lines.py <src.csv> <nvdisasm -g output> <kernel mangled name> <source.cu> [top]"""
import collections
import csv
import re
import sys

src_csv, dis, kname, srcfile = sys.argv[1:5]
top = int(sys.argv[5]) if len(sys.argv) > 5 else 40
lines = open(dis).read().split('\n')
start = next(i for i, ln in enumerate(lines) if ln.startswith('.text.' + kname + ':'))
addr2line, cur = {}, None
for ln in lines[start + 1:]:
    if ln.startswith('.text.') or '.section' in ln:
        break
    m = re.search(r'//## File "(.*?)", line (\d+)', ln)
    if m:
        cur = (m.group(1).split('/')[-1], int(m.group(2)))
        continue
    m = re.search(r'/\*([0-9a-f]{4,})\*/', ln)
    if m and cur is not None:
        addr2line[int(m.group(1), 16)] = cur
rows = list(csv.reader(open(src_csv)))
hdr = rows[1]
ia, iss, iex = hdr.index('Address'), hdr.index('Warp Stall Sampling (All Samples)'), hdr.index('Instructions Executed')
base = None
agg = collections.defaultdict(lambda: [0.0, 0.0])
tot = [0.0, 0.0]
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    try:
        a = int(r[ia], 16)
    except ValueError:
        continue
    if base is None:
        base = a
    s, e = float(r[iss] or 0), float(r[iex] or 0)
    key = addr2line.get(a - base, ('?', -1))
    agg[key][0] += s
    agg[key][1] += e
    tot[0] += s
    tot[1] += e
src = open(srcfile).read().split('\n')
print('total samples %d, warp instructions %d' % tuple(tot))
for key, (s, e) in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
    txt = src[key[1] - 1].strip()[:80] if key[0] == srcfile.split('/')[-1] else ''
    print(f"{key[0]}:{key[1]:5d} samp {s / tot[0] * 100:5.1f}% inst {e / tot[1] * 100:5.1f}%  {txt}")
