"""Dynamic instruction counts per source line: zip ncu's SASS page (executed
counts) with nvdisasm -g line info of the same cubin (analysis helper)."""
import csv, re, sys
from collections import Counter, defaultdict
listing, srccsv, kname, cells = sys.argv[1], sys.argv[2], sys.argv[3], float(sys.argv[4])
lines = open(listing).read().split('\n')
start = [i for i, l in enumerate(lines) if l.startswith(kname + ':')][0]
end = start + 1
while end < len(lines) and not re.match(r'^_Z\w+:', lines[end]) and not lines[end].startswith('.section'):
    end += 1
stat, cur = [], None
for ln in lines[start:end]:
    m = re.search(r'line (\d+)', ln)
    if '//##' in ln and m:
        f = re.search(r'File "([^"]+)"', ln)
        cur = ((f.group(1).split('/')[-1] if f else '?'), int(m.group(1)))
        continue
    m2 = re.match(r'\s+/\*([0-9a-f]{4})\*/\s+(@!?U?P\w+\s+)?([A-Z0-9_.]+)', ln)
    if m2:
        stat.append((cur, m2.group(3)))
L = open(srccsv).read().split('\n')
blocks, cb = [], None
for ln in L:
    if ln.startswith('"Kernel Name"'):
        cb = [ln]; blocks.append(cb)
    elif cb is not None:
        cb.append(ln)
want = sys.argv[5] if len(sys.argv) > 5 else 'stage_kernel<(int)1, (bool)0, (bool)0, (bool)1'
b = [x for x in blocks if want in x[0]][0]
rows = list(csv.reader(b[1:])); h = rows[0]; data = [r for r in rows[1:] if len(r) == len(h)]
ie = h.index('Instructions Executed')
dyn, ops, opc = Counter(), defaultdict(Counter), Counter()
for (loc, op), r in zip(stat, data):
    dyn[loc] += int(r[ie]); ops[loc][op.split('.')[0]] += int(r[ie]); opc[op if op.startswith('IMAD') else op.split('.')[0]] += int(r[ie])
print('static', len(stat), 'ncu', len(data), 'thread-inst/cell', round(sum(dyn.values()) * 32 / cells))
print(', '.join(f"{o} {c * 32 / cells:.0f}" for o, c in opc.most_common(24)))
src = open('paper_2305_18057_b200/csrc/sfv_kernels.cu').read().split('\n')
for loc, c in dyn.most_common(int(sys.argv[6]) if len(sys.argv) > 6 else 30):
    f, l = loc if loc else ('?', 0)
    line = src[l - 1].strip()[:58] if f == 'sfv_kernels.cu' else ''
    top = ', '.join(f"{o}{n * 32 / cells:.0f}" for o, n in ops[loc].most_common(4))
    print(f"{f[:14]}:{l:4d} {c * 32 / cells:6.1f}  {top:38s} {line}")
