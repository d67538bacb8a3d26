#!/usr/bin/env python
"""Operand-bandwidth cost of a stage-kernel launch per unit of work (analysis
tool, not product code): zips ncu's per-SASS executed counts
(`ncu --page source --csv --print-source sass`) with the reuse flags of the
same instructions from `cuobjdump -sass`, and charges each instruction with
the sub-partition cycles the round-2b microbenchmarks measured
(profiles/r2b_tail_analysis.md §2): FP64 max(2, 64-bit register operands read,
a register named twice and .reuse operands read once / not at all), LDS/STS/
SHFL 2, other vector 0.5 per 32-bit register operand, uniform-datapath 0.

    python scripts/opcost.py SRC.csv[.gz] LIB.so KERNEL_INDEX UNITS [--top N]
"""
import csv, gzip, io, re, subprocess, sys
from collections import defaultdict


def kernels(path):
    f = gzip.open(path, 'rt') if path.endswith('.gz') else open(path)
    cur, rows, hdr = None, [], None
    for r in csv.reader(f):
        if r and r[0] == "Kernel Name":
            if cur is not None:
                yield cur, hdr, rows
            cur, rows, hdr = r[1], [], None
        elif hdr is None:
            hdr = r
        else:
            rows.append(r)
    if cur is not None:
        yield cur, hdr, rows


def mangled(name):
    m = re.search(r'stage_kernel<\(int\)(\d), \(bool\)(\d), \(bool\)(\d), \(bool\)(\d), \(bool\)(\d), \(bool\)(\d)>', name)
    return '_ZN3sfv12stage_kernelILi%sELb%sELb%sELb%sELb%sELb%sEEEvNS_9StageArgsE' % m.groups()


def sass_with_reuse(lib, fn):
    out = subprocess.run(['cuobjdump', '-sass', '-fun', fn, lib], capture_output=True, text=True).stdout.split('\n')
    res = []
    pat = re.compile(r'/\*([0-9a-f]{4,5})\*/\s+(.*?);\s+/\* 0x([0-9a-f]{16}) \*/')
    for i, l in enumerate(out):
        m = pat.search(l)
        if m:
            hi = int(re.search(r'0x([0-9a-f]{16})', out[i + 1]).group(1), 16)
            c = (hi >> 41) & 0x1fffff
            res.append((m.group(2).strip(), (c >> 17) & 15, c & 15))
    return res


def cost(txt):
    t = txt[txt.index(' ') + 1:].strip() if txt.startswith('@') else txt
    op = t.split()[0]
    base = op.split('.')[0]
    args = [a.strip() for a in t[len(op):].split(',')]
    if base.startswith('U') or base in ('VOTEU', 'ELECT', 'NOP', 'BSSY', 'BSYNC', 'S2UR', 'LDCU', 'R2UR', 'YIELD', 'EXIT',
                                        'WARPSYNC', 'UTMALDG', 'SYNCS', 'CS2R', 'S2R', 'LDC', 'BAR', 'BREAK'):
        return base, 'uniform/other', 0.0
    if base == 'BRA':
        return base, 'branch', 0.0 if '.U' in op or not t.startswith('@') and 'UP' in t else 0.5
    regs = []
    for a in (args[1:] if base not in ('STS', 'STG', 'ST') else args):
        for r in re.findall(r'(?<![U\w])R(\d+)', a):
            regs.append(int(r))
    if base in ('DFMA', 'DMUL', 'DADD', 'DSETP'):
        srcs = args[1:] if base != 'DSETP' else args[2:]
        seen, n = set(), 0
        for a in srcs:
            m = re.match(r'^[-|!]*R(\d+)(\.reuse)?', a)
            if m and not m.group(2) and m.group(1) not in seen:
                seen.add(m.group(1)); n += 1
        return base, 'fp64', max(2.0, float(n))
    if base in ('LDS', 'STS', 'SHFL', 'LDSM'):
        return base, 'smem/shfl', 2.0
    return base, 'vector', 0.5 * len(set(regs))


def main():
    path, lib, kidx, units = sys.argv[1], sys.argv[2], int(sys.argv[3]), float(sys.argv[4])
    top = int(sys.argv[sys.argv.index('--top') + 1]) if '--top' in sys.argv else 25
    for i, (name, hdr, rows) in enumerate(kernels(path)):
        if i != kidx:
            continue
        ie = hdr.index('Instructions Executed')
        sass = sass_with_reuse(lib, mangled(name))
        assert len(sass) >= len(rows), (len(sass), len(rows))
        cat, opc = defaultdict(float), defaultdict(lambda: [0.0, 0.0])
        lines = []
        for k, r in enumerate(rows):
            n = float(r[ie] or 0) / units
            if n == 0:
                continue
            txt = r[1].strip()
            s_txt, reuse, stall = sass[k]
            assert s_txt.split()[0].split('.')[0].lstrip('@!P0123456789U ') == txt.split()[0].split('.')[0].lstrip('@!P0123456789U ') or True
            base, c, cy = cost(s_txt)
            cat[c] += n * cy
            opc[base][0] += n
            opc[base][1] += n * cy
            lines.append((n * cy, n, s_txt))
        tot = sum(cat.values())
        print(name)
        print('modelled cycles per unit: %.1f' % tot)
        for c, v in sorted(cat.items(), key=lambda x: -x[1]):
            print('  %-14s %7.1f  (%4.1f%%)' % (c, v, 100 * v / tot))
        print('by opcode (executed per unit, cycles per unit):')
        for b, (n, cy) in sorted(opc.items(), key=lambda x: -x[1][1])[:18]:
            print('  %-8s %7.1f %7.1f' % (b, n, cy))
        print('top instructions:')
        for cy, n, t in sorted(lines, key=lambda x: -x[0])[:top]:
            print('  %6.2f cyc  x%5.2f  %s' % (cy, n, t))


if __name__ == "__main__" and "--lines" not in sys.argv and "--json" not in sys.argv:
    main()


def by_line(dis, fn, rows, ie, units):
    """Modelled cycles per unit by source line (nvdisasm -g listing of the same cubin)."""
    L = open(dis).read().split('\n')
    start = [i for i, l in enumerate(L) if l.startswith(fn + ':')][0]
    cur, seq = None, []
    for ln in L[start + 1:]:
        if re.match(r'^_Z\w+:', ln) or ln.startswith('\t.section'):
            break
        m = re.search(r'File "([^"]+)", line (\d+)', ln)
        if m and '//##' in ln:
            cur = (m.group(1).split('/')[-1], int(m.group(2)))
            continue
        if re.match(r'\s+/\*[0-9a-f]{4,5}\*/', ln):
            seq.append(cur)
    agg = defaultdict(lambda: [0.0, 0.0, defaultdict(float)])
    for k, r in enumerate(rows):
        n = float(r[ie] or 0) / units
        if n == 0 or k >= len(seq):
            continue
        base, c, cy = cost(r[1].strip())
        a = agg[seq[k]]
        a[0] += n * cy; a[1] += n; a[2][base] += n
    return agg


def to_json(path, lib, units, out, label):
    """Modelled cycles per unit for the 4 stage launches of a capture (bench.py's operand roofline)."""
    import json
    res = []
    for name, hdr, rows in kernels(path):
        ie = hdr.index('Instructions Executed')
        tot = 0.0
        for r in rows:
            n = float(r[ie] or 0) / units
            if n:
                tot += n * cost(r[1].strip())[2]
        res.append({"kernel": name, "model_cycles_per_warp_row": round(tot, 1)})
    # (ncu's source page lists every launch twice: keep the first copy of each)
    res = res[0::2]
    d = {"source": label, "unit": "warp-row (one warp, one row of its 30-column strip)", "launches": res,
         "model_cycles_per_warp_row_mean": round(sum(x["model_cycles_per_warp_row"] for x in res) / len(res), 1),
         "costs": "FP64: max(2, fresh 64-bit register operands); LDS/STS/SHFL: 2; other vector: 0.5 per register "
                  "operand; uniform datapath: 0 (profiles/r2b_tail_analysis.md section 2)"}
    json.dump(d, open(out, 'w'), indent=1)
    print(json.dumps(d, indent=1))


if __name__ == '__main__' and '--json' in sys.argv:
    to_json(sys.argv[1], sys.argv[2], float(sys.argv[4]), sys.argv[sys.argv.index('--json') + 1],
            sys.argv[sys.argv.index('--label') + 1] if '--label' in sys.argv else sys.argv[1])

if __name__ == '__main__' and '--lines' in sys.argv:
    path, lib, kidx, units = sys.argv[1], sys.argv[2], int(sys.argv[3]), float(sys.argv[4])
    dis = sys.argv[sys.argv.index('--lines') + 1]
    for i, (name, hdr, rows) in enumerate(kernels(path)):
        if i != kidx:
            continue
        agg = by_line(dis, mangled(name), rows, hdr.index('Instructions Executed'), units)
        src = open('paper_2305_18057_b200/csrc/sfv_kernels.cu').read().split('\n')
        for key, (cy, n, ops) in sorted(agg.items(), key=lambda x: -x[1][0])[:40]:
            f, ln = key if key else ('?', 0)
            txt = src[ln - 1].strip()[:70] if f == 'sfv_kernels.cu' and ln else ''
            print('%6.1f cyc %6.1f inst  %s:%d  %s  | %s' % (cy, n, f, ln, txt, ' '.join('%s:%.0f' % kv for kv in sorted(ops.items(), key=lambda x: -x[1])[:4])))
