"""Join ncu per-SASS-instruction counts (--page source --print-source sass
CSV) with nvdisasm -gi inline chains: dynamic instruction counts per source
function.  Usage: sass_dyn.py ncu_sass.csv nvdisasm_dump kernel_substr src.cuh fn..."""
import bisect, collections, csv, os, re, sys
csvf, dump, kern, src = sys.argv[1:5]
want = sys.argv[5:]
# static attribution: offset -> function
lines = open(dump).read().split('\n')
start = next(i for i, l in enumerate(lines) if l.startswith('\t.section') and kern in l and '.text' in l)
srcl = open(src).read().split('\n')
ranges = []
for i, l in enumerate(srcl, 1):
    m = re.match(r'\s*(?:template <[^>]*>\s*)?(?:static\s+)?(?:DEV|__global__|__device__)[^(]*?\b(\w+)\(', l)
    if m and m.group(1) != '__launch_bounds__':
        ranges.append((i, m.group(1)))
    elif i > 1 and re.match(r'\s+(k_\w+)\(', l) and '__global__' in srcl[i - 2]:
        ranges.append((i, re.match(r'\s+(k_\w+)\(', l).group(1)))
starts = [r[0] for r in ranges]
fname = src.split('/')[-1]
def fn_of(ln):
    j = bisect.bisect_right(starts, ln) - 1
    return ranges[j][1] if j >= 0 else '?'
off2fn = {}; off2op = {}; chain = []; prev = False; n = 0; cur = 'other'
for l in lines[start + 1:]:
    if l.startswith('\t.section') and n > 10: break
    if '//## File' in l:
        if not prev: chain = []
        prev = True
        chain += re.findall(r'"([^"]+)", line (\d+)', l)
        names = [fn_of(int(ln)) for f, ln in chain if f.endswith(fname)]
        cur = next((x for x in names if x in want), names[-1] if names else 'other')
        continue
    prev = False
    m = re.match(r'\s+/\*([0-9a-f]{4,})\*/\s+(.*?);', l)
    if m and '.dword' not in l and '.word' not in l:
        n += 1; off = int(m.group(1), 16); off2fn[off] = cur; off2op[off] = m.group(2)
# dynamic counts
rows = list(csv.reader(open(csvf)))
sec = None; base = None; hdr = None
agg = collections.Counter(); aggop = collections.Counter(); conf = collections.Counter(); tot = 0
for r in rows:
    if not r: continue
    if r[0] == 'Kernel Name':
        sec = r[1]; base = None; continue
    if r[0] == 'Address':
        hdr = r; continue
    if sec is None or os.environ.get('SEC', kern) not in sec: continue
    a = int(r[0], 16)
    if base is None: base = a
    off = a - base
    ie = int(r[hdr.index('Instructions Executed')] or 0)
    f = off2fn.get(off, '?')
    agg[f] += ie; tot += ie
    op = off2op.get(off, '?').split()
    op = op[1] if op and op[0].startswith('@') and len(op) > 1 else (op[0] if op else '?')
    aggop[op] += ie
    try:
        conf[f] += int(r[hdr.index('L1 Conflicts Shared N-Way')] or 0)
    except (ValueError, IndexError):
        pass
print('dynamic warp instructions', tot)
for k, v in agg.most_common(): print(f'{v:12d} {100*v/tot:5.1f}%  {k}   (smem conflicts {conf[k]})')
print('top opcodes:')
for k, v in aggop.most_common(25): print(f'{v:12d} {100*v/tot:5.1f}%  {k}')
