"""Static SASS instruction counts per enclosing source function (uses
nvdisasm -gi inline chains).  Usage: sass_attrib.py dump.sass kernel_substr src.cuh [fn...]"""
import bisect, collections, re, sys
dump, kern, src = sys.argv[1:4]
want = set(sys.argv[4:])
lines = open(dump).read().split('\n')
start = next(i for i, l in enumerate(lines) if l.startswith('\t.section') and kern in l and '.text' in l)
srcl = open(src).read().split('\n')
ranges = []
for i, l in enumerate(srcl, 1):
    m = re.match(r'\s*(?:template <[^>]*>\s*)?(?:static\s+)?(?:DEV|__global__|__device__)[^(]*?\b(\w+)\(', l)
    if not m and i > 1 and re.match(r'\s+(k_\w+)\(', l) and '__global__' in srcl[i - 2]:
        m = re.match(r'\s+(k_\w+)\(', l)
    if m:
        ranges.append((i, m.group(1)))
starts = [r[0] for r in ranges]
fname = src.split('/')[-1]
def fn_of(ln):
    j = bisect.bisect_right(starts, ln) - 1
    return ranges[j][1] if j >= 0 else '?'
cnt = collections.Counter(); cur = '?'; n = 0; chain = []; prev_comment = False
for l in lines[start + 1:]:
    if l.startswith('\t.section') or l.startswith('//----'):
        if n > 10: break
    if '//## File' in l:
        if not prev_comment: chain = []
        prev_comment = True
        chain += re.findall(r'"([^"]+)", line (\d+)', l)
        names = [fn_of(int(ln)) for f, ln in chain if f.endswith(fname)]
        cur = next((x for x in names if x in want), names[-1] if names else 'other')
        continue
    prev_comment = False
    if re.match(r'\s+/\*[0-9a-f]{4,}\*/\s+\S', l) and '.dword' not in l and '.word' not in l:
        n += 1; cnt[cur] += 1
print('total', n)
for k, v in cnt.most_common(): print(f'{v:7d} {k}')
