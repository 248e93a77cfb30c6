"""List backward-branch loops of a SASS dump with instruction counts (hot-loop size check)."""
import re, sys
L = open(sys.argv[1]).read().splitlines()
ins = [l for l in L if re.search(r'/\*[0-9a-f]{4,}\*/', l)]
addr = lambda l: int(re.search(r'/\*([0-9a-f]{4,})\*/', l).group(1), 16)
for l in ins:
    m = re.search(r'BRA(\.\w+)* (0x[0-9a-f]+)', l)
    if m and 'BRA.DIV' not in l:
        tgt = int(m.group(2), 16)
        if tgt < addr(l):
            body = [x for x in ins if tgt <= addr(x) <= addr(l)]
            nw = sum('IMAD.WIDE' in x for x in body)
            if 16 <= nw <= 20 and len(body) < 400:
                from collections import Counter
                c = Counter(x.split(';')[0].split('*/')[1].split()[0 if not x.split('*/')[1].split()[0].startswith('@') else 1].split('.')[0] for x in body)
                print(hex(tgt), hex(addr(l)), len(body), 'per node', len(body) / 4, dict(c.most_common(14)))
