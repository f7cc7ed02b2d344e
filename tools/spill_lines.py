"""Count STL/LDL (register spills) per source line in one kernel of an nvdisasm --print-line-info
dump. Usage: python tools/spill_lines.py DUMP.sass NAME_SUBSTRING"""
import collections
import re
import sys

lines = open(sys.argv[1]).read().split('\n')
start = next(i for i, l in enumerate(lines) if l.startswith('.text.') and sys.argv[2] in l)
end = start + 1
while end < len(lines) and not lines[end].startswith('.text.'):
    end += 1
cnt = collections.Counter()
cur = None
for l in lines[start:end]:
    m = re.search(r'line (\d+)', l)
    if m:
        cur = m.group(1)
    if 'STL' in l or 'LDL' in l:
        cnt[(cur, 'STL' if 'STL' in l else 'LDL')] += 1
for k, v in sorted(cnt.items(), key=lambda x: -x[1])[:25]:
    print(k, v)
