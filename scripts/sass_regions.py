"""SASS instruction counts of one kernel by source region (code-size / I-cache
study).  usage: python scripts/sass_regions.py <nvdisasm -gi output> <kernel substr> <file> [top]
Attributes each instruction to the OUTERMOST line of <file> in its inline chain."""
import collections
import re
import sys

path, kern, srcfile = sys.argv[1], sys.argv[2], sys.argv[3]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
fn, cur = None, None
cnt = collections.Counter()
for line in open(path):
    m = re.match(r'\s*\.text\.(\S+):', line)
    if m:
        fn = m.group(1)
        continue
    if line.lstrip().startswith('//## File'):
        chain = re.findall(r'"([^"]+)", line (\d+)', line)
        lines = [int(l) for f, l in chain if f.endswith(srcfile)]
        cur = lines[-1] if lines else -1
        continue
    if fn and kern in fn and re.match(r'\s+/\*[0-9a-f]{4,}\*/', line):
        cnt[cur] += 1
print("total", sum(cnt.values()))
for l, c in cnt.most_common(top):
    print(f"{c:6d}  {srcfile}:{l}")
