"""Join an ncu SASS source page (per-instruction executions / stall samples)
with nvdisasm -gi line info of the same binary: hot code by source line.
usage: python scripts/hot_lines.py <ncu-rep> <nvdisasm -gi file> <kernel substr> <file> [top] [inner]"""
import collections
import csv
import re
import subprocess
import sys

rep, dis, kern, srcfile = sys.argv[1:5]
top = int(sys.argv[5]) if len(sys.argv) > 5 else 40
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
h = rows[1]
ie, sm = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
perf = [(int(r[ie] or 0), int(r[sm] or 0)) for r in rows[2:] if len(r) > ie]
fn, cur, lines = None, None, []
for line in open(dis):
    m = re.match(r'\s*\.text\.(\S+):', line)
    if m:
        fn = m.group(1)
        continue
    if line.lstrip().startswith('//## File'):
        chain = re.findall(r'"([^"]+)", line (\d+)', line)
        inner = f"{chain[0][0].split('/')[-1]}:{chain[0][1]}"
        outer = [int(l) for f, l in chain if f.endswith(srcfile)]
        cur = (outer[-1] if outer else -1, inner)
        continue
    if fn and kern in fn and re.match(r'\s+/\*[0-9a-f]{4,}\*/', line):
        lines.append(cur)
assert len(lines) == len(perf), (len(lines), len(perf))
ex, st, sz = collections.Counter(), collections.Counter(), collections.Counter()
key_inner = len(sys.argv) > 6 and sys.argv[6] == "inner"
for (o, i), (e, s) in zip(lines, perf):
    k = i if key_inner else o
    ex[k] += e
    st[k] += s
    sz[k] += 1
te, ts = sum(ex.values()), sum(st.values())
print(f"{'exec%':>6} {'stall%':>6} {'sass':>5}  line")
for o, s in st.most_common(top):
    print(f"{100*ex[o]/te:6.1f} {100*s/ts:6.1f} {sz[o]:5d}  {o}")
