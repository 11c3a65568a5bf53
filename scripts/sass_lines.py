"""Join an ncu SASS source page (per-instruction counts / stall samples)
with nvdisasm line info of the same cubin: per-source-line totals.

    python scripts/sass_lines.py <nvdisasm -g output> <ncu sass csv> <mangled-name-substring> [N]
"""
import collections, csv, re, sys
txt = open(sys.argv[1]).read().split('\n')
fn = None; line = None; seq = []
for l in txt:
    m = re.match(r'\s*\.text\.(\S+):', l)
    if m: fn = m.group(1); line = None; continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m: line = (m.group(1).split('/')[-1], int(m.group(2))); continue
    m = re.match(r'\s*/\*([0-9a-f]{4,})\*/\s+(.*?);', l)
    if m and fn and sys.argv[3] in fn:
        seq.append((line, m.group(2).strip()))
rows = list(csv.reader(open(sys.argv[2])))
hdr = rows[1]; data = rows[2:]
ie = hdr.index("Instructions Executed"); ss = hdr.index("Warp Stall Sampling (All Samples)")
assert len(seq) == len(data), (len(seq), len(data))
agg = collections.defaultdict(lambda: [0, 0])
for (ln, ins), r in zip(seq, data):
    agg[ln][0] += int(r[ie]); agg[ln][1] += int(r[ss])
tot = sum(v[0] for v in agg.values()); ts = sum(v[1] for v in agg.values())
n = int(sys.argv[4]) if len(sys.argv) > 4 else 40
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])[:n]:
    print(f"{str(k):32s} inst {100 * v[0] / tot:5.1f}%  stall {100 * v[1] / ts:5.1f}%")
