"""SASS-level hot spots of one ncu --set full capture (--import-source on):
executed-instruction mix per solved LP and the basic blocks ranked by
executed instructions, with their share of warp-stall samples.
usage: python profiles/ncu_hotspots.py report.ncu-rep N_LPS > profiles/rNN_cX_sass_hotspots.txt"""
import collections
import csv
import io
import re
import subprocess
import sys

rep, n_lp = sys.argv[1], int(sys.argv[2])
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
ie, src = h.index("Instructions Executed"), h.index("Source")
st = h.index("Warp Stall Sampling (All Samples)")
ins = [(int(r[0], 16), r[src].strip(), int(r[ie]), int(r[st])) for r in rows[2:]]
base = ins[0][0]
tot = sum(x[2] for x in ins)
tots = sum(x[3] for x in ins) or 1
print(rows[0][1])
print("executed warp instructions %d = %.0f per LP (%d LPs)" % (tot, tot / n_lp, n_lp))
op = collections.Counter()
for _, s, v, _ in ins:
    op[re.sub(r"^@!?U?P\w+\s+", "", s).split()[0]] += v
print("\nopcode mix (warp instructions per LP):")
for o, v in op.most_common(24):
    print("  %-22s %7.1f  %5.1f%%" % (o, v / n_lp, 100 * v / tot))
blocks, cur = [], None
for a, s, v, stl in ins:
    if cur and cur[1] == v and not cur[3]:
        cur[2].append(s)
        cur[4] += stl
    else:
        if cur:
            blocks.append(cur)
        cur = [a - base, v, [s], False, stl]
    if "BRA" in s.split()[0:2] or s.startswith("EXIT"):
        cur[3] = True
blocks.append(cur)
print("\nbasic blocks by executed instructions (offset, executions, length, share, stall share, top opcodes):")
for a, v, ss, _, stl in sorted(blocks, key=lambda b: -b[1] * len(b[2]))[:30]:
    c = collections.Counter(x.split()[1] if x.startswith("@") else x.split()[0] for x in ss)
    print("  %05x x%-9d len %3d  %5.2f%%  stall %5.2f%%  %s" % (
        a, v, len(ss), 100 * v * len(ss) / tot, 100 * stl / tots,
        " ".join("%s:%d" % kv for kv in c.most_common(6))))
