"""Map an ncu SASS page (scripts/ncu_source.sh *_sass.csv) onto source lines with the line
info of the local build of the same kernel: per line, share of stall samples / instructions
and the top opcodes.   python scripts/sass_hotspots.py SASS_CSV OBJ KERNEL_SUBSTR [N]"""
import collections
import csv
import os
import re
import subprocess
import sys
import tempfile


def main(sass_csv, obj, ksub, top=30):
    rows = list(csv.reader(open(sass_csv)))
    h = rows[1]
    ai, si, ni, src = (h.index(k) for k in ("Address", "Warp Stall Sampling (All Samples)",
                                           "Instructions Executed", "Source"))
    data = [(int(r[ai], 16), r[src].strip(), float(r[si] or 0), float(r[ni] or 0))
            for r in rows[2:] if len(r) > ni and r[ai].startswith("0x")]
    base = data[0][0]
    with tempfile.TemporaryDirectory() as d:
        subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=d, capture_output=True)
        cub = [f for f in os.listdir(d) if f.endswith(".cubin")][0]
        text = subprocess.run(["nvdisasm", "--print-line-info", os.path.join(d, cub)], capture_output=True,
                              text=True).stdout.split("\n")
    start = [i for i, l in enumerate(text) if l.startswith(".text.") and ksub in l][0]
    end = start + 1
    while end < len(text) and not text[end].startswith(".text."):
        end += 1
    cur, off2line = None, {}
    for l in text[start:end]:
        m = re.search(r'//## File "([^"]+)", line (\d+)', l)
        if m:
            cur = (m.group(1).split("/")[-1], int(m.group(2)))
            continue
        m = re.search(r"/\*([0-9a-f]{4,})\*/\s+\S", l)
        if m and cur:
            off2line[int(m.group(1), 16)] = cur
    S, N = collections.Counter(), collections.Counter()
    ops = collections.defaultdict(collections.Counter)
    ts = sum(x[2] for x in data) or 1
    tn = sum(x[3] for x in data) or 1
    for a, s, st, n in data:
        key = off2line.get(a - base, ("?", 0))
        S[key] += st
        N[key] += n
        op = s.split()[1] if s.startswith("@") else s.split()[0]
        ops[key][op.split(".")[0]] += n
    csrc = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "paper_2309_16849_b200", "csrc")
    for key, st in S.most_common(int(top)):
        f, ln = key
        p = os.path.join(csrc, f)
        txt = open(p).read().split("\n")[ln - 1].strip()[:64] if os.path.exists(p) and ln else ""
        topo = ",".join(f"{o}:{c / 1e6:.0f}M" for o, c in ops[key].most_common(3))
        print(f"{100 * st / ts:5.1f}% smp {100 * N[key] / tn:5.1f}% ins {f}:{ln:<4} {topo:34s} {txt}")
    tot = collections.Counter()
    for k in ops:
        tot.update(ops[k])
    print("opcodes:", ", ".join(f"{o} {100 * c / tn:.1f}%" for o, c in tot.most_common(14)))


if __name__ == "__main__":
    main(*sys.argv[1:])
