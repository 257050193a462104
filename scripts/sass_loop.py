"""Instruction mix of the hottest loop (most IMAD.WIDE.U32) of each matching kernel in a SASS dump."""
import re
import sys

txt = open(sys.argv[1]).read()
pat = sys.argv[2] if len(sys.argv) > 2 else "k_mc"
for f in re.split(r"\n\s+Function : ", txt)[1:]:
    name = f.split("\n")[0]
    if pat not in name:
        continue
    lines = [l for l in f.split("\n") if re.search(r"/\*[0-9a-f]{4,}\*/", l)]
    addr = [int(re.search(r"/\*([0-9a-f]{4,})\*/", l).group(1), 16) for l in lines]
    best = None
    for i, l in enumerate(lines):
        m = re.search(r"BRA\s+(0x[0-9a-f]+)", l)
        if m and int(m.group(1), 16) < addr[i] and int(m.group(1), 16) in addr:
            j = addr.index(int(m.group(1), 16))
            nw = sum("IMAD.WIDE.U32" in b for b in lines[j:i + 1])
            if best is None or nw > best[0]:
                best = (nw, j, i)
    if best is None:
        continue
    body = lines[best[1]:best[2] + 1]
    ops = {}
    for b in body:
        op = re.search(r"\*/\s+(@!?U?P\w+\s+)?([A-Z0-9_.]+)", b).group(2).split(".")[0]
        ops[op] = ops.get(op, 0) + 1
    print(name[40:90], "loop", len(body), sorted(ops.items(), key=lambda x: -x[1])[:14])
