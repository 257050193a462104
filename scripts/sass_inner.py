"""Innermost loops of a kernel in a SASS dump: every backward branch, its body
size and instruction mix (the Monte Carlo block loop is the one with the
Philox IMAD.WIDE.U32s).  python scripts/sass_inner.py dump.txt KERNEL_SUBSTR"""
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
    print(name.strip()[:120])
    for i, l in enumerate(lines):
        m = re.search(r"BRA\s+(?:`\(\.L_x_\d+\)\s*)?(0x[0-9a-f]+)", l)
        if not m:
            continue
        tgt = int(m.group(1), 16)
        if tgt >= addr[i] or tgt not in addr:
            continue
        j = addr.index(tgt)
        body = lines[j:i + 1]
        nw = sum("IMAD.WIDE.U32" in b for b in body)
        if nw < 8 or len(body) > 2000:
            continue
        ops = {}
        for b in body:
            op = re.search(r"\*/\s+(@!?U?P\w+\s+)?([A-Z0-9_.]+)", b).group(2).split(".")[0]
            ops[op] = ops.get(op, 0) + 1
        print(f"  loop {hex(tgt)}..{hex(addr[i])}: {len(body)} instr, IMAD.WIDE.U32 {nw}:",
              sorted(ops.items(), key=lambda x: -x[1])[:18])
