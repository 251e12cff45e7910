"""Decode scoreboard control fields from `cuobjdump -sass` output (Volta+ 128-bit encoding).
usage: sass_ctl.py obj function-substring [filter-regex]"""
import re, subprocess, sys
obj, fn = sys.argv[1], sys.argv[2]
flt = re.compile(sys.argv[3]) if len(sys.argv) > 3 else None
out = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout.splitlines()
infn = False; rows = []
i = 0
while i < len(out):
    l = out[i]
    if "Function :" in l:
        infn = fn in l
    elif infn:
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);\s+/\* 0x([0-9a-f]{16}) \*/", l)
        if m and i + 1 < len(out):
            m2 = re.match(r"\s+/\* 0x([0-9a-f]{16}) \*/", out[i + 1])
            if m2:
                hi = int(m2.group(1), 16)
                ctl = hi >> 41  # bits 105.. of the 128-bit word = bits 41.. of the high word
                stall = ctl & 0xf; yld = (ctl >> 4) & 1; wbar = (ctl >> 5) & 7; rbar = (ctl >> 8) & 7; wait = (ctl >> 11) & 0x3f
                rows.append((m.group(1), m.group(2), stall, yld, wbar, rbar, wait))
                i += 1
    i += 1
for a, ins, stall, yld, wbar, rbar, wait in rows:
    if flt and not flt.search(ins): continue
    w = "".join(str(b) for b in range(6) if wait >> b & 1)
    print(f"{a} W:{w or '-':6} wr:{wbar if wbar != 7 else '-'} rd:{rbar if rbar != 7 else '-'} st:{stall:2} {ins}")
