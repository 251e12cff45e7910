import numpy as np, sys
"""Bank-conflict wavefronts of a slab x block layout dump (SPK_DUMP_BLOCKED=path python bench.py ...):
per chunk, the half-warp rule measured by profiles/microbench/lds64_conflicts.cu.
  python profiles/scripts/blocked_layout_conflicts.py dump.bin"""
k = np.fromfile(sys.argv[1], dtype=np.uint32)
ng = len(k) // 128
k = k[:ng*128].reshape(ng, 32, 4)   # group, lane, chunk-in-group
tot = {"row":0, "col":0}; n=0
hist = np.zeros(20, int)
for g in range(min(ng, 4000)):
    for c in range(4):
        u = k[g, :, c]
        row = u >> 16; col = u & 0xfff
        for name, v in (("row", row), ("col", col)):
            w = 0
            for h in range(2):
                vv = v[16*h:16*h+16]
                # distinct addresses per bank pair
                mult = 0
                for b in range(16):
                    mult = max(mult, len(set(vv[(vv & 15) == b])))
                w += mult
            tot[name] += w
            if name == "row": hist[w] += 1
        n += 1
print("chunks", n, "row wavefronts/chunk %.2f col %.2f" % (tot["row"]/n, tot["col"]/n))
print("row hist", hist[:10])
u = k[5,:,0]; print("sample chunk rows&15:", (u>>16)&15); print("rows:", u>>16); print("cols&15:", u&15)
