import sys, hashlib, numpy as np
sys.path.insert(0, '.')
from paper_2306_06581_b200 import workloads as W
w = W.c4()
h = hashlib.sha256()
for arr in (w.x, w.y):
    h.update(np.ascontiguousarray(arr, np.float64).tobytes())
h.update(np.float64(w.scale).tobytes())
print("C4 digest", h.hexdigest(), w.scale)
