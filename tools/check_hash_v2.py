"""Prototype check: the device's v2 triangle hash equals a numpy restatement
over the device's own canonical list (run with TL_LIB_PATH=<v2 build>)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as O  # noqa: E402
from paper_2006_11494_b200 import capi  # noqa: E402

M = np.uint64


def fmix(z):
    with np.errstate(over="ignore"):
        z = (z ^ (z >> M(30))) * M(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> M(27))) * M(0x94D049BB133111EB)
        return z ^ (z >> M(31))


pairs = O.gen_rmat(9, 14, 16 << 14)
do = capi.DeviceGraph.from_pairs(pairs, 1 << 14).orient()
st = do.hash()
_, t = do.list(canonical=True)
g = [fmix(t[:, k].astype(M) ^ M(0xD6E8FEB86659FD93)) for k in range(3)]
with np.errstate(over="ignore"):
    h = fmix(g[0] + g[1] + g[2])
s = int(np.sum(h, dtype=M))
x = int(np.bitwise_xor.reduce(h))
print({"triangles": st["triangles"], "device": (st["hash_sum"], st["hash_xor"]), "numpy": (s, x),
       "equal": (st["hash_sum"], st["hash_xor"]) == (s, x)})
