"""Times the reference build (oracle/_ref) in both flavours on this host:
x86-64-v3 (libnasg_ref.so) and generic x86-64 (libnasg_ref_generic.so),
1 thread and all threads, on the same synthetic queries."""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle.oracle as O  # noqa: E402

res = {}
for lib in ("libnasg_ref.so", "libnasg_ref_generic.so"):
    O.LIBS["ref"] = os.path.join(O.HERE, "_ref", lib)
    o = O.Oracle("ref")
    w = o.init_network(0)
    x, wo, n, xi = o.synth_queries(1, 1 << 18)
    q9 = np.ascontiguousarray(np.concatenate([x[:, :3], wo[:, :3], n[:, :3]], 1))
    nt = len(os.sched_getaffinity(0))
    o.query_sample(w, q9[:4096], xi[:4096], threads=nt)
    for th in (1, nt):
        m = (1 << 14) if th == 1 else (1 << 18)
        t = time.perf_counter()
        o.query_sample(w, q9[:m], xi[:m], threads=th)
        res[f"{lib}_threads{th}"] = m / (time.perf_counter() - t)
print(json.dumps(res))
