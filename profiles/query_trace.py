"""Phase trace of the tensor-core query kernel (development build with
-DNASG_TRACE: clock64() stamps of pair 0 of CTA 0 over the first 32 tiles).
    make -C paper_2303_08064_b200/csrc OUT=$PWD/paper_2303_08064_b200/lib_exp/trace EXTRA=-DNASG_TRACE
    NASG_LIB=$PWD/paper_2303_08064_b200/lib_exp/trace/libnasg_b200.so python profiles/query_trace.py
Prints mean cycles per phase over tiles 4-29 for the MLP and the NASG warpgroup."""
import ctypes as C
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2303_08064_b200 as nasg  # noqa: E402

n = 1 << 22
g = nasg.Guide(nasg.TrainerConfig(seed=0, n_components=int(os.environ.get("TRACE_N", "8"))))
g.precision = nasg.NASG_MLP_BF16
dev = [torch.from_numpy(a).cuda() for a in nasg.synth_queries(5, n)]
for _ in range(2):
    g.query_sample(*dev)
torch.cuda.synchronize()
L = C.CDLL(nasg.LIB_PATH)
buf = np.zeros(2 * 32 * 16, np.uint64)
assert L.nasg_trace_read(buf.ctypes.data_as(C.c_void_p)) == 0
tr = buf.reshape(2, 32, 16).astype(np.int64)
ks = range(4, 30)
mlp = {"wait E + issue L0": [], "L0 wait": [], "drain h1 + issue": [], "L1 wait": [], "drain h2 + issue": [],
       "L2 wait": [], "drain h3 + issue out": [], "to next tile": []}
keys = list(mlp)
for k in ks:
    r = tr[0, k]
    seq = [r[0], r[1], r[2], r[3], r[4], r[5], r[6], r[7], tr[0, k + 1, 0]]
    for i, name in enumerate(keys):
        mlp[name].append(seq[i + 1] - seq[i])
nasg_ph = {"wait e_empty": [], "encode next": [], "wait raw_full": [], "epilogue": [], "to next tile": []}
for k in ks:
    r = tr[1, k]
    seq = [r[0], r[1], r[2], r[3], r[4], tr[1, k + 1, 0]]
    for i, name in enumerate(nasg_ph):
        nasg_ph[name].append(seq[i + 1] - seq[i])
out = {"mlp": {k: float(np.mean(v)) for k, v in mlp.items()}, "nasg": {k: float(np.mean(v)) for k, v in nasg_ph.items()}}
out["mlp_period"] = float(np.mean([tr[0, k + 1, 0] - tr[0, k, 0] for k in ks]))
out["nasg_period"] = float(np.mean([tr[1, k + 1, 0] - tr[1, k, 0] for k in ks]))
print(json.dumps(out, indent=1))
