"""Phase trace of the tensor-core trainer's K_fb (development build with
-DNASG_TRACE: clock64() stamps of warpgroup 0 of CTA 0 over its first tiles).
    make -C paper_2303_08064_b200/csrc OUT=$PWD/paper_2303_08064_b200/lib_exp/trace EXTRA=-DNASG_TRACE
    NASG_LIB=$PWD/paper_2303_08064_b200/lib_exp/trace/libnasg_b200.so AB_T=4096 python profiles/train_trace.py
Prints cycles per phase for the first tile (and the mean over tiles 1.. when there are several)."""
import ctypes as C
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2303_08064_b200 as nasg  # noqa: E402

for n in [int(v) for v in os.environ.get("AB_T", "4096").split(",")]:
    g = nasg.Guide(nasg.TrainerConfig(seed=3, sample_capacity=n, batch_size=n))
    g.train_precision = nasg.NASG_MLP_BF16
    s = torch.from_numpy(nasg.synth_samples(11, n)).cuda()
    for _ in range(3):
        g.train_iteration(s, 1.0, stats=False)
    torch.cuda.synchronize()
    L = C.CDLL(nasg.LIB_PATH)
    buf = np.zeros(16 * 16, np.uint64)
    assert L.nasg_fb_trace_read(buf.ctypes.data_as(C.c_void_p)) == 0
    tr = buf.reshape(16, 16).astype(np.int64)
    names = ["encode", "drain h1", "drain h2", "drain h3", "output layer wait", "KL gradient", "bwd delta3",
             "bwd delta2", "bwd delta1"]
    def phases(k):
        r = tr[k]
        seq = [r[0], r[1], r[2], r[3], r[4], r[5], r[6], r[7], r[8], r[9]]
        return {nm: int(seq[i + 1] - seq[i]) for i, nm in enumerate(names)}
    out = {"t": n, "launch_to_tile0": int(tr[0, 0] - tr[0, 15]), "weights_wait": int(tr[0, 14] - tr[0, 15]),
           "tile0": phases(0), "tile0_total": int(tr[0, 9] - tr[0, 0])}
    ks = [k for k in range(1, 16) if tr[k, 0] > 0 and tr[k, 9] > 0]
    if ks:
        out["mean_later_tiles"] = {nm: float(np.mean([phases(k)[nm] for k in ks])) for nm in names}
    print(json.dumps(out))
    g.close()
