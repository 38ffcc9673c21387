"""Does the early-started classification (it reads the samples before its
programmatic wait) respect a cross-stream event wait placed before the step?
Each step uploads a different sample set on a copy stream, the compute stream
waits on its event, then trains (stats read back); the per-step losses must equal
a run where every step is fully synchronised before the call."""
import sys, os
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2303_08064_b200 as nasg

n = 1 << 18
hosts = [torch.from_numpy(nasg.synth_samples(100 + k, n)).pin_memory() for k in range(4)]

def run(synced):
    g = nasg.Guide(nasg.TrainerConfig(seed=3, sample_capacity=n, batch_size=n))
    g.train_precision = nasg.NASG_MLP_BF16
    bufs = [torch.empty((n, 16), dtype=torch.float32, device="cuda") for _ in range(2)]
    cs, cur = torch.cuda.Stream(), torch.cuda.current_stream()
    copied = [torch.cuda.Event(), torch.cuda.Event()]
    trained = [torch.cuda.Event(), torch.cuda.Event()]
    losses = []
    for k in range(24):
        b = k % 2
        with torch.cuda.stream(cs):
            if k >= 2:
                cs.wait_event(trained[b])
            bufs[b].copy_(hosts[k % 4], non_blocking=True)
            copied[b].record(cs)
        if synced:
            torch.cuda.synchronize()
        cur.wait_event(copied[b])
        st = g.train_iteration(bufs[b], 1.0, stats=True)
        trained[b].record(cur)
        losses.append((st.mean_loss, st.dropped_samples))
    torch.cuda.synchronize()
    w = g.get_weights()
    g.close()
    return losses, w

a, wa = run(False)
b, wb = run(True)
same = a == b and np.array_equal(wa, wb)
print("event-ordered == synchronised:", same)
if not same:
    for k, (x, y) in enumerate(zip(a, b)):
        if x != y:
            print(k, x, y)
sys.exit(0 if same else 1)
