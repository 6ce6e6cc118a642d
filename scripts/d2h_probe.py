"""D2H of 630 MB: fresh np.empty vs pre-touched vs pinned destination (decompose e2e)."""
import time

import numpy as np
import torch

n = 630_000_000
d = torch.empty(n, dtype=torch.uint8, device="cuda")
d.fill_(7)
torch.cuda.synchronize()
for label in ("fresh", "touched", "pinned"):
    ts = []
    for _ in range(3):
        if label == "pinned":
            h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
        else:
            h = torch.from_numpy(np.empty(n, dtype=np.uint8))
            if label == "touched":
                h.numpy()[::4096] = 0
        t0 = time.perf_counter()
        h.copy_(d)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    print(label, "%.1f ms -> %.1f GB/s" % (min(ts) * 1e3, n / min(ts) / 1e9), flush=True)
