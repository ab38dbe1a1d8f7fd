"""Where the end-to-end step's time goes besides the iteration (bench.py e2e): times
pvr_set_transforms (host T) alone and an iteration after it vs a steady-state iteration, with
PVR_TRACE=1 printing the synced phase marks of set_transforms to stderr.

  PVR_TRACE=1 python tools/time_set_transforms.py [c3]
"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
from paper_1611_07289_b200 import Context, load_problem  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
prob = synth.make_problem(cfg)
ctx = Context(prob["dims"], prob["spacing"], prob["origin"], 0)
load_problem(ctx, prob)
ctx.init_volume()
ctx.sr_iterate(1, prob["alpha"], prob["lam"])
T = torch.from_numpy(np.ascontiguousarray(prob["T"].reshape(-1, 12))).pin_memory()
torch.cuda.synchronize()


def timed(fn, n=3):
    out = []
    for _ in range(n):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        out.append((time.perf_counter() - t0) * 1e3)
    return min(out), float(np.median(out))


print("set_transforms           min %.2f  median %.2f ms" % timed(lambda: ctx.set_transforms(T)), flush=True)
print("iteration (steady)       min %.2f  median %.2f ms" % timed(lambda: ctx.sr_iterate(1, prob["alpha"], prob["lam"])),
      flush=True)


def step():
    ctx.set_transforms(T)
    ctx.sr_iterate(1, prob["alpha"], prob["lam"])


print("set_transforms + iter    min %.2f  median %.2f ms" % timed(step), flush=True)
ctx.close()
