"""Print the lattice-kernel plans and per-kernel times for a config (GPU).

  python tools/plan_info.py CFG ['{"scale": [96, 96, 12], ...}'] ['{"bp_exact": 0, ...}']
"""
import json
import sys
import time

sys.path.insert(0, "."); sys.path.insert(0, "tests")
import synth  # noqa: E402
from helpers import make_gpu  # noqa: E402

cfg = sys.argv[1]
kw = json.loads(sys.argv[2]) if len(sys.argv) > 2 else {}
params = json.loads(sys.argv[3]) if len(sys.argv) > 3 else {}
if "scale" in kw:
    kw["scale"] = tuple(kw["scale"])
prob = synth.make_problem(cfg, **kw)
ctx = make_gpu(prob, dict(params, profile=1))
ctx.init_volume()
ctx.sr_iterate(2, 1.0, 0.02)
ctx.reset_stats()
n = 5
ctx.sr_iterate(n, 1.0, 0.02)
s = ctx.stats()
print(cfg, params, {k: s[k] for k in ("fwd_tile", "bp_tile", "fwd_groups", "bp_groups", "fwd_members", "bp_members",
                                      "fwd_smem", "bp_smem")})
print("ms/iter", {k: round(s[k] / n, 3) for k in ("ms_forward", "ms_backproject", "ms_update", "ms_estep", "ms_em")})
for _ in range(2):
    t0 = time.perf_counter()
    ctx.set_transforms(prob["T"])
    t1 = time.perf_counter()
    print("set_transforms %.1f ms" % ((t1 - t0) * 1e3))
s = ctx.stats()
print("replans device/host", s["device_replans"], s["host_replans"])
