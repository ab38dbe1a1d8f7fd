"""Per-orientation cost of the lattice kernels: c3 with all four stacks of one orientation
(ax / cor / sag), two iterations, for an ncu counter pass over the forward and backprojection
(shared-memory wavefronts per load / atomic by stack orientation).

  ncu --metrics ... -k regex:k_lattice python tools/orient_counters.py ax
"""
import sys

sys.path.insert(0, "."); sys.path.insert(0, "tests")
import synth  # noqa: E402
from helpers import make_gpu  # noqa: E402

tag = sys.argv[1]
prob = synth.make_problem("c3", stacks=[(tag, 0.0), (tag, 1.0), (tag, 2.0), (tag, 3.0)])
ctx = make_gpu(prob, {"profile": 1})
ctx.init_volume()
ctx.sr_iterate(2, 1.0, 0.02)
s = ctx.stats()
print(tag, {k: s[k] for k in ("fwd_tile", "bp_tile", "fwd_groups", "bp_groups")},
      {k: round(s[k] / 2, 3) for k in ("ms_forward", "ms_backproject")}, flush=True)
ctx.close()
