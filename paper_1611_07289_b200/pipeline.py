"""The PVR reconstruction loop over the C ABI (orchestration only: every step runs in the
library's kernels). P:157-158: "individual 2D patches are continuously rigidly
registered to the current 3D reconstruction of X and reintegrated into X using iterative
super-resolution"; P:147-153 (Eq. 4): patch scales may change per outer iteration.

    ctx = Context(dims, spacing_mm, origin_mm)
    for slices, G, thickness in stacks: ctx.add_stack(slices, G, thickness)
    ctx.extract_patches(64, 32)                       # or superpixel / explicit patches
    X, T, log = reconstruct(ctx, T0, outer=3, inner=5)
"""
import numpy as np


def reconstruct(ctx, T0, outer=3, inner=5, alpha=1.0, lam=0.02, register=True, levels=4,
                iters=20, schedule=None, init=True):
    """Run the PVR loop on a context whose patches are extracted.

    T0: [M][3][4] initial patch transforms. Each outer round runs `inner` SR iterations, then
    (when `register`) rigid patch-to-volume registration of every patch against the current X
    (pvr_register_patches, `levels` x `iters`) and installs the new transforms. `schedule`:
    optional list of callables, one per outer round, each re-extracting the patches of the
    context (f3 multi-scale: e.g. lambda c: c.superpixel_patches(S_i, m, 10, gamma_i)) and
    returning the new initial transforms for them (identity-relative: [M][3][4]); the volume
    carries over. Returns (X, T, log) with the per-round EM state and registration counts."""
    T = np.asarray(T0, np.float64).reshape(-1, 3, 4)
    ctx.set_transforms(T)
    if init:
        ctx.init_volume()
    log = []
    for r in range(outer):
        if schedule is not None and r < len(schedule) and schedule[r] is not None:
            T = np.asarray(schedule[r](ctx), np.float64).reshape(-1, 3, 4)
            ctx.set_transforms(T)
        ctx.sr_iterate(inner, alpha, lam)
        entry = {"round": r, "em": ctx.em_state()}
        if register:
            T, status, _ = ctx.register(levels, iters)
            ctx.set_transforms(T)
            entry["registered"] = int((status == 1).sum())
        log.append(entry)
    return ctx.volume(), T, log
