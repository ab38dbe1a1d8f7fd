#!/usr/bin/env python
"""bench.py — throughput of PVR's SR iteration (arXiv 1611.07289) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c3]

One step = one pvr_sr_iterate(1): forward simulate + residual + EM statistics, EM
parameters, E-step + patch weights, backprojection into (A, C), update + regulariser, over
every patch of the workload. Default workload: c3, the
whole-uterus configuration BASELINE.json's north_star quotes its target on.

Metric (BASELINE.json): PSF samples/s (value, whole job) and seconds per SR iteration
(ms_per_step), plus roofline fractions. Timing: W untimed warm-up steps, then exactly K steps
bracketed by barrier + cuda synchronize, CUDA events on the library's stream, max over ranks.
Inputs are larger than L2 (X 311 MB, A/C 623 MB, per-pixel arrays 577 MB at c3), so no
explicit flush is needed between iterations. For N > 1 launch with torchrun; patches are
sharded (strong scaling of a fixed workload) and (A, C) + EM statistics are allreduced.

--impl reference times the fp64 CPU oracle (oracle/, the "reference arm" of this tier) on a
bounded sample of the same workload on the host cores (rank 0 only under torchrun).
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "PSF samples/sec and s per SR iteration at 1/2/4/8 B200; % of HBM peak"
UNIT = "PSF samples/s"
# algorithmic FP32 FLOPs per PSF sample: forward = 3 (position) +
# 14 (trilinear, 7 lerps) + 2 (accumulate); adjoint = 3 + 12 (corner weights) + 16 (A and C)
# + 2 (scale)
FLOP_FWD, FLOP_ADJ = 19, 33


def peaks():
    p = {"hbm_gbs": 6538.6, "sm_max_mhz": 1965.0, "source": "fallback"}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            m = json.load(f)
        p.update(hbm_gbs=m["hbm_gbs"], sm_max_mhz=m.get("sm_max_mhz", 1965.0), source="measured")
    except Exception:
        pass
    # FP32 FFMA peak from the unit counts: 148 SMs x 128 FP32 lanes x 2 FLOP x max clock
    p["fp32_tflops"] = 148 * 128 * 2 * p["sm_max_mhz"] * 1e6 / 1e12
    return p


class Clocks:
    """nvidia-smi sampler running during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.Q,
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        self.lines = []
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            out, _ = self.proc.communicate(timeout=10)
            self.lines = [l for l in out.splitlines() if l.strip()]

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in getattr(self, "lines", []):
            f = [x.strip() for x in l.split(",")]
            try:
                sm.append(float(f[0]))
                mx = float(f[1])
            except ValueError:
                continue
            for n, v in zip(names, f[2:]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def dist_setup(n_gpus):
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws > 1 or n_gpus > 1:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        return ws, rank, local, dist
    return 1, 0, 0, None


# ---------------------------------------------------------------------------- reference arm
def oracle_sample(cfg, slices):
    """A bounded sample of workload `cfg` for the fp64 oracle: the same volume, stacks,
    PSF, patch layout and motion, but only `slices` slices per stack."""
    import synth
    c = synth.CONFIGS[cfg]
    return synth.make_problem(cfg, scale=(c["n"], c["W"], slices))


def time_oracle(cfg, steps, warmup, slices):
    import numpy as np
    import synth
    from oracle import Oracle
    slices = max(slices, synth.CONFIGS[cfg].get("depth", 1))  # 3D patches (c4) need >= depth slices
    prob = oracle_sample(cfg, slices)
    orc = Oracle(prob["dims"], prob["spacing"], prob["origin"])
    for st in prob["stacks"]:
        orc.add_stack(st["slices"], st["G"], st["thickness"])
    pp = prob["patch"]
    orc.extract_patches(pp["size"], pp["stride"], pp["depth"], pp["stride_z"])
    orc.set_transforms(prob["T"])
    orc.set_volume(np.full(orc.V, 300.0))
    _, kap, _, _ = orc.taps()
    S = len(orc.psf(0)[1])
    samples = int((kap >= 0.01).sum()) * S  # observed pixels (tau_obs = 0.01, Q25)
    for _ in range(warmup):
        orc.sr_iterate(1, prob["alpha"], prob["lam"])
    ts = []
    for _ in range(steps):
        t0 = time.perf_counter()
        orc.sr_iterate(1, prob["alpha"], prob["lam"])
        ts.append(time.perf_counter() - t0)
    t = statistics.mean(ts)
    cores = int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1))
    return dict(value=samples / t, unit=UNIT, cores=cores, kind="oracle", cpu_model=cpu_model(),
                sample=f"{cfg} with {slices} slice(s) per stack: M={orc.M} patches, "
                       f"{samples:.3e} observed PSF samples per iteration, full {prob['dims'][0]}^3 "
                       f"volume update; fp64, mean of {steps} iteration(s)",
                seconds_per_iteration=t)


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def config_block(cfg, prob=None, extra=None):
    import synth
    c = synth.CONFIGS[cfg]
    d = {"workload": c["name"], "config_id": cfg, "volume": [c["n"]] * 3, "spacing_mm": c["s"],
         "stacks": len(c["stacks"]), "stack_shape": [c["W"], c["W"], c["K"]],
         "patch": [c["size"], c["size"], c["depth"]], "stride": [c["stride"], c["stride"], c["stride_z"]],
         "l2_flush": "inputs larger than L2 (no explicit flush)"}
    if extra:
        d.update(extra)
    return d


def run_reference(args):
    ws, rank, _, _ = dist_setup(args.gpus)
    if rank != 0:
        return 0
    slices = args.ref_slices
    r = time_oracle(args.config, args.steps, args.warmup, slices)
    line = {"impl": "reference", "metric": METRIC, "value": r["value"], "unit": UNIT,
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": r["seconds_per_iteration"] * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded analytic phantom acquisition; synth/)",
            "config": config_block(args.config, extra={"reference_sample": r["sample"]}),
            "cpu_baseline": {k: r[k] for k in ("value", "unit", "cores", "kind", "sample", "cpu_model")},
            "e2e": {"value": r["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------- our arm
def run_ours(args):
    import numpy as np
    import torch

    import synth
    from paper_1611_07289_b200 import Context, load_problem, pvr

    ws, rank, local, dist = dist_setup(args.gpus)
    torch.cuda.set_device(local)
    if dist is not None:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    # a dedicated (non-NULL) torch stream: the library issues all work on it, and the timing
    # events below are recorded on the same stream
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    prob = synth.make_problem(args.config)
    ctx = Context(prob["dims"], prob["spacing"], prob["origin"], local, stream.cuda_stream)
    if ws > 1:
        # SURVEY 8(e) lever 3: reduce-scatter (A, C) over z slabs, slab update, all-gather X
        # (12 V (N-1)/N bytes per rank instead of the allreduce's 16 V (N-1)/N)
        ctx.set_param("exchange", pvr.EXCHANGE[args.exchange])
        uid = [pvr.pvr_comm_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        ctx.comm_init(ws, rank, uid[0])
    load_problem(ctx, prob, {"psf_quality": args.psf_quality} if args.psf_quality != 1 else None)
    ctx.init_volume()
    for _ in range(args.warmup):
        ctx.sr_iterate(1, prob["alpha"], prob["lam"])
    torch.cuda.synchronize()

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    # ---- timed region: K iterations, library-internal per-kernel events on the same stream
    ctx.set_param("profile", 1)
    ctx.reset_stats()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Clocks(local) as clk:
        barrier()
        ev0.record(stream)
        ctx.sr_iterate(args.steps, prob["alpha"], prob["lam"]) if args.one_call else \
            [ctx.sr_iterate(1, prob["alpha"], prob["lam"]) for _ in range(args.steps)]
        ev1.record(stream)
        barrier()
    ms = ev0.elapsed_time(ev1) / args.steps
    st = ctx.stats()
    ctx.set_param("profile", 0)
    ms_max = ms
    if dist is not None:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_max = float(t.item())
    samples = st["psf_samples"] / st["iterations"]          # global (all ranks) per iteration
    value = samples / (ms_max * 1e-3)

    # ---- roofline of the dominant kernel (average launch duration from the timed region)
    pk = peaks()
    kern = {
        "k_forward": (st["ms_forward"] / st["n_forward"], "alu", samples / ws * FLOP_FWD,
                      st["bytes_alg_forward"]),
        "k_backproject": (st["ms_backproject"] / st["n_backproject"], "alu", samples / ws * FLOP_ADJ,
                          st["bytes_alg_backproject"]),
        "k_update": (st["ms_update"] / st["n_update"], "hbm", None, st["bytes_alg_update"]),
        "k_estep": (st["ms_estep"] / st["n_estep"], "hbm", None, st["bytes_alg_estep"]),
    }
    name = max(kern, key=lambda k: kern[k][0])
    kms, bound, flops, bytes_alg = kern[name]
    traffic, counters = None, None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            tj = json.load(f)
        traffic = tj.get(args.config, {}).get(name)
        counters = tj.get(args.config + "_counters", {}).get(name)
    except Exception:
        pass
    if bound == "alu":
        ach = flops / (kms * 1e-3) / 1e12
        roof = {"kernel": name, "bound": "alu", "achieved": ach, "peak": pk["fp32_tflops"],
                "unit": "TFLOP/s", "frac": ach / pk["fp32_tflops"], "traffic": traffic,
                "peak_source": "FP32 FFMA: 148 SMs x 128 lanes x 2 x sm_max_mhz (DESIGN.md)",
                "ms_per_launch": kms, "flop_per_launch": flops}
        if counters:  # the limiters the kernel actually hits (ncu counts per launch / live time)
            fclk = pk["sm_max_mhz"] * 1e6
            roof["secondary"] = {
                "shared_lsu": {"achieved": counters["shared_wavefronts"] / (kms * 1e-3) / 1e9,
                               "peak": 148 * fclk / 1e9, "unit": "G wavefronts/s",
                               "frac": counters["shared_wavefronts"] / (kms * 1e-3) / (148 * fclk)},
                "issue": {"achieved": counters["warp_instructions"] / (kms * 1e-3) / 1e9,
                          "peak": 148 * 4 * fclk / 1e9, "unit": "G warp-instr/s",
                          "frac": counters["warp_instructions"] / (kms * 1e-3) / (148 * 4 * fclk)},
                "source": "ncu counts of one launch (profiles/ncu_traffic.json) over the live launch time"}
    else:
        ach = bytes_alg / (kms * 1e-3) / 1e9
        roof = {"kernel": name, "bound": "hbm", "achieved": ach, "peak": pk["hbm_gbs"],
                "unit": "GB/s", "frac": ach / pk["hbm_gbs"], "traffic": traffic,
                "peak_source": pk["source"], "ms_per_launch": kms, "bytes_per_launch": bytes_alg}
    breakdown = {k: {"ms": v[0], "share": v[0] / ms} for k, v in kern.items()}
    breakdown["em_params"] = {"ms": st["ms_em"] / st["n_em"], "share": st["ms_em"] / st["n_em"] / ms}
    if ws > 1:
        breakdown["allreduce_AC"] = {"ms": st["ms_allreduce"] / max(st["n_allreduce"], 1)}
    # iteration-level HBM fraction on SURVEY 8(d)'s B_alg = 24 P + 28 V + 48 M bytes (the fused
    # minimum per iteration), and, labelled apart, on the sum of the kernels' algorithmic bytes
    P_all = int(ctx.M) * prob["patch"]["size"] ** 2 * prob["patch"]["depth"]  # every window is full size
    V_all = int(st["voxels"])
    M_all = int(ctx.M)
    b_alg = 24 * P_all + 28 * V_all + 48 * M_all
    kernel_bytes = (st["bytes_alg_forward"] + st["bytes_alg_estep"] + st["bytes_alg_backproject"]
                    + st["bytes_alg_update"])
    hbm_iter = {"B_alg_bytes": b_alg, "frac": b_alg / (ms_max * 1e-3) / (pk["hbm_gbs"] * 1e9),
                "definition": "SURVEY 8(d): B_alg = 24 P + 28 V + 48 M bytes per iteration / t_iter / HBM peak",
                "kernel_bytes_sum": kernel_bytes,
                "kernel_bytes_frac": kernel_bytes / (ms * 1e-3) / (pk["hbm_gbs"] * 1e9)}
    plan = {k: st[k] for k in ("fwd_tile", "bp_tile", "fwd_groups", "bp_groups", "fwd_members", "bp_members",
                               "fwd_smem", "bp_smem", "bp_exact_groups", "fwd_split", "bp_split",
                               "device_replans", "host_replans", "replan_splits")}

    # ---- end to end through the C ABI with host buffers: per step the step's inputs (the
    # patch transforms from registration) go host -> device and the step's result metrics
    # (EM state: sigma^2, c, m, iteration, clamp range) come back, as a training step reads
    # back its loss; the volume itself is read once at the end (outside the steps)
    T_host = torch.from_numpy(np.ascontiguousarray(prob["T"].reshape(-1, 12))).pin_memory()
    e2e_steps = max(1, min(args.steps, 5))
    ctx.set_transforms(T_host)
    ctx.sr_iterate(1, prob["alpha"], prob["lam"])
    em_bytes = 6 * 8
    ctx.em_state()
    barrier()
    t0 = time.perf_counter()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(e2e_steps):
        ctx.set_transforms(T_host)
        ctx.sr_iterate(1, prob["alpha"], prob["lam"])
        ctx.em_state()
    e1.record(stream)
    barrier()
    e2e_ms = max(e0.elapsed_time(e1), (time.perf_counter() - t0) * 1e3) / e2e_steps
    if dist is not None:
        t = torch.tensor([e2e_ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    e2e = {"value": samples / (e2e_ms * 1e-3), "unit": UNIT, "ms_per_step": e2e_ms,
           "h2d_bytes_per_step": int(T_host.numel() * 8), "d2h_bytes_per_step": em_bytes,
           "calls": "pvr_set_transforms(host T) + pvr_sr_iterate(1) + pvr_get_em_state (host)"}
    # the same with the whole volume read back every step (311 MB at c3)
    X_host = torch.empty(prob["dims"][::-1], dtype=torch.float32).pin_memory()
    barrier()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    ev0.record(stream)
    for _ in range(e2e_steps):
        ctx.set_transforms(T_host)
        ctx.sr_iterate(1, prob["alpha"], prob["lam"])
        ctx.volume(X_host)
    ev1.record(stream)
    barrier()
    vol_ms = max(ev0.elapsed_time(ev1), (time.perf_counter() - t0) * 1e3) / e2e_steps
    e2e["with_volume_readback"] = {"ms_per_step": vol_ms, "d2h_bytes_per_step": int(X_host.numel() * 4)}

    # ---- f2 rigidity map: one pvr_rigidity_map call into a device buffer,
    # timed on the library's stream (one exact hi/lo backprojection + ratio + copy)
    R_dev = torch.empty(prob["dims"][::-1], dtype=torch.float32, device="cuda")
    ctx.rigidity_map(R_dev)  # builds the init plan once
    r0 = torch.cuda.Event(enable_timing=True)
    r1 = torch.cuda.Event(enable_timing=True)
    reps = 3
    r0.record(stream)
    for _ in range(reps):
        ctx.rigidity_map(R_dev)
    r1.record(stream)
    r1.synchronize()
    rig_ms = r0.elapsed_time(r1) / reps
    rigidity = {"ms_per_map": rig_ms, "psf_samples_per_s": samples / (rig_ms * 1e-3),
                "call": "pvr_rigidity_map(device out) after the timed iterations"}

    # ---- f1 rigid patch-to-volume registration: one pvr_register_patches
    # call (4 levels, <= 20 compass moves per level) of every patch against the current X
    torch.cuda.synchronize()
    t0r = time.perf_counter()
    _, reg_st, _ = ctx.register(levels=4, iters=20)
    reg_ms = (time.perf_counter() - t0r) * 1e3
    registration = {"ms_per_call": reg_ms, "patches": int(ctx.M), "patches_per_s": ctx.M / (reg_ms * 1e-3),
                    "registered": int((reg_st == 1).sum()),
                    "call": "pvr_register_patches(levels=4, iters=20), host outputs, wall clock"}

    # ---- f3 superpixel patches: SLIC on every slice of the same stacks
    # (S = 32 px, m = 20, 10 rounds, dilation 4 px), then one SR iteration on those patches
    superpixels = None
    if ws == 1 and not args.no_extras:
        sp = Context(prob["dims"], prob["spacing"], prob["origin"], local, stream.cuda_stream)
        for stk in prob["stacks"]:
            sp.add_stack(stk["slices"], stk["G"], stk["thickness"])
        torch.cuda.synchronize()
        t0s = time.perf_counter()
        Msp = sp.superpixel_patches(32, 20, 10, 4)
        sp_ms = (time.perf_counter() - t0s) * 1e3
        Tsp = np.tile(np.hstack([np.eye(3), np.zeros((3, 1))]), (Msp, 1, 1))
        sp.set_transforms(Tsp)
        sp.init_volume()
        sp.sr_iterate(1, prob["alpha"], prob["lam"])
        sp.reset_stats()
        s0 = torch.cuda.Event(enable_timing=True)
        s1 = torch.cuda.Event(enable_timing=True)
        s0.record(stream)
        sp.sr_iterate(3, prob["alpha"], prob["lam"])
        s1.record(stream)
        s1.synchronize()
        sst = sp.stats()
        it_ms = s0.elapsed_time(s1) / 3
        superpixels = {"ms_extract": sp_ms, "patches": int(Msp), "ms_per_iteration": it_ms,
                       "psf_samples_per_s": sst["psf_samples"] / 3 / (it_ms * 1e-3),
                       "call": "pvr_superpixel_patches(S=32, m=20, iters=10, gamma=4) (wall clock), "
                               "then pvr_sr_iterate on those patches (CUDA events)"}
        sp.close()
    ctx.close()

    line = None
    if rank == 0:
        cpu = None
        if ws == 1 and not args.no_cpu_baseline:
            r = time_oracle(args.config, 1, 0, args.ref_slices)
            cpu = {k: r[k] for k in ("value", "unit", "cores", "kind", "sample", "cpu_model")}
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_max, "s_per_iteration": ms_max * 1e-3,
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
                "data": "synthetic (seeded analytic phantom acquisition; synth/)",
                "config": config_block(args.config, extra={
                    "M": int(ctx.M), "P": int(st["pixels"]) if ws == 1 else None,
                    "psf_samples_per_iteration": samples,
                    "parallelism": f"patch-shard x{ws}" + (f", exchange {args.exchange}" if ws > 1 else ""),
                    "psf_quality": args.psf_quality}),
                "roofline": roof, "iteration_hbm": hbm_iter, "plan": plan,
                "kernels": breakdown, "clocks": clk.summary(), "e2e": e2e,
                "gpu_launches": int(st["kernel_launches"]), "cpu_baseline": cpu,
                "extras": {"f2_rigidity_map": rigidity, "f1_registration": registration,
                           "f3_superpixels": superpixels}}
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c3", choices=["c1", "c2", "c3", "c4", "c5"])
    ap.add_argument("--ref-slices", type=int, default=1,
                    help="slices per stack of the oracle's bounded sample")
    ap.add_argument("--one-call", action="store_true", help="time one pvr_sr_iterate(K) call")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="skip the f3 superpixel measurement")
    ap.add_argument("--exchange", default="slabs", choices=["allreduce", "slabs"],
                    help="multi-GPU (A, C) exchange (PVR_PARAM_EXCHANGE); default slabs")
    ap.add_argument("--psf-quality", type=float, default=1.0,
                    help="f4 PSF lattice density q (2 = the q = 2 quality mode); default 1")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        print("warning: --warmup < 3 violates the timing rules", file=sys.stderr)
    return run_reference(args) if args.impl == "reference" else run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
