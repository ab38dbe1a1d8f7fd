"""Multi-rank semantics on CPU (world size 2, gloo): the product's shard plan
(pvr_plan_shards, host-only) partitions the patches; each rank backprojects its shard and
computes its EM sufficient statistics with the oracle; SUM / MAX allreduces over gloo must
reproduce the single-rank result (P:233 with reading Q21: sum-allreduce, not averaging)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import synth


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _problem():
    return synth.make_problem("c3", scale=(40, 40, 6), size=16, stride=8)


def _oracle(prob):
    from oracle import Oracle
    orc = Oracle(prob["dims"], prob["spacing"], prob["origin"])
    for st in prob["stacks"]:
        orc.add_stack(st["slices"], st["G"], st["thickness"])
    pp = prob["patch"]
    orc.extract_patches(pp["size"], pp["stride"], pp["depth"], pp["stride_z"])
    orc.set_transforms(prob["T"])
    return orc


def _stats(e, live, p):
    """EM sufficient statistics of SURVEY 8(c) step 5 over one pixel subset."""
    m = live.astype(bool)
    if not m.any():
        return np.array([0.0, 0.0, 0.0]), np.array([-np.inf, -np.inf])
    return (np.array([(p[m] * e[m] ** 2).sum(), p[m].sum(), float(m.sum())]),
            np.array([e[m].max(), -e[m].min()]))


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1611_07289_b200 import pvr_plan_shards
    prob = _problem()
    orc = _oracle(prob)
    pt = orc.patches()
    S = len(orc.psf(0)[1])
    cost = (pt[:, 4] * pt[:, 5] * pt[:, 6]).astype(np.int64) * S
    bounds = pvr_plan_shards(cost, world)
    first, last = int(bounds[rank]), int(bounds[rank + 1])
    rng = np.random.default_rng(17)
    r = rng.normal(size=orc.P)
    e = rng.normal(0, 30, size=orc.P)
    p = rng.uniform(0, 1, size=orc.P)
    _, kap = orc.forward(np.zeros(orc.V))
    live = (kap >= 0.99).astype(np.uint8)
    pix0 = np.concatenate([[0], np.cumsum(pt[:, 4] * pt[:, 5] * pt[:, 6])])
    j0, j1 = pix0[first], pix0[last]
    # C2: backprojection of this rank's patches, SUM-allreduced
    part = torch.from_numpy(orc.adjoint(r, first, last - first).ravel())
    dist.all_reduce(part, op=dist.ReduceOp.SUM)
    # C1: EM statistics over this rank's pixels, SUM (3) and MAX (2)
    s, mx = _stats(e[j0:j1], live[j0:j1], p[j0:j1])
    ts, tm = torch.from_numpy(s), torch.from_numpy(mx)
    dist.all_reduce(ts, op=dist.ReduceOp.SUM)
    dist.all_reduce(tm, op=dist.ReduceOp.MAX)
    if rank == 0:
        full = orc.adjoint(r).ravel()
        s_all, mx_all = _stats(e, live, p)
        out.put((float(np.abs(part.numpy() - full).max() / np.abs(full).max()),
                 float(np.abs(ts.numpy() - s_all).max() / np.abs(s_all).max()),
                 float(np.abs(tm.numpy() - mx_all).max()), list(map(int, bounds))))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_sharded_reductions_match_single_rank(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = q.get(timeout=300)
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    d_ac, d_stats, d_max, bounds = res
    assert bounds[0] == 0 and bounds[-1] > bounds[1] > 0
    assert d_ac <= 1e-12 and d_stats <= 1e-12 and d_max == 0.0
