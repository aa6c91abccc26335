"""Distributed Newton-step solve (slab finest level + agglomerated coarse
levels + CGS2 GMRES) against the single-GPU solver.  The ranks are separate
processes on one GPU talking gloo (host-staged ghost exchange): the kernels of
different ranks never wait on each other, so sharing the device is safe."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import block_rel

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _problem(level, split):
    import bench
    return bench.baseline_inputs(2, level, split, seed=0, notch=True)


def _worker(rank, world, port, level, split, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import paper_2005_00331_b200 as P
        from paper_2005_00331_b200.distributed import DistributedGmg, distributed_gmres
        h, params, U, pt, act, dirn, x = _problem(level, split)
        n = h.dof_map(level).n_scalar
        dmask = np.zeros(n, dtype=bool)
        dmask[dirn] = True
        gmg = DistributedGmg(h, level, rank, world, coarse_level=2,
                             cheb=P.ChebyshevConfig(sweeps=3))
        gmg.setup(params, split, U, pt, pt, act, dmask)
        part = gmg.part
        rhs = x.copy()
        rhs[np.concatenate([dmask, dmask, act])] = 0.0
        rl = torch.from_numpy(part.scatter(rhs, rank, 3)).cuda()
        gmg.fine.halo.zero_ghosts(rl, 3)
        z = gmg(rl)
        zg = np.zeros(3 * n)
        part.gather_into(zg, z.cpu().numpy(), rank, 3)
        res = distributed_gmres(gmg, rl, P.KrylovConfig(relative_tolerance=1e-8, restart=50))
        xg = np.zeros(3 * n)
        part.gather_into(xg, res.solution.cpu().numpy(), rank, 3)
        out = torch.from_numpy(np.concatenate([zg, xg]))
        dist.all_reduce(out)
        if rank == 0:
            q.put(("ok", out.numpy(), res.iterations,
                   {L.level: L.ranges for L in gmg.lv}))
        dist.barrier()
        dist.destroy_process_group()
    except Exception:  # pragma: no cover
        import traceback
        q.put(("err", traceback.format_exc(), None, None))


@pytest.mark.parametrize("world,level,split", [(2, 6, "miehe"), (4, 7, "miehe"), (2, 7, "none"),
                                                (2, 8, "miehe"), (4, 8, "none")])
def test_distributed_newton_step_matches_single_gpu(world, level, split):
    """Slab levels: (2, 6) the finest only; (4, 7) / (2, 7) two; (2, 8) three
    (256^2 -> 128^2 -> 64^2 in slabs, 32^2 agglomerated); (4, 8) three (256^2 -> 64^2 at 16 rows per rank)."""
    import paper_2005_00331_b200 as P
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, level, split, q))
             for r in range(world)]
    for p in procs:
        p.start()
    status, out, iters, ranges = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
    assert status == "ok", out
    h, params, U, pt, act, dirn, x = _problem(level, split)
    st = P.LinearizationState(h, level, params, split=split)
    st.set_solution(U); st.set_phi_tilde(pt); st.set_phi_old(pt); st.set_active(act)
    st.set_dirichlet_nodes(dirn)
    st.refresh_cache()
    gmg = P.GmgPreconditioner(h, coarse_level=2, cheb=P.ChebyshevConfig(sweeps=3))
    gmg.setup(st)
    n = st.n_scalar
    expect_slabs = {(2, 6): 1, (4, 7): 2, (2, 7): 2, (2, 8): 3, (4, 8): 3}[(world, level)]
    assert len(ranges) == expect_slabs
    for l, rg in ranges.items():   # every slab level's Lanczos ranges
        for blk in ("uu", "phiphi"):
            assert np.allclose(rg[blk], gmg.ranges[l][blk], rtol=1e-10, atol=0), (l, blk)
    rhs = x.copy()
    rhs[st.constrained_mask()] = 0.0
    zg = out[:3 * n]
    assert max(block_rel(zg, gmg.apply(rhs), n)) <= 1e-12
    res = P.gmres_solve(P.JacobianOperator(st), rhs,
                        P.KrylovConfig(relative_tolerance=1e-8, restart=50),
                        preconditioner=gmg.apply)
    assert abs(iters - res.iterations) <= 1
    assert max(block_rel(out[3 * n:], res.solution, n)) <= 1e-7
