"""Slab decomposition: partition bookkeeping on CPU, the
ghost-row exchange and the distributed operator/dot over gloo with world
size 2 and 4 (the local cell kernel replaced by the C oracle on CPU), and the
slab-window CUDA kernel against the whole-mesh kernel on one GPU."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import block_rel
from oracle import oracle as O
from paper_2005_00331_b200 import _lib
from paper_2005_00331_b200.parallel import HaloExchange, SlabPartition, SlabState, owned_dot


@pytest.mark.parametrize("world", [1, 2, 4, 8])
@pytest.mark.parametrize("p,level", [(2, 4), (2, 6), (1, 5), (3, 4)])
def test_partition_covers_every_node_once(world, p, level):
    part = SlabPartition(p, level, world)
    count = np.zeros(part.n, dtype=np.int64)
    for r in range(world):
        idx = part.local_index(r)
        assert idx.size == part.local_n(r)
        count[idx[part.owned_mask(r)]] += 1
        lo, hi = part.rows(r)
        olo, ohi = part.own_rows(r)
        assert lo <= olo < ohi <= hi + 1
        if r > 0:
            assert olo - lo == p            # p ghost rows below
        if r < world - 1:
            assert hi == ohi                 # one ghost row above
    assert np.all(count == 1)
    # the slit copies belong to exactly one rank, the one owning row i_mid
    owners = [r for r in range(world) if part.owns_dup(r)]
    assert len(owners) == 1


def test_partition_rejects_bad_worlds():
    with pytest.raises(ValueError):
        SlabPartition(2, 4, 3)
    with pytest.raises(ValueError):
        SlabPartition(2, 2, 4)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


class OracleSlab(SlabState):
    """SlabState whose local cell kernel is the C oracle (CPU test double):
    the local slab (owned + ghost rows) is embedded in a zero global vector,
    the whole-mesh oracle operator applied, and the owned rows kept -- so the
    owned rows near the slab edges are right only if the ghosts are."""

    def __init__(self, ost, *a, **k):
        super().__init__(*a, **k)
        self.ost = ost

    def _local_apply(self, mode, src, dst, rhs):
        part, n = self.part, self.part.n
        idx = part.local_index(self.rank)
        ln = idx.size
        ncomp_in = {0: 3, 1: 2, 2: 1, 3: 3}[mode]
        g = np.zeros(3 * n)
        comps = {0: (0, 1, 2), 1: (0, 1), 2: (2,), 3: (0, 1, 2)}[mode]
        s = src.numpy()
        for k, c in enumerate(comps):
            g[c * n + idx] = s[k * ln:(k + 1) * ln]
        fn = {0: O.apply_jacobian, 1: lambda st, v: O.apply_block_uu(st, v[:2 * n]),
              2: lambda st, v: O.apply_block_phiphi(st, v[2 * n:]), 3: O.apply_phi_row}[mode]
        out = fn(self.ost, g)
        own = part.owned_mask(self.rank)
        d = dst.numpy()
        ncomp_out = {0: 3, 1: 2, 2: 1, 3: 1}[mode]
        for k in range(ncomp_out):
            loc = out[k * n + idx]
            blk = d[k * ln:(k + 1) * ln]
            blk[own] = loc[own]
            if rhs is not None:
                blk[own] = rhs.numpy()[k * ln:(k + 1) * ln][own] - loc[own]


def _worker(rank, world, port, level, split, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        part = SlabPartition(2, level, world)
        ost, x = O.baseline_state(2, level, split, seed=3)
        ost.refresh_cache()
        cpu = torch.device("cpu")
        st = OracleSlab(ost, part, rank, ost.params, split, ost.U, ost.phi_tilde, ost.active,
                        ost.dirichlet, device=cpu)
        n, ln = part.n, part.local_n(rank)
        own = np.tile(part.owned_mask(rank), 3)
        # 1. ghost exchange: start from owned values only, ghosts must arrive
        full = torch.from_numpy(part.scatter(x, rank, 3))
        v = torch.where(torch.from_numpy(own), full, torch.zeros((), dtype=torch.float64))
        st.halo.exchange(v, 3)
        lo, hi = part.rows(rank)
        grid_part = np.tile(np.r_[np.ones((hi - lo + 1) * part.np1, bool),
                                  np.zeros(ln - (hi - lo + 1) * part.np1, bool)], 1)
        for c in range(3):
            blk = slice(c * ln, c * ln + (hi - lo + 1) * part.np1)
            assert torch.equal(v[blk], full[blk]), ("ghost rows", rank, c)
        # 2. distributed operator, every mode, plain and fused
        results = {}
        for mode, nin, nout in ((0, 3, 3), (1, 2, 2), (2, 1, 1), (3, 3, 1)):
            comps = {0: (0, 1, 2), 1: (0, 1), 2: (2,), 3: (0, 1, 2)}[mode]
            src = torch.cat([torch.from_numpy(part.scatter(x[c * n:(c + 1) * n], rank, 1))
                             * torch.from_numpy(part.owned_mask(rank)).double() for c in comps])
            dst = st.empty(nout)
            st.apply_into(mode, src, dst)
            glob = np.zeros(nout * n)
            part.gather_into(glob, dst.numpy(), rank, nout)
            t = torch.from_numpy(glob)
            dist.all_reduce(t)
            results[mode] = t.numpy()
        # 3. distributed dot over owned entries
        xl = torch.from_numpy(part.scatter(x, rank, 3))
        dot = owned_dot(part, rank, xl, xl, 3)
        if rank == 0:
            q.put(("ok", results, dot))
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover - reported to the parent
        import traceback
        q.put(("err", traceback.format_exc(), None))


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("split", ["miehe", "none"])
def test_gloo_distributed_operator(world, split):
    level = 4
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, level, split, q))
             for r in range(world)]
    for pr in procs:
        pr.start()
    status, results, dot = q.get(timeout=300)
    for pr in procs:
        pr.join(timeout=60)
    assert status == "ok", results
    ost, x = O.baseline_state(2, level, split, seed=3)
    ost.refresh_cache()
    n = ost.n
    want = {0: O.apply_jacobian(ost, x), 1: O.apply_block_uu(ost, x[:2 * n]),
            2: O.apply_block_phiphi(ost, x[2 * n:]), 3: O.apply_phi_row(ost, x)}
    for mode, w in want.items():
        assert max(block_rel(results[mode], w, n)) <= 1e-14, mode
    assert dot == pytest.approx(float(x @ x), rel=1e-13)


@pytest.mark.gpu
@pytest.mark.parametrize("split", ["miehe", "none"])
@pytest.mark.parametrize("world,level", [(2, 8), (4, 9), (8, 9)])
def test_slab_window_kernel_matches_whole_mesh(split, world, level):
    """Emulate the ranks one after another on one GPU (ghosts taken from the
    global arrays): owned rows of every slab == the whole-mesh application."""
    import paper_2005_00331_b200 as P
    ost, x = O.baseline_state(2, level, split, seed=4)
    h = P.build_hierarchy(level, 2)
    gst = P.LinearizationState(h, level, ost.params, split=split)
    gst.set_solution(ost.U)
    gst.set_phi_tilde(ost.phi_tilde)
    gst.set_active(ost.active)
    gst.set_dirichlet_nodes(np.flatnonzero(ost.dirichlet))
    gst.refresh_cache()
    n = gst.n_scalar
    part = SlabPartition(2, level, world)
    rhs = np.random.default_rng(2).standard_normal(3 * n)
    for mode, nin, nout in ((0, 3, 3), (1, 2, 2), (2, 1, 1), (3, 3, 1)):
        comps = {0: (0, 1, 2), 1: (0, 1), 2: (2,), 3: (0, 1, 2)}[mode]
        xin = np.concatenate([x[c * n:(c + 1) * n] for c in comps])
        xd = torch.from_numpy(xin).cuda()
        want = torch.empty(nout * n, dtype=torch.float64, device="cuda")
        gst.apply_into(mode, xd, want)
        wantf = torch.empty_like(want)
        rhd = torch.from_numpy(rhs[:nout * n]).cuda()
        gst.apply_into(mode, xd, wantf, rhd)
        got = np.zeros(nout * n)
        gotf = np.zeros(nout * n)
        for r in range(world):
            st = SlabState(part, r, ost.params, split, ost.U, ost.phi_tilde, ost.active,
                           ost.dirichlet)
            st.refresh_cache()
            src = torch.from_numpy(part.scatter(xin, r, nin)).cuda()
            dst = st.empty(nout)
            st.apply_into(mode, src, dst, exchange=False)
            part.gather_into(got, dst.cpu().numpy(), r, nout)
            rl = torch.from_numpy(part.scatter(rhs[:nout * n], r, nout)).cuda()
            st.apply_into(mode, src, dst, rl, exchange=False)
            part.gather_into(gotf, dst.cpu().numpy(), r, nout)
        assert max(block_rel(got, want.cpu().numpy(), n)) <= 1e-15, mode
        assert max(block_rel(gotf, wantf.cpu().numpy(), n)) <= 1e-15, mode


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 8])
def test_overlapped_slab_decomposition_bitwise(world):
    """The NCCL path of SlabState.apply_into runs the interior cell rows while
    the ghost rows are in flight, then the two boundary rows: the three
    pff_apply_rows launches must give exactly the single-launch result."""
    import paper_2005_00331_b200 as P
    from paper_2005_00331_b200._lib import call, ptr, stream_handle
    level = 7
    ost, x = O.baseline_state(2, level, "miehe", seed=6)
    part = SlabPartition(2, level, world)
    rhs = np.random.default_rng(3).standard_normal(3 * ost.n)
    for r in range(world):
        st = SlabState(part, r, ost.params, "miehe", ost.U, ost.phi_tilde, ost.active,
                       ost.dirichlet)
        st.refresh_cache()
        src = torch.from_numpy(part.scatter(x, r, 3)).cuda()
        rl = torch.from_numpy(part.scatter(rhs, r, 3)).cuda()
        c0, c1 = part.cells(r)
        for fused in (None, rl):
            want = st.empty(3)
            st.apply_into(0, src, want, fused, exchange=False)
            got = st.empty(3)
            h = st.handle()
            for a, b in ((c0 + 1, c1 - 1), (c0, c0 + 1), (c1 - 1, c1)):
                call("pff_apply_rows", h, 0, ptr(src), ptr(got), ptr(fused), a, b, stream_handle())
            own = torch.from_numpy(np.tile(part.owned_mask(r), 3)).cuda()
            assert torch.equal(got[own], want[own])


def _restrict_worker(rank, world, port, p, level, q):
    """Slab -> slab restriction on CPU: each rank restricts its OWNED fine rows
    (the oracle's P^T with the other rows zeroed) into its coarse window, the
    reverse ghost-row sum completes the boundary rows; then the forward
    exchange + prolongation of the coarse window into the owned fine rows."""
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_2005_00331_b200.parallel import HaloExchange
        pf, pc = SlabPartition(p, level, world), SlabPartition(p, level - 1, world)
        T = O.Transfer(p, level)
        rng = np.random.default_rng(7)
        y = rng.uniform(-1, 1, 3 * pf.n)
        # restriction of the owned fine entries only
        own_f = np.zeros(pf.n, bool)
        own_f[pf.local_index(rank)[pf.owned_mask(rank)]] = True
        part_glob = T.restrict(np.where(np.tile(own_f, 3), y, 0.0))
        # the window must hold every nonzero partial: nothing outside it, zero
        # on its bottom ghost rows
        idx_c = pc.local_index(rank)
        inwin = np.zeros(pc.n, bool)
        inwin[idx_c] = True
        assert np.all(part_glob.reshape(3, pc.n)[:, ~inwin] == 0.0)
        loc = torch.from_numpy(pc.scatter(part_glob, rank, 3))
        lo, _ = pc.rows(rank)
        olo, _ = pc.own_rows(rank)
        lnc = pc.local_n(rank)
        for c in range(3):
            assert torch.all(loc[c * lnc:c * lnc + (olo - lo) * pc.np1] == 0.0)
        halo = HaloExchange(pc, rank)
        halo.reverse_add(loc, 3)
        rc = np.zeros(3 * pc.n)
        pc.gather_into(rc, loc.numpy(), rank, 3)
        t = torch.from_numpy(rc)
        dist.all_reduce(t)
        # prolongation from the coarse window (after the forward exchange)
        xc = rng.uniform(-1, 1, 3 * pc.n)
        own_c = torch.from_numpy(np.tile(pc.owned_mask(rank), 3))
        zc = torch.where(own_c, torch.from_numpy(pc.scatter(xc, rank, 3)),
                         torch.zeros((), dtype=torch.float64))
        halo.exchange(zc, 3)
        full_c = np.zeros(3 * pc.n)
        for c in range(3):
            full_c[c * pc.n + idx_c] = zc.numpy()[c * lnc:(c + 1) * lnc]
        pz = T.prolongate(full_c)
        zf = np.zeros(3 * pf.n)
        pf.gather_into(zf, pf.scatter(pz, rank, 3), rank, 3)
        tz = torch.from_numpy(zf)
        dist.all_reduce(tz)
        if rank == 0:
            q.put(("ok", t.numpy(), tz.numpy()))
        dist.barrier()
        dist.destroy_process_group()
    except Exception:  # pragma: no cover - reported to the parent
        import traceback
        q.put(("err", traceback.format_exc(), None))


@pytest.mark.parametrize("world,p,level", [(2, 2, 5), (4, 2, 5), (4, 1, 6), (2, 4, 4)])
def test_gloo_slab_to_slab_transfers(world, p, level):
    """The slab V-cycle's transfers (distributed.py): restriction of the owned
    fine rows into the coarse window + reverse ghost-row sum == P^T y, and
    prolongation from an exchanged coarse window == P x on the owned fine rows
    (src/multigrid.py:97-120)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_restrict_worker, args=(r, world, port, p, level, q))
             for r in range(world)]
    for pr in procs:
        pr.start()
    status, rc, zf = q.get(timeout=300)
    for pr in procs:
        pr.join(timeout=60)
    assert status == "ok", rc
    T = O.Transfer(p, level)
    rng = np.random.default_rng(7)
    y = rng.uniform(-1, 1, 3 * T.nf)
    xc = rng.uniform(-1, 1, 3 * T.nc)
    want = T.restrict(y)
    assert np.max(np.abs(rc - want)) <= 1e-13 * np.max(np.abs(want))
    wz = T.prolongate(xc)
    assert np.max(np.abs(zf - wz)) <= 1e-14 * np.max(np.abs(wz))
