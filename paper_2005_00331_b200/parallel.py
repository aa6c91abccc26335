"""Cell-row slab decomposition across GPUs.

One process per GPU.  Rank g owns cell rows [r_g, r_{g+1}) of the 2^l x 2^l
mesh and the node rows [p r_g, p r_{g+1}) (the top rank also node row p 2^l);
the owner of node row i_mid = p 2^l / 2 owns the upper slit copies too.  To
write its rows exactly once, a rank recomputes the cell row r_g - 1 below its
slab, so it holds LOCAL vectors with node rows [p (r_g - 1), p r_{g+1}]:
p ghost rows below (owned by rank g-1) and one ghost row above (owned by
rank g+1), followed by the slit copies when row i_mid is in range (the
layout of ``pff_level_set_window``, include/pff_b200.h).

Before every operator application the ghost rows of the source vector are
exchanged with the two neighbours (torch.distributed point-to-point: NCCL on
GPUs, gloo in the CPU tests); dot products are local sums over owned rows
followed by one all-reduce.  There is no other data-path collective.

The reference has no parallel path; the partition follows
the paper's distributed setting restricted to slabs.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist

from . import _lib
from ._lib import call, ptr, stream_handle
from .basis import MaterialParams, shape_data


@dataclass(frozen=True)
class SlabPartition:
    """Equal cell-row slabs of one mesh level over ``world`` ranks."""

    degree: int
    level: int
    world: int

    def __post_init__(self):
        ns = 2 ** self.level
        if self.world < 1 or self.world & (self.world - 1) or ns % self.world:
            raise ValueError("world size must be a power of two dividing 2^level")
        if self.world > 1 and ns // self.world < 2:
            raise ValueError("each slab needs at least two cell rows")

    # -- geometry ---------------------------------------------------------------
    @property
    def nside(self) -> int:
        return 2 ** self.level

    @property
    def np1(self) -> int:
        return self.degree * self.nside + 1

    @property
    def n_grid(self) -> int:
        return self.np1 * self.np1

    @property
    def i_mid(self) -> int:
        return self.degree * self.nside // 2

    @property
    def n_dup(self) -> int:
        return self.i_mid if self.level >= 1 else 0

    @property
    def n(self) -> int:
        return self.n_grid + self.n_dup

    def cells(self, rank: int):
        ns, w = self.nside, self.world
        return rank * ns // w, (rank + 1) * ns // w

    def rows(self, rank: int):
        """(j_lo, j_hi) local node rows incl. ghosts, inclusive."""
        c0, c1 = self.cells(rank)
        return self.degree * max(c0 - 1, 0), self.degree * c1

    def own_rows(self, rank: int):
        """[lo, hi) node rows owned by the rank."""
        c0, c1 = self.cells(rank)
        hi = self.degree * c1 + (1 if c1 == self.nside else 0)
        return self.degree * c0, hi

    def has_dup(self, rank: int) -> bool:
        lo, hi = self.rows(rank)
        return self.n_dup > 0 and lo <= self.i_mid <= hi

    def owns_dup(self, rank: int) -> bool:
        lo, hi = self.own_rows(rank)
        return self.n_dup > 0 and lo <= self.i_mid < hi

    def local_n(self, rank: int) -> int:
        lo, hi = self.rows(rank)
        return (hi - lo + 1) * self.np1 + (self.n_dup if self.has_dup(rank) else 0)

    # -- global <-> local (host arrays; setup and tests) ---------------------------
    def local_index(self, rank: int) -> np.ndarray:
        """Global scalar ids of the local entries, in local order."""
        lo, hi = self.rows(rank)
        idx = np.arange(lo * self.np1, (hi + 1) * self.np1, dtype=np.int64)
        if self.has_dup(rank):
            idx = np.concatenate([idx, self.n_grid + np.arange(self.n_dup, dtype=np.int64)])
        return idx

    def owned_mask(self, rank: int) -> np.ndarray:
        """Mask over the local entries: True where this rank owns the node."""
        lo, hi = self.rows(rank)
        olo, ohi = self.own_rows(rank)
        rows = np.repeat(np.arange(lo, hi + 1), self.np1)
        m = (rows >= olo) & (rows < ohi)
        if self.has_dup(rank):
            m = np.concatenate([m, np.full(self.n_dup, self.owns_dup(rank))])
        return m

    def scatter(self, glob: np.ndarray, rank: int, ncomp: int) -> np.ndarray:
        idx = self.local_index(rank)
        return np.concatenate([glob[c * self.n + idx] for c in range(ncomp)])

    def gather_into(self, glob: np.ndarray, local: np.ndarray, rank: int, ncomp: int):
        idx = self.local_index(rank)
        own = self.owned_mask(rank)
        ln = idx.size
        for c in range(ncomp):
            glob[c * self.n + idx[own]] = local[c * ln:(c + 1) * ln][own]


class HaloExchange:
    """Ghost-row exchange of a local slab vector with the two neighbours."""

    def __init__(self, part: SlabPartition, rank: int, group=None):
        self.part, self.rank, self.group = part, rank, group
        p, np1 = part.degree, part.np1
        lo, hi = part.rows(rank)
        olo, ohi = part.own_rows(rank)
        self.ln = part.local_n(rank)
        # (peer, local row range [a, b)) to send / receive, per component
        self.sends, self.recvs = [], []
        if rank > 0:
            self.recvs.append((rank - 1, lo, olo))            # p ghost rows below
            self.sends.append((rank - 1, olo, olo + 1))       # my bottom row -> their ghost above
        if rank < part.world - 1:
            self.recvs.append((rank + 1, hi, hi + 1))         # 1 ghost row above
            self.sends.append((rank + 1, ohi - p, ohi))       # my top p rows -> their ghosts below
        self.lo, self.np1 = lo, np1

    def zero_ghosts(self, vec: torch.Tensor, ncomp: int):
        """Zero the ghost rows and a non-owned slit-copy segment, so local dots
        over the whole local vector are owned dots."""
        part, rank = self.part, self.rank
        if part.world == 1:
            return
        dup0 = (part.rows(rank)[1] - self.lo + 1) * self.np1
        for c in range(ncomp):
            for _, a, b in self.recvs:
                self._view(vec, c, a, b).zero_()
            if part.has_dup(rank) and not part.owns_dup(rank):
                vec[c * self.ln + dup0:(c + 1) * self.ln].zero_()

    def _view(self, vec: torch.Tensor, comp: int, a: int, b: int) -> torch.Tensor:
        base = comp * self.ln
        return vec[base + (a - self.lo) * self.np1: base + (b - self.lo) * self.np1]

    def overlappable(self, vec: torch.Tensor) -> bool:
        """True when the exchange runs asynchronously on the device (NCCL)."""
        return (self.part.world > 1 and vec.is_cuda
                and dist.get_backend(self.group) != "gloo")

    def start(self, vec: torch.Tensor, ncomp: int) -> "_PendingHalo":
        """Post the ghost-row sends/receives (NCCL), one packed message per
        neighbour and direction; ``wait()`` on the result orders the current
        stream after the transfers and unpacks the ghost rows."""
        ops, unpack = [], []
        for peer, a, b in self.recvs:
            buf = torch.empty(ncomp * (b - a) * self.np1, dtype=vec.dtype, device=vec.device)
            ops.append(dist.P2POp(dist.irecv, buf, peer, self.group))
            unpack.append((buf, a, b))
        for peer, a, b in self.sends:
            buf = torch.cat([self._view(vec, c, a, b) for c in range(ncomp)])
            ops.append(dist.P2POp(dist.isend, buf, peer, self.group))
        return _PendingHalo(dist.batch_isend_irecv(ops) if ops else [], unpack, self, vec, ncomp)

    def exchange(self, vec: torch.Tensor, ncomp: int):
        """Ghost rows <- the neighbours' owned rows.  One message per neighbour
        and direction: the rows of all ``ncomp`` components are packed into one
        contiguous buffer."""
        if self.part.world == 1:
            return
        if vec.is_cuda and dist.get_backend(self.group) == "gloo":
            host = vec.cpu()          # gloo point-to-point is host-only (test/debug path)
            self.exchange(host, ncomp)
            vec.copy_(host)
            return
        ops, unpack = [], []
        for peer, a, b in self.recvs:
            buf = torch.empty(ncomp * (b - a) * self.np1, dtype=vec.dtype, device=vec.device)
            ops.append(dist.P2POp(dist.irecv, buf, peer, self.group))
            unpack.append((buf, a, b))
        for peer, a, b in self.sends:
            buf = torch.cat([self._view(vec, c, a, b) for c in range(ncomp)])
            ops.append(dist.P2POp(dist.isend, buf, peer, self.group))
        for req in dist.batch_isend_irecv(ops):
            req.wait()
        for buf, a, b in unpack:
            w = (b - a) * self.np1
            for c in range(ncomp):
                self._view(vec, c, a, b).copy_(buf[c * w:(c + 1) * w])

    def reverse_add(self, vec: torch.Tensor, ncomp: int):
        """Reverse ghost-row sum of a slab-to-slab restriction: the partial
        sums this rank computed for its top ghost row (the next rank's bottom
        owned row) go up and are added there, in one message per neighbour;
        the ghost rows are zeroed afterwards."""
        part, rank = self.part, self.rank
        if part.world == 1:
            return
        if vec.is_cuda and dist.get_backend(self.group) == "gloo":
            host = vec.cpu()
            self.reverse_add(host, ncomp)
            vec.copy_(host)
            return
        lo, hi = part.rows(rank)
        olo, _ = part.own_rows(rank)
        ops = []
        recv = None
        if rank > 0:
            recv = torch.empty(ncomp * self.np1, dtype=vec.dtype, device=vec.device)
            ops.append(dist.P2POp(dist.irecv, recv, rank - 1, self.group))
        if rank < part.world - 1:
            send = torch.cat([self._view(vec, c, hi, hi + 1) for c in range(ncomp)])
            ops.append(dist.P2POp(dist.isend, send, rank + 1, self.group))
        for req in dist.batch_isend_irecv(ops):
            req.wait()
        if recv is not None:
            for c in range(ncomp):
                self._view(vec, c, olo, olo + 1).add_(recv[c * self.np1:(c + 1) * self.np1])
        self.zero_ghosts(vec, ncomp)


class _PendingHalo:
    def __init__(self, reqs, unpack, halo, vec, ncomp):
        self.reqs, self.unpack, self.halo, self.vec, self.ncomp = reqs, unpack, halo, vec, ncomp

    def wait(self):
        for r in self.reqs:
            r.wait()
        for buf, a, b in self.unpack:
            w = (b - a) * self.halo.np1
            for c in range(self.ncomp):
                self.halo._view(self.vec, c, a, b).copy_(buf[c * w:(c + 1) * w])


class SlabState:
    """Rank-local linearisation point of one level (FULL operator family on a
    slab): the local arrays of ``pff_level_set_window`` and the window handle."""

    def __init__(self, part: SlabPartition, rank: int, params: MaterialParams, split: str,
                 U, phi_tilde, active, dirichlet, device=None, group=None):
        if split not in ("none", "miehe"):
            raise ValueError("split must be 'none' or 'miehe'")
        self.part, self.rank, self.params, self.split = part, rank, params, split
        self.device = device or torch.device("cuda", torch.cuda.current_device())
        self.ln = part.local_n(rank)
        self.halo = HaloExchange(part, rank, group)
        flags = (np.asarray(dirichlet, dtype=np.uint8) | (np.asarray(active, dtype=np.uint8) << 1))
        self.U = self._local(U, 3, np.float64)
        self.pt = self._local(phi_tilde, 1, np.float64)
        fl = self._local(flags, 1, np.uint8)   # + 16 bytes: the sweep's 16-byte flag-row copies
        self.flags = torch.zeros(fl.numel() + 16, dtype=torch.uint8, device=self.device)[:fl.numel()]
        self.flags.copy_(fl)
        self._handle = None
        self._qc = None

    def _local(self, arr, ncomp, dtype):
        arr = np.asarray(arr)
        if arr.size == ncomp * self.part.n:          # global array: take this rank's rows
            loc = self.part.scatter(arr, self.rank, ncomp)
        elif arr.size == ncomp * self.ln:            # already local
            loc = arr
        else:
            raise ValueError("array is neither global nor local for this slab")
        return torch.from_numpy(np.ascontiguousarray(loc, dtype=dtype)).to(self.device)

    def handle(self):
        if self._handle is None:
            s = shape_data(self.part.degree)
            h = ctypes.c_void_p()
            mat = _lib.material(self.params)
            E = s.embedding()
            call("pff_level_create", ctypes.byref(h), self.part.degree, self.part.level,
                 1 if self.split == "miehe" else 0, ctypes.byref(mat), s.values.ctypes.data,
                 s.derivatives.ctypes.data, s.quad_weights.ctypes.data, E.ctypes.data)
            c0, c1 = self.part.cells(self.rank)
            call("pff_level_set_window", h, c0, c1)
            assert _lib.load().pff_level_n_scalar(h) == self.ln
            self._qc = torch.empty(_lib.load().pff_level_qcache_len(h), dtype=torch.float64,
                                   device=self.device)
            call("pff_level_bind", h, ptr(self.U), ptr(self.pt), ptr(self.flags), ptr(self._qc))
            self._handle = h
        return self._handle

    def __del__(self):
        try:
            h = getattr(self, "_handle", None)
            if h is not None and _lib._lib is not None:
                _lib._lib.pff_level_destroy(h)
        except Exception:
            pass

    def refresh_cache(self):
        call("pff_level_refresh", self.handle(), stream_handle())

    def empty(self, ncomp: int) -> torch.Tensor:
        return torch.zeros(ncomp * self.ln, dtype=torch.float64, device=self.device)

    def apply_into(self, mode: int, src: torch.Tensor, dst: torch.Tensor,
                   rhs: torch.Tensor | None = None, exchange: bool = True):
        """dst(owned rows) = G src  (or rhs - G src); src ghost rows are
        refreshed from the neighbours first.  With NCCL the exchange overlaps
        the interior cell rows (they read owned node rows only); the two
        boundary cell rows run once the ghost rows have arrived."""
        ncomp = {_lib.MODE_FULL: 3, _lib.MODE_UU: 2, _lib.MODE_PHIPHI: 1,
                 _lib.MODE_PHIROW: 3}[mode]
        c0, c1 = self.part.cells(self.rank)
        if exchange and c1 - c0 >= 3 and self.halo.overlappable(src) \
                and type(self)._local_apply is SlabState._local_apply:
            pending = self.halo.start(src, ncomp)
            h, st = self.handle(), stream_handle()
            call("pff_apply_rows", h, mode, ptr(src), ptr(dst), ptr(rhs), c0 + 1, c1 - 1, st)
            pending.wait()
            call("pff_apply_rows", h, mode, ptr(src), ptr(dst), ptr(rhs), c0, c0 + 1, st)
            call("pff_apply_rows", h, mode, ptr(src), ptr(dst), ptr(rhs), c1 - 1, c1, st)
            return dst
        if exchange:
            self.halo.exchange(src, ncomp)
        self._local_apply(mode, src, dst, rhs)
        return dst

    def _local_apply(self, mode, src, dst, rhs):
        call("pff_apply", self.handle(), mode, ptr(src), ptr(dst), ptr(rhs), stream_handle())


def owned_dot(part: SlabPartition, rank: int, x: torch.Tensor, y: torch.Tensor, ncomp: int,
              group=None) -> float:
    """Global dot product of two local slab vectors (owned entries only)."""
    own = torch.from_numpy(np.tile(part.owned_mask(rank), ncomp)).to(x.device)
    local = torch.sum(torch.where(own, x * y, torch.zeros((), dtype=x.dtype, device=x.device)))
    if dist.is_available() and dist.is_initialized() and part.world > 1:
        dist.all_reduce(local, group=group)
    return float(local.item())
