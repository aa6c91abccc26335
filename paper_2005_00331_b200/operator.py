"""Linearisation state and the matrix-free Jacobian family on the B200.

Drop-in for src/pff_operator.py (fracturekit 0.1.0): same names, argument
meaning, constraint conventions and exceptions.  Vectors may be numpy arrays
(copied to the device, results returned as numpy) or CUDA float64 torch
tensors (zero-copy, results returned as CUDA tensors).  All arithmetic runs
in libpff_b200.so; there is no CPU path.
"""

from __future__ import annotations

import ctypes
import time
import warnings
from dataclasses import dataclass
from functools import cached_property

import numpy as np
import torch

from . import _lib
from ._lib import call, ptr, stream_handle
from .basis import LANE_WIDTHS, MaterialParams, ShapeData, shape_data
from .mesh import MeshHierarchy


class StaleCacheError(RuntimeError):
    """Raised when the Jacobian is applied at an outdated linearization."""


class BlockVector:
    """Monolithic (u_x | u_y | phi) host vector with per-component views
    (src/pff_operator.py:32-59): ``data`` is the flat array the operator API
    takes, the views alias it."""

    __slots__ = ("data", "n_scalar")

    def __init__(self, data, n_scalar: int):
        arr = np.asarray(data, dtype=np.float64)
        if arr.ndim != 1 or arr.size != 3 * n_scalar:
            raise ValueError(f"a block vector of {n_scalar} scalar nodes has {3 * n_scalar} entries")
        self.data, self.n_scalar = arr, n_scalar

    @classmethod
    def zeros(cls, n_scalar: int) -> "BlockVector":
        return cls(np.zeros(3 * n_scalar), n_scalar)

    def _part(self, k: int) -> np.ndarray:
        return self.data[k * self.n_scalar:(k + 1) * self.n_scalar]

    u_x = property(lambda self: self._part(0))
    u_y = property(lambda self: self._part(1))
    phi = property(lambda self: self._part(2))

    def copy(self) -> "BlockVector":
        return BlockVector(self.data.copy(), self.n_scalar)


class AssemblyMemoryError(MemoryError):
    """Raised when the assembled (sparse) Jacobian does not fit into memory
    (src/pff_operator.py:28-29)."""


def _dev():
    _lib.require_cuda()
    return torch.device("cuda", torch.cuda.current_device())


def as_device(v, n: int | None = None, name: str = "vector"):
    """(CUDA float64 contiguous tensor, origin) with origin False for CUDA
    tensors, True for numpy input, or the host torch tensor it came from."""
    if isinstance(v, torch.Tensor):
        t = v
        was_np = False
        if t.device.type != "cuda":
            was_np = t
            t = t.to(device=_dev(), dtype=torch.float64, non_blocking=t.is_pinned())
        elif t.dtype != torch.float64 or not t.is_contiguous():
            t = t.to(dtype=torch.float64).contiguous()
    else:
        a = np.ascontiguousarray(np.asarray(v, dtype=np.float64))
        t = torch.from_numpy(a).to(_dev(), non_blocking=False)
        was_np = True
    if n is not None and t.numel() != n:
        raise ValueError(f"{name} must have {n} entries, got {t.numel()}")
    return t.reshape(-1), was_np


def back(t: torch.Tensor, was_np):
    """Return the result in the caller's array kind (numpy / host tensor /
    CUDA tensor); a pinned host input gets a pinned host result."""
    if isinstance(was_np, torch.Tensor):
        out = torch.empty(t.shape, dtype=t.dtype, pin_memory=was_np.is_pinned())
        out.copy_(t, non_blocking=False)
        return out
    return t.cpu().numpy() if was_np else t


_PINNED_MIN = 1 << 20   # host mirrors with at least this many entries are pinned


class _Dual:
    """A host numpy array and its device mirror, synchronised lazily.

    Reading the host side marks it possibly modified (callers may write into
    it in place, as the reference's own code does), so the next device use
    re-uploads; device writes mark the host side stale."""

    def __init__(self, n: int, dtype, fill, tail=None):
        self._n, self._dtype, self._fill = n, dtype, fill
        self._tail = tail       # (start, value): entries [start:] start as value
        self._h = None          # host array, made on first host access
        self._d = None
        self._host_new = True
        self._dev_new = False
        self.stamp = 0   # bumped on every (possible) modification

    def _tdtype(self):
        return torch.bool if self._dtype is bool else torch.from_numpy(
            np.empty(0, dtype=self._dtype)).dtype

    def _alloc_host(self) -> np.ndarray:
        # large mirrors live in pinned memory: their uploads then run at the
        # full PCIe rate (torch's caching host allocator recycles the blocks)
        if self._n >= _PINNED_MIN and torch.cuda.is_available():
            return torch.empty(self._n, dtype=self._tdtype(), pin_memory=True).numpy()
        return np.empty(self._n, dtype=self._dtype)

    def _host_array(self) -> np.ndarray:
        if self._h is None:
            self._h = self._alloc_host()
            self._h[:] = self._fill
            if self._tail is not None:
                self._h[self._tail[0]:] = self._tail[1]
        return self._h

    def host(self) -> np.ndarray:
        if self._dev_new:
            h = self._alloc_host()        # a fresh array, as before (callers may hold the old one)
            torch.from_numpy(h).copy_(self._d)
            self._h = h
            self._dev_new = False
        self._host_array()
        self._host_new = True
        self.stamp += 1
        return self._h

    def device(self) -> torch.Tensor:
        if self._d is None:
            if self._h is None:     # never touched on the host: fill on the device
                self._d = torch.full((self._n,), self._fill, dtype=self._tdtype(), device=_dev())
                if self._tail is not None:
                    self._d[self._tail[0]:] = self._tail[1]
            else:
                self._d = torch.from_numpy(self._h).to(_dev())
            self._host_new = False
        elif self._host_new:
            self._d.copy_(torch.from_numpy(self._h))
            self._host_new = False
        return self._d

    def set(self, value, index=None):
        if isinstance(value, torch.Tensor) and value.is_cuda and index is None:
            if self._d is None:
                self._d = torch.empty(self._n, dtype=self._tdtype(), device=value.device)
            d = self._d
            d.copy_(value.reshape(-1).to(d.dtype))
            self._host_new, self._dev_new = False, True
            self.stamp += 1
        else:
            h = self.host()
            if index is None:
                h[:] = np.asarray(value.cpu() if isinstance(value, torch.Tensor) else value)
            else:
                h[:] = False
                h[np.asarray(index)] = True
            self._host_new = True


class LinearizationState:
    """Frozen evaluation point (u, phi, phi_tilde, active set) on one level
    (src/pff_operator.py:64-196).

    ``refresh_cache()`` uploads the linearisation point and rebuilds the
    device q-point cache; applying at a stale cache raises
    :class:`StaleCacheError` exactly like the reference.  ``lane_width`` and
    ``cache_tensors`` are validated and kept for API compatibility (the GPU
    has no SIMD lanes; the tangent is always built from the cache)."""

    def __init__(self, hierarchy: MeshHierarchy, level: int, params: MaterialParams,
                 split: str = "miehe", lane_width: int = 8, cache_tensors: bool = False):
        if split not in ("none", "miehe"):
            raise ValueError("split must be 'none' or 'miehe'")
        if lane_width not in LANE_WIDTHS:
            raise ValueError(f"lane_width must be one of {LANE_WIDTHS}")
        self.hierarchy = hierarchy
        self.level = level
        self.params = params
        self.split = split
        self.lane_width = lane_width
        self.cache_tensors = cache_tensors
        self.dof_map = hierarchy.dof_map(level)
        self.mesh = hierarchy.level(level)
        self.shape: ShapeData = shape_data(hierarchy.degree)
        n = self.dof_map.n_scalar
        self._U = _Dual(3 * n, np.float64, 0.0, tail=(2 * n, 1.0))   # u = 0, phi = 1
        self._pt = _Dual(n, np.float64, 1.0)
        self._po = _Dual(n, np.float64, 1.0)
        self._act = _Dual(n, bool, False)
        self._dir = _Dual(n, bool, False)
        self._flags = None
        self._flags_stamp = None
        self._bound_key = None
        self._qcache = None
        self._handle = None
        self._version = 0
        self._cache_version = -1

    # -- sizes and views ----------------------------------------------------
    @property
    def n_scalar(self) -> int:
        return self.dof_map.n_scalar

    @property
    def U(self) -> np.ndarray:
        return self._U.host()

    @property
    def u_x(self) -> np.ndarray:
        return self.U[: self.n_scalar]

    @property
    def u_y(self) -> np.ndarray:
        return self.U[self.n_scalar: 2 * self.n_scalar]

    @property
    def phi(self) -> np.ndarray:
        return self.U[2 * self.n_scalar:]

    @property
    def phi_tilde(self) -> np.ndarray:
        return self._pt.host()

    @property
    def phi_old(self) -> np.ndarray:
        return self._po.host()

    @property
    def active(self) -> np.ndarray:
        return self._act.host()

    @property
    def dirichlet_nodes(self) -> np.ndarray:
        return self._dir.host()

    @property
    def version(self) -> int:
        return self._version

    # -- mutation (bumps the version) ----------------------------------------
    def set_solution(self, U):
        self._U.set(U)
        self._version += 1

    def set_phi_tilde(self, phi_tilde):
        self._pt.set(phi_tilde)
        self._version += 1

    def set_phi_old(self, phi_old):
        self._po.set(phi_old)
        self._version += 1

    def set_active(self, active):
        self._act.set(active)
        self._version += 1

    def set_dirichlet_nodes(self, nodes):
        if isinstance(nodes, torch.Tensor) and nodes.dtype == torch.bool:
            self._dir.set(nodes)
        else:
            self._dir.set(None, index=nodes)
        self._version += 1

    def uses_sweep_kernel(self) -> bool:
        """True when this level's applications run the Q2 sweep kernel."""
        return _lib.load().pff_level_uses_sweep(self._level_handle()) == 1

    def constrained_mask(self) -> np.ndarray:
        d = self.dirichlet_nodes
        return np.concatenate([d, d, self.active])

    # -- device side ----------------------------------------------------------
    def _level_handle(self):
        if self._handle is None:
            s = self.shape
            h = ctypes.c_void_p()
            mat = _lib.material(self.params)
            N, D, w, E = s.values, s.derivatives, s.quad_weights, s.embedding()
            call("pff_level_create", ctypes.byref(h), self.hierarchy.degree,
                 self.level, 1 if self.split == "miehe" else 0, ctypes.byref(mat),
                 N.ctypes.data, D.ctypes.data, w.ctypes.data, E.ctypes.data)
            self._handle = h
            self._keep = (N, D, w, E)
        return self._handle

    def __del__(self):
        try:
            h = getattr(self, "_handle", None)
            if h is not None and _lib._lib is not None:
                _lib._lib.pff_level_destroy(h)
        except Exception:   # interpreter shutdown: modules may already be gone
            pass

    def _sync_flags(self):
        stamp = (self._dir.stamp, self._act.stamp)
        if self._flags is None or stamp != self._flags_stamp:
            d = self._dir.device()
            a = self._act.device()
            if self._flags is None:
                # 16 bytes of padding: the sweeps stage flag bytes in aligned units
                # (Q2: 16-byte TMA rows, Q4: 4-byte cp.async words) that may extend
                # past the final node
                buf = torch.zeros(d.numel() + 16, dtype=torch.uint8, device=d.device)
                self._flags = buf[:d.numel()]
            call("pff_flags", d.numel(), ptr(d), ptr(a), ptr(self._flags), 0, stream_handle())
            self._flags_stamp = (self._dir.stamp, self._act.stamp)
        return self._flags

    def _bind_key(self):
        return (self._U.stamp, self._pt.stamp, self._dir.stamp, self._act.stamp,
                self._U._host_new, self._pt._host_new)

    def bind(self):
        """Bind the current device buffers to the level handle; returns it."""
        key = self._bind_key()
        if self._handle is not None and self._qcache is not None and key == self._bound_key:
            return self._handle
        h = self._level_handle()
        if self._qcache is None:
            qlen = _lib.load().pff_level_qcache_len(h)
            self._qcache = torch.empty(qlen, dtype=torch.float64, device=_dev())
        call("pff_level_bind", h, ptr(self._U.device()), ptr(self._pt.device()),
             ptr(self._sync_flags()), ptr(self._qcache))
        self._bound_key = self._bind_key()
        return h

    def device_U(self) -> torch.Tensor:
        return self._U.device()

    def device_flags(self) -> torch.Tensor:
        return self._sync_flags()

    def device_phi_old(self) -> torch.Tensor:
        return self._po.device()

    def touch_solution(self):
        """The device copy of U was modified in place (a kernel wrote it):
        the host mirror is stale and the version moves on."""
        self._U.device()
        self._U._host_new, self._U._dev_new = False, True
        self._U.stamp += 1
        self._version += 1

    def add_to_solution(self, dU):
        """U += dU on the device (state.set_solution(state.U + dU) without
        the host round trip)."""
        n3 = 3 * self.n_scalar
        d, _ = as_device(dU, n3)
        U = self._U.device()
        call("pff_axpby", n3, 1.0, ptr(d), 1.0, ptr(U), stream_handle())
        self.touch_solution()

    def refresh_cache(self):
        call("pff_level_refresh", self.bind(), stream_handle())
        self._cache_version = self._version

    def _check_cache(self):
        if self._qcache is None or self._cache_version != self._version:
            raise StaleCacheError(
                f"quadrature cache at version {self._cache_version}, state at {self._version}")

    def cache(self):
        """Device q-point cache as a dict of (n_cells, q, q) views
        (src/pff_operator.py:186-191 names; stored cell-fastest on device)."""
        self._check_cache()
        q, nc = self.shape.q, self.mesh.n_cells
        qc = self._qcache[:6 * q * q * nc].view(6, q, q, nc)
        names = ("e11", "e22", "e12", "gt", "dg", "pc")
        return {k: qc[i].permute(2, 0, 1) for i, k in enumerate(names)}

    def cache_bytes(self) -> int:
        return 0 if self._qcache is None else self._qcache.numel() * 8

    # -- operator entry points used by the solvers (device tensors) ----------
    def apply_into(self, mode: int, src: torch.Tensor, dst: torch.Tensor,
                   rhs: torch.Tensor | None = None):
        self._check_cache()
        call("pff_apply", self.bind(), mode, ptr(src), ptr(dst), ptr(rhs), stream_handle())
        return dst


_NC_IN = {_lib.MODE_FULL: 3, _lib.MODE_UU: 2, _lib.MODE_PHIPHI: 1, _lib.MODE_PHIROW: 3}
_NC_OUT = {_lib.MODE_FULL: 3, _lib.MODE_UU: 2, _lib.MODE_PHIPHI: 1, _lib.MODE_PHIROW: 1}


def _pipelined(state: LinearizationState, mode: int, xh: torch.Tensor, nchunks: int = 0) -> torch.Tensor:
    """Host (pinned) -> device -> host application through pff_apply_host: the
    library queues the H2D of every cell-row chunk on one copy stream, sweeps
    chunk k on the current stream once its rows are resident and copies it
    back on a second copy stream, so both PCIe directions and the kernel
    overlap and no per-chunk work is left to the host.  Same arithmetic as the
    one-shot path (nchunks 0: the library's ramp of chunk sizes)."""
    n = state.dof_map.n_scalar
    dev = _dev()
    xd = torch.empty(_NC_IN[mode] * n, dtype=torch.float64, device=dev)
    yd = torch.empty(_NC_OUT[mode] * n, dtype=torch.float64, device=dev)
    yh = torch.empty(_NC_OUT[mode] * n, dtype=torch.float64, pin_memory=True)
    main = torch.cuda.current_stream()
    call("pff_apply_host", state.bind(), mode, xh.data_ptr(), yh.data_ptr(), xd.data_ptr(),
         yd.data_ptr(), nchunks, main.cuda_stream)
    main.synchronize()
    return yh


def _run(state: LinearizationState, mode: int, v, n_in: int, n_out: int):
    state._check_cache()
    if (isinstance(v, torch.Tensor) and not v.is_cuda and v.is_pinned()
            and v.dtype == torch.float64 and v.is_contiguous() and v.numel() == n_in
            and state.hierarchy.degree == 2 and state.uses_sweep_kernel()):
        return _pipelined(state, mode, v.reshape(-1))
    x, was_np = as_device(v, n_in)
    out = torch.empty(n_out, dtype=torch.float64, device=x.device)
    state.apply_into(mode, x, out)
    return back(out, was_np)


def apply_jacobian(state: LinearizationState, dU):
    """Matrix-free Jacobian action with identity rows/columns on constraints
    (src/pff_operator.py:262-270)."""
    n = state.n_scalar
    return _run(state, _lib.MODE_FULL, dU, 3 * n, 3 * n)


def apply_block_uu(state: LinearizationState, du):
    """Displacement block on a (2n,) vector (src/pff_operator.py:273-282)."""
    n = state.n_scalar
    return _run(state, _lib.MODE_UU, du, 2 * n, 2 * n)


def apply_block_phiphi(state: LinearizationState, dphi):
    """Phase-field block on an (n,) vector (src/pff_operator.py:285-291)."""
    n = state.n_scalar
    return _run(state, _lib.MODE_PHIPHI, dphi, n, n)


def apply_phi_row(state: LinearizationState, dU):
    """phi-row (coupling plus phi block) on a full vector (src/pff_operator.py:294-302)."""
    n = state.n_scalar
    return _run(state, _lib.MODE_PHIROW, dU, 3 * n, n)


def block_diagonal(state: LinearizationState, block: str, invert: bool = False,
                   as_numpy: bool = True):
    """Matrix-free diagonal of the uu or phiphi block; constrained rows get 1
    (src/pff_operator.py:305-327).  One kernel computes both blocks."""
    if block not in ("uu", "phiphi"):
        raise ValueError("block must be 'uu' or 'phiphi'")
    duu, dpp = block_diagonals(state, invert)
    out = duu if block == "uu" else dpp
    return out.cpu().numpy() if as_numpy else out


def block_diagonals(state: LinearizationState, invert: bool = False):
    """Both block diagonals (device tensors) from one diagonal kernel."""
    state._check_cache()
    n = state.n_scalar
    dev = _dev()
    duu = torch.empty(2 * n, dtype=torch.float64, device=dev)
    dpp = torch.empty(n, dtype=torch.float64, device=dev)
    call("pff_diagonal", state.bind(), ptr(duu), ptr(dpp), int(invert), stream_handle())
    return duu, dpp


def extrapolate_phase(phi_nm1, phi_nm2, t_n: float, t_nm1: float, t_nm2: float):
    """Linear extrapolation of the phase field from two previous steps
    (src/pff_operator.py:208-215); device tensors stay on the device."""
    if not (t_nm2 < t_nm1 < t_n):
        raise ValueError("time points must be strictly increasing")
    factor = (t_n - t_nm1) / (t_nm1 - t_nm2)
    if isinstance(phi_nm1, torch.Tensor) and phi_nm1.is_cuda:
        return phi_nm1 + factor * (phi_nm1 - phi_nm2)
    phi_nm1 = np.asarray(phi_nm1, dtype=float)
    phi_nm2 = np.asarray(phi_nm2, dtype=float)
    return phi_nm1 + factor * (phi_nm1 - phi_nm2)


def residual(state: LinearizationState, mask_dirichlet: bool = True, mask_active: bool = False,
             as_numpy: bool = True):
    """Nonlinear residual (src/pff_operator.py:218-241)."""
    n = state.n_scalar
    out = torch.empty(3 * n, dtype=torch.float64, device=_dev())
    call("pff_residual", state.bind(), ptr(out), int(mask_dirichlet), int(mask_active),
         stream_handle())
    return out.cpu().numpy() if as_numpy else out


# ------------------------------------------------------------ assembled path
# the assembled Jacobian the paper compares the matrix-free
# application against (src/pff_operator.py:199-205, 328-377), built on the device.

@dataclass
class SparseOracle:
    """Assembled CSR Jacobian with identity constraint rows/columns.  ``device``
    is a CUDA sparse-CSR tensor (cuSPARSE SpMV via ``matvec``); ``matrix`` a
    scipy CSR copy on the host, made on first access (the reference's field)."""

    device: torch.Tensor
    state_version: int
    assembly_seconds: float

    @property
    def shape(self):
        return tuple(self.device.shape)

    @property
    def nnz(self) -> int:
        return int(self.device._nnz())

    @cached_property
    def matrix(self):
        import scipy.sparse as sp
        A = self.device
        return sp.csr_matrix((A.values().cpu().numpy(), A.col_indices().cpu().numpy(),
                              A.crow_indices().cpu().numpy()), shape=self.shape)

    def matvec(self, x):
        """A x (cuSPARSE); numpy in -> numpy out, CUDA tensor in -> CUDA out."""
        xd, was_np = as_device(x, self.shape[1])
        return back(torch.mv(self.device, xd), was_np)


def cell_matrices(state: LinearizationState, as_numpy: bool = True):
    """Dense local Jacobian matrices G_k of every cell, (n_cells, 3 nloc, 3 nloc)
    (src/pff_operator.py:328-340), from ``pff_cell_matrices``."""
    state._check_cache()
    nl = 3 * state.dof_map.n_local
    gk = torch.empty((state.mesh.n_cells, nl, nl), dtype=torch.float64, device=_dev())
    call("pff_cell_matrices", state.bind(), ptr(gk), stream_handle())
    return gk.cpu().numpy() if as_numpy else gk


def assemble_oracle(state: LinearizationState) -> SparseOracle:
    """Scatter the cellwise dense matrices into CSR with identity constraints
    (src/pff_operator.py:343-377), entirely on the device; running out of
    device memory raises :class:`AssemblyMemoryError`."""
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    dm = state.dof_map
    n, nloc = dm.n_scalar, dm.n_local
    dev = _dev()
    try:
        gk = cell_matrices(state, as_numpy=False)
        conn = torch.from_numpy(dm.conn).to(dev)
        full = torch.cat([conn + c * n for c in range(3)], dim=1)         # (cells, 3 nloc)
        rows = full.repeat_interleave(3 * nloc, dim=1).reshape(-1)
        cols = full.repeat(1, 3 * nloc).reshape(-1)
        vals = gk.reshape(-1)                                              # (cell, row, col)
        del gk, full
        mask = torch.from_numpy(state.constrained_mask()).to(dev)
        keep = ~(mask[rows] | mask[cols])
        rows, cols, vals = rows[keep], cols[keep], vals[keep]
        cd = torch.nonzero(mask).reshape(-1)
        idx = torch.stack([torch.cat([rows, cd]), torch.cat([cols, cd])])
        del rows, cols, keep
        vals = torch.cat([vals, torch.ones(cd.numel(), dtype=torch.float64, device=dev)])
        with warnings.catch_warnings():   # torch flags sparse CSR as beta
            warnings.simplefilter("ignore", UserWarning)
            A = torch.sparse_coo_tensor(idx, vals, (3 * n, 3 * n),
                                        check_invariants=False).coalesce().to_sparse_csr()
        torch.cuda.synchronize()
    except torch.cuda.OutOfMemoryError as exc:
        raise AssemblyMemoryError(
            f"sparse oracle at level {state.level}, degree {dm.degree} does not fit in "
            "device memory") from exc
    return SparseOracle(device=A, state_version=state.version,
                        assembly_seconds=time.perf_counter() - t0)


def restrict_state_to_level(state: LinearizationState, target: int) -> LinearizationState:
    """Nodal injection of the linearisation point (src/pff_operator.py:380-400),
    done on device level by level."""
    if not 0 <= target <= state.level:
        raise ValueError("target level out of range")
    if target == state.level:
        return state
    cur = state
    for l in range(state.level - 1, target - 1, -1):
        cur = _inject_once(cur, l)
    return cur


def _inject_once(fine: LinearizationState, level: int) -> LinearizationState:
    coarse = LinearizationState(fine.hierarchy, level, fine.params, split=fine.split,
                                lane_width=fine.lane_width, cache_tensors=fine.cache_tensors)
    hf, hc = fine.bind(), coarse._level_handle()
    n = coarse.n_scalar
    dev = _dev()
    U = torch.empty(3 * n, dtype=torch.float64, device=dev)
    pt = torch.empty(n, dtype=torch.float64, device=dev)
    po = torch.empty(n, dtype=torch.float64, device=dev)
    fl = torch.empty(n, dtype=torch.uint8, device=dev)
    s = stream_handle()
    call("pff_inject_f64", hf, hc, ptr(fine._U.device()), ptr(U), 3, s)
    call("pff_inject_f64", hf, hc, ptr(fine._pt.device()), ptr(pt), 1, s)
    call("pff_inject_f64", hf, hc, ptr(fine._po.device()), ptr(po), 1, s)
    call("pff_inject_u8", hf, hc, ptr(fine._sync_flags()), ptr(fl), s)
    coarse.set_solution(U)
    coarse.set_phi_tilde(pt)
    coarse.set_phi_old(po)
    dmask = torch.empty(n, dtype=torch.bool, device=dev)
    amask = torch.empty(n, dtype=torch.bool, device=dev)
    call("pff_flags", n, ptr(dmask), ptr(amask), ptr(fl), 1, s)
    coarse.set_active(amask)
    coarse._dir.set(dmask)   # reference: no version bump
    return coarse


class JacobianOperator:
    """Device callable ``v -> apply_jacobian(state, v)`` with an in-place entry
    point the device GMRES uses to fuse ``rhs - A x``."""

    def __init__(self, state: LinearizationState):
        self.state = state
        self.n = 3 * state.n_scalar

    def __call__(self, v):
        return apply_jacobian(self.state, v)

    def apply_into(self, src, dst, rhs=None):
        return self.state.apply_into(_lib.MODE_FULL, src, dst, rhs)
