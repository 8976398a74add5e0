"""Python mirror of the reference's operator-level interfaces over the C ABI
(include/stmg_b200.h). Vectors are CUDA torch tensors (float64) in the
reference layout; torch is used only for device memory and streams.

  Mesh                ~ stmg::MeshHierarchy   (include/stmg/mesh.hpp:38-60)
  SpaceTimeOperator   ~ stmg::SpaceTimeOperator (space_time_operator.hpp:34-105)
  ASMSmoother         ~ stmg::ASMSmoother      (asm_smoother.hpp:16-45)
  Transfer            ~ stmg::Transfer         (transfer.hpp:22-40)
  SpaceTimeMultigrid  ~ stmg::SpaceTimeMultigrid (multigrid.hpp:61-113)
  gmres / solve       ~ stmg::gmres            (gmres.hpp:9-33)
"""
from __future__ import annotations

import ctypes as C
from typing import Callable, Optional, Sequence

import numpy as np

from . import native as N

HEAT, WAVE = 0, 1
DG, CGP = 0, 1
SPACE_H, SPACE_P, TIME_TAU, TIME_K = 0, 1, 2, 3
COARSENING_NAMES = {0: "space-h", 1: "space-p", 2: "time-tau", 3: "time-k", -1: "finest"}


def _torch():
    import torch
    return torch


def _stream():
    return C.c_void_p(_torch().cuda.current_stream().cuda_stream)


def _ptr(t, n: Optional[int] = None) -> C.c_void_p:
    """Device pointer of a tensor argument: contiguous float64 on the current
    CUDA device, and exactly n entries when n is given (the C side reads or
    writes n doubles; a short or foreign tensor would be out of bounds)."""
    torch = _torch()
    if not isinstance(t, torch.Tensor) or not t.is_cuda or t.dtype != torch.float64 or not t.is_contiguous():
        raise N.StmgInvalidArgument("expected a contiguous float64 CUDA tensor")
    if t.device.index != torch.cuda.current_device():
        raise N.StmgInvalidArgument(f"tensor on cuda:{t.device.index}, current device is cuda:{torch.cuda.current_device()}")
    if n is not None and t.numel() != n:
        raise N.StmgInvalidArgument(f"size mismatch: {t.numel()} entries, expected {n}")
    return C.c_void_p(t.data_ptr())


def _host(a, n: int, writable: bool = False) -> np.ndarray:
    """Host buffer argument: contiguous float64 numpy array of n entries."""
    if writable:
        if not (isinstance(a, np.ndarray) and a.dtype == np.float64 and a.flags.c_contiguous and a.flags.writeable):
            raise N.StmgInvalidArgument("output must be a writable contiguous float64 numpy array")
    else:
        a = np.ascontiguousarray(a, dtype=np.float64)
    if a.size != n:
        raise N.StmgInvalidArgument(f"size mismatch: {a.size} entries, expected {n}")
    return a


def _dbl(a: Optional[np.ndarray]):
    if a is None:
        return None
    a = np.ascontiguousarray(a, dtype=np.float64)
    return a, a.ctypes.data_as(N.c_double_p)


class Mesh:
    """MeshHierarchy of make_cartesian (mesh.cpp:148-187). base_cells is the
    reference's cube count per axis, or a per-axis triple (x, y, z) for the
    box meshes of the weak-scaling study (stmg_mesh_create_box)."""

    def __init__(self, dim: int, lo, hi, base_cells, refinements: int, vertices: Optional[np.ndarray] = None):
        lib = N.load()
        self.dim, self.refinements = dim, refinements
        if np.ndim(base_cells) == 0:
            self.base = (int(base_cells),) * 3
        else:
            self.base = tuple(int(c) for c in base_cells) + (1,) * (3 - len(base_cells))
        self.base_cells = self.base[0]
        lo_a, lo_p = _dbl(np.asarray(lo, dtype=np.float64))
        hi_a, hi_p = _dbl(np.asarray(hi, dtype=np.float64))
        v = _dbl(vertices)
        if v is not None and v[0].size != 3 * self.n_verts(refinements):
            raise N.StmgInvalidArgument("Mesh: vertices must hold 3 doubles per finest-level vertex")
        h = C.c_void_p()
        if np.ndim(base_cells) == 0:
            N.check(lib.stmg_mesh_create(dim, lo_p, hi_p, int(base_cells), refinements, v[1] if v else None,
                                         C.byref(h)))
        else:
            bc = (C.c_longlong * 3)(*self.base)
            N.check(lib.stmg_mesh_create_box(dim, lo_p, hi_p, bc, refinements, v[1] if v else None, C.byref(h)))
        self._h = h

    def cells_axis(self, level: int):
        return tuple((self.base[a] << level) if a < self.dim else 1 for a in range(3))

    def cells(self, level: int) -> int:
        return int(np.prod(self.cells_axis(level)))

    def n_verts(self, level: int) -> int:
        return int(np.prod([c + 1 for c in self.cells_axis(level)[:self.dim]]))

    def __del__(self):
        if getattr(self, "_h", None):
            N.load().stmg_mesh_destroy(self._h)
            self._h = None


class SpaceTimeOperator:
    def __init__(self, mesh: Mesh, mesh_level: int, p: int, equation: int, scheme: int, k: int, tau: float,
                 n_steps: int, rho: Optional[np.ndarray] = None, _handle=None, _owner=None):
        lib = N.load()
        self.mesh = mesh
        if _handle is not None:
            self._h, self._owned, self._owner = C.c_void_p(_handle), False, _owner
        else:
            r = _dbl(rho)
            h = C.c_void_p()
            N.check(lib.stmg_st_operator_create(mesh._h, mesh_level, p, equation, scheme, k, tau, n_steps,
                                                r[1] if r else None, C.byref(h)))
            self._h, self._owned = h, True
        self.n_dofs = lib.stmg_st_operator_n_dofs(self._h)
        self.n_space = lib.stmg_st_operator_n_space(self._h)
        self.n_t = lib.stmg_st_operator_n_t(self._h)

    def apply(self, u, y=None):
        """y = S u (overwrite)."""
        torch = _torch()
        if u.numel() != self.n_dofs:
            raise N.StmgInvalidArgument("SpaceTimeOperator::apply: size mismatch")
        if y is None:
            y = torch.empty_like(u)
        N.check(N.load().stmg_st_operator_apply(self._h, _ptr(u, self.n_dofs), _ptr(y, self.n_dofs), _stream()))
        return y

    def apply_host(self, u: np.ndarray, y: Optional[np.ndarray] = None) -> np.ndarray:
        """y = S u on host buffers (H2D/D2H inside the C ABI call)."""
        u = _host(u, self.n_dofs)
        y = np.empty_like(u) if y is None else _host(y, self.n_dofs, writable=True)
        N.check(N.load().stmg_st_operator_apply_host(self._h, u.ctypes.data_as(N.c_double_p),
                                                     y.ctypes.data_as(N.c_double_p)))
        return y

    def residual(self, f, u, r=None):
        """r = f - S u (one fused pass)."""
        if r is None:
            r = _torch().empty_like(u)
        n = self.n_dofs
        N.check(N.load().stmg_st_operator_residual(self._h, _ptr(f, n), _ptr(u, n), _ptr(r, n), _stream()))
        return r

    def interpolate(self, kind: int, frequency: float = 0.5, t: float = 0.0, centre=(0.5, 0.5, 0.5),
                    width: float = 0.05, zero_boundary: bool = False):
        """Nodal interpolant on the Q_p lattice (kind: 0 heat source, 1 wave
        source, 2 Gaussian, 3 manufactured u, 4 manufactured v)."""
        out = _torch().empty(self.n_space, dtype=_torch().float64, device="cuda")
        c = np.ascontiguousarray(centre, dtype=np.float64)
        N.check(N.load().stmg_st_operator_interpolate(self._h, kind, frequency, t, c.ctypes.data_as(N.c_double_p),
                                                      width, 1 if zero_boundary else 0, _ptr(out), _stream()))
        return out

    def assemble_rhs(self, source_kind: int, frequency: float, t0: float, u0, v0=None):
        """Slab right-hand side (SpaceTimeOperator::assemble_rhs)."""
        rhs = _torch().empty(self.n_dofs, dtype=_torch().float64, device="cuda")
        N.check(N.load().stmg_st_operator_assemble_rhs(self._h, source_kind, frequency, t0, _ptr(u0),
                                                       _ptr(v0) if v0 is not None else None, _ptr(rhs), _stream()))
        return rhs

    def extract_final(self, u, u0, v0=None):
        """State after the slab (SpaceTimeOperator::extract_final) -> (u, v or None)."""
        torch = _torch()
        uf = torch.empty(self.n_space, dtype=torch.float64, device="cuda")
        vf = torch.empty(self.n_space, dtype=torch.float64, device="cuda") if v0 is not None else None
        N.check(N.load().stmg_st_operator_extract_final(self._h, _ptr(u), _ptr(u0),
                                                        _ptr(v0) if v0 is not None else None, _ptr(uf),
                                                        _ptr(vf) if vf is not None else None, _stream()))
        return uf, vf

    def error_norms(self, x, u0, frequency: float = 0.5, t0: float = 0.0):
        """error_norms (driver.cpp:83-92) of one batch vs the manufactured
        solution -> (L2(L2), Linf(L2), Linf(Linf))."""
        out = (C.c_double * 3)()
        _torch().cuda.synchronize()
        N.check(N.load().stmg_st_operator_error_norms(self._h, _ptr(x), _ptr(u0), frequency, t0, out))
        return tuple(out)

    def spatial_apply(self, kind: int, u, y=None):
        torch = _torch()
        if y is None:
            y = torch.empty_like(u)
        N.check(N.load().stmg_spatial_apply(self._h, kind, _ptr(u, self.n_space), _ptr(y, self.n_space), _stream()))
        return y

    def __del__(self):
        if getattr(self, "_owned", False) and self._h:
            N.load().stmg_st_operator_destroy(self._h)
            self._h = None


class ASMSmoother:
    def __init__(self, op: SpaceTimeOperator):
        h = C.c_void_p()
        N.check(N.load().stmg_asm_create(op._h, C.byref(h)))
        self._h, self.op = h, op

    def add_correction(self, r, z):
        """z += W sum_T R_T^T B_T^-1 R_T r (accumulate)."""
        n = self.op.n_dofs
        N.check(N.load().stmg_asm_add_correction(self._h, _ptr(r, n), _ptr(z, n), _stream()))
        return z

    def __del__(self):
        if getattr(self, "_h", None):
            N.load().stmg_asm_destroy(self._h)
            self._h = None


class Transfer:
    def __init__(self, fine: SpaceTimeOperator, coarse: SpaceTimeOperator):
        h = C.c_void_p()
        N.check(N.load().stmg_transfer_create(fine._h, coarse._h, C.byref(h)))
        self._h, self.fine, self.coarse = h, fine, coarse

    def prolong(self, c, f=None):
        if f is None:
            f = _torch().empty(self.fine.n_dofs, dtype=c.dtype, device=c.device)
        N.check(N.load().stmg_transfer_prolong(self._h, _ptr(c, self.coarse.n_dofs), _ptr(f, self.fine.n_dofs),
                                               _stream()))
        return f

    def restrict_(self, f, c=None):
        if c is None:
            c = _torch().empty(self.coarse.n_dofs, dtype=f.dtype, device=f.device)
        N.check(N.load().stmg_transfer_restrict(self._h, _ptr(f, self.fine.n_dofs), _ptr(c, self.coarse.n_dofs),
                                                _stream()))
        return c

    def __del__(self):
        if getattr(self, "_h", None):
            N.load().stmg_transfer_destroy(self._h)
            self._h = None


def mg_options(**kw) -> N.MgOptions:
    o = N.MgOptions()
    N.load().stmg_mg_options_default(C.byref(o))
    for k, v in kw.items():
        setattr(o, k, v)
    return o


def gmres_options(**kw) -> N.GmresOptions:
    o = N.GmresOptions()
    N.load().stmg_gmres_options_default(C.byref(o))
    for k, v in kw.items():
        setattr(o, k, v)
    return o


class SpaceTimeMultigrid:
    def __init__(self, equation: int, scheme: int, mesh: Mesh, rho: Optional[np.ndarray], fine_level: int, p: int,
                 k: int, n_steps: int, tau: float, strategy: Optional[Sequence[int]] = None, **options):
        lib = N.load()
        r = _dbl(rho)
        strat = None
        ns = -1
        if strategy is not None:
            ns = len(strategy)
            strat = (C.c_int * max(ns, 1))(*strategy)
        o = mg_options(**options)
        h = C.c_void_p()
        N.check(lib.stmg_multigrid_create(equation, scheme, mesh._h, r[1] if r else None, fine_level, p, k, n_steps,
                                          tau, ns, strat, C.byref(o), C.byref(h)))
        self._h, self.mesh = h, mesh
        self.n_levels = lib.stmg_multigrid_n_levels(h)
        self._ops = [SpaceTimeOperator(mesh, 0, 1, 0, 0, 0, 1.0, 1, _handle=lib.stmg_multigrid_operator_at(h, l),
                                       _owner=self) for l in range(self.n_levels)]

    def operator_at(self, l: int) -> SpaceTimeOperator:
        return self._ops[l]

    def _n(self, l: int) -> int:
        if not 0 <= l < self.n_levels:
            raise N.StmgInvalidArgument(f"bad level {l}")
        return self._ops[l].n_dofs

    def level_info(self):
        out = []
        for l in range(self.n_levels):
            ints = (C.c_int * 5)()
            n = C.c_longlong()
            w = C.c_double()
            N.check(N.load().stmg_multigrid_level_info(self._h, l, ints, C.byref(n), C.byref(w)))
            out.append({"coarsening": COARSENING_NAMES[ints[4]], "mesh_level": ints[0], "p": ints[1], "k": ints[2],
                        "n_steps": ints[3], "n_dofs": n.value, "omega": w.value})
        return out

    def smoother_kind(self, l: int) -> int:
        """bit 0 tensor FDM, bit 1 per-cell eigenbasis, bit 2 temporal fast
        diagonalisation (-1: coarsest level, no smoother)."""
        return int(N.load().stmg_multigrid_smoother_kind(self._h, l))

    def smoother_bytes(self, l: int) -> int:
        """Bytes of per-cell smoother data streamed by one level-l sweep."""
        return int(N.load().stmg_multigrid_smoother_bytes(self._h, l))

    def vcycle_bytes(self, n_smooth: int = 1) -> int:
        """Algorithmic HBM bytes of one V-cycle: per level l
        with N_l dofs, 2 n_smooth smoother sweeps streaming the level's cell
        data plus ~112 N_l bytes of vector traffic (smoother in/out, residual,
        restriction, prolongation); the coarsest level's dense solve n_c^2."""
        info = self.level_info()
        total = 0
        for l, li in enumerate(info):
            n = li["n_dofs"]
            if l + 1 < len(info):
                total += 2 * n_smooth * max(self.smoother_bytes(l), 0) + 112 * n
            else:
                total += 8 * n * n
        return total

    def omega_at(self, l: int) -> float:
        return self.level_info()[l]["omega"]

    def set_omega(self, l: int, w: float):
        N.check(N.load().stmg_multigrid_set_omega(self._h, l, w))

    def apply(self, r, z=None):
        if z is None:
            z = _torch().empty_like(r)
        n = self._n(0)
        N.check(N.load().stmg_multigrid_apply(self._h, _ptr(r, n), _ptr(z, n), _stream()))
        return z

    def apply_host(self, r: np.ndarray, z: np.ndarray) -> np.ndarray:
        """One V-cycle on host buffers (H2D/D2H inside the C ABI call)."""
        r, z = _host(r, self._n(0)), _host(z, self._n(0), writable=True)
        N.check(N.load().stmg_multigrid_apply_host(self._h, r.ctypes.data_as(N.c_double_p),
                                                   z.ctypes.data_as(N.c_double_p)))
        return z

    def smooth(self, l: int, f, u):
        N.check(N.load().stmg_multigrid_smooth(self._h, l, _ptr(f, self._n(l)), _ptr(u, self._n(l)), _stream()))
        return u

    def asm_add_correction(self, l: int, r, z):
        N.check(N.load().stmg_multigrid_asm_add_correction(self._h, l, _ptr(r, self._n(l)), _ptr(z, self._n(l)),
                                                           _stream()))
        return z

    def prolong(self, l: int, c, f=None):
        if f is None:
            f = _torch().empty(self._ops[l].n_dofs, dtype=c.dtype, device=c.device)
        N.check(N.load().stmg_multigrid_prolong(self._h, l, _ptr(c, self._n(l + 1)), _ptr(f, self._n(l)), _stream()))
        return f

    def restrict_(self, l: int, f, c=None):
        if c is None:
            c = _torch().empty(self._ops[l + 1].n_dofs, dtype=f.dtype, device=f.device)
        N.check(N.load().stmg_multigrid_restrict(self._h, l, _ptr(f, self._n(l)), _ptr(c, self._n(l + 1)),
                                                 _stream()))
        return c

    def device_bytes(self) -> int:
        return N.load().stmg_multigrid_device_bytes(self._h)

    def solve(self, b, x, precondition: bool = True, history_cap: int = 1100, **opts):
        """GMRES(op = finest operator, precond = one V-cycle) as march() plugs
        them (driver.cpp:193-203); x is the initial guess and the result."""
        o = gmres_options(**opts)
        res = N.GmresResult()
        hist = np.zeros(history_cap)
        N.check(N.load().stmg_solve(self._h, 1 if precondition else 0, _ptr(b, self._n(0)), _ptr(x, self._n(0)),
                                    C.byref(o), C.byref(res),
                                    hist.ctypes.data_as(N.c_double_p), history_cap, _stream()))
        return _result(res, hist)

    def march(self, n_batches: int, u, v=None, source_kind: int = 1, frequency: float = 0.5, errors: bool = True,
              **opts) -> dict:
        """march (driver.cpp:95-260) on the device: n_batches slabs of the
        finest operator; u (v for the wave) is the entering state and becomes
        the final state. Returns the per-batch GMRES iterations and the
        manufactured-solution error norms of u."""
        o = gmres_options(**opts)
        its = (C.c_int * n_batches)()
        err = (C.c_double * 3)()
        N.check(N.load().stmg_march(self._h, n_batches, source_kind, frequency, _ptr(u),
                                    _ptr(v) if v is not None else None, C.byref(o), its,
                                    err if errors else None, _stream()))
        return {"iterations": list(its), "error_u": tuple(err) if errors else None}

    def march_probes(self, n_batches: int, u, points, v=None, samples_per_step: int = 16, source_kind: int = 1,
                     frequency: float = 0.5, **opts) -> dict:
        """march with probe time series (driver.cpp:146-236): returns the
        iterations, error norms, sample times and one series per point."""
        pts = np.ascontiguousarray(points, dtype=np.float64).reshape(-1, 3)
        n_samples = 1 + n_batches * self.level_info()[0]["n_steps"] * samples_per_step
        times = np.zeros(n_samples)
        vals = np.zeros((pts.shape[0], n_samples))
        o = gmres_options(**opts)
        its = (C.c_int * n_batches)()
        err = (C.c_double * 3)()
        N.check(N.load().stmg_march_probes(self._h, n_batches, source_kind, frequency, _ptr(u),
                                           _ptr(v) if v is not None else None, C.byref(o), its, err, pts.shape[0],
                                           pts.ctypes.data_as(N.c_double_p), samples_per_step,
                                           times.ctypes.data_as(N.c_double_p), vals.ctypes.data_as(N.c_double_p),
                                           _stream()))
        return {"iterations": list(its), "error_u": tuple(err), "times": times, "values": vals}

    def solve_host(self, b: np.ndarray, x: np.ndarray, precondition: bool = True, history_cap: int = 1100, **opts):
        o = gmres_options(**opts)
        res = N.GmresResult()
        hist = np.zeros(history_cap)
        b, x = _host(b, self._n(0)), _host(x, self._n(0), writable=True)
        N.check(N.load().stmg_solve_host(self._h, 1 if precondition else 0, b.ctypes.data_as(N.c_double_p),
                                         x.ctypes.data_as(N.c_double_p), C.byref(o), C.byref(res),
                                         hist.ctypes.data_as(N.c_double_p), history_cap))
        return _result(res, hist)

    def __del__(self):
        if getattr(self, "_h", None):
            self._ops = []
            N.load().stmg_multigrid_destroy(self._h)
            self._h = None


class Comm:
    """Communicator of the partitioned solve. Comm(world, rank, uid): NCCL
    (rank 0 draws the unique id, torch.distributed broadcasts it, every rank
    joins, stmg_comm_create). Comm.host(group): the host-staged transport
    (stmg_comm_create_host) over a torch.distributed process group, e.g. gloo
    -- interface planes and allreduces cross page-locked host memory."""

    def __init__(self, world: int, rank: int, uid: Optional[bytes] = None, _handle=None):
        if _handle is not None:
            self._h, self.world, self.rank = _handle, world, rank
            return
        h = C.c_void_p()
        N.check(N.load().stmg_comm_create(world, rank, uid, C.byref(h)))
        self._h, self.world, self.rank = h, world, rank

    @classmethod
    def host(cls, group=None) -> "Comm":
        import torch
        import torch.distributed as dist
        world, rank = dist.get_world_size(group), dist.get_rank(group)

        def view(p, n):
            return torch.from_numpy(np.ctypeslib.as_array(p, shape=(n,)))

        def allreduce(ctx, h, n):
            try:
                dist.all_reduce(view(h, n), op=dist.ReduceOp.SUM, group=group)
                return 0
            except Exception:  # noqa: BLE001 - reported as a C status
                return 1

        def sendrecv(ctx, peer, hs, hr, n):
            try:
                send = view(hs, n).clone()
                recv = torch.empty(n, dtype=torch.float64)
                reqs = [dist.isend(send, peer, group=group), dist.irecv(recv, peer, group=group)]
                for q in reqs:
                    q.wait()
                view(hr, n).copy_(recv)
                return 0
            except Exception:  # noqa: BLE001
                return 1

        t = N.HostTransport(None, N.HOST_ALLREDUCE(allreduce), N.HOST_SENDRECV(sendrecv))
        h = C.c_void_p()
        N.check(N.load().stmg_comm_create_host(world, rank, C.byref(t), C.byref(h)))
        c = cls(world, rank, _handle=h)
        c._transport = t  # the callbacks must outlive the communicator
        return c

    @staticmethod
    def unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        N.check(N.load().stmg_nccl_unique_id(buf))
        return buf.raw

    def __del__(self):
        if getattr(self, "_h", None):
            N.load().stmg_comm_destroy(self._h)
            self._h = None


def slab_plan(scheme: int, fine_level: int, p: int, k: int, n_steps: int, cells_z: int, n_parts: int):
    """(partitioned levels, total levels) of the default plan (host only)."""
    d, n = C.c_int(), C.c_int()
    N.check(N.load().stmg_slab_plan(scheme, fine_level, p, k, n_steps, cells_z, n_parts, C.byref(d), C.byref(n)))
    return d.value, n.value


class SlabMultigrid:
    """STMG solve on a z-slab partition of the finest mesh: the
    process holds parts [first_part, first_part + local_parts) of n_parts;
    comm (a Comm, or None for one process) joins the processes over NCCL.
    Local vectors are the concatenation of the local parts' slab vectors."""

    def __init__(self, equation: int, scheme: int, mesh: Mesh, rho: Optional[np.ndarray], fine_level: int, p: int,
                 k: int, n_steps: int, tau: float, n_parts: int, first_part: int = 0,
                 local_parts: Optional[int] = None, comm: Optional[Comm] = None,
                 strategy: Optional[Sequence[int]] = None, **options):
        lib = N.load()
        r = _dbl(rho)
        strat, ns = None, -1
        if strategy is not None:
            ns = len(strategy)
            strat = (C.c_int * max(ns, 1))(*strategy)
        o = mg_options(**options)
        if local_parts is None:
            local_parts = n_parts - first_part
        h = C.c_void_p()
        N.check(lib.stmg_slab_multigrid_create(equation, scheme, mesh._h, r[1] if r else None, fine_level, p, k,
                                               n_steps, tau, ns, strat, C.byref(o), n_parts, first_part,
                                               local_parts, comm._h if comm is not None else None, C.byref(h)))
        self._h, self.mesh, self.comm = h, mesh, comm
        self.n_local = lib.stmg_slab_multigrid_local_dofs(h)
        info = (C.c_int * 2)()
        N.check(lib.stmg_slab_multigrid_info(h, info))
        self.dist_levels, self.n_levels = info[0], info[1]
        self.parts = []
        for i in range(local_parts):
            off, nd, p0 = C.c_longlong(), C.c_longlong(), C.c_longlong()
            N.check(lib.stmg_slab_multigrid_part(h, i, C.byref(off), C.byref(nd), C.byref(p0)))
            self.parts.append({"offset": off.value, "n_dofs": nd.value, "plane0": p0.value})
        # full-length finest-level vector (scatter / gather)
        self.n_full = (n_steps * (k + 1 if scheme == DG else k)) * int(np.prod(
            [((mesh.base[a] << fine_level) * p + 1) for a in range(mesh.dim)]))

    def omega_at(self, l: int) -> float:
        return float(N.load().stmg_slab_multigrid_omega(self._h, l))

    def set_omega(self, l: int, w: float):
        N.check(N.load().stmg_slab_multigrid_set_omega(self._h, l, w))

    def apply(self, u, y=None):
        y = _torch().empty_like(u) if y is None else y
        N.check(N.load().stmg_slab_multigrid_apply(self._h, _ptr(u, self.n_local), _ptr(y, self.n_local), _stream()))
        return y

    def vcycle(self, r, z=None):
        z = _torch().empty_like(r) if z is None else z
        N.check(N.load().stmg_slab_multigrid_vcycle(self._h, _ptr(r, self.n_local), _ptr(z, self.n_local), _stream()))
        return z

    def asm_add_correction(self, r, z):
        N.check(N.load().stmg_slab_multigrid_asm_add_correction(self._h, _ptr(r, self.n_local), _ptr(z, self.n_local),
                                                                _stream()))
        return z

    def solve(self, b, x, **opts):
        o = gmres_options(**opts)
        res = N.GmresResult()
        N.check(N.load().stmg_slab_multigrid_solve(self._h, _ptr(b, self.n_local), _ptr(x, self.n_local), C.byref(o),
                                                   C.byref(res), _stream()))
        return _result(res, np.zeros(0))

    def dot(self, a, b) -> float:
        out = C.c_double()
        _torch().cuda.synchronize()
        N.check(N.load().stmg_slab_multigrid_dot(self._h, _ptr(a, self.n_local), _ptr(b, self.n_local), C.byref(out)))
        return out.value

    def scatter(self, full, local=None):
        torch = _torch()
        local = torch.empty(self.n_local, dtype=full.dtype, device=full.device) if local is None else local
        N.check(N.load().stmg_slab_multigrid_scatter(self._h, _ptr(full, self.n_full), _ptr(local, self.n_local),
                                                     _stream()))
        return local

    def gather(self, local, full):
        N.check(N.load().stmg_slab_multigrid_gather(self._h, _ptr(local, self.n_local), _ptr(full, self.n_full),
                                                    _stream()))
        return full

    def __del__(self):
        if getattr(self, "_h", None):
            N.load().stmg_slab_multigrid_destroy(self._h)
            self._h = None


def _result(res: N.GmresResult, hist: np.ndarray) -> dict:
    n = min(res.history_len, hist.size)
    return {"converged": bool(res.converged), "iterations": res.iterations,
            "initial_residual": res.initial_residual, "final_residual": res.final_residual,
            "residual_history": hist[:n].tolist()}


def gmres(op: Callable, b, x, precond: Optional[Callable] = None, history_cap: int = 1100, **opts) -> dict:
    """stmg::gmres with Python callables op(in, out) / precond(in, out) on CUDA
    tensors of length n (include/stmg/gmres.hpp:31-33)."""
    torch = _torch()
    n = b.numel()

    def wrap(fn):
        def cb(ctx, din, dout, stream):
            try:
                # zero-copy views of the device buffers
                tin = _view(din, n)
                tout = _view(dout, n)
                fn(tin, tout)
                return 0
            except Exception:  # noqa: BLE001 - reported as a failed callback
                return -1
        return N.LINEAR_MAP(cb)

    cop = wrap(op)
    cpc = wrap(precond) if precond is not None else N.LINEAR_MAP()
    o = gmres_options(**opts)
    res = N.GmresResult()
    hist = np.zeros(history_cap)
    torch.cuda.synchronize()
    N.check(N.load().stmg_gmres(n, cop, None, cpc, None, _ptr(b), _ptr(x), C.byref(o), C.byref(res),
                                hist.ctypes.data_as(N.c_double_p), history_cap, _stream()))
    return _result(res, hist)


_VIEW_CACHE: dict = {}


def _view(ptr, n):
    """float64 CUDA tensor aliasing device memory at ptr (no copy)."""
    torch = _torch()
    key = (ptr, n)
    t = _VIEW_CACHE.get(key)
    if t is None:
        class _Cai:
            __cuda_array_interface__ = {"shape": (n,), "typestr": "<f8", "data": (ptr, False), "version": 3}
        t = torch.as_tensor(_Cai(), device="cuda")
        _VIEW_CACHE[key] = t
    return t
