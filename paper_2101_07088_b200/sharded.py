"""One system solved on several GPUs (one process per GPU).

The charges are split by index into contiguous shards, one per rank
(SURVEY.md section 8e, step 1).  Each rank

1. spreads its own charges (and their first images) into a full copy of the
   grids (``se_shard_spread``),
2. sums the grids over ranks (``torch.distributed`` collectives, NCCL over
   NVLink on the solver's stream),
3. runs the grid pipeline -- xy FFTs, z DCT-I, mode BVPs, correction, inverse
   transforms -- on the summed grids: replicated on every rank
   (``se_shard_fields``), or with ``decompose=True`` distributed as the
   prescribed scheme: reduce-scatter into z slabs, slab xy FFTs, all-to-all
   to (kx, ky) pencils, pencil z transforms + BVPs, all-to-all back, slab
   inverse FFTs, all-gather of the field grid (``se_dist_*``),
4. interpolates the fields and evaluates the near field at its own charges,
   with every charge as a near-field source (``se_shard_charges``),

then the parts of the energy are summed (all-reduce of one double) and, for
the host API, potentials and fields are gathered to every rank.  Spreading is
linear in the charges and the per-charge stages are independent, so the
result equals the single-GPU solve up to the order of the grid sums.

The host logic here is backend-neutral: ``ShardedSlabSolver`` drives an
engine with the three phases.  The product engine is ``CudaShardEngine``
(the C-ABI in include/slabewald.h); the CPU tests drive the same host logic
over ``gloo`` with a checker engine built on the test oracle.
"""

import ctypes

import numpy as np
import torch
import torch.distributed as dist

from . import _lib
from .slab import STAGES, SlabSolver, SolveResult, _flags


# exception type <-> the library's error codes (include/slabewald.h), so a
# failure seen by one rank is raised with the same type on every rank
_ERR_TYPES = ((ValueError, _lib.SE_ERR_VALUE), (FloatingPointError, _lib.SE_ERR_FLOAT),
              (np.linalg.LinAlgError, _lib.SE_ERR_LINALG), (MemoryError, _lib.SE_ERR_MEMORY),
              (RuntimeError, _lib.SE_ERR_CUDA))


def _error_code(exc):
    for typ, code in _ERR_TYPES:
        if isinstance(exc, typ):
            return code
    return _lib.SE_ERR_CUDA


def _error_type(code):
    for typ, c in _ERR_TYPES:
        if c == code:
            return typ
    return RuntimeError


def shard_range(n, rank, world):
    """Contiguous index range [first, first + count) of ``rank``."""
    first = (n * rank) // world
    last = (n * (rank + 1)) // world
    return first, last - first


def cell_destinations(x, Lx, world, halo):
    """Ranks that need each charge for the cell-routed near field: the owner
    of its x slab ([r Lx/P, (r+1) Lx/P), as a target) and the slabs within
    ``halo`` of it across a slab face (as a source; periodic in x).
    Returns (charge index, destination rank, is_target) rows, each charge
    sent at most once to a rank.  Needs a slab width >= halo."""
    w = Lx / world
    xw = torch.remainder(x, Lx)
    owner = torch.clamp((xw / w).floor().to(torch.int64), 0, world - 1)
    idx = torch.arange(x.shape[0], device=x.device)
    rows = [(idx, owner, torch.ones_like(owner, dtype=torch.bool))]
    if world > 1:
        lo = owner.to(x.dtype) * w
        left = (owner - 1) % world
        right = (owner + 1) % world
        near_lo = (xw - lo) < halo
        near_hi = (lo + w - xw) <= halo
        rows.append((idx[near_lo], left[near_lo], torch.zeros_like(left[near_lo], dtype=torch.bool)))
        # with two ranks the right neighbour is the left one: send once
        keep = near_hi & ~(near_lo & (right == left))
        rows.append((idx[keep], right[keep], torch.zeros_like(right[keep], dtype=torch.bool)))
    ci = torch.cat([r[0] for r in rows])
    dest = torch.cat([r[1] for r in rows])
    tgt = torch.cat([r[2] for r in rows])
    return ci, dest, tgt


def _exchange(rows, dest, world, group):
    """all-to-all of float64 record rows by destination rank (sorted send,
    counts exchanged first).  Returns the received rows."""
    order = torch.argsort(dest, stable=True)
    rows = rows[order].contiguous()
    counts = torch.bincount(dest, minlength=world)
    if world == 1:
        return rows
    recv_counts = torch.empty_like(counts)
    dist.all_to_all_single(recv_counts, counts, group=group)
    sc, rc = counts.tolist(), recv_counts.tolist()
    out = torch.empty((sum(rc), rows.shape[1]), dtype=rows.dtype, device=rows.device)
    dist.all_to_all_single(out, rows, output_split_sizes=rc, input_split_sizes=sc, group=group)
    return out


class _DeviceArray:
    """Zero-copy view of a library-owned device buffer for torch."""

    def __init__(self, ptr, n):
        self.__cuda_array_interface__ = {
            "shape": (int(n),), "typestr": "<f8", "data": (int(ptr), False),
            "version": 3, "strides": None}


class CudaShardEngine:
    """The three solve phases of one rank on its GPU (se_shard_*)."""

    def __init__(self, system, params, refine=1, device=0, precision="fp64"):
        self.device = torch.device("cuda", device)
        self.solver = SlabSolver(system, params, refine=refine, device=device,
                                 precision=precision)
        self.solver.set_stream(torch.cuda.current_stream(self.device).cuda_stream)
        self._lib = self.solver._lib

    def positions(self, positions):
        if isinstance(positions, torch.Tensor):
            pos = positions.to(torch.float64)
        else:
            pos = torch.as_tensor(np.ascontiguousarray(positions,
                                                       dtype=np.float64))
        return pos.to(self.device, non_blocking=True).contiguous()

    def spread(self, pos_all, first, count, flags):
        ptr = ctypes.c_void_p()
        size = ctypes.c_int64()
        _lib.check(self._lib.se_shard_spread(
            self.solver._plan, ctypes.c_void_p(pos_all.data_ptr()),
            pos_all.shape[0], first, count, flags, ctypes.byref(ptr),
            ctypes.byref(size)))
        return torch.as_tensor(_DeviceArray(ptr.value, size.value),
                               device=self.device)

    def fields(self):
        _lib.check(self._lib.se_shard_fields(self.solver._plan))

    # -- distributed grid pipeline (se_dist_*) ---------------------------
    def dist_setup(self, rank, world):
        """Decompose the grid pipeline over ``world`` ranks; returns the
        library buffers the collectives act on (torch views)."""
        sizes = (ctypes.c_int64 * 7)()
        _lib.check(self._lib.se_dist_setup(self.solver._plan, rank, world, sizes))
        ptrs = (ctypes.c_void_p * 7)()
        _lib.check(self._lib.se_dist_buffers(self.solver._plan, ptrs))
        names = ("rho", "rho_slab", "a2a_fwd_send", "a2a_back_send",
                 "fields_slab", "fields", "dsc")
        view = lambda ptr, n: torch.as_tensor(_DeviceArray(ptr, n), device=self.device)
        buf = {
            "rho": view(ptrs[0], sizes[0]),
            "rho_slab": view(ptrs[1], sizes[1]),
            "send_fwd": view(ptrs[2], sizes[2]),
            "recv_fwd": view(ptrs[3], sizes[2]),
            "send_back": view(ptrs[2], sizes[3]),
            "recv_back": view(ptrs[3], sizes[3]),
            "fields_slab": view(ptrs[4], sizes[4]),
            "fields": view(ptrs[5], sizes[5]),
            "dsc": view(ptrs[6], sizes[6]),
        }
        del names
        return buf

    def dist_forward(self):
        _lib.check(self._lib.se_dist_forward(self.solver._plan))

    def dist_modes(self):
        _lib.check(self._lib.se_dist_modes(self.solver._plan))

    def dist_fields(self):
        _lib.check(self._lib.se_dist_fields(self.solver._plan))

    def charges(self, pos_all, count, need_forces):
        phi = torch.empty(count, dtype=torch.float64, device=self.device)
        E = torch.zeros((count, 3), dtype=torch.float64, device=self.device)
        U = ctypes.c_double(0.0)
        diag = _lib.SeDiag()
        _lib.check(self._lib.se_shard_charges(
            self.solver._plan, ctypes.c_void_p(pos_all.data_ptr()),
            ctypes.c_void_p(phi.data_ptr()),
            ctypes.c_void_p(E.data_ptr() if need_forces else 0),
            ctypes.byref(U), ctypes.byref(diag)))
        return phi, E, float(U.value), diag

    # -- cell-routed near field (near="cell") ---------------------------
    def spread_own(self, pos_own, first, count, flags):
        ptr = ctypes.c_void_p()
        size = ctypes.c_int64()
        _lib.check(self._lib.se_shard_spread_own(
            self.solver._plan, ctypes.c_void_p(pos_own.data_ptr()), self.solver._q.size,
            first, count, flags, ctypes.byref(ptr), ctypes.byref(size)))
        return torch.as_tensor(_DeviceArray(ptr.value, size.value), device=self.device)

    def near(self, src_pos, src_q, nt, gauge, zsrc_min, stream=None):
        """Near-field sums at the first ``nt`` of the routed sources, on
        ``stream`` (concurrent with the grid pipeline)."""
        out = torch.empty((4, max(nt, 1)), dtype=torch.float64, device=self.device)
        near0 = torch.zeros(1, dtype=torch.float64, device=self.device)
        npairs = torch.zeros(1, dtype=torch.int64, device=self.device)
        st = (stream or torch.cuda.current_stream(self.device)).cuda_stream
        _lib.check(self._lib.se_shard_near(
            self.solver._plan, ctypes.c_void_p(st), ctypes.c_void_p(src_pos.data_ptr()),
            ctypes.c_void_p(src_q.data_ptr()), src_pos.shape[0], nt, 1 if gauge else 0,
            ctypes.c_void_p(zsrc_min.data_ptr()), ctypes.c_void_p(out.data_ptr()),
            ctypes.c_void_p(near0.data_ptr()), ctypes.c_void_p(npairs.data_ptr())))
        return out[:, :nt], near0, npairs

    def charges_own(self, pos_own, near_own, near0, need_forces):
        count = pos_own.shape[0]
        phi = torch.empty(count, dtype=torch.float64, device=self.device)
        E = torch.zeros((count, 3), dtype=torch.float64, device=self.device)
        near_own = near_own.contiguous()
        U = ctypes.c_double(0.0)
        diag = _lib.SeDiag()
        _lib.check(self._lib.se_shard_charges_own(
            self.solver._plan, ctypes.c_void_p(pos_own.data_ptr()),
            ctypes.c_void_p(near_own.data_ptr()), ctypes.c_void_p(near0.data_ptr()),
            ctypes.c_void_p(phi.data_ptr()),
            ctypes.c_void_p(E.data_ptr() if need_forces else 0),
            ctypes.byref(U), ctypes.byref(diag)))
        return phi, E, float(U.value), diag

    def diagnostics(self, diag):
        return self.solver._diagnostics(diag)

    def close(self):
        self.solver.close()


class ShardedSlabSolver:
    """``SlabSolver`` API over a process group: every rank constructs it with
    the same system; ``solve`` returns the full result on every rank."""

    def __init__(self, system, params, threads=1, refine=1, group=None,
                 device=None, engine=None, precision="fp64", decompose=False,
                 near="index"):
        if not dist.is_initialized():
            raise RuntimeError("ShardedSlabSolver needs torch.distributed "
                               "initialised (one process per GPU)")
        self.system, self.params = system, params
        self.threads = threads
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        n = system.charges.size
        self.first, self.count = shard_range(n, self.rank, self.world)
        self.counts = [shard_range(n, r, self.world)[1]
                       for r in range(self.world)]
        if engine is None:
            if device is None:
                device = torch.cuda.current_device()
            engine = CudaShardEngine(system, params, refine, device, precision)
        self.engine = engine
        self.precision = precision
        self.decompose = decompose
        if near not in ("index", "cell"):
            raise ValueError("near must be 'index' or 'cell'")
        geo = system.geometry
        # the cell-routed near field: x slabs of width Lx / P, halo r_cut
        # (the query radius of the charges; the gauge's r_nf is smaller)
        self.halo = float(params.r_cut)
        if near == "cell" and (geo.Lx / self.world < self.halo or
                               not system.surface.is_zero or np.isinf(params.xi)):
            raise ValueError("near='cell' needs Lx / ranks >= r_cut, zero surface "
                             "charge and a finite xi")
        self.near_mode = near
        self.buf = engine.dist_setup(self.rank, self.world) if self.decompose else None
        self.last_timings = None
        self._side = None

    def close(self):
        self.engine.close()

    def solve_shard(self, pos_all, need_energy=True, need_forces=True,
                    need_potential=True, subtract_self=False,
                    include_correction=True, force_general=False,
                    timings=False):
        """The sharded solve on engine-resident positions of ALL charges.
        Returns (phi, E, U, diag) with phi, E for this rank's charges
        ``first .. first+count-1`` and U the total energy."""
        flags = _flags(need_energy, need_forces, need_potential,
                       subtract_self, include_correction, force_general,
                       timings, self.precision == "fp32")
        rho = self.engine.spread(pos_all, self.first, self.count, flags)
        if self.decompose:
            self._grid_pipeline_distributed()
        else:
            if self.world > 1:
                dist.all_reduce(rho, group=self.group)
            self.engine.fields()
        # Some input errors are detected by one rank only (a charge of its own
        # shard outside the z domain, its own near-field buffers): agree on
        # the outcome before the next collective, so every rank raises the
        # same exception instead of the others blocking in the all-reduce.
        try:
            phi, E, u_part, diag = self.engine.charges(pos_all, self.count,
                                                       need_forces)
            err = None
        except (ValueError, FloatingPointError, ArithmeticError, MemoryError,
                RuntimeError) as exc:
            err = exc
        self._agree(err)
        U = u_part
        if self.world > 1:
            u = torch.tensor([u_part], dtype=torch.float64, device=phi.device)
            dist.all_reduce(u, group=self.group)
            U = float(u.item())
        if timings and hasattr(diag, "t_ms"):
            self.last_timings = dict(zip(STAGES, list(diag.t_ms)[:len(STAGES)]))
        return phi, E, U, diag

    # -- cell-routed near field --------------------------------------------
    def _route_sources(self, pos_own):
        """Send each own charge to the rank owning its x slab (target) and to
        the neighbouring slabs within r_cut (halo source).  Returns the
        received (positions [ns][3], charges [ns], global indices of the
        nt targets), targets first.  One sort of the destination keys, one
        row gather and one all-to-all: rows go out grouped by destination,
        targets before halo copies, and the receiver concatenates the
        senders' target blocks, then their halo blocks."""
        dev = pos_own.device
        if getattr(self, "_qg", None) is None or self._qg.device != dev:
            q = torch.as_tensor(self.system.charges[self.first:self.first + self.count],
                                dtype=torch.float64, device=dev)
            g = torch.arange(self.first, self.first + self.count, dtype=torch.float64,
                             device=dev)
            self._qg = torch.stack([q, g], dim=1)
        if self.world == 1:                       # every charge is an own target
            return (pos_own.contiguous(), self._qg[:, 0].contiguous(),
                    self._qg[:, 1].to(torch.int64))
        own = torch.cat([pos_own, self._qg], dim=1)                 # [count][5]
        ci, dest, tgt = cell_destinations(pos_own[:, 0], self.system.geometry.Lx,
                                          self.world, self.halo)
        key = dest * 2 + (~tgt).to(torch.int64)                     # (rank, halo?)
        order = torch.argsort(key, stable=True)
        rows = own.index_select(0, ci[order])
        counts = torch.bincount(key, minlength=2 * self.world)
        recv = torch.empty_like(counts)
        dist.all_to_all_single(recv, counts, group=self.group)
        sc = counts.view(self.world, 2).sum(1).tolist()
        rc2 = recv.view(self.world, 2).tolist()
        rc = [a + b for a, b in rc2]
        got = torch.empty((sum(rc), 5), dtype=torch.float64, device=dev)
        dist.all_to_all_single(got, rows, output_split_sizes=rc, input_split_sizes=sc,
                               group=self.group)
        blocks_t, blocks_h, off = [], [], 0
        for nt_s, nh_s in rc2:
            blocks_t.append(got[off:off + nt_s])
            blocks_h.append(got[off + nt_s:off + nt_s + nh_s])
            off += nt_s + nh_s
        got = torch.cat(blocks_t + blocks_h)
        nt = sum(b[0] for b in rc2)
        return (got[:, 0:3].contiguous(), got[:, 3].contiguous(),
                got[:nt, 4].to(torch.int64))

    def _route_back(self, near_t, tgt_gidx):
        """Near sums of this rank's targets -> the ranks holding those
        charges' index shards, in shard order ([4][count])."""
        dev = near_t.device
        if self.world == 1:                       # targets are the shard, in order
            out = torch.zeros((4, self.count), dtype=torch.float64, device=dev)
            out[:, tgt_gidx - self.first] = near_t
            return out
        firsts = torch.tensor([shard_range(self.system.charges.size, r, self.world)[0]
                               for r in range(self.world)], dtype=torch.int64, device=dev)
        dest = torch.searchsorted(firsts, tgt_gidx, right=True) - 1
        rows = torch.cat([tgt_gidx[:, None].to(torch.float64), near_t.T], dim=1)
        got = _exchange(rows, dest, self.world, self.group)
        out = torch.zeros((4, self.count), dtype=torch.float64, device=dev)
        out[:, got[:, 0].to(torch.int64) - self.first] = got[:, 1:5].T
        return out

    def _zsrc_min(self, pos_own):
        """Minimum z over all near-field sources of all ranks (charges and
        mirror layers), the reference KD tree's z origin (slab.py:120)."""
        geo = self.system.geometry
        z = pos_own[:, 2]
        dev = pos_own.device
        big = torch.tensor(1e300, dtype=torch.float64, device=dev)
        zmin = z.min() if z.numel() else big
        zmax = z.max() if z.numel() else -big
        t = torch.stack([zmin, -zmax])
        if self.world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MIN, group=self.group)
        zmin, zmax = t[0], -t[1]
        cands = [zmin]
        if geo.eps_b != geo.eps:
            cands.append(-zmax)
        if geo.eps_t != geo.eps:
            cands.append(2.0 * geo.H - zmax)
        return torch.stack(cands).min().reshape(1)

    def solve_shard_own(self, pos_own, need_energy=True, need_forces=True,
                        need_potential=True, subtract_self=False,
                        include_correction=True, force_general=False, timings=False):
        """The sharded solve with only this rank's index-shard positions
        (``pos_own`` [count][3] on the engine's device) and the near field
        routed by cell: the routed near field runs on a side stream while
        the grid pipeline's collectives and kernels run on the main one.
        Returns (phi, E, U, diag) of the own shard; diag["n_pairs"] summed."""
        flags = _flags(need_energy, need_forces, need_potential,
                       subtract_self, include_correction, force_general,
                       timings, self.precision == "fp32")
        rho = self.engine.spread_own(pos_own, self.first, self.count, flags)
        src_pos, src_q, tgt_gidx = self._route_sources(pos_own)
        zsrc = self._zsrc_min(pos_own)
        nt = int(tgt_gidx.numel())
        gauge = need_potential and self.rank == 0     # rank 0's slab holds x = 0
        cuda = pos_own.is_cuda
        if cuda:
            main = torch.cuda.current_stream(pos_own.device)
            if self._side is None:
                self._side = torch.cuda.Stream(pos_own.device)
            self._side.wait_stream(main)
            with torch.cuda.stream(self._side):
                near_t, near0, npairs = self.engine.near(src_pos, src_q, nt, gauge, zsrc,
                                                         self._side)
        else:
            near_t, near0, npairs = self.engine.near(src_pos, src_q, nt, gauge, zsrc)
        if self.decompose:
            self._grid_pipeline_distributed()
        else:
            if self.world > 1:
                dist.all_reduce(rho, group=self.group)
            self.engine.fields()
        if cuda:
            main.wait_stream(self._side)
        near_own = self._route_back(near_t, tgt_gidx)
        stat = torch.cat([near0.reshape(1), npairs.to(torch.float64).reshape(1)])
        if self.world > 1:
            dist.all_reduce(stat, group=self.group)
        try:
            phi, E, u_part, diag = self.engine.charges_own(pos_own, near_own, stat[0:1],
                                                           need_forces)
            err = None
        except (ValueError, FloatingPointError, ArithmeticError, MemoryError,
                RuntimeError) as exc:
            err = exc
        self._agree(err)
        U = u_part
        if self.world > 1:
            u = torch.tensor([u_part], dtype=torch.float64, device=phi.device)
            dist.all_reduce(u, group=self.group)
            U = float(u.item())
        self.last_pairs = int(stat[1].item())
        if timings and hasattr(diag, "t_ms"):
            self.last_timings = dict(zip(STAGES, list(diag.t_ms)[:len(STAGES)]))
        return phi, E, U, diag

    def _agree(self, err):
        """All-reduce (MAX) the error code of this rank's phase; raise the
        local exception, or one of the same type naming the failing rank."""
        code = _error_code(err) if err is not None else 0
        if self.world > 1:
            dev = self.engine.device if dist.get_backend(self.group) == "nccl" \
                else torch.device("cpu")
            t = torch.tensor([code, self.rank if code else -1], dtype=torch.int64,
                             device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX, group=self.group)
            if err is None and int(t[0]) != 0:
                raise _error_type(int(t[0]))(
                    "sharded solve failed on rank %d (see that rank's error)" % int(t[1]))
        if err is not None:
            raise err

    def _grid_pipeline_distributed(self):
        """Reduce-scatter of the spread grids into z slabs, xy FFT, all-to-all
        to (kx, ky) pencils, mode stage, all-to-all back, inverse xy FFT,
        all-gather of the fields."""
        b, g = self.buf, self.group
        dist.reduce_scatter_tensor(b["rho_slab"], b["rho"], group=g)
        self.engine.dist_forward()
        dist.all_to_all_single(b["recv_fwd"], b["send_fwd"], group=g)
        self.engine.dist_modes()
        dist.all_to_all_single(b["recv_back"], b["send_back"], group=g)
        dist.all_reduce(b["dsc"], group=g)
        self.engine.dist_fields()
        dist.all_gather_into_tensor(b["fields"], b["fields_slab"], group=g)

    def _gather(self, local, width):
        if self.world == 1:
            return local
        cap = max(self.counts)
        buf = torch.zeros((cap, width), dtype=local.dtype, device=local.device)
        buf[:local.shape[0]] = local.reshape(-1, width)
        parts = [torch.empty_like(buf) for _ in range(self.world)]
        dist.all_gather(parts, buf, group=self.group)
        return torch.cat([p[:c] for p, c in zip(parts, self.counts)])

    def solve(self, positions=None, need_energy=True, need_forces=True,
              need_potential=True, subtract_self=False,
              include_correction=True, force_general=False, timings=False):
        """Same call and result as ``SlabSolver.solve`` (reference
        slab.py:259-394), computed across the group."""
        pos = self.system.positions if positions is None else positions
        pos = np.atleast_2d(np.asarray(pos, dtype=float))
        if pos.ndim != 2 or (pos.size and pos.shape[1] != 3):
            raise ValueError("positions must be (N, 3)")
        if pos.shape[0] != self.system.charges.size:
            raise ValueError("positions and charges disagree on N")
        if self.near_mode == "cell":
            # only this rank's index shard goes to the device
            pos_own = self.engine.positions(pos[self.first:self.first + self.count])
            phi, E, U, diag = self.solve_shard_own(
                pos_own, need_energy, need_forces, need_potential, subtract_self,
                include_correction, force_general, timings)
        else:
            pos_all = self.engine.positions(pos)
            phi, E, U, diag = self.solve_shard(
                pos_all, need_energy, need_forces, need_potential, subtract_self,
                include_correction, force_general, timings)
        phi_all = self._gather(phi.reshape(-1, 1), 1).reshape(-1)
        E_all = self._gather(E, 3) if need_forces else \
            torch.zeros((pos.shape[0], 3), dtype=torch.float64)
        out = self.engine.diagnostics(diag)
        if self.near_mode == "cell" and isinstance(out, dict):
            out["n_pairs"] = self.last_pairs
        if timings and self.last_timings is not None:
            out["timings_ms"] = self.last_timings
        return SolveResult(phi_bar=phi_all.cpu().numpy(),
                           E_bar=E_all.cpu().numpy(), U=U, diagnostics=out)


__all__ = ["ShardedSlabSolver", "CudaShardEngine", "shard_range"]
