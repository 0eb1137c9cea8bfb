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

    def diagnostics(self, diag):
        return self.solver._diagnostics(diag)

    def close(self):
        self.solver.close()


class ShardedSlabSolver:
    """``SlabSolver`` API over a process group: every rank constructs it with
    the same system; ``solve`` returns the full result on every rank."""

    def __init__(self, system, params, threads=1, refine=1, group=None,
                 device=None, engine=None, precision="fp64", decompose=False):
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
        self.buf = engine.dist_setup(self.rank, self.world) if self.decompose else None
        self.last_timings = None

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
        pos_all = self.engine.positions(pos)
        phi, E, U, diag = self.solve_shard(
            pos_all, need_energy, need_forces, need_potential, subtract_self,
            include_correction, force_general, timings)
        phi_all = self._gather(phi.reshape(-1, 1), 1).reshape(-1)
        E_all = self._gather(E, 3) if need_forces else \
            torch.zeros((pos.shape[0], 3), dtype=torch.float64)
        out = self.engine.diagnostics(diag)
        if timings and self.last_timings is not None:
            out["timings_ms"] = self.last_timings
        return SolveResult(phi_bar=phi_all.cpu().numpy(),
                           E_bar=E_all.cpu().numpy(), U=U, diagnostics=out)


__all__ = ["ShardedSlabSolver", "CudaShardEngine", "shard_range"]
