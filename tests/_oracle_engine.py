"""Test-only shard engine: the three solve phases of one rank computed by
the CPU oracle, so the host logic of ``ShardedSlabSolver`` (shard ranges,
grid all-reduce, energy sum, gathers) runs over ``gloo`` without a GPU.
Never used by the product path (which takes ``CudaShardEngine``)."""

import numpy as np
import torch

from oracle import slab_oracle as O
from paper_2101_07088_b200 import _lib


class OracleShardEngine:
    def __init__(self, system, params, refine=1):
        self.oracle = O.OracleSlabSolver(system, params, refine=refine)
        self.q = system.charges

    def positions(self, positions):
        return torch.from_numpy(np.ascontiguousarray(positions,
                                                     dtype=np.float64))

    def spread(self, pos_all, first, count, flags):
        self.flags, self.first = flags, first
        own = slice(first, first + count)
        rho = self.oracle.spread_phase(
            pos_all.numpy()[own], self.q[own],
            bool(flags & _lib.CORRECTION), bool(flags & _lib.FORCE_GENERAL))
        self.shape = rho.shape
        self.rho = torch.from_numpy(np.ascontiguousarray(rho)).reshape(-1)
        return self.rho                     # summed in place by the host

    def fields(self):
        f = self.flags
        self.state = self.oracle.field_phase(
            self.rho.numpy().reshape(self.shape), bool(f & _lib.NEED_FORCES),
            bool(f & _lib.CORRECTION), bool(f & _lib.FORCE_GENERAL))

    def charges(self, pos_all, count, need_forces):
        f = self.flags
        first = self.first
        phi, E, U, diag = self.oracle.charge_phase(
            self.state, pos_all.numpy(), self.q, first, count,
            bool(f & _lib.NEED_ENERGY), need_forces,
            bool(f & _lib.NEED_POTENTIAL), bool(f & _lib.SUBTRACT_SELF))
        return torch.from_numpy(phi), torch.from_numpy(np.asarray(E)), U, diag

    def diagnostics(self, diag):
        return diag

    def close(self):
        pass
