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

    # -- cell-routed near field (ShardedSlabSolver(near="cell")) ----------
    device = torch.device("cpu")

    def spread_own(self, pos_own, first, count, flags):
        self.flags, self.first, self.count = flags, first, count
        self.pos_own = pos_own.numpy()
        own = slice(first, first + count)
        rho = self.oracle.spread_phase(
            self.pos_own, self.q[own],
            bool(flags & _lib.CORRECTION), bool(flags & _lib.FORCE_GENERAL))
        self.shape = rho.shape
        self.rho = torch.from_numpy(np.ascontiguousarray(rho)).reshape(-1)
        return self.rho

    def near(self, src_pos, src_q, nt, gauge, zsrc_min, stream=None):
        sp, sq = src_pos.numpy(), src_q.numpy()
        nf = O.NearSources(sp, sq, self.oracle.system.geometry, self.oracle.params)
        out = np.zeros((4, nt))
        if nt:
            phi, E = nf.evaluate(sp[:nt], "avg",
                                 subtract_unsplit=bool(self.flags & _lib.SUBTRACT_SELF))
            out[0], out[1:4] = phi, np.asarray(E).T
        near0 = 0.0
        if gauge:
            near0 = nf.evaluate(np.zeros((1, 3)), "point", need_field=False)[0]
        return (torch.from_numpy(out), torch.tensor([near0], dtype=torch.float64),
                torch.tensor([0], dtype=torch.int64))

    def charges_own(self, pos_own, near_own, near0, need_forces):
        f = self.flags
        n = self.q.size
        pos = np.zeros((n, 3))
        pos[self.first:self.first + self.count] = pos_own.numpy()
        phi, E, U, diag = self.oracle.charge_phase(
            self.state, pos, self.q, self.first, self.count,
            bool(f & _lib.NEED_ENERGY), need_forces, bool(f & _lib.NEED_POTENTIAL),
            bool(f & _lib.SUBTRACT_SELF), near_ext=near_own.numpy(),
            near0_ext=float(near0.reshape(-1)[0]))
        return torch.from_numpy(phi), torch.from_numpy(np.asarray(E)), U, diag

    def diagnostics(self, diag):
        return diag

    def close(self):
        pass


class MirrorDistEngine:
    """Test-only engine for the distributed grid pipeline's host plumbing:
    numpy stand-ins for the se_dist_* phases with the library's buffer
    layouts (z slabs of zc planes, mode pencils of mc modes, all-to-all
    blocks [P][zc][F][mc]) and a simple invertible per-mode operation in
    place of the physics, so the result after the real torch.distributed
    collectives can be checked against the same operations on the full
    grid.  The physics of the phases is covered on the GPU."""

    def __init__(self, nz=5, nxy=(4, 6), seed=0):
        self.Nz = nz
        self.Nx, self.Ny = nxy
        self.NXY = self.Nx * self.Ny
        self.M = self.Nx * (self.Ny // 2 + 1)
        self.seed = seed

    def dist_setup(self, rank, world):
        self.rank, self.P = rank, world
        self.zc = -(-self.Nz // world)
        self.mc = -(-self.M // world)
        self.Nz_pad = self.zc * world
        z = lambda n: torch.zeros(n, dtype=torch.float64)
        self.b = {"rho": z(2 * self.Nz_pad * self.NXY),
                  "rho_slab": z(2 * self.zc * self.NXY),
                  "send": z(2 * world * self.zc * 4 * self.mc),
                  "recv": z(2 * world * self.zc * 4 * self.mc),
                  "fields_slab": z(4 * self.zc * self.NXY),
                  "fields": z(4 * self.Nz_pad * self.NXY),
                  "dsc": z(16)}
        nf = 2 * world * self.zc * 2 * self.mc
        b = self.b
        return {"rho": b["rho"], "rho_slab": b["rho_slab"],
                "send_fwd": b["send"][:nf], "recv_fwd": b["recv"][:nf],
                "send_back": b["send"], "recv_back": b["recv"],
                "fields_slab": b["fields_slab"], "fields": b["fields"],
                "dsc": b["dsc"]}

    def rank_rho(self, rank):
        rng = np.random.default_rng(self.seed + rank)
        rho = np.zeros((self.Nz_pad, 2, self.NXY))
        rho[:self.Nz] = rng.standard_normal((self.Nz, 2, self.NXY))
        return rho

    def positions(self, positions):
        return torch.from_numpy(np.ascontiguousarray(positions, dtype=np.float64))

    def spread(self, pos_all, first, count, flags):
        self.b["rho"].copy_(torch.from_numpy(self.rank_rho(self.rank).ravel()))
        return self.b["rho"]

    def hat_of(self, rho_planes):           # [k][2][NXY] -> [k][2][M] complex
        hat = np.zeros(rho_planes.shape[:2] + (self.M,), dtype=complex)
        hat[...] = rho_planes[..., np.arange(self.M) % self.NXY]
        return hat

    @staticmethod
    def mode_op(pen, m_glob):               # [Nz][2][m] -> [Nz][4][m]
        out = np.zeros((pen.shape[0], 4, pen.shape[2]), dtype=complex)
        for f in range(4):
            out[:, f] = pen[:, f % 2] * (f + 1) * (m_glob + 1) * (1 + 1j)
        return out

    def fields_of(self, spec_planes):       # [k][4][M] -> [k][4][NXY]
        return spec_planes[..., np.arange(self.NXY) % self.M].real

    def dist_forward(self):
        zc, mc, P, M = self.zc, self.mc, self.P, self.M
        hat = self.hat_of(self.b["rho_slab"].numpy().reshape(zc, 2, self.NXY))
        send = np.zeros((P, zc, 2, mc), dtype=complex)
        for q in range(P):
            for l in range(mc):
                if q * mc + l < M:
                    send[q, :, :, l] = hat[:, :, q * mc + l]
        self.b["send"][:send.size * 2].copy_(torch.from_numpy(send.view(np.float64).ravel()))

    def dist_modes(self):
        zc, mc, P, Nz = self.zc, self.mc, self.P, self.Nz
        recv = self.b["recv"][:2 * P * zc * 2 * mc].numpy().view(complex).reshape(P, zc, 2, mc)
        pen = np.zeros((Nz, 2, mc), dtype=complex)
        for s in range(P):
            for j in range(zc):
                if s * zc + j < Nz:
                    pen[s * zc + j] = recv[s, j]
        m_glob = self.rank * mc + np.arange(mc)
        spec = self.mode_op(pen, m_glob)
        send = np.zeros((P, zc, 4, mc), dtype=complex)
        for q in range(P):
            for j in range(zc):
                if q * zc + j < Nz:
                    send[q, j] = spec[q * zc + j]
        self.b["send"].copy_(torch.from_numpy(send.view(np.float64).ravel()))
        self.b["dsc"].zero_()
        if self.rank == 0:
            self.b["dsc"][0] = 42.0

    def dist_fields(self):
        zc, mc, P, M = self.zc, self.mc, self.P, self.M
        assert float(self.b["dsc"][0]) == 42.0       # the summed scalars arrived
        recv = self.b["recv"].numpy().view(complex).reshape(P, zc, 4, mc)
        spec = np.zeros((zc, 4, M), dtype=complex)
        for s in range(P):
            for l in range(mc):
                if s * mc + l < M:
                    spec[:, :, s * mc + l] = recv[s, :, :, l]
        self.b["fields_slab"].copy_(torch.from_numpy(self.fields_of(spec).ravel()))

    def charges(self, pos_all, count, need_forces):
        return (torch.zeros(count, dtype=torch.float64),
                torch.zeros((count, 3), dtype=torch.float64), 0.0, {})

    def expected_fields(self):
        total = sum(self.rank_rho(r) for r in range(self.P))[:self.Nz]
        pen = self.hat_of(total)
        spec = self.mode_op(pen, np.arange(self.M))
        return self.fields_of(spec)

    def diagnostics(self, diag):
        return diag

    def close(self):
        pass
