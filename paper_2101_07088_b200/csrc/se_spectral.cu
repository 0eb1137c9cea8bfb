// Fourier x Chebyshev transforms and the per-mode boundary value problems.
//
// Reference: SlabSolver._forward / _modes_to_grid (slab.py:240-251),
// cheb_transform / cheb_inverse / cheb_derivative (chebyshev.py:46-79),
// DtnSolver.solve (dpsolver.py:47-71) -> BvpFactor (bvp.py:142-278),
// solve_k0_dirichlet (bvp.py:281-296), the mismatch assembly
// (slab.py:302-318), HarmonicCorrection (dpsolver.py:89-155) and the k = 0
// combination (slab.py:397-445, dpsolver.py:166-218).
//
// B200 design.  The xy transforms are batched cuFFT D2Z / C2R over the
// Chebyshev planes of the z-slowest layout.  The DCT-I along z (Nz = 258 at
// the north-star size, 2(Nz-1) = 2*257: Bluestein for an FFT) is a matrix
// product over all modes at once, folded by the node reflection into two
// half-order products (even / odd coefficient rows) that hand-written
// kernels run on the FP64 tensor pipe (mma.sync m8n8k4): the fold is fused
// into the forward kernel's staging, the node recombination, harmonic
// correction and i k multipliers into the inverse kernel's epilogue.
// The BVP is a lane pair per (kx, ky) mode of the half spectrum (over /
// in-slab grid): sweeps along z touch row n of all modes together, so every
// global access is coalesced across the warp; factors are precomputed per
// distinct |k| at plan time.  The
// mismatch, harmonic-correction moments and the k = 0 combination are fused
// into the same kernel (a mode needs only its own wall values), and the
// correction values themselves are evaluated on the fly while assembling
// the four spectral fields, so no (mode x node) correction table is stored.
#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "se_internal.cuh"

namespace se {

namespace {

__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cscale(double2 a, double s) { return make_double2(a.x * s, a.y * s); }
__device__ __forceinline__ double2 cfma(double s, double2 a, double2 acc) {
    return make_double2(fma(s, a.x, acc.x), fma(s, a.y, acc.y));
}

// k-independent integration maps (bvp.py:21-54) and BC column sums
// (bvp.py:104-121), uploaded once.
struct Maps {
    const double *e_lo, *e_hi, *q_lo, *q_dg, *q_hi;   // [Nz]
    const double *ue, *uq, *ve, *vq;                  // [Nz]
};

// ---------------------------------------------------------------------------
// per-|k| factorisation                                    bvp.py:145-198
// ---------------------------------------------------------------------------
struct FactorArgs {
    Maps mp; int Nz; int n_uniq; double half;
    const double* kuniq; double* fac; double* sinv; double* kappa;
    int* bad;
};

__global__ void factor_kernel(FactorArgs a) {
    int u = blockIdx.x * blockDim.x + threadIdx.x;
    if (u >= a.n_uniq) return;
    const int n = a.Nz;
    const double kap = a.kuniq[u] * a.half;
    const double k2 = kap * kap;
    a.kappa[u] = kap;
    double* cp = a.fac + ((int64_t)u * FAC_ROWS + FAC_CP) * n;
    double* inv = a.fac + ((int64_t)u * FAC_ROWS + FAC_INV) * n;
    double* aib = a.fac + ((int64_t)u * FAC_ROWS + FAC_AINVB) * n;
    double* c0 = a.fac + ((int64_t)u * FAC_ROWS + FAC_C0) * n;
    double* c1 = a.fac + ((int64_t)u * FAC_ROWS + FAC_C1) * n;
    // Thomas factorisation of each parity chain (rows m = 2j + par)
    for (int par = 0; par < 2; ++par) {
        double cprev = 0.0;
        for (int m = par; m < n; m += 2) {
            double dg = 1.0 - k2 * a.mp.q_dg[m];
            double lo = -k2 * a.mp.q_lo[m];
            double up = -k2 * a.mp.q_hi[m];
            double den = (m == par) ? dg : dg - lo * cprev;
            double iv = 1.0 / den;
            inv[m] = iv;
            double c = (m + 2 < n) ? up * iv : 0.0;
            cp[m] = c;
            cprev = c;
        }
        // A^{-1} B column: rhs = -kappa^2 at the chain's first row
        double dprev = 0.0;
        for (int m = par; m < n; m += 2) {
            double lo = -k2 * a.mp.q_lo[m];
            double r = (m == par) ? -k2 : 0.0;
            double d = (m == par) ? r * inv[m] : (r - lo * dprev) * inv[m];
            aib[m] = d;
            dprev = d;
        }
        int last = par + 2 * ((n - 1 - par) / 2);
        for (int m = last - 2; m >= par; m -= 2) aib[m] -= cp[m] * aib[m + 2];
    }
    // BC rows C and the Schur complement S = C A^{-1} B - D
    double s00 = 0, s01 = 0, s10 = 0, s11 = 0;
    for (int m = 0; m < n; ++m) {
        double r0 = a.mp.ue[m] + kap * a.mp.uq[m];
        double r1 = a.mp.ve[m] - kap * a.mp.vq[m];
        c0[m] = r0;
        c1[m] = r1;
        if ((m & 1) == 0) { s00 += r0 * aib[m]; s10 += r1 * aib[m]; }
        else { s01 += r0 * aib[m]; s11 += r1 * aib[m]; }
    }
    s00 -= kap; s01 -= 1.0 + kap; s10 -= -kap; s11 -= 1.0 + kap;
    double det = s00 * s11 - s01 * s10;
    double scale = fabs(s00) + fabs(s01) + fabs(s10) + fabs(s11);
    if (fabs(det) * 1e12 < scale * scale) atomicAdd(a.bad, 1);
    a.sinv[4 * u + 0] = s11 / det;
    a.sinv[4 * u + 1] = -s01 / det;
    a.sinv[4 * u + 2] = -s10 / det;
    a.sinv[4 * u + 3] = s00 / det;
}

// ---------------------------------------------------------------------------
// the per-mode solve
// ---------------------------------------------------------------------------
struct BvpArgs {
    Maps mp;
    int Nz, Nx, Nyh; int64_t M;  // M: mode stride of the scratch / ext columns
    int64_t Mv;                  // modes to solve (< M on the last pencil rank)
    double half, eps, eps_b, eps_t, cb, ct, z0, z1, k_max, k0_scale;
    int refine, two, mode;       // mode 0 jump, 1 plain+sigma, 2 plain
    int correction;              // compute correction moments
    const int* kidx; const double* kmag; const unsigned char* sel;
    const double* fac; const double* sinv; const double* kappa;
    const double* tw0; const double* twH;
    const double2* sbh; const double2* sth;
    double2* ext;                // [2N][2][M] in: raw DCT, out: iDCT inputs
    double2* scrA; double2* scrB;   // [Nz][2][M] each
    double2* bst;                // split kernels: [6][2][M] c0, c1, deferred dc0, dc1, r2
    int iter;                    // split kernels: the refinement iteration
    double inv_nxy;
    double2* mom;                // [M][2]  M_b/den, M_t/den
    double2* mism;               // [4][M] (debug, may be null)
    double2* keep;               // [Nz][2][M] psi coefficients (debug, may be null)
    double* k0out;               // [16]
    double* scal;                // scal[0] = A_i
    int* flags;
    double rb, rt, H;
};

__device__ __forceinline__ bool finite2(double2 v) { return isfinite(v.x) && isfinite(v.y); }

// The mode's wall data -> mismatch, correction moments and (mode k = 0) the
// linear k = 0 coefficients (slab.py:302-318,397-445; dpsolver.py:131-138,
// 189-218).  wi / ei: in-slab grid's wall values / ends, wo / eo: the
// over grid's (zero when only the in-slab grid is solved).
__device__ __forceinline__ void finish_mode(const BvpArgs& a, int64_t m, const double2 (&wi)[4],
                                            const double2 (&ei)[2], const double2 (&wo)[4],
                                            const double2 (&eo)[2]) {
    double2 sb = a.sbh[m], st = a.sth[m];
    double2 phib, eb, phit, et;
    if (a.mode == 0) {                                   // slab.py:306-316
        phib = csub(wi[0], cscale(wo[0], a.cb));
        eb = cadd(csub(cscale(wi[2], a.eps), cscale(wo[2], a.eps_b * a.cb)), sb);
        phit = csub(wi[1], cscale(wo[1], a.ct));
        et = csub(csub(cscale(wi[3], a.eps), cscale(wo[3], a.eps_t * a.ct)), st);
    } else {                                             // slab.py:322-324
        phib = make_double2(0, 0); eb = sb;
        phit = make_double2(0, 0); et = cscale(st, -1.0);
    }
    if (a.mism) {
        a.mism[m] = phib; a.mism[a.M + m] = eb;
        a.mism[2 * a.M + m] = phit; a.mism[3 * a.M + m] = et;
    }
    if (a.correction) {
        if (!(finite2(phib) && finite2(eb) && finite2(phit) && finite2(et)))
            atomicOr(a.flags, FLAG_NONFINITE);
        double2 mb = make_double2(0, 0), mt = make_double2(0, 0);
        if (a.sel[m]) {                                  // dpsolver.py:131-138
            double k = a.kmag[m];
            mb = cscale(csub(eb, cscale(phib, a.eps_b * k)), 1.0 / a.eps);
            mt = cscale(cadd(cscale(phit, a.eps_t * k), et), 1.0 / a.eps);
            double den = k * ((1.0 + a.rb) * (1.0 + a.rt)
                              - (1.0 - a.rb) * (1.0 - a.rt) * exp(-2.0 * k * a.H));
            mb = cscale(mb, 1.0 / den);
            mt = cscale(mt, 1.0 / den);
        }
        a.mom[2 * m] = mb;
        a.mom[2 * m + 1] = mt;
    }
    if (a.kidx[m] >= 0) return;
    // ---- k = 0 linear modes                       slab.py:400-445, dpsolver.py:189-218
    double* o = a.k0out;
    double ai1, ai2, A_b, A_t, pib = wi[0].x, pit = wi[1].x, pbb, ptt;
    int check = 0;
    if (a.mode == 0) {
        A_b = -(a.cb * eo[0].x);
        A_t = -(a.ct * eo[1].x);
        ai1 = (a.eps_b * (a.cb * wo[2].x + A_b) - a.eps * wi[2].x - sb.x) / a.eps;
        ai2 = (a.eps_t * (a.ct * wo[3].x + A_t) - a.eps * wi[3].x + st.x) / a.eps;
        pbb = a.cb * wo[0].x;
        ptt = a.ct * wo[1].x;
        check = 1;
    } else {
        double s0b = (a.mode == 1) ? sb.x : 0.0, s0t = (a.mode == 1) ? st.x : 0.0;
        ai1 = -ei[0].x - s0b / a.eps;
        ai2 = -ei[1].x + s0t / a.eps;
        A_b = ai1; A_t = ai2;
        pbb = pib; ptt = pit;
    }
    double ref = fmax(fmax(fabs(ai1), fabs(ai2)), fabs(a.k0_scale));
    double disc = ref > 0 ? fabs(ai1 - ai2) / ref : 0.0;
    if (check && disc > 1e-2) atomicOr(a.flags, FLAG_K0_FAIL);
    else if (check && disc > 1e-3) atomicOr(a.flags, FLAG_K0_WARN);
    double A_i = 0.5 * (ai1 + ai2);
    o[0] = ai1; o[1] = ai2; o[2] = disc; o[3] = A_i; o[4] = A_b; o[5] = A_t;
    o[6] = pib; o[7] = pit; o[8] = pbb; o[9] = ptt;
    a.scal[0] = A_i;
}

// ---------------------------------------------------------------------------
// The per-mode solve, one thread per (mode, grid) column, split over kernels
// so each holds only its own pass's registers (one fused kernel needed 254
// registers and 8 warps / SM; split: 1.22 -> 1.10 ms at C4).  Scratch
// columns (row stride 2M of [Nz][2][M]): A = y'' (ypp), B = Thomas d / x
// (the scaled rhs f_sc is re-derived from the raw DCT column where needed:
// 1.10 -> 1.06 ms against keeping a third column); the column state -- c0, c1, the refinement's Schur rhs r2 and the
// deferred last update dc -- is carried in a.bst between the kernels:
//   pass 0: forward sweep + descend -> c (or the k = 0 solve, bvp.py:281-296);
//   pass 1: a refinement's forward pass (the first materialises y'' as it
//           reads it) -> r2                              bvp.py:229-246
//   pass 3: its descend -> dc; the last refinement's y'' update is deferred
//   pass 2: y'' (+ the deferred update) -> y = Q y'' + c0 T0 + c1 T1, y'
//           (downward recurrence, chebyshev.py:68-79), wall values and the
//           iDCT inputs (in-slab grid), then the lane-pair finish of
//           bvp_final_kernel (mismatch, moments, k = 0; finish_mode).
// ---------------------------------------------------------------------------
template <int PASS>
__device__ __forceinline__ void solve_mode_pass(const BvpArgs& a, int64_t m, int g,
                                                double2 wv[4], double2 ends[2], bool emit) {
    const int n = a.Nz;
    const int64_t M = a.M, RS = 2 * M;
    const double2* __restrict__ raw = a.ext + g * M + m;
    double2* __restrict__ A = a.scrA + g * M + m;
    double2* __restrict__ B = a.scrB + g * M + m;
    double2* __restrict__ st = a.bst + g * M + m;          // state s at st[s * RS]
    const double* __restrict__ q_lo = a.mp.q_lo;
    const double* __restrict__ q_dg = a.mp.q_dg;
    const double* __restrict__ q_hi = a.mp.q_hi;
    const double* __restrict__ e_lo = a.mp.e_lo;
    const double* __restrict__ e_hi = a.mp.e_hi;
    const double base = -(a.half * a.half) / a.eps * a.inv_nxy;
    auto fsc_at = [&](int k) -> double2 { return cscale(raw[(int64_t)k * RS], base); };
    const int u = a.kidx[m];
    const bool defer = u >= 0 && a.refine > 0;
    const double* __restrict__ cp = nullptr; const double* __restrict__ iv = nullptr;
    const double* __restrict__ aib = nullptr; const double* __restrict__ cr0 = nullptr;
    const double* __restrict__ cr1 = nullptr;
    double kap = 0, k2 = 0, S00 = 0, S01 = 0, S10 = 0, S11 = 0;
    if (u >= 0) {
        cp = a.fac + ((int64_t)u * FAC_ROWS + FAC_CP) * n;
        iv = a.fac + ((int64_t)u * FAC_ROWS + FAC_INV) * n;
        aib = a.fac + ((int64_t)u * FAC_ROWS + FAC_AINVB) * n;
        cr0 = a.fac + ((int64_t)u * FAC_ROWS + FAC_C0) * n;
        cr1 = a.fac + ((int64_t)u * FAC_ROWS + FAC_C1) * n;
        kap = a.kappa[u]; k2 = kap * kap;
        S00 = a.sinv[4 * u]; S01 = a.sinv[4 * u + 1];
        S10 = a.sinv[4 * u + 2]; S11 = a.sinv[4 * u + 3];
    }
    constexpr int CH = 4;
    auto descend = [&](double2& s0, double2& s1) {
        double2 xp1 = make_double2(0, 0), xp2 = make_double2(0, 0);
        s0 = make_double2(0, 0); s1 = make_double2(0, 0);
        for (int k0 = n - 1; k0 >= 0; k0 -= CH) {
            double2 dv[CH]; double cpv[CH], c0r[CH], c1r[CH];
#pragma unroll
            for (int j = 0; j < CH; ++j) {
                const int k = k0 - j;
                if (k >= 0) { dv[j] = B[(int64_t)k * RS]; cpv[j] = cp[k]; c0r[j] = cr0[k]; c1r[j] = cr1[k]; }
            }
#pragma unroll
            for (int j = 0; j < CH; ++j) {
                const int k = k0 - j;
                if (k >= 0) {
                    const double2 x = (k + 2 < n) ? cfma(-cpv[j], xp2, dv[j]) : dv[j];
                    B[(int64_t)k * RS] = x;
                    s0 = cfma(c0r[j], x, s0);
                    s1 = cfma(c1r[j], x, s1);
                    xp2 = xp1; xp1 = x;
                }
            }
        }
    };
    auto update_a = [&](double2 v0, double2 v1, bool accumulate) {
        for (int k0 = 0; k0 < n; k0 += CH) {
            double2 bv[CH], av[CH]; double ab[CH];
#pragma unroll
            for (int j = 0; j < CH; ++j) {
                const int k = k0 + j;
                if (k < n) {
                    bv[j] = B[(int64_t)k * RS]; ab[j] = aib[k];
                    if (accumulate) av[j] = A[(int64_t)k * RS];
                }
            }
#pragma unroll
            for (int j = 0; j < CH; ++j) {
                const int k = k0 + j;
                if (k < n) {
                    double2 y = cfma(-ab[j], (k & 1) ? v1 : v0, bv[j]);
                    if (accumulate) y = cadd(av[j], y);
                    A[(int64_t)k * RS] = y;
                }
            }
        }
    };
    if constexpr (PASS == 0) {
        double2 c0v = make_double2(0, 0), c1v = make_double2(0, 0);
        if (u < 0) {                           // k = 0: y'' = f, y(z0) = y(z1) = 0   bvp.py:281-296
            for (int k = 0; k < n; ++k) A[(int64_t)k * RS] = fsc_at(k);
            double2 P = make_double2(0, 0), Qs = make_double2(0, 0);
            for (int k = 1; k < n; ++k) {
                double2 y = cscale(A[(int64_t)k * RS], q_dg[k]);
                if (k >= 2) y = cadd(y, cscale(A[(int64_t)(k - 2) * RS], q_lo[k]));
                if (k + 2 < n) y = cadd(y, cscale(A[(int64_t)(k + 2) * RS], q_hi[k]));
                P = cadd(P, y);
                Qs = (k & 1) ? csub(Qs, y) : cadd(Qs, y);
            }
            c0v = cscale(cadd(P, Qs), -0.5);
            c1v = cscale(csub(Qs, P), 0.5);
        } else {
            double2 dm1 = make_double2(0, 0), dm2 = make_double2(0, 0);
            for (int k0 = 0; k0 < n; k0 += CH) {
                double2 rv[CH]; double ivv[CH];
#pragma unroll
                for (int j = 0; j < CH; ++j) {
                    const int k = k0 + j;
                    if (k < n) { rv[j] = fsc_at(k); ivv[j] = iv[k]; }
                }
#pragma unroll
                for (int j = 0; j < CH; ++j) {
                    const int k = k0 + j;
                    if (k < n) {
                        const double2 r = rv[j];
                        const double2 d = (k < 2) ? cscale(r, ivv[j])
                                                  : cscale(cfma(k2 * q_lo[k], dm2, r), ivv[j]);
                        B[(int64_t)k * RS] = d;
                        dm2 = dm1; dm1 = d;
                    }
                }
            }
            double2 s0, s1;
            descend(s0, s1);
            c0v = make_double2(S00 * s0.x + S01 * s1.x, S00 * s0.y + S01 * s1.y);
            c1v = make_double2(S10 * s0.x + S11 * s1.x, S10 * s0.y + S11 * s1.y);
            if (a.refine <= 0) update_a(c0v, c1v, false);
        }
        st[0] = c0v; st[RS] = c1v;
    } else if constexpr (PASS == 1) {
        // one refinement's forward pass (iteration a.iter): y'' window,
        // residual, Thomas forward sweep; the Schur rhs r2 into the state
        if (!defer) return;
        const double2 c0v = st[0], c1v = st[RS];
        {
            const bool mat = a.iter == 0;
            auto ypp0 = [&](int k) -> double2 {
                return cfma(-aib[k], (k & 1) ? c1v : c0v, B[(int64_t)k * RS]);
            };
            double2 yq_sum = make_double2(0, 0), yq_sgn = make_double2(0, 0);
            double2 ye_sum = make_double2(0, 0), ye_sgn = make_double2(0, 0);
            double2 ym2 = make_double2(0, 0), ym1 = make_double2(0, 0);
            double2 y0 = mat ? ypp0(0) : A[0];
            double2 yp1 = (n > 1) ? (mat ? ypp0(1) : A[RS]) : make_double2(0, 0);
            double2 dm1 = make_double2(0, 0), dm2 = make_double2(0, 0);
            for (int k0 = 0; k0 < n; k0 += CH) {
                double2 ap[CH], fv[CH]; double ivv[CH], abv[CH];
#pragma unroll
                for (int j = 0; j < CH; ++j) {
                    const int k = k0 + j;
                    if (k < n) {
                        ap[j] = (k + 2 < n) ? (mat ? B : A)[(int64_t)(k + 2) * RS]
                                            : make_double2(0, 0);
                        abv[j] = (mat && k + 2 < n) ? aib[k + 2] : 0.0;
                        fv[j] = fsc_at(k);            // f_sc re-derived from the raw column
                        ivv[j] = iv[k];
                    }
                }
#pragma unroll
                for (int j = 0; j < CH; ++j) {
                    const int k = k0 + j;
                    if (k < n) {
                        double2 yp2 = ap[j];
                        if (mat && k + 2 < n) yp2 = cfma(-abv[j], (k & 1) ? c1v : c0v, yp2);
                        if (mat) A[(int64_t)k * RS] = y0;
                        double2 yq = make_double2(0, 0), ye = make_double2(0, 0);
                        if (k > 0) {
                            yq = cscale(y0, q_dg[k]);
                            if (k >= 2) yq = cadd(yq, cscale(ym2, q_lo[k]));
                            if (k + 2 < n) yq = cadd(yq, cscale(yp2, q_hi[k]));
                            ye = cscale(ym1, e_lo[k]);
                            if (k + 1 < n) ye = cadd(ye, cscale(yp1, e_hi[k]));
                        }
                        double2 r = csub(fv[j], csub(y0, cscale(yq, k2)));
                        if (k == 0) r = cadd(r, cscale(c0v, k2));
                        if (k == 1) r = cadd(r, cscale(c1v, k2));
                        yq_sum = cadd(yq_sum, yq); ye_sum = cadd(ye_sum, ye);
                        if (k & 1) { yq_sgn = csub(yq_sgn, yq); ye_sgn = csub(ye_sgn, ye); }
                        else { yq_sgn = cadd(yq_sgn, yq); ye_sgn = cadd(ye_sgn, ye); }
                        const double2 d = (k < 2) ? cscale(r, ivv[j])
                                                  : cscale(cfma(k2 * q_lo[k], dm2, r), ivv[j]);
                        B[(int64_t)k * RS] = d;
                        dm2 = dm1; dm1 = d;
                        ym2 = ym1; ym1 = y0; y0 = yp1; yp1 = yp2;
                    }
                }
            }
            st[4 * RS] = cscale(cadd(cadd(ye_sum, cscale(yq_sum, kap)),
                                     cadd(cscale(c0v, kap), cscale(c1v, 1.0 + kap))), -1.0);
            st[5 * RS] = cscale(cadd(csub(ye_sgn, cscale(yq_sgn, kap)),
                                     cadd(cscale(c0v, -kap), cscale(c1v, 1.0 + kap))), -1.0);
        }
    } else if constexpr (PASS == 3) {
        // the refinement's descend and correction dc; the last one's y''
        // update is deferred into pass 2
        if (!defer) return;
        double2 t0, t1;
        descend(t0, t1);
        t0 = csub(t0, st[4 * RS]); t1 = csub(t1, st[5 * RS]);
        const double2 dc0 = make_double2(S00 * t0.x + S01 * t1.x, S00 * t0.y + S01 * t1.y);
        const double2 dc1 = make_double2(S10 * t0.x + S11 * t1.x, S10 * t0.y + S11 * t1.y);
        if (a.iter + 1 < a.refine) update_a(dc0, dc1, true);
        else { st[2 * RS] = dc0; st[3 * RS] = dc1; }   // applied by pass 2
        st[0] = cadd(st[0], dc0);
        st[RS] = cadd(st[RS], dc1);
    } else {
        const double2 c0v = st[0], c1v = st[RS];
        const double2 pd0 = defer ? st[2 * RS] : make_double2(0, 0);
        const double2 pd1 = defer ? st[3 * RS] : make_double2(0, 0);
        auto ypp = [&](int k) -> double2 {
            const double2 av = A[(int64_t)k * RS];
            if (!defer) return av;
            return cadd(av, cfma(-aib[k], (k & 1) ? pd1 : pd0, B[(int64_t)k * RS]));
        };
        const double dscale = 2.0 / (a.z1 - a.z0);
        double2 w_y0 = make_double2(0, 0), w_yH = make_double2(0, 0);
        double2 w_d0 = make_double2(0, 0), w_dH = make_double2(0, 0);
        double2 d_sum = make_double2(0, 0), d_sgn = make_double2(0, 0);
        double2 bp1 = make_double2(0, 0), bp2 = make_double2(0, 0);
        double2 ynext = make_double2(0, 0);
        double2* out_y = a.ext + 0 * M + m;
        double2* out_d = a.ext + 1 * M + m;
        constexpr int CHF = 4;
        double2 ap2 = make_double2(0, 0), ap1 = make_double2(0, 0);
        double2 a0 = ypp(n - 1);
        double2 am1 = (n >= 2) ? ypp(n - 2) : make_double2(0, 0);
        for (int k0 = n - 1; k0 >= 0; k0 -= CHF) {
            double2 amv[CHF];
#pragma unroll
            for (int j = 0; j < CHF; ++j) {
                const int k = k0 - j;
                amv[j] = (k >= 2) ? ypp(k - 2) : make_double2(0, 0);
            }
#pragma unroll
            for (int j = 0; j < CHF; ++j) {
                const int k = k0 - j;
                if (k < 0) break;
                const double2 am2 = amv[j];
                double2 y = make_double2(0, 0);
                if (k > 0) {
                    y = cscale(a0, q_dg[k]);
                    if (k >= 2) y = cadd(y, cscale(am2, q_lo[k]));
                    if (k + 2 < n) y = cadd(y, cscale(ap2, q_hi[k]));
                }
                if (k == 0) y = cadd(y, c0v);
                if (k == 1) y = cadd(y, c1v);
                double2 b;
                if (k == n - 1) b = make_double2(0, 0);
                else if (k == n - 2) b = cscale(ynext, 2.0 * (n - 1));
                else b = cadd(bp2, cscale(ynext, 2.0 * (k + 1)));
                const double2 bs = cscale((k == 0) ? cscale(b, 0.5) : b, dscale);
                w_y0 = cfma(a.tw0[k], y, w_y0);
                w_yH = cfma(a.twH[k], y, w_yH);
                w_d0 = cfma(a.tw0[k], bs, w_d0);
                w_dH = cfma(a.twH[k], bs, w_dH);
                d_sum = cadd(d_sum, bs);
                d_sgn = (k & 1) ? csub(d_sgn, bs) : cadd(d_sgn, bs);
                if (a.keep) a.keep[((int64_t)k * 2 + g) * M + m] = y;
                if (emit) {
                    out_y[(int64_t)k * RS] = y;
                    out_d[(int64_t)k * RS] = bs;
                }
                bp2 = bp1; bp1 = b; ynext = y;
                ap2 = ap1; ap1 = a0; a0 = am1; am1 = am2;
            }
        }
        wv[0] = w_y0; wv[1] = w_yH; wv[2] = w_d0; wv[3] = w_dH;
        ends[0] = d_sgn; ends[1] = d_sum;
    }
}

template <int PASS, int MINB>
__global__ void __launch_bounds__(128, MINB) bvp_pass_kernel(BvpArgs a) {
    const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int g = (int)(tid & 1);
    const int64_t m = tid >> 1;
    if (m >= a.Mv || !(a.two || g == 1)) return;
    double2 w[4], e[2];
    solve_mode_pass<PASS>(a, m, g, w, e, false);
}

template <int MINB>
__global__ void __launch_bounds__(64, MINB) bvp_final_kernel(BvpArgs a) {
    const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int g = (int)(tid & 1);
    const int64_t mm = tid >> 1;
    const bool valid = mm < a.Mv;
    const int64_t m = valid ? mm : (a.Mv > 0 ? a.Mv - 1 : 0);
    double2 w[4], e[2];
    for (int q = 0; q < 4; ++q) w[q] = make_double2(0, 0);
    e[0] = e[1] = make_double2(0, 0);
    if (valid && (a.two || g == 1)) solve_mode_pass<2>(a, m, g, w, e, g == 1);
    double2 wo[4], eo[2], wi[4], ei[2];
    for (int q = 0; q < 4; ++q) {
        double2 o;
        o.x = __shfl_xor_sync(0xffffffffu, w[q].x, 1);
        o.y = __shfl_xor_sync(0xffffffffu, w[q].y, 1);
        wo[q] = o; wi[q] = w[q];
    }
    for (int q = 0; q < 2; ++q) {
        double2 o;
        o.x = __shfl_xor_sync(0xffffffffu, e[q].x, 1);
        o.y = __shfl_xor_sync(0xffffffffu, e[q].y, 1);
        eo[q] = o; ei[q] = e[q];
    }
    if (!valid || g == 0) return;
    finish_mode(a, m, wi, ei, wo, eo);
}


// ---------------------------------------------------------------------------
// Small problems: the mode BVP with a WARP per (mode, grid) column.  With a
// few thousand modes (the paper's N_xy = 88: 3960) the lane-pair kernel runs
// ~8000 threads, one or two warps per SM, each walking ~14 dependent sweeps
// of Nz rows -- latency, not bandwidth.  Here the parity-split Thomas sweeps
// (bvp.py:76-90, 216-227), the derivative recurrence (chebyshev.py:68-79)
// and the Schur / wall sums are chunked warp scans: lane l owns rows
// [l C, (l+1) C), C = ceil(Nz / 32), composes its chunk's affine maps, one
// 5-step shuffle scan carries each chain into every chunk, and the chunk is
// swept again.  The column, its y'' and Thomas scratch, the k-only maps and
// the mode's per-|k| factor rows are staged in shared memory (coalesced), so
// a sweep costs ~C + 5 dependent steps instead of Nz.  At the north-star
// size (33 K modes) the lane-pair kernel is faster (1.27 vs 1.61 ms): the
// dispatch takes this kernel below BVPW_MAX_MODES.
// ---------------------------------------------------------------------------
constexpr int BVPW_MODES = 2;                   // modes per CTA (x 2 grids = warps)
constexpr int64_t BVPW_MAX_MODES = 12000;
constexpr int BVPW_MAPS = 7;                    // q_lo q_dg q_hi e_lo e_hi tw0 twH
constexpr int BVPW_FACS = 5;                    // cp inv aib c0 c1 (FAC_* order)
constexpr unsigned BFULL = 0xffffffffu;

__host__ __device__ inline int bvpw_dbl(int n) {         // maps + factors, 16 B aligned
    return ((BVPW_MAPS + BVPW_MODES * BVPW_FACS) * n + 1) & ~1;
}
__host__ __device__ inline size_t bvpw_smem(int n) {
    return (size_t)bvpw_dbl(n) * 8 + (size_t)2 * BVPW_MODES * 3 * n * 16;
}

__device__ __forceinline__ double2 shfl_up2(double2 v, int o) {
    return make_double2(__shfl_up_sync(BFULL, v.x, o), __shfl_up_sync(BFULL, v.y, o));
}
__device__ __forceinline__ double2 shfl_down2(double2 v, int o) {
    return make_double2(__shfl_down_sync(BFULL, v.x, o), __shfl_down_sync(BFULL, v.y, o));
}
__device__ __forceinline__ double2 warp_sum2(double2 v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        v.x += __shfl_xor_sync(BFULL, v.x, o);
        v.y += __shfl_xor_sync(BFULL, v.y, o);
    }
    return v;
}

// Carry of an affine chain x_next = a x_prev + b across the warp's chunks:
// (a, b) is the composition of this lane's chunk for each parity; returns
// the value entering this lane's chunk (the chain starts from 0).  up: the
// chain runs with the lane index (forward sweep), else against it.
__device__ __forceinline__ void chain_carry(double (&a)[2], double2 (&b)[2], bool up, int lane,
                                            double2 (&in)[2]) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
#pragma unroll
        for (int q = 0; q < 2; ++q) {
            const double ap = up ? __shfl_up_sync(BFULL, a[q], o) : __shfl_down_sync(BFULL, a[q], o);
            const double2 bp = up ? shfl_up2(b[q], o) : shfl_down2(b[q], o);
            if (up ? lane >= o : lane + o < 32) {
                b[q] = make_double2(fma(a[q], bp.x, b[q].x), fma(a[q], bp.y, b[q].y));
                a[q] *= ap;
            }
        }
    }
#pragma unroll
    for (int q = 0; q < 2; ++q) {
        const double2 v = up ? shfl_up2(b[q], 1) : shfl_down2(b[q], 1);
        const bool first = up ? lane == 0 : lane == 31;
        in[q] = first ? make_double2(0, 0) : v;
    }
}

// exclusive suffix sums of the lane totals, per parity (against the lane index)
__device__ __forceinline__ void suffix_carry(double2 (&t)[2], int lane, double2 (&in)[2]) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
#pragma unroll
        for (int q = 0; q < 2; ++q) {
            const double2 v = shfl_down2(t[q], o);
            if (lane + o < 32) t[q] = cadd(t[q], v);
        }
    }
#pragma unroll
    for (int q = 0; q < 2; ++q) {
        const double2 v = shfl_down2(t[q], 1);
        in[q] = lane == 31 ? make_double2(0, 0) : v;
    }
}

__global__ void __launch_bounds__(64 * BVPW_MODES) bvp_warp_kernel(BvpArgs a) {
    extern __shared__ double2 bsm[];
    __shared__ double2 wall[2 * BVPW_MODES][6];
    const int n = a.Nz;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g = warp & 1, mi = warp >> 1;
    const int64_t mb = (int64_t)blockIdx.x * BVPW_MODES;
    const int64_t m = mb + mi;
    const bool valid = m < a.Mv;
    double* maps = reinterpret_cast<double*>(bsm);
    double* facs = maps + BVPW_MAPS * n;
    double2* cols = reinterpret_cast<double2*>(maps + bvpw_dbl(n));
    const double* srcmap[BVPW_MAPS] = {a.mp.q_lo, a.mp.q_dg, a.mp.q_hi, a.mp.e_lo, a.mp.e_hi,
                                       a.tw0, a.twH};
    constexpr int U = 8;                         // loads in flight per thread
    {
        const int tot = BVPW_MAPS * n;
        for (int b0 = 0; b0 < tot; b0 += U * blockDim.x) {
            double v[U];
#pragma unroll
            for (int j = 0; j < U; ++j) {
                const int e = b0 + j * blockDim.x + tid;
                v[j] = e < tot ? __ldg(srcmap[e / n] + e % n) : 0.0;
            }
#pragma unroll
            for (int j = 0; j < U; ++j) {
                const int e = b0 + j * blockDim.x + tid;
                if (e < tot) maps[e] = v[j];
            }
        }
    }
    {
        const int tot = BVPW_MODES * BVPW_FACS * n;
        for (int b0 = 0; b0 < tot; b0 += U * blockDim.x) {
            double v[U];
#pragma unroll
            for (int j = 0; j < U; ++j) {
                const int e = b0 + j * blockDim.x + tid;
                const int md = e / (BVPW_FACS * n), r = e - md * BVPW_FACS * n;
                const int64_t mm = mb + md;
                const int u = (e < tot && mm < a.Mv) ? a.kidx[mm] : -1;
                v[j] = u >= 0 ? __ldg(a.fac + (int64_t)u * FAC_ROWS * n + r) : 0.0;
            }
#pragma unroll
            for (int j = 0; j < U; ++j) {
                const int e = b0 + j * blockDim.x + tid;
                if (e < tot) facs[e] = v[j];
            }
        }
    }
    // the columns' Chebyshev coefficients: row k holds 2 grids x the CTA's
    // modes (two contiguous runs)
    const int64_t RS = 2 * a.M;
    const double base = -(a.half * a.half) / a.eps * a.inv_nxy;
    {
        const int tot = n * 2 * BVPW_MODES;
        for (int b0 = 0; b0 < tot; b0 += U * blockDim.x) {
            double2 v[U];
#pragma unroll
            for (int j = 0; j < U; ++j) {
                const int e = b0 + j * blockDim.x + tid;
                const int k = e / (2 * BVPW_MODES), r = e - k * 2 * BVPW_MODES;
                const int gg = r / BVPW_MODES, md = r - gg * BVPW_MODES;
                const int64_t mm = mb + md;
                v[j] = (e < tot && mm < a.Mv) ? a.ext[(int64_t)k * RS + gg * a.M + mm]
                                              : make_double2(0, 0);
            }
#pragma unroll
            for (int j = 0; j < U; ++j) {
                const int e = b0 + j * blockDim.x + tid;
                if (e < tot) {
                    const int k = e / (2 * BVPW_MODES), r = e - k * 2 * BVPW_MODES;
                    const int gg = r / BVPW_MODES, md = r - gg * BVPW_MODES;
                    cols[(size_t)(2 * md + gg) * 3 * n + k] = cscale(v[j], base);
                }
            }
        }
    }
    __syncthreads();
    const double* q_lo = maps;
    const double* q_dg = maps + n;
    const double* q_hi = maps + 2 * n;
    const double* e_lo = maps + 3 * n;
    const double* e_hi = maps + 4 * n;
    const double* tw0 = maps + 5 * n;
    const double* twH = maps + 6 * n;
    double2* F = cols + (size_t)warp * 3 * n;    // right-hand side f_sc
    double2* A = F + n;                          // y''
    double2* B = A + n;                          // Thomas d / x
    const int C = (n + 31) / 32, k0 = lane * C, k1 = min(n, k0 + C);
    double2 w_out[4], e_out[2];
    for (int q = 0; q < 4; ++q) w_out[q] = make_double2(0, 0);
    e_out[0] = e_out[1] = make_double2(0, 0);
    const bool solve = valid && (a.two || g == 1);
    if (solve) {                                  // warp-uniform
        const int u = a.kidx[m];
        double2 c0v = make_double2(0, 0), c1v = make_double2(0, 0);
        auto yq_at = [&](int k) -> double2 {      // (Q y'')_k, k > 0
            double2 y = cscale(A[k], q_dg[k]);
            if (k >= 2) y = cadd(y, cscale(A[k - 2], q_lo[k]));
            if (k + 2 < n) y = cadd(y, cscale(A[k + 2], q_hi[k]));
            return y;
        };
        if (u < 0) {
            // ---- k = 0: y'' = f, y(z0) = y(z1) = 0           bvp.py:281-296
            for (int k = k0; k < k1; ++k) A[k] = F[k];
            __syncwarp();
            double2 P = make_double2(0, 0), Qs = make_double2(0, 0);
            for (int k = max(k0, 1); k < k1; ++k) {
                const double2 y = yq_at(k);
                P = cadd(P, y);
                Qs = (k & 1) ? csub(Qs, y) : cadd(Qs, y);
            }
            P = warp_sum2(P); Qs = warp_sum2(Qs);
            c0v = cscale(cadd(P, Qs), -0.5);
            c1v = cscale(csub(Qs, P), 0.5);
        } else {
            const double* fm = facs + (size_t)mi * BVPW_FACS * n;
            const double* cp = fm + FAC_CP * n;
            const double* iv = fm + FAC_INV * n;
            const double* aib = fm + FAC_AINVB * n;
            const double* cr0 = fm + FAC_C0 * n;
            const double* cr1 = fm + FAC_C1 * n;
            const double kap = a.kappa[u], k2 = kap * kap;
            const double S00 = a.sinv[4 * u], S01 = a.sinv[4 * u + 1];
            const double S10 = a.sinv[4 * u + 2], S11 = a.sinv[4 * u + 3];
            // forward sweep d_k = alpha_k d_{k-2} + beta_k, alpha_k = k^2 q_lo
            // iv, beta_k = r_k iv; r = F (first) or the residual in B
            auto forward = [&](bool from_f) {
                double ca[2] = {1.0, 1.0};
                double2 cb[2] = {make_double2(0, 0), make_double2(0, 0)};
                for (int k = k0; k < k1; ++k) {
                    const int q = k & 1;
                    const double al = k >= 2 ? k2 * q_lo[k] * iv[k] : 0.0;
                    const double2 be = cscale(from_f ? F[k] : B[k], iv[k]);
                    cb[q] = make_double2(fma(al, cb[q].x, be.x), fma(al, cb[q].y, be.y));
                    ca[q] *= al;
                }
                double2 in[2];
                chain_carry(ca, cb, true, lane, in);
                for (int k = k0; k < k1; ++k) {
                    const int q = k & 1;
                    const double al = k >= 2 ? k2 * q_lo[k] * iv[k] : 0.0;
                    const double2 be = cscale(from_f ? F[k] : B[k], iv[k]);
                    const double2 d = make_double2(fma(al, in[q].x, be.x), fma(al, in[q].y, be.y));
                    B[k] = d;
                    in[q] = d;
                }
                __syncwarp();
            };
            // backward sweep x_k = -cp_k x_{k+2} + d_k; Schur rhs C.x
            auto backward = [&](double2& s0, double2& s1) {
                double ca[2] = {1.0, 1.0};
                double2 cb[2] = {make_double2(0, 0), make_double2(0, 0)};
                for (int k = k1 - 1; k >= k0; --k) {
                    const int q = k & 1;
                    const double ga = k + 2 < n ? -cp[k] : 0.0;
                    const double2 d = B[k];
                    cb[q] = make_double2(fma(ga, cb[q].x, d.x), fma(ga, cb[q].y, d.y));
                    ca[q] *= ga;
                }
                double2 in[2];
                chain_carry(ca, cb, false, lane, in);
                s0 = make_double2(0, 0); s1 = make_double2(0, 0);
                for (int k = k1 - 1; k >= k0; --k) {
                    const int q = k & 1;
                    const double ga = k + 2 < n ? -cp[k] : 0.0;
                    const double2 d = B[k];
                    const double2 x = make_double2(fma(ga, in[q].x, d.x), fma(ga, in[q].y, d.y));
                    B[k] = x;
                    in[q] = x;
                    s0 = cfma(cr0[k], x, s0);
                    s1 = cfma(cr1[k], x, s1);
                }
                s0 = warp_sum2(s0); s1 = warp_sum2(s1);
                __syncwarp();
            };
            auto update = [&](double2 v0, double2 v1, bool accumulate) {
                for (int k = k0; k < k1; ++k) {
                    double2 y = cfma(-aib[k], (k & 1) ? v1 : v0, B[k]);
                    if (accumulate) y = cadd(A[k], y);
                    A[k] = y;
                }
                __syncwarp();
            };
            double2 s0, s1;
            forward(true);
            backward(s0, s1);
            c0v = make_double2(S00 * s0.x + S01 * s1.x, S00 * s0.y + S01 * s1.y);
            c1v = make_double2(S10 * s0.x + S11 * s1.x, S10 * s0.y + S11 * s1.y);
            update(c0v, c1v, false);
            for (int it = 0; it < a.refine; ++it) {     // bvp.py:229-246,268-273
                double2 yq_sum = make_double2(0, 0), yq_sgn = make_double2(0, 0);
                double2 ye_sum = make_double2(0, 0), ye_sgn = make_double2(0, 0);
                for (int k = k0; k < k1; ++k) {
                    double2 yq = make_double2(0, 0), ye = make_double2(0, 0);
                    if (k > 0) {
                        yq = yq_at(k);
                        ye = cscale(A[k - 1], e_lo[k]);
                        if (k + 1 < n) ye = cadd(ye, cscale(A[k + 1], e_hi[k]));
                    }
                    double2 r = csub(F[k], csub(A[k], cscale(yq, k2)));
                    if (k == 0) r = cadd(r, cscale(c0v, k2));
                    if (k == 1) r = cadd(r, cscale(c1v, k2));
                    yq_sum = cadd(yq_sum, yq); ye_sum = cadd(ye_sum, ye);
                    if (k & 1) { yq_sgn = csub(yq_sgn, yq); ye_sgn = csub(ye_sgn, ye); }
                    else { yq_sgn = cadd(yq_sgn, yq); ye_sgn = cadd(ye_sgn, ye); }
                    B[k] = r;
                }
                yq_sum = warp_sum2(yq_sum); ye_sum = warp_sum2(ye_sum);
                yq_sgn = warp_sum2(yq_sgn); ye_sgn = warp_sum2(ye_sgn);
                __syncwarp();
                const double2 r20 = cscale(cadd(cadd(ye_sum, cscale(yq_sum, kap)),
                                                cadd(cscale(c0v, kap), cscale(c1v, 1.0 + kap))), -1.0);
                const double2 r21 = cscale(cadd(csub(ye_sgn, cscale(yq_sgn, kap)),
                                                cadd(cscale(c0v, -kap), cscale(c1v, 1.0 + kap))), -1.0);
                forward(false);
                double2 t0, t1;
                backward(t0, t1);
                t0 = csub(t0, r20); t1 = csub(t1, r21);
                const double2 dc0 = make_double2(S00 * t0.x + S01 * t1.x, S00 * t0.y + S01 * t1.y);
                const double2 dc1 = make_double2(S10 * t0.x + S11 * t1.x, S10 * t0.y + S11 * t1.y);
                update(dc0, dc1, true);
                c0v = cadd(c0v, dc0);
                c1v = cadd(c1v, dc1);
            }
        }
        // ---- y = Q y'' + c0 T0 + c1 T1 (into F), the derivative b by suffix
        // sums of w_j = 2 j y_j over each parity chain (into B), wall values
        for (int k = k0; k < k1; ++k) {
            double2 y = k > 0 ? yq_at(k) : make_double2(0, 0);
            if (k == 0) y = cadd(y, c0v);
            if (k == 1) y = cadd(y, c1v);
            F[k] = y;
        }
        __syncwarp();
        double2 tot[2] = {make_double2(0, 0), make_double2(0, 0)};
        for (int k = k0; k < k1; ++k) tot[k & 1] = cfma(2.0 * k, F[k], tot[k & 1]);
        double2 run[2];
        suffix_carry(tot, lane, run);
        const double dscale = 2.0 / (a.z1 - a.z0);
        double2 w_y0 = make_double2(0, 0), w_yH = make_double2(0, 0);
        double2 w_d0 = make_double2(0, 0), w_dH = make_double2(0, 0);
        double2 d_sum = make_double2(0, 0), d_sgn = make_double2(0, 0);
        for (int k = k1 - 1; k >= k0; --k) {
            const double2 y = F[k];
            const double2 b = run[(k + 1) & 1];       // sum of w_j, j > k, j = k+1 mod 2
            run[k & 1] = cfma(2.0 * k, y, run[k & 1]);
            const double2 bs = cscale(k == 0 ? cscale(b, 0.5) : b, dscale);
            B[k] = bs;
            w_y0 = cfma(tw0[k], y, w_y0);
            w_yH = cfma(twH[k], y, w_yH);
            w_d0 = cfma(tw0[k], bs, w_d0);
            w_dH = cfma(twH[k], bs, w_dH);
            d_sum = cadd(d_sum, bs);
            d_sgn = (k & 1) ? csub(d_sgn, bs) : cadd(d_sgn, bs);
        }
        w_out[0] = warp_sum2(w_y0); w_out[1] = warp_sum2(w_yH);
        w_out[2] = warp_sum2(w_d0); w_out[3] = warp_sum2(w_dH);
        e_out[0] = warp_sum2(d_sgn); e_out[1] = warp_sum2(d_sum);
    }
    if (lane == 0) {
        for (int q = 0; q < 4; ++q) wall[warp][q] = w_out[q];
        wall[warp][4] = e_out[0]; wall[warp][5] = e_out[1];
    }
    __syncthreads();
    // coalesced stores: psi (F) and dpsi (B) coefficients of the in-slab
    // columns for the iDCT (slot 0 / 1 of ext), the debug copy of both grids
    for (int e = tid; e < n * 2 * BVPW_MODES; e += blockDim.x) {
        const int k = e / (2 * BVPW_MODES), r = e - k * 2 * BVPW_MODES;
        const int slot = r / BVPW_MODES, md = r - slot * BVPW_MODES;
        const int64_t mm = mb + md;
        if (mm >= a.Mv) continue;
        const double2* col = cols + (size_t)(2 * md + 1) * 3 * n;
        a.ext[(int64_t)k * RS + slot * a.M + mm] = slot ? col[2 * n + k] : col[k];
        if (a.keep && (slot == 1 || a.two))
            a.keep[((int64_t)k * 2 + slot) * a.M + mm] = cols[(size_t)(2 * md + slot) * 3 * n + k];
    }
    if (!valid || g == 0 || lane != 0) return;
    double2 wi[4], ei[2], wo[4], eo[2];
    for (int q = 0; q < 4; ++q) { wi[q] = wall[warp][q]; wo[q] = wall[warp - 1][q]; }
    ei[0] = wall[warp][4]; ei[1] = wall[warp][5];
    eo[0] = wall[warp - 1][4]; eo[1] = wall[warp - 1][5];
    finish_mode(a, m, wi, ei, wo, eo);
}

// ---------------------------------------------------------------------------
// z DCT-I (chebyshev.py:46-65) as hand-written FP64 tensor-core products.
// With the node reflection j -> N - j the (Nz x Nz) transform splits into
// an even-coefficient half acting on s_c = v_c + v_{N-c} and an odd half
// acting on d_c = v_c - v_{N-c}, each of order ~Nz/2 (half the flops).
// A CTA owns DCT_COLS real columns (of the [Nz][W] row layout, W = 4 M:
// two grids x M modes x re/im) for all Nz rows: the folded / coefficient
// columns are staged in shared memory column-major (k contiguous, so the
// B fragments of mma.sync.m8n8k4 are bank-conflict free), the transform
// matrices (zero-padded to multiples of 8 x 4, row-major, L2 resident) feed
// the A fragments.  8 warps: warp w computes parity w / 4 and a quarter of
// its 8-row tiles against all DCT_COLS columns.
// ---------------------------------------------------------------------------
constexpr int DCT_COLS = 32;
constexpr int DCT_MT = 20;                 // max m-tiles per parity (Nz <= 320)

__device__ __forceinline__ void dmma884(double (&c)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c[0]), "+d"(c[1]) : "d"(a), "d"(b));
}

struct DctArgs {
    int n, Pe, Po, P8, P4;       // Nz, parity sizes, padded rows / k
    int tmap;                    // warp -> (parity, tiles) map (zdct_fwd_kernel)
    int64_t W;                   // real columns per row
    const double* De; const double* Do;    // [P8][P4] row-major, zero padded
};

// C[tile rows][0:DCT_COLS] = D[rows][k] * S[k][cols] for this warp's 8-row
// tiles mt0 + ts * i (i < MW)
// parity and half of the row tiles: per k step MW A fragments (global, L2
// resident matrix; prefetched one step ahead) and 4 B fragments (shared)
// feed 4 MW DMMAs.
template <int MW>
__device__ __forceinline__ void dct_mma(const double* __restrict__ D, int P4, int mrows,
                                        const double* __restrict__ Sc, int lane, int mt0, int ts,
                                        double (&acc)[MW][4][2]) {
#pragma unroll
    for (int mt = 0; mt < MW; ++mt)
#pragma unroll
        for (int t = 0; t < 4; ++t) acc[mt][t][0] = acc[mt][t][1] = 0.0;
    const int ar = lane >> 2, ak = lane & 3;
    const double* bp = Sc + ar * P4 + ak;                    // column-major [col][k]
    const double* ap = D + (mt0 * 8 + ar) * P4 + ak;
    const int rs = ts * 8 * P4;                                // row stride between tiles
    double an[MW];
#pragma unroll
    for (int mt = 0; mt < MW; ++mt)
        an[mt] = (mt0 + ts * mt) * 8 < mrows ? __ldg(ap + mt * rs) : 0.0;
    for (int k0 = 0; k0 < P4; k0 += 4) {
        double av[MW];
#pragma unroll
        for (int mt = 0; mt < MW; ++mt) av[mt] = an[mt];
        if (k0 + 4 < P4) {
#pragma unroll
            for (int mt = 0; mt < MW; ++mt)
                an[mt] = (mt0 + ts * mt) * 8 < mrows ? __ldg(ap + mt * rs + k0 + 4) : 0.0;
        }
        double bv[4];
#pragma unroll
        for (int t = 0; t < 4; ++t) bv[t] = bp[t * 8 * P4 + k0];
        // m-tiles past the matrix rows (the last warp's slice) issue no MMA
#pragma unroll
        for (int mt = 0; mt < MW; ++mt)
            if ((mt0 + ts * mt) * 8 < mrows) {
#pragma unroll
                for (int t = 0; t < 4; ++t) dmma884(acc[mt][t], av[mt], bv[t]);
            }
    }
}

// forward: hat rows [n][W] (xy spectra per plane) -> ext rows [n][W]
// (Chebyshev coefficient n in row n, unnormalised as the GEMM form was)
template <int MT, typename TIn = double>
__global__ void __launch_bounds__(256, 2) zdct_fwd_kernel(DctArgs a, const TIn* __restrict__ in,
                                                         double* __restrict__ out) {
    extern __shared__ double sm[];
    double* Se = sm;                                   // [DCT_COLS][P4]
    double* So = sm + DCT_COLS * a.P4;
    const int64_t w0 = (int64_t)blockIdx.x * DCT_COLS;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int N = a.n - 1;
    // fold (s_c, d_c) while staging: lanes run along the columns (coalesced);
    // STG_U items per thread are loaded before any is stored, so 2 STG_U
    // loads are in flight per thread
    constexpr int STG_U = 6;
    const int total = a.P4 * DCT_COLS;
    for (int base = 0; base < total; base += 256 * STG_U) {
        double xv[STG_U], yv[STG_U];
#pragma unroll
        for (int u = 0; u < STG_U; ++u) {
            const int e = base + u * 256 + tid;
            const int c = e / DCT_COLS, col = e - c * DCT_COLS;
            const int64_t w = w0 + col;
            const bool ok = e < total && w < a.W && c < a.Pe;
            xv[u] = ok ? (double)in[(int64_t)c * a.W + w] : 0.0;
            yv[u] = (ok && c < a.Po) ? (double)in[(int64_t)(N - c) * a.W + w] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < STG_U; ++u) {
            const int e = base + u * 256 + tid;
            if (e < total) {
                const int c = e / DCT_COLS, col = e - c * DCT_COLS;
                Se[col * a.P4 + c] = xv[u] + yv[u];
                So[col * a.P4 + c] = xv[u] - yv[u];
            }
        }
    }
    __syncthreads();
    constexpr int MW = (MT + 3) / 4;
    // tmap 1: warp w takes parity w & 1 and the tiles w / 2 + 4 i, so the
    // two warps on each SM sub-partition (w, w + 4) share its DMMA unit with
    // balanced tile counts (9 / 9 / 8 / 8 of the 34 at Nz = 258, where the
    // contiguous split (tmap 0) gives 10 / 10 / 10 / 4)
    const int par = a.tmap ? (warp & 1) : (warp >> 2);
    const int mt0 = a.tmap ? (warp >> 1) : (warp & 3) * MW, ts = a.tmap ? 4 : 1;
    const int rows = par ? a.Po : a.Pe;
    double acc[MW][4][2];
    dct_mma<MW>(par ? a.Do : a.De, a.P4, a.P8, par ? So : Se, lane, mt0, ts, acc);
#pragma unroll
    for (int mt = 0; mt < MW; ++mt) {
        const int i = (mt0 + ts * mt) * 8 + (lane >> 2);
        if (i >= rows) continue;
        const int64_t row = 2 * (int64_t)i + par;
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            const int64_t w = w0 + t * 8 + 2 * (lane & 3);
            if (w + 1 < a.W)
                *reinterpret_cast<double2*>(out + row * a.W + w) =
                    make_double2(acc[mt][t][0], acc[mt][t][1]);
            else if (w < a.W)
                out[row * a.W + w] = acc[mt][t][0];
        }
    }
}

// inverse + assembly: the iDCT of the psi and dpsi/dz coefficient columns of
// DCT_COLS / 4 modes (ext rows [n][W]: slot 0 = psi, slot 1 = dpsi at column
// offset 2 M), the node values v_j = E_j + O_j, v_{N-j} = E_j - O_j, the
// harmonic correction on the fly and the i k multipliers -> spec [n][4][M]
// (slab.py:335-353)
struct AsmArgs2 {
    const double2* mom; const double* kx; const double* ky; const double* kmag;
    const unsigned char* sel; const double* z;
    int Nx, Ny, Nyh; int64_t M, Mv, m0;
    int w0, w1, corr, forces;
    double rb, rt, H;
};

template <int MT, typename TOut = double2>
__global__ void __launch_bounds__(256, 2) zdct_inv_kernel(DctArgs a, AsmArgs2 q,
                                                         const double* __restrict__ ext,
                                                         TOut* __restrict__ spec) {
    extern __shared__ double sm[];
    constexpr int MPB = DCT_COLS / 4;                  // modes per CTA
    double* Ce = sm;                                   // [DCT_COLS][P4] even coefficients
    double* Co = sm + DCT_COLS * a.P4;                 // odd
    const int64_t mb = (int64_t)blockIdx.x * MPB;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    // column col: slot = col / 16 (psi, dpsi), mode mb + (col % 16) / 2, re/im
    constexpr int STG_U = 6;
    const int total = a.P4 * DCT_COLS;
    for (int base = 0; base < total; base += 256 * STG_U) {
        double cev[STG_U], cov[STG_U];
#pragma unroll
        for (int u = 0; u < STG_U; ++u) {
            const int e = base + u * 256 + tid;
            const int i = e / DCT_COLS, col = e - i * DCT_COLS;
            const int slot = col >> 4, r = col & 15;
            const int64_t m = mb + (r >> 1);
            const int64_t w = slot * 2 * q.M + 2 * m + (r & 1);
            const bool ok = e < total && m < q.Mv;
            cev[u] = (ok && i < a.Pe) ? ext[(2 * (int64_t)i) * a.W + w] : 0.0;
            cov[u] = (ok && i < a.Po) ? ext[(2 * (int64_t)i + 1) * a.W + w] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < STG_U; ++u) {
            const int e = base + u * 256 + tid;
            if (e < total) {
                const int i = e / DCT_COLS, col = e - i * DCT_COLS;
                Ce[col * a.P4 + i] = cev[u];
                Co[col * a.P4 + i] = cov[u];
            }
        }
    }
    __syncthreads();
    constexpr int MW = (MT + 3) / 4;
    const int par = a.tmap ? (warp & 1) : (warp >> 2);
    const int mt0 = a.tmap ? (warp >> 1) : (warp & 3) * MW, ts = a.tmap ? 4 : 1;
    double acc[MW][4][2];
    dct_mma<MW>(par ? a.Do : a.De, a.P4, a.P8, par ? Co : Ce, lane, mt0, ts, acc);
    __syncthreads();                                   // coefficients consumed
    // E (par 0) / O (par 1) node halves back to shared memory, row-major
    double* EO = sm;                                   // [2][P8][DCT_COLS]
#pragma unroll
    for (int mt = 0; mt < MW; ++mt) {
        const int j = (mt0 + ts * mt) * 8 + (lane >> 2);
        if (j >= a.P8) continue;
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            const int col = t * 8 + 2 * (lane & 3);
            double* dst = EO + ((int64_t)par * a.P8 + j) * DCT_COLS + col;
            dst[0] = acc[mt][t][0];
            dst[1] = acc[mt][t][1];
        }
    }
    // per-mode constants of the CTA's MPB modes, once per CTA (the i k
    // multipliers need a 64-bit division of the mode index)
    __shared__ double s_ik[MPB][2];
    if (tid < MPB) {
        const int64_t m = mb + tid;
        double ikx = 0.0, iky = 0.0;
        if (q.forces && m < q.Mv) {
            const int64_t gm = q.m0 + m;
            const int ix = (int)(gm / q.Nyh), iy = (int)(gm % q.Nyh);
            ikx = (q.Nx % 2 == 0 && ix == q.Nx / 2) ? 0.0 : q.kx[ix];
            iky = (q.Ny % 2 == 0 && iy == q.Ny / 2) ? 0.0 : q.ky[iy];
        }
        s_ik[tid][0] = ikx; s_ik[tid][1] = iky;
    }
    __syncthreads();
    const int N = a.n - 1;
    for (int e = tid; e < a.n * MPB; e += blockDim.x) {
        const int j = e / MPB, mi = e - j * MPB;
        const int64_t m = mb + mi;
        if (m >= q.Mv) continue;
        const bool lo = j < a.Pe;
        const int r = lo ? j : N - j;
        const double* Er = EO + (int64_t)r * DCT_COLS;
        const double* Or = EO + ((int64_t)a.P8 + r) * DCT_COLS;
        double2 v = make_double2(Er[2 * mi], Er[2 * mi + 1]);
        double2 d = make_double2(Er[16 + 2 * mi], Er[16 + 2 * mi + 1]);
        if (r < a.Po) {
            const double2 ov = make_double2(Or[2 * mi], Or[2 * mi + 1]);
            const double2 od = make_double2(Or[16 + 2 * mi], Or[16 + 2 * mi + 1]);
            v = lo ? cadd(v, ov) : csub(v, ov);
            d = lo ? cadd(d, od) : csub(d, od);
        }
        if (q.corr && q.sel[m] && j >= q.w0 && j < q.w1) {
            const double k = q.kmag[m], z = q.z[j];
            // exp(-u) by exp_neg (valid for |u| <= 700; clamped: beyond it the
            // terms are < 1e-304 of the others) instead of libm exp
            auto ex = [](double u) { return exp_neg(fmin(fmax(u, -700.0), 700.0)); };
            const double e1 = ex(k * z), e2 = ex(k * (q.H - z));
            const double e3 = ex(k * (q.H + z)), e4 = ex(k * (2.0 * q.H - z));
            const double pb = (q.rt + 1.0) * e1 - (q.rt - 1.0) * e4;
            const double pt = -(q.rb + 1.0) * e2 + (q.rb - 1.0) * e3;
            const double db = -k * ((q.rt + 1.0) * e1 + (q.rt - 1.0) * e4);
            const double dt = -k * ((q.rb + 1.0) * e2 + (q.rb - 1.0) * e3);
            const double2 mbv = q.mom[2 * m], mtv = q.mom[2 * m + 1];
            v = cadd(v, cadd(cscale(mbv, pb), cscale(mtv, pt)));
            d = cadd(d, cadd(cscale(mbv, db), cscale(mtv, dt)));
        }
        TOut* out = spec + (int64_t)j * 4 * q.M + m;
        auto mk = [](double re, double im) {
            TOut o;
            o.x = re; o.y = im;
            return o;
        };
        out[0] = mk(v.x, v.y);
        if (q.forces) {
            const double ikx = s_ik[mi][0], iky = s_ik[mi][1];
            out[q.M] = mk(-ikx * v.y, ikx * v.x);            // i kx v
            out[2 * q.M] = mk(-iky * v.y, iky * v.x);        // i ky v
            out[3 * q.M] = mk(d.x, d.y);
        }
    }
}

Maps maps_of(Plan* p, const double* base) {
    const int n = p->Nz;
    Maps mp;
    mp.e_lo = base; mp.e_hi = base + n; mp.q_lo = base + 2 * n;
    mp.q_dg = base + 3 * n; mp.q_hi = base + 4 * n;
    mp.ue = base + 5 * n; mp.uq = base + 6 * n; mp.ve = base + 7 * n; mp.vq = base + 8 * n;
    return mp;
}

}  // namespace

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
void factor_bvp(Plan* p) {
    const int n = p->Nz;
    // integration maps (bvp.py:21-54) and BC column sums (bvp.py:110-121)
    std::vector<double> h(9 * (size_t)n, 0.0);
    double *e_lo = &h[0], *e_hi = &h[n], *q_lo = &h[2 * n], *q_dg = &h[3 * n], *q_hi = &h[4 * n];
    if (n > 1) { e_lo[1] = 1.0; e_hi[1] = -0.5; q_dg[1] = -0.125; q_hi[1] = 0.125; }
    if (n > 2) { e_lo[2] = 0.25; e_hi[2] = -0.25; q_lo[2] = 0.25; q_dg[2] = -1.0 / 6.0; q_hi[2] = 1.0 / 24.0; }
    for (int m = 3; m < n; ++m) {
        e_lo[m] = 0.5 / m;
        e_hi[m] = -0.5 / m;
        q_lo[m] = 1.0 / (4.0 * m * (m - 1));
        q_dg[m] = -0.5 / ((double)m * m - 1.0);
        q_hi[m] = 1.0 / (4.0 * m * (m + 1));
    }
    auto colsums = [&](const std::vector<double>& w, double* ue, double* uq) {
        for (int j = 0; j < n - 1; ++j) ue[j] += w[j + 1] * e_lo[j + 1];
        for (int j = 1; j < n; ++j) ue[j] += w[j - 1] * e_hi[j - 1];
        for (int j = 0; j < n - 2; ++j) uq[j] += w[j + 2] * q_lo[j + 2];
        for (int j = 0; j < n; ++j) uq[j] += w[j] * q_dg[j];
        for (int j = 2; j < n; ++j) uq[j] += w[j - 2] * q_hi[j - 2];
    };
    std::vector<double> ones(n, 1.0), sgn(n);
    for (int j = 0; j < n; ++j) sgn[j] = (j % 2 == 0) ? 1.0 : -1.0;
    colsums(ones, &h[5 * n], &h[6 * n]);
    colsums(sgn, &h[7 * n], &h[8 * n]);
    p->d_maps = dalloc<double>(p, h.size());
    SE_CUDA(cudaMemcpy(p->d_maps, h.data(), h.size() * sizeof(double), cudaMemcpyHostToDevice));
    // DCT-I matrices, chebyshev.py:46-65 with the node flip:
    //  a_n = w_n/(2N) sum_j g_j cos(pi n (N-j)/N) v_j,  g = 1 at the ends else 2,
    //        w_n = 2 for interior n else 1
    //  v_j = sum_n cos(pi n (N-j)/N) a_n
    // Both are split by the node reflection j -> N - j (F[n][N-j] = (-1)^n
    // F[n][j], I[N-j][n] = (-1)^n I[j][n]): even / odd coefficient rows
    // need only the symmetric / antisymmetric node combinations, so each
    // transform is two GEMMs of half the order (half the flops).
    {
        const int N = n - 1;
        const int Pe = (n + 1) / 2, Po = n / 2;
        auto Fv = [&](int r, int c) {
            const long long nm = (long long)r * (N - c) % (2 * N);
            const double g = (c == 0 || c == N) ? 1.0 : 2.0;
            const double w = (r == 0 || r == N) ? 1.0 : 2.0;
            return w / (2.0 * N) * g * std::cos(M_PI * (double)nm / N);
        };
        auto Iv = [&](int r, int c) {
            const long long nm = (long long)c * (N - r) % (2 * N);
            return std::cos(M_PI * (double)nm / N);
        };
        // row-major, zero padded to P8 rows x P4 columns (the DMMA tiles):
        // forward even / odd (coefficient rows, folded-node columns) and
        // inverse even / odd (node rows, coefficient columns)
        const int P8 = ((Pe + 7) / 8) * 8, P4 = ((Pe + 3) / 4) * 4;
        if (P8 / 8 > DCT_MT) throw Error(SE_ERR_VALUE, "Nz too large for the z transform kernels");
        p->dct_p8 = P8; p->dct_p4 = P4;
        const size_t blk = (size_t)P8 * P4;
        std::vector<double> F(2 * blk, 0.0), I(2 * blk, 0.0);
        for (int i = 0; i < Pe; ++i)
            for (int c = 0; c < Pe; ++c) F[(size_t)i * P4 + c] = Fv(2 * i, c);
        for (int i = 0; i < Po; ++i)
            for (int c = 0; c < Po; ++c) F[blk + (size_t)i * P4 + c] = Fv(2 * i + 1, c);
        for (int r = 0; r < Pe; ++r)
            for (int i = 0; i < Pe; ++i) I[(size_t)r * P4 + i] = Iv(r, 2 * i);
        for (int r = 0; r < Po; ++r)
            for (int i = 0; i < Po; ++i) I[blk + (size_t)r * P4 + i] = Iv(r, 2 * i + 1);
        p->d_dct_fwd = dalloc<double>(p, F.size());
        p->d_dct_inv = dalloc<double>(p, I.size());
        SE_CUDA(cudaMemcpy(p->d_dct_fwd, F.data(), F.size() * sizeof(double), cudaMemcpyHostToDevice));
        SE_CUDA(cudaMemcpy(p->d_dct_inv, I.data(), I.size() * sizeof(double), cudaMemcpyHostToDevice));
    }
    const int nu = std::max(p->n_uniq, 1);
    p->d_fac = dalloc<double>(p, (size_t)nu * FAC_ROWS * n);
    p->d_sinv = dalloc<double>(p, 4 * (size_t)nu);
    p->d_kappa = dalloc<double>(p, (size_t)nu);
    int* d_bad = dalloc<int>(p, 1);
    SE_CUDA(cudaMemset(d_bad, 0, sizeof(int)));
    if (p->n_uniq > 0) {
        FactorArgs a{maps_of(p, p->d_maps), n, p->n_uniq, 0.5 * (p->P.z1 - p->P.z0),
                     p->d_kuniq, p->d_fac, p->d_sinv, p->d_kappa, d_bad};
        factor_kernel<<<(p->n_uniq + 127) / 128, 128, 0, p->stream>>>(a);
        SE_LAUNCHED(p);
    }
    int bad = 0;
    SE_CUDA(cudaMemcpyAsync(&bad, d_bad, sizeof(int), cudaMemcpyDeviceToHost, p->stream));
    SE_CUDA(cudaStreamSynchronize(p->stream));
    if (bad) throw Error(SE_ERR_LINALG, "ill-conditioned Schur block in the mode BVP factorisation");
}

static DctArgs dct_args(Plan* p, const double* mats, int64_t W) {
    DctArgs a{};
    a.n = p->Nz; a.Pe = (p->Nz + 1) / 2; a.Po = p->Nz / 2;
    a.P8 = p->dct_p8; a.P4 = p->dct_p4; a.W = W;
    a.De = mats; a.Do = mats + (size_t)a.P8 * a.P4;
    static const int tmap = [] {
        const char* e = std::getenv("SE_DCT_TMAP");
        return e ? std::atoi(e) : 1;
    }();
    a.tmap = tmap;
    return a;
}

// dispatch on the number of 8-row tiles per parity (accumulators in registers)
#define SE_DCT_LAUNCH(KERNEL, MT, GRID, SMEM, ST, ...)                                   \
    do {                                                                                  \
        auto kfn = KERNEL<MT, DCT_T>;                                                     \
        SE_CUDA(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize,     \
                                     (int)(SMEM)));                                       \
        kfn<<<GRID, 256, SMEM, ST>>>(__VA_ARGS__);                                        \
    } while (0)

#define SE_DCT_DISPATCH(KERNEL, MTV, GRID, SMEM, ST, ...)                                 \
    switch (MTV) {                                                                        \
        case 1: SE_DCT_LAUNCH(KERNEL, 1, GRID, SMEM, ST, __VA_ARGS__); break;             \
        case 2: SE_DCT_LAUNCH(KERNEL, 2, GRID, SMEM, ST, __VA_ARGS__); break;             \
        case 3: SE_DCT_LAUNCH(KERNEL, 3, GRID, SMEM, ST, __VA_ARGS__); break;             \
        case 4: SE_DCT_LAUNCH(KERNEL, 4, GRID, SMEM, ST, __VA_ARGS__); break;             \
        case 5: SE_DCT_LAUNCH(KERNEL, 5, GRID, SMEM, ST, __VA_ARGS__); break;             \
        case 6: SE_DCT_LAUNCH(KERNEL, 6, GRID, SMEM, ST, __VA_ARGS__); break;             \
        case 7: SE_DCT_LAUNCH(KERNEL, 7, GRID, SMEM, ST, __VA_ARGS__); break;             \
        case 8: SE_DCT_LAUNCH(KERNEL, 8, GRID, SMEM, ST, __VA_ARGS__); break;             \
        case 9: SE_DCT_LAUNCH(KERNEL, 9, GRID, SMEM, ST, __VA_ARGS__); break;             \
        case 10: SE_DCT_LAUNCH(KERNEL, 10, GRID, SMEM, ST, __VA_ARGS__); break;           \
        case 11: SE_DCT_LAUNCH(KERNEL, 11, GRID, SMEM, ST, __VA_ARGS__); break;           \
        case 12: SE_DCT_LAUNCH(KERNEL, 12, GRID, SMEM, ST, __VA_ARGS__); break;           \
        case 13: SE_DCT_LAUNCH(KERNEL, 13, GRID, SMEM, ST, __VA_ARGS__); break;           \
        case 14: SE_DCT_LAUNCH(KERNEL, 14, GRID, SMEM, ST, __VA_ARGS__); break;           \
        case 15: SE_DCT_LAUNCH(KERNEL, 15, GRID, SMEM, ST, __VA_ARGS__); break;           \
        case 16: SE_DCT_LAUNCH(KERNEL, 16, GRID, SMEM, ST, __VA_ARGS__); break;           \
        case 17: SE_DCT_LAUNCH(KERNEL, 17, GRID, SMEM, ST, __VA_ARGS__); break;           \
        case 18: SE_DCT_LAUNCH(KERNEL, 18, GRID, SMEM, ST, __VA_ARGS__); break;           \
        case 19: SE_DCT_LAUNCH(KERNEL, 19, GRID, SMEM, ST, __VA_ARGS__); break;           \
        case 20: SE_DCT_LAUNCH(KERNEL, 20, GRID, SMEM, ST, __VA_ARGS__); break;           \
        default: throw Error(SE_ERR_VALUE, "Nz outside the z transform kernels' range"); \
    }

// z DCT-I of the xy spectra in d_hat ([Nz][2][M] for the mode view) into
// the Chebyshev coefficients d_ext (same layout)
void z_forward(Plan* p, const ModeView& v) {
    const int64_t W = 4 * v.M;
    const DctArgs a = dct_args(p, p->d_dct_fwd, W);
    const size_t smem = 2 * (size_t)DCT_COLS * a.P4 * sizeof(double);
    const unsigned grid = (unsigned)((W + DCT_COLS - 1) / DCT_COLS);
    double* out = reinterpret_cast<double*>(p->d_ext);
    if (p->g32) {
        using DCT_T = float;
        const float* in = reinterpret_cast<const float*>(p->d_hat32);
        SE_DCT_DISPATCH(zdct_fwd_kernel, a.P8 / 8, grid, smem, p->stream, a, in, out);
    } else {
        using DCT_T = double;
        const double* in = reinterpret_cast<const double*>(p->d_hat);
        SE_DCT_DISPATCH(zdct_fwd_kernel, a.P8 / 8, grid, smem, p->stream, a, in, out);
    }
    SE_LAUNCHED(p);
}

void forward_transforms(Plan* p, bool two_grids) {
    NvtxRange nv("se.forward_transforms");
    (void)two_grids;
    if (p->g32) SE_CUFFT(cufftExecR2C(p->fft_fwd2_f, p->d_rho32, p->d_hat32));
    else SE_CUFFT(cufftExecD2Z(p->fft_fwd2, p->d_rho, p->d_hat));
    z_forward(p, ModeView{p->M, p->M, 0});
}

void bvp_solve(Plan* p, bool two_grids, int mode, bool correction) {
    bvp_solve_view(p, two_grids, mode, correction, ModeView{p->M, p->M, 0});
}

void bvp_solve_view(Plan* p, bool two_grids, int mode, bool correction, const ModeView& v) {
    NvtxRange nv("se.mode_bvp");
    BvpArgs a{};
    const bool whole = v.m0 == 0 && v.M == p->M;
    a.mp = maps_of(p, p->d_maps);
    a.Nz = p->Nz; a.Nx = p->Nx; a.Nyh = p->Nyh; a.M = v.M; a.Mv = v.Mv;
    a.half = 0.5 * (p->P.z1 - p->P.z0);
    a.eps = p->P.eps; a.eps_b = p->P.eps_b; a.eps_t = p->P.eps_t;
    a.cb = 2.0 * p->P.eps / (p->P.eps_b + p->P.eps);
    a.ct = 2.0 * p->P.eps / (p->P.eps_t + p->P.eps);
    a.z0 = p->P.z0; a.z1 = p->P.z1; a.k_max = p->P.k_max; a.k0_scale = p->k0_scale;
    a.refine = p->P.refine; a.two = two_grids ? 1 : 0; a.mode = mode;
    a.correction = correction ? 1 : 0;
    // per-mode tables seen from the view's first mode
    a.kidx = p->d_kidx + v.m0; a.kmag = p->d_kmag + v.m0; a.sel = p->d_sel + v.m0;
    a.fac = p->d_fac; a.sinv = p->d_sinv; a.kappa = p->d_kappa;
    a.tw0 = p->d_tw0; a.twH = p->d_twH;
    a.sbh = reinterpret_cast<const double2*>(p->d_sbh) + v.m0;
    a.sth = reinterpret_cast<const double2*>(p->d_sth) + v.m0;
    a.ext = reinterpret_cast<double2*>(p->d_ext);
    a.scrA = reinterpret_cast<double2*>(p->d_scr);
    a.scrB = a.scrA + (int64_t)p->Nz * 2 * v.M;
    a.inv_nxy = 1.0 / (double)p->NXY;
    a.mom = reinterpret_cast<double2*>(p->d_mom);
    a.mism = whole ? reinterpret_cast<double2*>(p->d_mism) : nullptr;
    a.keep = (whole && p->keep_stages) ? reinterpret_cast<double2*>(p->d_keep) : nullptr;
    a.k0out = p->d_k0; a.scal = p->d_scal; a.flags = p->d_flags;
    a.rb = p->P.eps_b / p->P.eps; a.rt = p->P.eps_t / p->P.eps; a.H = p->P.H;
    p->ktic(1);
    const size_t wsmem = bvpw_smem(p->Nz);
    if (v.Mv <= BVPW_MAX_MODES && wsmem <= 200 * 1024) {
        SE_CUDA(cudaFuncSetAttribute(bvp_warp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)wsmem));
        bvp_warp_kernel<<<(unsigned)((v.Mv + BVPW_MODES - 1) / BVPW_MODES), 64 * BVPW_MODES,
                          wsmem, p->stream>>>(a);
    } else {
        // the lane-per-column solve split over kernels (passes 0, then 1 + 3
        // per refinement, then the final pass with the lane-pair finish):
        // 1.22 -> 1.10 ms at C4 against the fused 254-register kernel
        a.bst = reinterpret_cast<double2*>(p->d_bst);
        const unsigned nb128 = (unsigned)((2 * v.M + 127) / 128);
        const unsigned nb64 = (unsigned)((2 * v.M + 63) / 64);
        bvp_pass_kernel<0, 4><<<nb128, 128, 0, p->stream>>>(a);
        for (int it = 0; it < a.refine; ++it) {
            a.iter = it;
            bvp_pass_kernel<1, 4><<<nb128, 128, 0, p->stream>>>(a);
            bvp_pass_kernel<3, 4><<<nb128, 128, 0, p->stream>>>(a);
        }
        bvp_final_kernel<8><<<nb64, 64, 0, p->stream>>>(a);
    }
    p->ktoc(1);
    SE_LAUNCHED(p);
}

// inverse z DCT-I of the mode view and the assembly of the four spectral
// fields into d_spec ([Nz][4][M] of the view)
void z_inverse_assemble(Plan* p, bool forces, bool correction, const ModeView& v) {
    const int64_t W = 4 * v.M;
    const DctArgs a = dct_args(p, p->d_dct_inv, W);
    AsmArgs2 q{};
    q.mom = reinterpret_cast<const double2*>(p->d_mom);
    q.kx = p->d_kx; q.ky = p->d_ky; q.kmag = p->d_kmag + v.m0; q.sel = p->d_sel + v.m0;
    q.z = p->d_z; q.Nx = p->Nx; q.Ny = p->Ny; q.Nyh = p->Nyh; q.M = v.M;
    q.Mv = v.Mv; q.m0 = v.m0;
    q.w0 = p->win0; q.w1 = p->win1; q.corr = correction ? 1 : 0; q.forces = forces ? 1 : 0;
    q.rb = p->P.eps_b / p->P.eps; q.rt = p->P.eps_t / p->P.eps; q.H = p->P.H;
    const size_t smem = std::max(2 * (size_t)DCT_COLS * a.P4, 2 * (size_t)a.P8 * DCT_COLS) *
                        sizeof(double);
    const unsigned grid = (unsigned)((v.Mv + DCT_COLS / 4 - 1) / (DCT_COLS / 4));
    const double* ext = reinterpret_cast<const double*>(p->d_ext);
    if (grid > 0) {
        if (p->g32) {
            using DCT_T = float2;
            float2* spec = reinterpret_cast<float2*>(p->d_spec32);
            SE_DCT_DISPATCH(zdct_inv_kernel, a.P8 / 8, grid, smem, p->stream, a, q, ext, spec);
        } else {
            using DCT_T = double2;
            double2* spec = reinterpret_cast<double2*>(p->d_spec);
            SE_DCT_DISPATCH(zdct_inv_kernel, a.P8 / 8, grid, smem, p->stream, a, q, ext, spec);
        }
        SE_LAUNCHED(p);
    }
}

void inverse_transforms(Plan* p, bool forces, bool correction) {
    NvtxRange nv("se.inverse_transforms");
    z_inverse_assemble(p, forces, correction, ModeView{p->M, p->M, 0});
    if (p->g32) {
        if (forces) SE_CUFFT(cufftExecC2R(p->fft_inv4_f, p->d_spec32, p->d_fields32));
        else SE_CUFFT(cufftExecC2R(p->fft_inv1_f, p->d_spec32, p->d_fields32));
    } else if (forces) {
        SE_CUFFT(cufftExecZ2D(p->fft_inv4, p->d_spec, p->d_fields));
    } else {
        SE_CUFFT(cufftExecZ2D(p->fft_inv1, p->d_spec, p->d_fields));
    }
}

}  // namespace se
