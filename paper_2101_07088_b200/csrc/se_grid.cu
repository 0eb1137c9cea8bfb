// Spreading and interpolation on the uniform-xy x Chebyshev-z grid.
//
// Reference: FourierChebGrid.spread / .interpolate (gridops.py:80-133) with
// the stencils of gridops.py:18-44, called from SlabSolver.solve
// (slab.py:282-289 spread, slab.py:359 interpolate, slab.py:253-256 gamma).
//
// B200 design.  fp64 shared-memory atomics are CAS loops on sm_100a and
// global fp64 atomics cost ~1 op/clk/SM, so the spread is a GATHER: each CTA
// owns an 8x8-column x 32-node tile of the output grid in registers (one
// column x 8 nodes per thread) and streams every source whose stencil
// touches the tile through shared memory, 64 at a time.  The tensor-product
// weights are staged as 8 x-, 8 y- and 32 z-weights per source; a warp skips
// a source whose stencil misses the warp's 4x8-column x 8-node sub-tile
// (uniform branch), so the FMA pipe only sees sources that touch it.  No
// atomics, deterministic order, coalesced stores.  The interpolation is the
// adjoint on the same tiling (4 fields x 4 nodes per thread in registers,
// warp-shuffle reduction, one global atomic per source and tile).
//
// Stencil membership is computed with the reference's exact operation order
// (no FMA contraction: __dmul_rn / __dsub_rn) so the set of grid nodes each
// charge touches is bit-identical to numpy's (gridops.py:20-25, 31-38).
#include <cub/cub.cuh>

#include <cmath>

#include "se_internal.cuh"

namespace se {

namespace {

__device__ __forceinline__ int lower_bound_d(const double* a, int n, double v) {
    int lo = 0, hi = n;              // first k with a[k] >= v
    while (lo < hi) {
        int mid = (lo + hi) >> 1;
        if (a[mid] < v) lo = mid + 1; else hi = mid;
    }
    return lo;
}

__device__ __forceinline__ int upper_bound_d(const double* a, int n, double v) {
    int lo = 0, hi = n;              // first k with a[k] > v
    while (lo < hi) {
        int mid = (lo + hi) >> 1;
        if (a[mid] <= v) lo = mid + 1; else hi = mid;
    }
    return lo;
}

__device__ __forceinline__ int pmod(long long a, int n) {
    long long r = a % n;
    return (int)(r < 0 ? r + n : r);
}

// ---------------------------------------------------------------------------
// source construction: charges (class 0 near a wall / class 1 mid-slab) and
// first images of near-wall charges (class 1)         slab.py:51-82,280-289
// ---------------------------------------------------------------------------
struct SrcArgs {
    const double* pos; const double* q; int64_t n;
    double H, two_HE, fb, ft; int two_grids;
    double4* src; int* cls; int* owner;
};

__global__ void make_sources_kernel(SrcArgs a) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= a.n) return;
    double x = a.pos[3 * i], y = a.pos[3 * i + 1], z = a.pos[3 * i + 2];
    double qi = a.q[i];
    int64_t base = 3 * i;
    if (!a.two_grids) {
        a.src[base] = make_double4(x, y, z, qi);
        a.cls[base] = 1; a.owner[base] = (int)i;
        a.cls[base + 1] = -1; a.cls[base + 2] = -1;
        return;
    }
    bool nb = z < a.two_HE;                       // slab.py:59
    bool nt = z > __dsub_rn(a.H, a.two_HE);       // slab.py:60
    bool over = nb || nt;
    a.src[base] = make_double4(x, y, z, qi);
    a.cls[base] = over ? 0 : 1;
    a.owner[base] = (int)i;
    if (nb && a.fb != 0.0) {                       // bottom image  :67-72
        a.src[base + 1] = make_double4(x, y, -z, a.fb * qi);
        a.cls[base + 1] = 1; a.owner[base + 1] = -1;
    } else {
        a.cls[base + 1] = -1;
    }
    if (nt && a.ft != 0.0) {                       // top image     :73-78
        a.src[base + 2] = make_double4(x, y, __dsub_rn(2.0 * a.H, z), a.ft * qi);
        a.cls[base + 2] = 1; a.owner[base + 2] = -1;
    } else {
        a.cls[base + 2] = -1;
    }
}

struct KeyArgs {
    const double4* src; const int* cls; int64_t total;
    const double* znodes; int Nz; double hx, hy; int Nx, Ny, nbx;
    double rad, z0, z1; int zbits; uint32_t invalid;
    uint32_t* keys; int* perm; int* flags;
};

__global__ void source_keys_kernel(KeyArgs a) {
    int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (s >= a.total) return;
    a.perm[s] = (int)s;
    int c = a.cls[s];
    if (c < 0) { a.keys[s] = a.invalid; return; }
    double4 v = a.src[s];
    if (v.z < a.z0 || v.z > a.z1) atomicOr(a.flags, FLAG_Z_OUTSIDE);
    int cx = pmod((long long)floor(v.x / a.hx), a.Nx);
    int cy = pmod((long long)floor(v.y / a.hy), a.Ny);
    int bin = (cy / TILE) * a.nbx + (cx / TILE);
    int lo = lower_bound_d(a.znodes, a.Nz, __dsub_rn(v.z, a.rad));
    uint32_t seg = (uint32_t)(bin * 2 + c);
    a.keys[s] = (seg << a.zbits) | (uint32_t)lo;
}

__global__ void segment_offsets_kernel(const uint32_t* keys, int64_t total,
                                       int zbits, int nseg, int64_t* seg) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i > total) return;
    int cur = (i < total) ? (int)(keys[i] >> zbits) : nseg + 1;
    int prev = (i == 0) ? -1 : (int)(keys[i - 1] >> zbits);
    if (cur > nseg) cur = nseg + 1;
    for (int k = prev + 1; k <= cur && k <= nseg; ++k) seg[k] = i;
}

// Per-source stencil tables (sorted order).  gridops.py:18-44
struct StencilArgs {
    const double4* src; const int* owner_in; const int* perm;
    const uint32_t* keys; uint32_t invalid_major; int zbits; int64_t total;
    const double* znodes; int Nz;
    double hx, hy, rad, rad_keep, width, norm; int mx, my, wz;
    Stencils st;
};

__global__ void stencil_kernel(StencilArgs a) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= a.total) return;
    if ((a.keys[i] >> a.zbits) >= a.invalid_major) return;
    int s = a.perm[i];
    double4 v = a.src[s];
    const int64_t S = a.st.S;
    // x axis: j0 = floor(x/h); delta = x - (j0+off)*h; keep |delta| <= r(1+1e-12)
    long long jx = (long long)floor(v.x / a.hx);
    for (int o = 0; o <= 2 * a.mx; ++o) {
        double xj = __dmul_rn((double)(jx + o - a.mx), a.hx);
        double d = __dsub_rn(v.x, xj);
        double wt = 0.0;
        if (fabs(d) <= a.rad_keep) {
            double t = d / a.width;
            wt = exp(-0.5 * (t * t)) / a.norm;
        }
        a.st.wx[o * S + i] = wt;
    }
    long long jy = (long long)floor(v.y / a.hy);
    for (int o = 0; o <= 2 * a.my; ++o) {
        double yj = __dmul_rn((double)(jy + o - a.my), a.hy);
        double d = __dsub_rn(v.y, yj);
        double wt = 0.0;
        if (fabs(d) <= a.rad_keep) {
            double t = d / a.width;
            wt = exp(-0.5 * (t * t)) / a.norm;
        }
        a.st.wy[o * S + i] = wt;
    }
    // z axis: nodes in [searchsorted(z-r, left), searchsorted(z+r, right))
    int lo = lower_bound_d(a.znodes, a.Nz, __dsub_rn(v.z, a.rad));
    int hi = upper_bound_d(a.znodes, a.Nz, __dadd_rn(v.z, a.rad));
    for (int t = 0; t < a.wz; ++t) {
        int k = lo + t;
        double wt = 0.0;
        if (k < hi && k < a.Nz) {
            double d = __dsub_rn(v.z, a.znodes[k]);
            if (fabs(d) <= a.rad) {
                double u = d / a.width;
                wt = exp(-0.5 * (u * u)) / a.norm;
            }
        }
        a.st.wzt[t * S + i] = wt;
    }
    a.st.j0x[i] = (int)jx;
    a.st.j0y[i] = (int)jy;
    a.st.lo[i] = lo;
    a.st.q[i] = v.w;
    a.st.owner[i] = a.owner_in[s];
}

// ---------------------------------------------------------------------------
// tile helpers shared by spread and interp
// ---------------------------------------------------------------------------
struct TileArgs {
    Stencils st;
    const int64_t* seg; int nbx, nby;
    int Nx, Ny, Nz; int64_t NXY;
    int Rx, Ry;                  // neighbour bin radius
};

constexpr int MAX_BINS = 49;     // (2*3+1)^2

// Build the list of candidate (bin, class) source ranges for the tile.
template <int TZ>
__device__ void tile_ranges(const TileArgs& a, int bx, int by, int k0, int cls,
                            int* s_lo, int* s_len, int* s_nr, int* s_total) {
    // bins along x / y (deduplicated when the ring wraps onto itself)
    int nxb = (2 * a.Rx + 1 >= a.nbx) ? a.nbx : 2 * a.Rx + 1;
    int nyb = (2 * a.Ry + 1 >= a.nby) ? a.nby : 2 * a.Ry + 1;
    int nr = nxb * nyb;
    int t = threadIdx.x;
    if (t < nr) {
        int ix = t % nxb, iy = t / nxb;
        int bxx = (nxb == a.nbx) ? ix : pmod(bx - a.Rx + ix, a.nbx);
        int byy = (nyb == a.nby) ? iy : pmod(by - a.Ry + iy, a.nby);
        int sg = (byy * a.nbx + bxx) * 2 + cls;
        int64_t b = a.seg[sg], e = a.seg[sg + 1];
        // sources sorted by first node lo: keep lo in [k0 - wz + 1, k0 + TZ - 1]
        int want_lo = k0 - a.st.wz + 1, want_hi = k0 + TZ - 1;
        int64_t l = b, h = e;
        while (l < h) { int64_t mid = (l + h) >> 1; if (a.st.lo[mid] < want_lo) l = mid + 1; else h = mid; }
        int64_t first = l;
        h = e;
        while (l < h) { int64_t mid = (l + h) >> 1; if (a.st.lo[mid] <= want_hi) l = mid + 1; else h = mid; }
        s_lo[t] = (int)first;
        s_len[t] = (int)(l - first);
    }
    __syncthreads();
    if (t == 0) {
        int tot = 0;
        for (int r = 0; r < nr; ++r) tot += s_len[r];
        *s_nr = nr;
        *s_total = tot;
    }
    __syncthreads();
}

__device__ __forceinline__ int map_candidate(int idx, const int* s_lo,
                                             const int* s_len, int nr) {
    for (int r = 0; r < nr; ++r) {
        if (idx < s_len[r]) return s_lo[r] + idx;
        idx -= s_len[r];
    }
    return -1;
}

// x (or y) weights of source i at the TILE columns starting at g0.
__device__ __forceinline__ unsigned axis_tile_weights(
        const double* w, int64_t S, int64_t i, int j0, int m, int n, int g0,
        double scale, double* out) {
    unsigned mask = 0;
#pragma unroll
    for (int c = 0; c < TILE; ++c) {
        int g = g0 + c;
        double acc = 0.0;
        if (g < n) {
            int o = pmod((long long)g - j0 + m, n);
            for (; o <= 2 * m; o += n) acc += w[o * S + i];
        }
        acc *= scale;
        out[c] = acc;
        if (acc != 0.0) mask |= 1u << c;
    }
    return mask;
}

// ---------------------------------------------------------------------------
// spread: gather into register tiles                    gridops.py:80-103
// ---------------------------------------------------------------------------
struct SpreadArgs {
    TileArgs t;
    double* rho;                 // [Nz][2][Nx][Ny]
    int two;                     // slot 0 (over) as well as slot 1 (in)
};

__global__ void __launch_bounds__(256) spread_kernel(SpreadArgs a) {
    constexpr int TZ = SPREAD_TZ;       // 32 nodes = 4 groups of 8
    __shared__ double s_wx[CHUNK][TILE];
    __shared__ double s_wy[CHUNK][TILE];
    __shared__ double s_wz[CHUNK][TZ];
    __shared__ unsigned s_xm[CHUNK], s_ym[CHUNK], s_zm[2][CHUNK];
    __shared__ int s_lo[MAX_BINS], s_len[MAX_BINS], s_nr, s_total;

    const TileArgs& A = a.t;
    const int bx = blockIdx.x, by = blockIdx.y, k0 = blockIdx.z * TZ;
    const int gx0 = bx * TILE, gy0 = by * TILE;
    const int t = threadIdx.x;
    const int col = t & 63, tx = col >> 3, ty = col & 7, zg = t >> 6;
    const int warp = t >> 5;
    const unsigned wxbits = 0xFu << (4 * (warp & 1));
    const unsigned wzbit = 1u << zg;
    const int64_t S = A.st.S;

    double acc[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) acc[r] = 0.0;

    const int gx = gx0 + tx, gy = gy0 + ty;
    for (int cls = a.two ? 0 : 1; cls < 2; ++cls) {
        tile_ranges<TZ>(A, bx, by, k0, cls, s_lo, s_len, &s_nr, &s_total);
        const int total = s_total, nr = s_nr;
        for (int base = 0; base < total; base += CHUNK) {
            // ---- stage CHUNK sources: 4 parts (x, y, z lo half, z hi half)
            const int slot = t & (CHUNK - 1), part = t >> 6;
            const int idx = base + slot;
            int i = (idx < total) ? map_candidate(idx, s_lo, s_len, nr) : -1;
            if (part == 0) {
                unsigned m = 0;
                if (i >= 0) m = axis_tile_weights(A.st.wx, S, i, A.st.j0x[i], A.st.mx,
                                                  A.Nx, gx0, A.st.q[i], s_wx[slot]);
                else for (int c = 0; c < TILE; ++c) s_wx[slot][c] = 0.0;
                s_xm[slot] = m;
            } else if (part == 1) {
                unsigned m = 0;
                if (i >= 0) m = axis_tile_weights(A.st.wy, S, i, A.st.j0y[i], A.st.my,
                                                  A.Ny, gy0, 1.0, s_wy[slot]);
                else for (int c = 0; c < TILE; ++c) s_wy[slot][c] = 0.0;
                s_ym[slot] = m;
            } else {
                const int h = part - 2;            // nodes k0 + 16h .. +16
                unsigned m = 0;
                int lo = (i >= 0) ? A.st.lo[i] : 0;
#pragma unroll 4
                for (int r = 0; r < 16; ++r) {
                    int k = k0 + 16 * h + r;
                    int tt = k - lo;
                    double w = 0.0;
                    if (i >= 0 && tt >= 0 && tt < A.st.wz && k < A.Nz)
                        w = A.st.wzt[tt * S + i];
                    s_wz[slot][16 * h + r] = w;
                    if (w != 0.0) m |= 1u << ((16 * h + r) >> 3);
                }
                s_zm[h][slot] = m;
            }
            __syncthreads();
            // ---- accumulate
            const int nloc = min(CHUNK, total - base);
            for (int s = 0; s < nloc; ++s) {
                if ((s_xm[s] & wxbits) && ((s_zm[0][s] | s_zm[1][s]) & wzbit) && s_ym[s]) {
                    const double cxy = s_wx[s][tx] * s_wy[s][ty];
                    const double* wz = &s_wz[s][8 * zg];
#pragma unroll
                    for (int r = 0; r < 8; ++r) acc[r] = fma(cxy, wz[r], acc[r]);
                }
            }
            __syncthreads();
        }
        // ---- store this class's running sum (slot 0 after class 0, 1 after 1)
        if (gx < A.Nx && gy < A.Ny) {
            double* base_ptr = a.rho + (int64_t)(cls) * A.NXY + (int64_t)gx * A.Ny + gy;
#pragma unroll
            for (int r = 0; r < 8; ++r) {
                int k = k0 + 8 * zg + r;
                if (k < A.Nz) base_ptr[(int64_t)k * 2 * A.NXY] = acc[r];
            }
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------
// interpolation of the field stack at the charges (adjoint)   gridops.py:105-133
// ---------------------------------------------------------------------------
struct InterpArgs {
    TileArgs t;
    const double* fields;        // [Nz][4][Nx][Ny]
    const double* znodes; const double* wcc;
    const double* scal;          // scal[0] = A_i
    double* out;                 // [4][N] raw sums
    int64_t N;
    int nf;                      // 1 (potential only) or 4
};

template <int NF>
__global__ void __launch_bounds__(256) interp_kernel(InterpArgs a) {
    constexpr int TZ = INTERP_TZ;       // 16 nodes = 4 groups of 4
    __shared__ double s_wx[CHUNK][TILE];
    __shared__ double s_wy[CHUNK][TILE];
    __shared__ double s_wz[CHUNK][TZ];
    __shared__ unsigned s_xm[CHUNK], s_ym[CHUNK], s_zm[CHUNK];
    __shared__ int s_own[CHUNK];
    __shared__ double s_red[8][CHUNK][NF];
    __shared__ int s_lo[MAX_BINS], s_len[MAX_BINS], s_nr, s_total;

    const TileArgs& A = a.t;
    const int bx = blockIdx.x, by = blockIdx.y, k0 = blockIdx.z * TZ;
    const int gx0 = bx * TILE, gy0 = by * TILE;
    const int t = threadIdx.x;
    const int col = t & 63, tx = col >> 3, ty = col & 7, zg = t >> 6;
    const int warp = t >> 5, lane = t & 31;
    const unsigned wxbits = 0xFu << (4 * (warp & 1));
    const unsigned wzbit = 1u << zg;
    const int64_t S = A.st.S;
    const int gx = gx0 + tx, gy = gy0 + ty;
    const double A_i = a.scal[0];

    // field values of this thread's column x 4 nodes, CC-weighted, with the
    // k = 0 linear terms folded in (psi + A_i z, dpsi + A_i; slab.py:340-352)
    double F[NF][4];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
        int k = k0 + 4 * zg + r;
        bool ok = (k < A.Nz) && (gx < A.Nx) && (gy < A.Ny);
        double wq = ok ? a.wcc[k] : 0.0;
#pragma unroll
        for (int c = 0; c < NF; ++c) {
            double v = 0.0;
            if (ok) {
                v = a.fields[((int64_t)k * 4 + c) * A.NXY + (int64_t)gx * A.Ny + gy];
                if (c == 0) v = v + A_i * a.znodes[k];
                if (c == 3) v = v + A_i;
            }
            F[c][r] = v * wq;
        }
    }

    for (int cls = 0; cls < 2; ++cls) {
        tile_ranges<TZ>(A, bx, by, k0, cls, s_lo, s_len, &s_nr, &s_total);
        const int total = s_total, nr = s_nr;
        for (int base = 0; base < total; base += CHUNK) {
            const int slot = t & (CHUNK - 1), part = t >> 6;
            const int idx = base + slot;
            int i = (idx < total) ? map_candidate(idx, s_lo, s_len, nr) : -1;
            int own = (i >= 0) ? A.st.owner[i] : -1;
            if (own < 0) i = -1;                       // images are not targets
            if (part == 0) {
                unsigned m = 0;
                if (i >= 0) m = axis_tile_weights(A.st.wx, S, i, A.st.j0x[i], A.st.mx,
                                                  A.Nx, gx0, 1.0, s_wx[slot]);
                else for (int c = 0; c < TILE; ++c) s_wx[slot][c] = 0.0;
                s_xm[slot] = m;
                s_own[slot] = own;
            } else if (part == 1) {
                unsigned m = 0;
                if (i >= 0) m = axis_tile_weights(A.st.wy, S, i, A.st.j0y[i], A.st.my,
                                                  A.Ny, gy0, 1.0, s_wy[slot]);
                else for (int c = 0; c < TILE; ++c) s_wy[slot][c] = 0.0;
                s_ym[slot] = m;
            } else if (part == 2) {
                unsigned m = 0;
                int lo = (i >= 0) ? A.st.lo[i] : 0;
#pragma unroll
                for (int r = 0; r < TZ; ++r) {
                    int k = k0 + r;
                    int tt = k - lo;
                    double w = 0.0;
                    if (i >= 0 && tt >= 0 && tt < A.st.wz && k < A.Nz)
                        w = A.st.wzt[tt * S + i];
                    s_wz[slot][r] = w;
                    if (w != 0.0) m |= 1u << (r >> 2);
                }
                s_zm[slot] = m;
            }
            // zero the per-warp reduction slots
            for (int e = t; e < 8 * CHUNK * NF; e += 256) (&s_red[0][0][0])[e] = 0.0;
            __syncthreads();
            const int nloc = min(CHUNK, total - base);
            for (int s = 0; s < nloc; ++s) {
                if ((s_xm[s] & wxbits) && (s_zm[s] & wzbit) && s_ym[s]) {
                    const double wxy = s_wx[s][tx] * s_wy[s][ty];
                    const double* wz = &s_wz[s][4 * zg];
                    double part_c[NF];
#pragma unroll
                    for (int c = 0; c < NF; ++c) {
                        double v = 0.0;
#pragma unroll
                        for (int r = 0; r < 4; ++r) v = fma(wz[r], F[c][r], v);
                        part_c[c] = v * wxy;
                    }
#pragma unroll
                    for (int c = 0; c < NF; ++c) {
#pragma unroll
                        for (int off = 16; off > 0; off >>= 1)
                            part_c[c] += __shfl_xor_sync(0xffffffffu, part_c[c], off);
                    }
                    if (lane == 0) {
#pragma unroll
                        for (int c = 0; c < NF; ++c) s_red[warp][s][c] = part_c[c];
                    }
                }
            }
            __syncthreads();
            // combine the 8 warps and push one atomic per (source, field)
            for (int e = t; e < CHUNK * NF; e += 256) {
                int s = e / NF, c = e % NF;
                if (s < nloc && s_own[s] >= 0) {
                    double v = 0.0;
#pragma unroll
                    for (int w = 0; w < 8; ++w) v += s_red[w][s][c];
                    if (v != 0.0) atomicAdd(&a.out[(int64_t)c * a.N + s_own[s]], v);
                }
            }
            __syncthreads();
        }
    }
}

// ---------------------------------------------------------------------------
// pointwise interpolation of field 0 (psi + A_i z) at arbitrary points with
// an arbitrary width: the gauge (slab.py:253-256,377-384) and the wall nodes
// of the surface-charge energy (slab.py:448-461).  One warp per point.
// ---------------------------------------------------------------------------
struct PointArgs {
    const double* pts; int64_t n;
    const double* fields; const double* znodes; const double* wcc;
    const double* scal; int Nx, Ny, Nz; int64_t NXY;
    double hx, hy, width, rad, rad_keep, norm; int mx, my;
    double* out; int* flags; double z0, z1;
};

__global__ void point_interp_kernel(PointArgs a) {
    int64_t wid = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    int lane = threadIdx.x & 31;
    if (wid >= a.n) return;
    double px = a.pts[3 * wid], py = a.pts[3 * wid + 1], pz = a.pts[3 * wid + 2];
    if (pz < a.z0 || pz > a.z1) { if (lane == 0) atomicOr(a.flags, FLAG_Z_OUTSIDE); }
    const double A_i = a.scal[0];
    long long jx = (long long)floor(px / a.hx), jy = (long long)floor(py / a.hy);
    int lo = lower_bound_d(a.znodes, a.Nz, __dsub_rn(pz, a.rad));
    int hi = upper_bound_d(a.znodes, a.Nz, __dadd_rn(pz, a.rad));
    const int wx = 2 * a.mx + 1, wy = 2 * a.my + 1;
    double sum = 0.0;
    for (int e = lane; e < wx * wy; e += 32) {
        int ox = e / wy, oy = e % wy;
        double dx = __dsub_rn(px, __dmul_rn((double)(jx + ox - a.mx), a.hx));
        double dy = __dsub_rn(py, __dmul_rn((double)(jy + oy - a.my), a.hy));
        if (fabs(dx) > a.rad_keep || fabs(dy) > a.rad_keep) continue;
        double tx = dx / a.width, ty = dy / a.width;
        double wxy = (exp(-0.5 * (tx * tx)) / a.norm) * (exp(-0.5 * (ty * ty)) / a.norm);
        int gx = pmod(jx + ox - a.mx, a.Nx), gy = pmod(jy + oy - a.my, a.Ny);
        double col = 0.0;
        for (int k = lo; k < hi; ++k) {
            double dz = __dsub_rn(pz, a.znodes[k]);
            if (fabs(dz) > a.rad) continue;
            double tz = dz / a.width;
            double wz = exp(-0.5 * (tz * tz)) / a.norm * a.wcc[k];
            double f = a.fields[((int64_t)k * 4) * a.NXY + (int64_t)gx * a.Ny + gy]
                       + A_i * a.znodes[k];
            col += wz * f;
        }
        sum += wxy * col;
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, off);
    if (lane == 0) a.out[wid] = a.hx * a.hy * sum;
}

int zbits_for(int Nz) {
    int b = 1;
    while ((1 << b) <= Nz) ++b;
    return b;
}

}  // namespace

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
void ensure_sources(Plan* p, int64_t n) {
    int64_t cap = 3 * n;
    if (cap <= p->src_cap) return;
    cap = cap < 64 ? 64 : cap;
    Stencils& st = p->ss.st;
    void* olds[] = {p->d_src, p->d_src_cls, p->d_src_owner, p->d_keys,
                    p->d_keys2, p->d_perm, p->d_perm2, p->d_cub, st.j0x,
                    st.j0y, st.lo, st.q, st.wx, st.wy, st.wzt, st.owner};
    for (void* o : olds) dfree(p, o);
    p->d_src = dalloc<double4>(p, cap);
    p->d_src_cls = dalloc<int>(p, cap);
    p->d_src_owner = dalloc<int>(p, cap);
    p->d_keys = dalloc<uint32_t>(p, cap);
    p->d_keys2 = dalloc<uint32_t>(p, cap);
    p->d_perm = dalloc<int>(p, cap);
    p->d_perm2 = dalloc<int>(p, cap);
    size_t bytes = 0;
    SE_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, (uint32_t*)nullptr,
                                            (uint32_t*)nullptr, (int*)nullptr,
                                            (int*)nullptr, (int)cap, 0, 32,
                                            p->stream));
    p->cub_bytes = bytes;
    p->d_cub = dalloc<char>(p, bytes);
    st.S = cap;
    st.mx = p->mx;
    st.my = p->my;
    st.wz = p->wz_max;
    st.j0x = dalloc<int>(p, cap);
    st.j0y = dalloc<int>(p, cap);
    st.lo = dalloc<int>(p, cap);
    st.q = dalloc<double>(p, cap);
    st.wx = dalloc<double>(p, (size_t)(2 * p->mx + 1) * cap);
    st.wy = dalloc<double>(p, (size_t)(2 * p->my + 1) * cap);
    st.wzt = dalloc<double>(p, (size_t)p->wz_max * cap);
    st.owner = dalloc<int>(p, cap);
    p->src_cap = cap;
}

static void launch_make_sources(Plan* p, const double* d_pos, int64_t n, bool two_grids) {
    const int TB = 256;
    SrcArgs sa{d_pos, p->d_q, n, p->P.H, 2.0 * p->P.H_E,
               -(p->P.eps_b - p->P.eps) / (p->P.eps_b + p->P.eps),
               -(p->P.eps_t - p->P.eps) / (p->P.eps_t + p->P.eps),
               two_grids ? 1 : 0, p->d_src, p->d_src_cls, p->d_src_owner};
    if (n > 0) {
        make_sources_kernel<<<(unsigned)((n + TB - 1) / TB), TB, 0, p->stream>>>(sa);
        SE_LAUNCHED(p);
    }
}

void partition_sources(Plan* p, const double* d_pos, int64_t n) {
    int64_t cap = 3 * n;
    if (cap > p->src_cap) {
        void* olds[] = {p->d_src, p->d_src_cls, p->d_src_owner};
        for (void* o : olds) dfree(p, o);
        p->d_src = dalloc<double4>(p, cap);
        p->d_src_cls = dalloc<int>(p, cap);
        p->d_src_owner = dalloc<int>(p, cap);
        p->src_cap = 0;          // the sort buffers were not resized
    }
    launch_make_sources(p, d_pos, n, true);
}

void build_sources(Plan* p, const double* d_pos, int64_t n, bool two_grids) {
    ensure_sources(p, n);
    const int64_t total = 3 * n;
    const int TB = 256;
    launch_make_sources(p, d_pos, n, two_grids);
    SourceSet& ss = p->ss;
    ss.nbx = (p->Nx + TILE - 1) / TILE;
    ss.nby = (p->Ny + TILE - 1) / TILE;
    const int nseg = ss.nbx * ss.nby * 2;
    const int zb = zbits_for(p->Nz);
    uint32_t invalid = (uint32_t)nseg << zb;
    int end_bit = 1;
    while (end_bit < 32 && ((uint64_t)invalid >> end_bit) != 0) ++end_bit;
    if (!ss.seg) ss.seg = dalloc<int64_t>(p, (size_t)nseg + 1);
    uint32_t* keys = p->d_keys;
    uint32_t* keys2 = p->d_keys2;
    if (total > 0) {
        KeyArgs ka{p->d_src, p->d_src_cls, total, p->d_z, p->Nz, p->hx, p->hy,
                   p->Nx, p->Ny, ss.nbx, p->rad, p->P.z0, p->P.z1, zb, invalid,
                   keys, p->d_perm, p->d_flags};
        source_keys_kernel<<<(unsigned)((total + TB - 1) / TB), TB, 0, p->stream>>>(ka);
        SE_LAUNCHED(p);
        size_t bytes = p->cub_bytes;
        SE_CUDA(cub::DeviceRadixSort::SortPairs(p->d_cub, bytes, keys, keys2,
                                                p->d_perm, p->d_perm2, (int)total,
                                                0, end_bit, p->stream));
    }
    segment_offsets_kernel<<<(unsigned)((total + 1 + TB - 1) / TB), TB, 0, p->stream>>>(
        keys2, total, zb, nseg, ss.seg);
    SE_LAUNCHED(p);
    ss.S = total;
    Stencils st = ss.st;
    if (total > 0) {
        StencilArgs sta{p->d_src, p->d_src_owner, p->d_perm2, keys2, (uint32_t)nseg,
                        zb, total, p->d_z, p->Nz, p->hx, p->hy, p->rad,
                        p->rad_keep, p->width, p->norm, p->mx, p->my, p->wz_max, st};
        stencil_kernel<<<(unsigned)((total + TB - 1) / TB), TB, 0, p->stream>>>(sta);
        SE_LAUNCHED(p);
    }
}

static TileArgs tile_args(Plan* p) {
    TileArgs t{};
    t.st = p->ss.st;
    t.seg = p->ss.seg;
    t.nbx = p->ss.nbx;
    t.nby = p->ss.nby;
    t.Nx = p->Nx; t.Ny = p->Ny; t.Nz = p->Nz; t.NXY = p->NXY;
    t.Rx = (p->mx + TILE - 1) / TILE + ((p->Nx % TILE) ? 1 : 0);
    t.Ry = (p->my + TILE - 1) / TILE + ((p->Ny % TILE) ? 1 : 0);
    if ((2 * t.Rx + 1) * (2 * t.Ry + 1) > MAX_BINS)
        throw Error(SE_ERR_VALUE, "stencil half width too large for the tile kernels");
    return t;
}

void spread(Plan* p, bool two_grids) {
    SpreadArgs a{tile_args(p), p->d_rho, two_grids ? 1 : 0};
    dim3 grid(p->ss.nbx, p->ss.nby, (p->Nz + SPREAD_TZ - 1) / SPREAD_TZ);
    spread_kernel<<<grid, 256, 0, p->stream>>>(a);
    SE_LAUNCHED(p);
}

void interp_charges(Plan* p, int64_t n, bool forces) {
    SE_CUDA(cudaMemsetAsync(p->d_far, 0, sizeof(double) * 4 * (size_t)n, p->stream));
    if (n == 0) return;
    InterpArgs a{tile_args(p), p->d_fields, p->d_z, p->d_wcc, p->d_scal, p->d_far,
                 n, forces ? 4 : 1};
    dim3 grid(p->ss.nbx, p->ss.nby, (p->Nz + INTERP_TZ - 1) / INTERP_TZ);
    if (forces) interp_kernel<4><<<grid, 256, 0, p->stream>>>(a);
    else interp_kernel<1><<<grid, 256, 0, p->stream>>>(a);
    SE_LAUNCHED(p);
}

void interp_points(Plan* p, const double* d_pts, int64_t npts, double width,
                   double radius, double* d_out) {
    if (npts == 0) return;
    PointArgs a{};
    a.pts = d_pts; a.n = npts; a.fields = p->d_fields; a.znodes = p->d_z;
    a.wcc = p->d_wcc; a.scal = p->d_scal; a.Nx = p->Nx; a.Ny = p->Ny;
    a.Nz = p->Nz; a.NXY = p->NXY; a.hx = p->hx; a.hy = p->hy;
    a.width = width; a.rad = radius; a.rad_keep = radius + 1e-12 * radius;
    a.norm = std::sqrt(2.0 * M_PI * width * width);
    a.mx = (int)std::floor(radius / p->hx + 1e-12);
    a.my = (int)std::floor(radius / p->hy + 1e-12);
    a.out = d_out; a.flags = p->d_flags; a.z0 = p->P.z0; a.z1 = p->P.z1;
    int64_t threads = npts * 32;
    point_interp_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, p->stream>>>(a);
    SE_LAUNCHED(p);
}

}  // namespace se
