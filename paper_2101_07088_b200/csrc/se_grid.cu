// Spreading and interpolation on the uniform-xy x Chebyshev-z grid.
//
// Reference: FourierChebGrid.spread / .interpolate (gridops.py:80-133) with
// the stencils of gridops.py:18-44, called from SlabSolver.solve
// (slab.py:282-289 spread, slab.py:359 interpolate, slab.py:253-256 gamma).
//
// B200 design.  fp64 shared-memory atomics are CAS loops on sm_100a and
// global fp64 atomics cost ~1 op/clk/SM, so the spread is a GATHER: each CTA
// owns an 8x8-column x 16-node tile of the output grid in DMMA accumulator
// fragments (one warp per 8-node z group, FP64 tensor pipe) and streams every
// source whose stencil touches the tile through shared memory, 64 at a time
// (candidates from the neighbour bins, compacted with warp ballots, weights
// staged with cp.async).  No atomics, deterministic order.  The
// interpolation is charge-stationary instead: warps own groups of 4 charges
// of one 4x4-column bin and walk the union of their stencils, loading each
// field node once for the group; the weights are recomputed exactly.
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
    const double* pos; const double* q; int64_t n; int64_t first;   // charges first..first+n
    double H, two_HE, fb, ft; int two_grids;
    double4* src; int* cls; int* owner;
};

__global__ void make_sources_kernel(SrcArgs a) {
    int64_t li = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (li >= a.n) return;
    const int64_t i = a.first + li;                    // global charge index
    double x = a.pos[3 * i], y = a.pos[3 * i + 1], z = a.pos[3 * i + 2];
    double qi = a.q[i];
    int64_t base = 3 * li;
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
    double hx, hy, rad, rad_keep, inv_width, inv_norm; int mx, my, wz;
    Stencils st;
};

// Two passes per CTA of STENCIL_TB sorted sources: one thread per source
// finds its x / y base columns and z node range (binary searches) and writes
// the per-source arrays; then the CTA computes the record elements
// (wx | wy | wz, one Gaussian each) element-parallel and writes the records
// coalesced -- every exp in flight at once instead of 44 in one thread.
constexpr int STENCIL_TB = 256;

__global__ void __launch_bounds__(STENCIL_TB) stencil_kernel(StencilArgs a) {
    __shared__ double sx[STENCIL_TB], sy[STENCIL_TB], sz[STENCIL_TB];
    __shared__ int sjx[STENCIL_TB], sjy[STENCIL_TB], slo[STENCIL_TB], shi[STENCIL_TB];
    const int t = threadIdx.x;
    const int64_t i0 = blockIdx.x * (int64_t)STENCIL_TB;
    const int64_t i = i0 + t;
    const int rs = a.st.rs;
    // invalid slots sort to the end: the valid ones are a prefix of the CTA
    const bool valid = i < a.total && (a.keys[i] >> a.zbits) < a.invalid_major;
    if (valid) {
        const int s = a.perm[i];
        const double4 v = a.src[s];
        // x / y: j0 = floor(x/h); z: nodes in
        // [searchsorted(z-r, left), searchsorted(z+r, right))   gridops.py:18-44
        const long long jx = (long long)floor(v.x / a.hx);
        const long long jy = (long long)floor(v.y / a.hy);
        const int lo = lower_bound_d(a.znodes, a.Nz, __dsub_rn(v.z, a.rad));
        const int hi = upper_bound_d(a.znodes, a.Nz, __dadd_rn(v.z, a.rad));
        sx[t] = v.x; sy[t] = v.y; sz[t] = v.z;
        sjx[t] = (int)jx; sjy[t] = (int)jy; slo[t] = lo; shi[t] = hi;
        a.st.j0x[i] = (int)jx;
        a.st.j0y[i] = (int)jy;
        a.st.lo[i] = lo;
        a.st.hi[i] = hi < lo + a.wz ? hi : lo + a.wz;
        a.st.q[i] = v.w;
        a.st.owner[i] = a.owner_in[s];
    }
    const int nvalid = __syncthreads_count(valid);
    const int SX = 2 * a.mx + 1, SXY = SX + 2 * a.my + 1;
    // half a warp per record: lanes over its elements, records in turn; the
    // record's scalars are read once per record, not per element
    const int h = t >> 4, hl = t & 15;
    const double hx = a.hx, hy = a.hy, rk = a.rad_keep, rz = a.rad;
    const double iw = a.inv_width, inrm = a.inv_norm;
    const int wz = a.wz, Nz = a.Nz;
    double* const rec0 = a.st.rec + i0 * rs;
    for (int r = h; r < nvalid; r += STENCIL_TB / 16) {
        const double px = sx[r], py = sy[r], pz = sz[r];
        const int bx = sjx[r] - a.mx, by = sjy[r] - a.my - SX, lo = slo[r] - SXY;
        const int zend = min(min(shi[r], Nz), slo[r] + wz) + SXY;   // element bound of z
        double* const out = rec0 + (int64_t)r * rs;
        for (int c = hl; c < rs; c += 16) {
            // one converged Gaussian per element: x / y offsets select their
            // axis, z elements their node (|delta| <= r (1 + 1e-12) on x / y)
            double d, lim;
            bool ok = true;
            if (c < SXY) {
                const bool y = c >= SX;
                const double node = __dmul_rn((double)((y ? by : bx) + c), y ? hy : hx);
                d = __dsub_rn(y ? py : px, node);
                lim = rk;
            } else {
                ok = c < zend;
                d = __dsub_rn(pz, ok ? a.znodes[lo + c] : 0.0);
                lim = rz;
            }
            out[c] = (ok && fabs(d) <= lim) ? gauss_w(d, iw, inrm) : 0.0;
        }
    }
}

// ---------------------------------------------------------------------------
// tile helpers shared by spread and interp
// ---------------------------------------------------------------------------
struct TileArgs {
    Stencils st;
    const int64_t* seg; int nbx, nby;
    int Nx, Ny, Nz; int64_t NXY;
    int Rx, Ry;                  // neighbour bin radius
    int TZ;                      // z nodes per tile of the calling kernel
    int SX, SY, SZ;              // interp partial slots per dimension
};

constexpr int MAX_BINS = 49;     // (2*3+1)^2

// Candidate (bin, class) source ranges of the tile: sources are sorted by
// first z node within each segment, so those that can reach nodes
// [k0, k0 + TZ) form one contiguous range per bin (two binary searches).
template <int TZ>
__device__ void tile_ranges(const TileArgs& a, int bx, int by, int k0, int cls,
                            int* s_lo, int* s_len, int* s_nr, int* s_total) {
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

__device__ __forceinline__ int imod(int a, int n) { int r = a % n; return r < 0 ? r + n : r; }

// 8-byte asynchronous global -> shared copy (LDGSTS) and its completion wait
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
    unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" :: "r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_wait_all() {
    asm volatile("cp.async.wait_all;\n" ::: "memory");
}

// Shared-memory staging of up to CAP sources that touch the CTA tile.
// Rows are per source so the compute loop reads a source's weights with
// broadcast (vector) loads; the fill maps consecutive threads to consecutive
// addresses both in shared memory and in the AoS stencil records.
template <int TZ, int CAP, bool ZW = true>
struct Stage {
    double wx[CAP][TILE];
    double wy[CAP][TILE];
    double wz[ZW ? CAP : 1][TZ];       // ZW = false: the z weights are read from the records
    double q[CAP];
    int idx[CAP], lo[CAP], ox[CAP], oy[CAP];
    unsigned xm[CAP], zm[CAP];
    int wcount[8];
};

// Mask of the TILE columns g0.. lying in the periodic stencil j0-m..j0+m;
// *o0 returns the stencil offset of column g0.
__device__ __forceinline__ unsigned axis_mask(int j0, int m, int n, int g0, int* o0) {
    int o = g0 - j0 + m;
    if ((unsigned)o >= (unsigned)n) o = imod(o, n);
    *o0 = o;
    const int w = 2 * m + 1;
    if (w < 32 && n >= w + TILE) {
        // the stencil covers each column at most once: bits c with
        // o + c <= 2m, and after the periodic wrap those with o + c - n <= 2m
        const unsigned full = (1u << w) - 1u;
        unsigned mask = 0;
        if (o < w) mask = full >> o;
        if (o > n - TILE) mask |= full << (n - o);
        mask &= (1u << TILE) - 1u;
        const int rem = n - g0;
        if (rem < TILE) mask &= (1u << rem) - 1u;
        return mask;
    }
    unsigned mask = 0;
#pragma unroll
    for (int c = 0; c < TILE; ++c) {
        if (g0 + c < n && o <= 2 * m) mask |= 1u << c;
        if (++o == n) o = 0;
    }
    return mask;
}

// One staging round: candidates [cursor, cursor + CAP) are tested against
// the tile, the touching ones are compacted (warp ballots + block prefix)
// and their tile-restricted weights staged.  Returns the staged count.
template <int TZ, int NG, int CAP, bool FOLD_Q, bool ZW = true>
__device__ int stage_round(Stage<TZ, CAP, ZW>& sm, const TileArgs& A, int cursor,
                           int total, const int* s_lo, const int* s_len, int nr,
                           int gx0, int gy0, int k0) {
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    constexpr int NW = CAP / 32;
    bool touch = false;
    int i = -1, lo = 0, ox = 0, oy = 0;
    unsigned xm = 0, zm = 0;
    if (t < CAP && cursor + t < total) {
        i = map_candidate(cursor + t, s_lo, s_len, nr);
        if (i >= 0) {
            lo = A.st.lo[i];
            const int hi = A.st.hi[i];
            xm = axis_mask(A.st.j0x[i], A.st.mx, A.Nx, gx0, &ox);
            const unsigned ym = axis_mask(A.st.j0y[i], A.st.my, A.Ny, gy0, &oy);
            constexpr int per = TZ / NG;
#pragma unroll
            for (int g = 0; g < NG; ++g) {
                const int a0 = k0 + g * per, a1 = a0 + per;
                if (lo < a1 && hi > a0) zm |= 1u << g;
            }
            touch = xm && ym && zm;
        }
    }
    unsigned b = 0;
    if (warp < NW) {
        b = __ballot_sync(0xffffffffu, touch);
        if (lane == 0) sm.wcount[warp] = __popc(b);
    }
    __syncthreads();
    int base = 0, n = 0;
#pragma unroll
    for (int w = 0; w < NW; ++w) {
        const int c = sm.wcount[w];
        if (w < warp) base += c;
        n += c;
    }
    if (touch) {
        const int sl = base + __popc(b & ((1u << lane) - 1u));
        sm.idx[sl] = i; sm.lo[sl] = lo; sm.ox[sl] = ox; sm.oy[sl] = oy;
        sm.xm[sl] = xm; sm.zm[sl] = zm;
        sm.q[sl] = FOLD_Q ? A.st.q[i] : 1.0;
    }
    __syncthreads();
    const int rs = A.st.rs, mx = A.st.mx, my = A.st.my;
    const int yoff = 2 * mx + 1, zoff = yoff + 2 * my + 1;
    const bool simple = A.Nx >= 2 * mx + 1 && A.Ny >= 2 * my + 1;
    // x / y weights: one stencil offset per column when the grid is wider
    // than the stencil (async copies); otherwise sum the wrapped offsets
    for (int e = threadIdx.x; e < n * TILE; e += blockDim.x) {
        const int sl = e / TILE, c = e % TILE;
        const double* rec = A.st.rec + (int64_t)sm.idx[sl] * rs;
        int ox = sm.ox[sl] + c; if (ox >= A.Nx) ox -= A.Nx;
        int oy = sm.oy[sl] + c; if (oy >= A.Ny) oy -= A.Ny;
        const bool inx = gx0 + c < A.Nx, iny = gy0 + c < A.Ny;
        if (simple) {
            if (inx && ox <= 2 * mx) cp_async8(&sm.wx[sl][c], rec + ox); else sm.wx[sl][c] = 0.0;
            if (iny && oy <= 2 * my) cp_async8(&sm.wy[sl][c], rec + yoff + oy); else sm.wy[sl][c] = 0.0;
        } else {
            double wxv = 0.0, wyv = 0.0;
            if (inx) for (; ox <= 2 * mx; ox += A.Nx) wxv += rec[ox];
            if (iny) for (; oy <= 2 * my; oy += A.Ny) wyv += rec[yoff + oy];
            sm.wx[sl][c] = wxv;
            sm.wy[sl][c] = wyv;
        }
    }
    if (ZW)
    for (int e = threadIdx.x; e < n * TZ; e += blockDim.x) {
        const int sl = e / TZ, r = e % TZ;
        const int k = k0 + r, tt = k - sm.lo[sl];
        if (tt >= 0 && tt < A.st.wz && k < A.Nz)
            cp_async8(&sm.wz[sl][r], A.st.rec + (int64_t)sm.idx[sl] * rs + zoff + tt);
        else
            sm.wz[sl][r] = 0.0;
    }
    cp_async_wait_all();
    __syncthreads();
    return n;
}

// ---------------------------------------------------------------------------
// spread: gather into register tiles                    gridops.py:80-103
// ---------------------------------------------------------------------------
struct SpreadArgs {
    TileArgs t;
    double* rho;                 // [Nz][2][Nx][Ny]
    int two;                     // slot 0 (over) as well as slot 1 (in)
    float* rho32;                // fp32 mode: the same grids in single precision
};

// ---------------------------------------------------------------------------
// interpolation of the field stack at the charges         gridops.py:105-133
//
// Charge-stationary: the charges are sorted by (4x4-column xy bin, first z
// node) and cut into groups of IG consecutive charges of one bin.  One warp
// owns a group: its window is the union of the group's stencils (at most
// (3 + 2 mx + 1) x (3 + 2 my + 1) columns x the union z range), each lane
// walks window columns and for every z node loads the NF field values once
// and applies them to all IG charges (IG x NF FMAs per NF loads).  Weights
// are recomputed in the reference's operation order (bit-identical to the
// spread's stencils).  The k = 0 linear terms (psi + A_i z, dpsi/dz + A_i)
// are separable and added analytically.  The per-charge sums are reduced
// across the warp and written once: no atomics, no partial buffers.
// ---------------------------------------------------------------------------
constexpr int IG_MAX = 8;        // charges per warp group (template IG <= IG_MAX)
constexpr int IBIN = 4;          // xy bin width (columns)
constexpr int IZC = 32;          // z nodes per weight-table chunk
constexpr int IWARPS = 8;

struct ChargeKeyArgs {
    const double* pos; int64_t first, count;
    const double* znodes; int Nz; double hx, hy, rad; int Nx, Ny, nbx; int zbits;
    uint32_t* keys; int* perm;
};

__global__ void charge_keys_kernel(ChargeKeyArgs a) {
    int64_t li = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (li >= a.count) return;
    const int64_t i = a.first + li;
    const double x = a.pos[3 * i], y = a.pos[3 * i + 1], z = a.pos[3 * i + 2];
    const int cx = pmod((long long)floor(x / a.hx), a.Nx);
    const int cy = pmod((long long)floor(y / a.hy), a.Ny);
    const uint32_t bin = (uint32_t)((cy / IBIN) * a.nbx + cx / IBIN);
    const int lo = lower_bound_d(a.znodes, a.Nz, __dsub_rn(z, a.rad));
    a.keys[li] = (bin << a.zbits) | (uint32_t)lo;
    a.perm[li] = (int)i;
}

// groups of <= IG consecutive sorted charges within each bin: per-bin
// counts, an exclusive scan (cub), then one thread per bin writes its groups
__global__ void group_count_kernel(const int64_t* seg, int nbins, int IG, int* cnt) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b > nbins) return;
    cnt[b] = (b < nbins) ? (int)((seg[b + 1] - seg[b] + IG - 1) / IG) : 0;
}

__global__ void group_fill_kernel(const int64_t* seg, const int* off, int nbins, int IG,
                                  int2* groups, int* ngroups) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b == nbins) *ngroups = off[nbins];
    if (b >= nbins) return;
    const int64_t s0 = seg[b], n = seg[b + 1] - s0;
    int o = off[b];
    for (int64_t j = 0; j < n; j += IG)
        groups[o++] = make_int2((int)(s0 + j), (int)(n - j < IG ? n - j : IG));
}

template <typename T>
struct InterpArgsT {
    const T* fields;             // [Nz][4][Nx][Ny]
    const double* pos; const double* znodes; const double* wcc;
    const double* scal;          // scal[0] = A_i
    const int* perm; const int2* groups; const int* ngroups;
    int Nx, Ny, Nz; int64_t NXY;
    double hx, hy, rad, rad_keep, inv_width, inv_norm; int mx, my;
    double* out; int64_t N;      // [NF][N] raw sums (global charge index)
};
using InterpArgs = InterpArgsT<double>;

struct GroupInfo {
    double x[IG_MAX], y[IG_MAX], z[IG_MAX];
    long long jx[IG_MAX], jy[IG_MAX];
    int jxw[IG_MAX], jyw[IG_MAX], lo[IG_MAX], hi[IG_MAX], idx[IG_MAX];
    double sx[IG_MAX], sy[IG_MAX], sz0[IG_MAX], sz1[IG_MAX];   // k = 0 separable sums
};

// T = float (fp32 mode): single-precision field loads and FMAs (weights
// rounded to fp32), the k = 0 terms and the final sums in fp64
template <int NF, int IG, int MINB, int UNR, typename T = double, int IW = IWARPS>
__global__ void __launch_bounds__(IW * 32, MINB) interp_kernel(InterpArgsT<T> a) {
    extern __shared__ __align__(16) double ism[];
    __shared__ GroupInfo ginfo[IW];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g = blockIdx.x * IW + warp;
    if (g >= *a.ngroups) return;
    const int SX = 2 * a.mx + 1, SY = 2 * a.my + 1;
    double* swx = ism + (size_t)warp * IG * (SX + SY + IZC);
    double* swy = swx + IG * SX;
    double* swz = swy + IG * SY;
    // the inner loop's z weights in the field precision (fp32 mode: fp32)
    float* swzf = reinterpret_cast<float*>(ism + (size_t)IW * IG * (SX + SY + IZC)) +
                  (size_t)warp * IG * IZC;
    GroupInfo& gi = ginfo[warp];
    const int2 gr = a.groups[g];
    const int cnt = gr.y;
    if (lane < IG) {
        int i = -1, lo = 0, hi = 0, jxw = 0, jyw = 0;
        long long jx = 0, jy = 0;
        double x = 0, y = 0, z = 0;
        if (lane < cnt) {
            i = a.perm[gr.x + lane];
            x = a.pos[3 * i]; y = a.pos[3 * i + 1]; z = a.pos[3 * i + 2];
            jx = (long long)floor(x / a.hx);
            jy = (long long)floor(y / a.hy);
            jxw = pmod(jx, a.Nx); jyw = pmod(jy, a.Ny);
            lo = lower_bound_d(a.znodes, a.Nz, __dsub_rn(z, a.rad));
            hi = upper_bound_d(a.znodes, a.Nz, __dadd_rn(z, a.rad));
        }
        gi.x[lane] = x; gi.y[lane] = y; gi.z[lane] = z;
        gi.jx[lane] = jx; gi.jy[lane] = jy; gi.jxw[lane] = jxw; gi.jyw[lane] = jyw;
        gi.lo[lane] = lo; gi.hi[lane] = hi; gi.idx[lane] = i;
    }
    __syncwarp();
    // the group's window; per-charge data stays in shared memory (GroupInfo)
    // so the column loop holds only its accumulators in registers
    int xmin = 1 << 30, xmax = -1, ymin = 1 << 30, ymax = -1, zlo = 1 << 30, zhi = 0;
#pragma unroll
    for (int m = 0; m < IG; ++m) {
        if (m < cnt) {
            xmin = min(xmin, gi.jxw[m]); xmax = max(xmax, gi.jxw[m]);
            ymin = min(ymin, gi.jyw[m]); ymax = max(ymax, gi.jyw[m]);
            zlo = min(zlo, gi.lo[m]); zhi = max(zhi, gi.hi[m]);
        }
    }
    // x / y weights: offsets o = 0 .. 2m of each charge (gridops.py:20-25)
    for (int e = lane; e < IG * SX; e += 32) {
        const int m = e / SX, o = e - m * SX;
        double wt = 0.0;
        if (m < cnt) {
            const double xj = __dmul_rn((double)(gi.jx[m] + o - a.mx), a.hx);
            const double d = __dsub_rn(gi.x[m], xj);
            if (fabs(d) <= a.rad_keep) wt = gauss_w(d, a.inv_width, a.inv_norm);
        }
        swx[e] = wt;
    }
    for (int e = lane; e < IG * SY; e += 32) {
        const int m = e / SY, o = e - m * SY;
        double wt = 0.0;
        if (m < cnt) {
            const double yj = __dmul_rn((double)(gi.jy[m] + o - a.my), a.hy);
            const double d = __dsub_rn(gi.y[m], yj);
            if (fabs(d) <= a.rad_keep) wt = gauss_w(d, a.inv_width, a.inv_norm);
        }
        swy[e] = wt;
    }
    __syncwarp();
    // separable sums for the k = 0 linear terms (lane m: charge m)
    if (lane < IG) {
        double sx = 0.0, sy = 0.0;
        for (int o = 0; o < SX; ++o) sx += swx[lane * SX + o];
        for (int o = 0; o < SY; ++o) sy += swy[lane * SY + o];
        gi.sx[lane] = sx; gi.sy[lane] = sy; gi.sz0[lane] = 0.0; gi.sz1[lane] = 0.0;
    }
    T acc[IG][NF];
#pragma unroll
    for (int m = 0; m < IG; ++m)
#pragma unroll
        for (int c = 0; c < NF; ++c) acc[m][c] = T(0);
    const int Wx = xmax - xmin + SX, Wy = ymax - ymin + SY;
    const int sx32 = 32 / Wy, sy32 = 32 - sx32 * Wy;
    const int64_t zstride = 4 * a.NXY;
    for (int zc = zlo; zc < zhi; zc += IZC) {
        const int nz = min(IZC, zhi - zc);
        __syncwarp();
        // z weights x Clenshaw-Curtis weights (gridops.py:29-39, 128-129)
        // layout [r][m]: the inner loop reads a node's IG weights with
        // vector loads
        for (int e = lane; e < IG * IZC; e += 32) {
            const int r = e / IG, m = e - r * IG, k = zc + r;
            double wt = 0.0;
            if (m < cnt && k >= gi.lo[m] && k < gi.hi[m] && k < a.Nz) {
                const double d = __dsub_rn(gi.z[m], a.znodes[k]);
                if (fabs(d) <= a.rad) wt = gauss_w(d, a.inv_width, a.inv_norm);
                wt = wt * a.wcc[k];
            }
            swz[e] = wt;
            if (sizeof(T) == sizeof(float)) swzf[e] = (float)wt;
        }
        __syncwarp();
        if (lane < IG) {
            double sz0 = gi.sz0[lane], sz1 = gi.sz1[lane];
            for (int r = 0; r < nz; ++r) {
                const double w = swz[r * IG + lane];
                sz1 += w;
                sz0 += w * a.znodes[zc + r];
            }
            gi.sz0[lane] = sz0; gi.sz1[lane] = sz1;
        }
        // fp64: (ux, uy) of this lane's column advanced by 32 columns per
        // step without an integer division per column (3.51 -> 3.48 ms; the
        // fp32 kernel keeps the division: 2.66 vs 2.69 ms)
        int cux = lane / Wy, cuy = lane - cux * Wy;
        for (int p = lane; p < Wx * Wy; p += 32) {
            int ux, uy;
            if constexpr (sizeof(T) == sizeof(double)) {
                ux = cux; uy = cuy;
                cux += sx32; cuy += sy32;
                if (cuy >= Wy) { cuy -= Wy; ++cux; }
            } else {
                ux = p / Wy; uy = p - ux * Wy;
            }
            T wxy[IG];
            bool any = false;
#pragma unroll
            for (int m = 0; m < IG; ++m) {
                const int ox = xmin + ux - gi.jxw[m], oy = ymin + uy - gi.jyw[m];
                double w = 0.0;
                if (m < cnt && ox >= 0 && ox < SX && oy >= 0 && oy < SY)
                    w = swx[m * SX + ox] * swy[m * SY + oy];
                wxy[m] = (T)w;
                any |= (w != 0.0);
            }
            if (!any) continue;
            int gx = xmin - a.mx + ux, gy = ymin - a.my + uy;
            gx %= a.Nx; if (gx < 0) gx += a.Nx;
            gy %= a.Ny; if (gy < 0) gy += a.Ny;
            const T* F = a.fields + (int64_t)zc * zstride + (int64_t)gx * a.Ny + gy;
#pragma unroll UNR
            for (int r = 0; r < nz; ++r) {
                T f[NF];
#pragma unroll
                for (int c = 0; c < NF; ++c) f[c] = __ldg(F + (int64_t)r * zstride + c * a.NXY);
                T wz[IG];
                if constexpr (IG == 4 && sizeof(T) == sizeof(float)) {
                    const float4 v = *reinterpret_cast<const float4*>(swzf + r * IG);
                    wz[0] = v.x; wz[1] = v.y; wz[2] = v.z; wz[3] = v.w;
                } else if constexpr (IG == 4) {
                    const double2 v0 = *reinterpret_cast<const double2*>(swz + r * IG);
                    const double2 v1 = *reinterpret_cast<const double2*>(swz + r * IG + 2);
                    wz[0] = (T)v0.x; wz[1] = (T)v0.y; wz[2] = (T)v1.x; wz[3] = (T)v1.y;
                } else {
#pragma unroll
                    for (int m = 0; m < IG; ++m)
                        wz[m] = (sizeof(T) == sizeof(float)) ? (T)swzf[r * IG + m] : (T)swz[r * IG + m];
                }
#pragma unroll
                for (int m = 0; m < IG; ++m) {
                    const T W = wxy[m] * wz[m];
#pragma unroll
                    for (int c = 0; c < NF; ++c) acc[m][c] = fma(W, f[c], acc[m][c]);
                }
            }
        }
    }
    // warp sums; lane m * NF + c ends up holding (m, c)
    double mine = 0.0;
#pragma unroll
    for (int m = 0; m < IG; ++m)
#pragma unroll
        for (int c = 0; c < NF; ++c) {
            double v = (double)acc[m][c];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
            if (lane == m * NF + c) mine = v;
        }
    // analytic k = 0 terms: sum_nodes W * (A_i z) and W * A_i
    const double A_i = a.scal[0];
    const int src = lane / NF;
    __syncwarp();
    const double Sx = gi.sx[src % IG], Sy = gi.sy[src % IG];
    const double Sz0 = gi.sz0[src % IG], Sz1 = gi.sz1[src % IG];
    if (lane < IG * NF && src < cnt) {
        const int c = lane - src * NF;
        double v = mine;
        if (c == 0) v += A_i * ((Sx * Sy) * Sz0);
        if (c == 3) v += A_i * ((Sx * Sy) * Sz1);
        a.out[(int64_t)c * a.N + gi.idx[src]] = v;
    }
}

// ---------------------------------------------------------------------------
// pointwise interpolation of field 0 (psi + A_i z) at arbitrary points with
// an arbitrary width: the gauge (slab.py:253-256,377-384) and the wall nodes
// of the surface-charge energy (slab.py:448-461).  One warp per point.
// ---------------------------------------------------------------------------
struct PointArgs {
    const double* pts; int64_t n;
    const double* fields; const float* fields32;      // one of them (fp32 mode: fields32)
    const double* znodes; const double* wcc;
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
            const int64_t at = ((int64_t)k * 4) * a.NXY + (int64_t)gx * a.Ny + gy;
            double f = (a.fields32 ? (double)a.fields32[at] : a.fields[at]) + A_i * a.znodes[k];
            col += wz * f;
        }
        sum += wxy * col;
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, off);
    if (lane == 0) a.out[wid] = a.hx * a.hy * sum;
}

// the same for a few points (the gauge origin): one CTA per point, a thread
// per stencil column, block reduction -- a single warp walking 169 columns x
// ~17 nodes of exp() is latency-bound (~55 us at the paper configuration)
__global__ void __launch_bounds__(256) point_interp_cta_kernel(PointArgs a) {
    __shared__ double red[8];
    const int64_t pt = blockIdx.x;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const double px = a.pts[3 * pt], py = a.pts[3 * pt + 1], pz = a.pts[3 * pt + 2];
    if (tid == 0 && (pz < a.z0 || pz > a.z1)) atomicOr(a.flags, FLAG_Z_OUTSIDE);
    const double A_i = a.scal[0];
    const long long jx = (long long)floor(px / a.hx), jy = (long long)floor(py / a.hy);
    const int lo = lower_bound_d(a.znodes, a.Nz, __dsub_rn(pz, a.rad));
    const int hi = upper_bound_d(a.znodes, a.Nz, __dadd_rn(pz, a.rad));
    const int wx = 2 * a.mx + 1, wy = 2 * a.my + 1;
    double sum = 0.0;
    for (int e = tid; e < wx * wy; e += blockDim.x) {
        const int ox = e / wy, oy = e % wy;
        const double dx = __dsub_rn(px, __dmul_rn((double)(jx + ox - a.mx), a.hx));
        const double dy = __dsub_rn(py, __dmul_rn((double)(jy + oy - a.my), a.hy));
        if (fabs(dx) > a.rad_keep || fabs(dy) > a.rad_keep) continue;
        const double tx = dx / a.width, ty = dy / a.width;
        const double wxy = (exp(-0.5 * (tx * tx)) / a.norm) * (exp(-0.5 * (ty * ty)) / a.norm);
        const int gx = pmod(jx + ox - a.mx, a.Nx), gy = pmod(jy + oy - a.my, a.Ny);
        double col = 0.0;
        for (int k = lo; k < hi; ++k) {
            const double dz = __dsub_rn(pz, a.znodes[k]);
            if (fabs(dz) > a.rad) continue;
            const double tz = dz / a.width;
            const double wz = exp(-0.5 * (tz * tz)) / a.norm * a.wcc[k];
            const int64_t at = ((int64_t)k * 4) * a.NXY + (int64_t)gx * a.Ny + gy;
            const double f = (a.fields32 ? (double)a.fields32[at] : a.fields[at]) + A_i * a.znodes[k];
            col += wz * f;
        }
        sum += wxy * col;
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, off);
    if (lane == 0) red[warp] = sum;
    __syncthreads();
    if (tid == 0) {
        double t = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
        a.out[pt] = a.hx * a.hy * t;
    }
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
                    st.j0y, st.lo, st.hi, st.q, st.rec, st.owner};
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
    st.hi = dalloc<int>(p, cap);
    st.rs = (2 * p->mx + 1) + (2 * p->my + 1) + p->wz_max;
    st.rs += st.rs & 1;
    // records exist for the valid sources only, which sort first: a charge
    // has at most one mirror image unless it lies within 2 H_E of both walls
    // (H < 4 H_E), so 2n records suffice then (C5: 12 GB instead of 18)
    const int64_t rec_cap = (p->P.H >= 4.0 * p->P.H_E) ? std::max<int64_t>(64, 2 * n) : cap;
    st.rec = dalloc<double>(p, (size_t)st.rs * rec_cap);
    st.owner = dalloc<int>(p, cap);
    p->src_cap = cap;
}

static void launch_make_sources(Plan* p, const double* d_pos, int64_t n, bool two_grids,
                                int64_t first = 0) {
    const int TB = 256;
    SrcArgs sa{d_pos, p->d_q, n, first, p->P.H, 2.0 * p->P.H_E,
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

void build_sources(Plan* p, const double* d_pos, int64_t first, int64_t n, bool two_grids) {
    NvtxRange nv("se.sources");
    ensure_sources(p, n);
    const int64_t total = 3 * n;
    const int TB = 256;
    launch_make_sources(p, d_pos, n, two_grids, first);
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
                        p->rad_keep, 1.0 / p->width, 1.0 / p->norm, p->mx, p->my, p->wz_max, st};
        stencil_kernel<<<(unsigned)((total + STENCIL_TB - 1) / STENCIL_TB), STENCIL_TB, 0,
                         p->stream>>>(sta);
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

// Accumulation on the FP64 tensor pipe (DMMA m8n8k4): a warp owns the
// tile's 64 columns x one 8-node z group as eight 8x8 accumulator fragments
// (one per x column: rows y, columns z); four staged sources form one
// k-step with A[y][s] = q_s wx_s(x) wy_s(y) and B[s][z] = wz_s(z), so one
// mma.sync does the 256 FMAs that would cost eight DFMAs per lane.  A warp
// skips k-steps whose sources all miss its z group.
__device__ __forceinline__ void dmma_8x8x4(double (&c)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c[0]), "+d"(c[1]) : "d"(a), "d"(b));
}

template <int TZ, int CAP, int MINB, bool ZW>
__global__ void __launch_bounds__(4 * TZ, MINB) spread_mma_kernel(SpreadArgs a) {
    constexpr int NG = TZ / 8;
    extern __shared__ __align__(16) unsigned char dsm[];
    Stage<TZ, CAP, ZW>& sm = *reinterpret_cast<Stage<TZ, CAP, ZW>*>(dsm);
    __shared__ int s_lo[MAX_BINS], s_len[MAX_BINS], s_nr, s_total;

    const TileArgs& A = a.t;
    const int bx = blockIdx.x, by = blockIdx.y, k0 = blockIdx.z * TZ;
    const int gx0 = bx * TILE, gy0 = by * TILE;
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const int zg = warp, kk = lane & 3, rr = lane >> 2;
    const unsigned wzbit = 1u << zg;
    const int kz = k0 + 8 * zg + rr;                       // this lane's B row (z node)
    const int zoffr = (2 * A.st.mx + 1) + (2 * A.st.my + 1);   // wz offset in a record

    double c[TILE][2];
#pragma unroll
    for (int mb = 0; mb < TILE; ++mb) { c[mb][0] = 0.0; c[mb][1] = 0.0; }

    for (int cls = a.two ? 0 : 1; cls < 2; ++cls) {
        tile_ranges<TZ>(A, bx, by, k0, cls, s_lo, s_len, &s_nr, &s_total);
        const int total = s_total, nr = s_nr;
        for (int cursor = 0; cursor < total; cursor += CAP) {
            const int n = stage_round<TZ, NG, CAP, true, ZW>(
                sm, A, cursor, total, s_lo, s_len, nr, gx0, gy0, k0);
            for (int s0 = 0; s0 < n; s0 += 4) {
                const int sidx = s0 + kk;
                const bool ok = sidx < n && (sm.zm[sidx] & wzbit);
                if (!__any_sync(0xffffffffu, ok)) continue;
                // B = wz_s(z) straight from the source's record (zeros past
                // its last node); lanes rr read 8 consecutive doubles
                double b = 0.0;
                if (ZW) {
                    if (ok) b = sm.wz[sidx][8 * zg + rr];
                } else if (ok) {
                    const int tt = kz - sm.lo[sidx];
                    if (tt >= 0 && tt < A.st.wz && kz < A.Nz)
                        b = __ldg(A.st.rec + (int64_t)sm.idx[sidx] * A.st.rs + zoffr + tt);
                }
                const double qwy = ok ? sm.q[sidx] * sm.wy[sidx][rr] : 0.0;
                const int sl = ok ? sidx : 0;
                const double2* wx2 = reinterpret_cast<const double2*>(&sm.wx[sl][0]);
#pragma unroll
                for (int h = 0; h < TILE / 2; ++h) {
                    const double2 w = wx2[h];
                    dmma_8x8x4(c[2 * h], qwy * w.x, b);
                    dmma_8x8x4(c[2 * h + 1], qwy * w.y, b);
                }
            }
            __syncthreads();
        }
        // store this class's running sum (slot 0 after class 0, slot 1 after 1):
        // fragment mb = column x, row rr = y, columns 2kk, 2kk+1 = z
        const int gy = gy0 + rr;
#pragma unroll
        for (int mb = 0; mb < TILE; ++mb) {
            const int gx = gx0 + mb;
            if (gx < A.Nx && gy < A.Ny) {
                const int64_t off = (int64_t)(cls) * A.NXY + (int64_t)gx * A.Ny + gy;
#pragma unroll
                for (int i = 0; i < 2; ++i) {
                    const int k = k0 + 8 * zg + 2 * kk + i;
                    if (k < A.Nz) {
                        if (a.rho32) a.rho32[off + (int64_t)k * 2 * A.NXY] = (float)c[mb][i];
                        else a.rho[off + (int64_t)k * 2 * A.NXY] = c[mb][i];
                    }
                }
            }
        }
    }
}

template <int TZ, int CAP, int MINB, bool ZW>
static void launch_spread_mma(Plan* p, const SpreadArgs& a) {
    dim3 grid(p->ss.nbx, p->ss.nby, (p->Nz + TZ - 1) / TZ);
    const int smem = (int)sizeof(Stage<TZ, CAP, ZW>);
    SE_CUDA(cudaFuncSetAttribute(spread_mma_kernel<TZ, CAP, MINB, ZW>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    spread_mma_kernel<TZ, CAP, MINB, ZW><<<grid, 4 * TZ, smem, p->stream>>>(a);
}



void spread(Plan* p, bool two_grids) {
    NvtxRange nv("se.spread");
    SpreadArgs a{tile_args(p), p->d_rho, two_grids ? 1 : 0, p->g32 ? p->d_rho32 : nullptr};
    // 8x8-column x 16-node tiles, 2 warps (one per 8-node z group), DMMA
    // accumulation, 64 staged sources per round: measured best among tile
    // heights {16, 32}, rounds {32..256}, scalar lane shapes and 2..16 CTAs
    // per SM (scalar 2.67 ms -> DMMA 2.08 ms at C4).  Round 2: the z weights
    // are read from the records inside the k-steps instead of being staged
    // (10 KB of shared memory per CTA instead of 18), which lets 18 CTAs
    // share an SM (56 registers): 2.13 -> 1.94 ms (10 / 12 / 14 / 16 / 20
    // CTAs: 2.27 / 2.10 / 1.98 / 2.02 / 2.19 ms).  Grids of less than ~16
    // tiles per SM (the paper's configuration: 726 tiles) are latency-bound
    // on those loads instead and keep the staged z weights (0.171 vs
    // 0.242 ms there)
    p->ktic(0);
    const int64_t tiles = (int64_t)p->ss.nbx * p->ss.nby * ((p->Nz + 15) / 16);
    if (tiles >= 16 * (int64_t)p->num_sms) launch_spread_mma<16, 64, 18, false>(p, a);
    else launch_spread_mma<16, 64, 10, true>(p, a);
    p->ktoc(0);
    SE_LAUNCHED(p);
}

void interp_charges(Plan* p, int64_t n, int64_t first, int64_t count, bool forces) {
    if (count == 0) return;
    NvtxRange nv("se.interpolate");
    const int TB = 256;
    const int nbx = (p->Nx + IBIN - 1) / IBIN, nby = (p->Ny + IBIN - 1) / IBIN;
    const int nbins = nbx * nby;
    const int zb = zbits_for(p->Nz);
    int end_bit = zb;
    while (end_bit < 32 && ((uint64_t)nbins >> (end_bit - zb)) != 0) ++end_bit;
    if (((uint64_t)nbins << zb) >> 32)
        throw Error(SE_ERR_VALUE, "grid too large for the interpolation sort keys");
    ensure_sources(p, n);               // key / permutation / sort scratch (>= 3n)
    // charges per group: 5 (round 2: fp64 3.51 ms vs 3.90 with 4 and 4.01
    // with 6; fp32 2.68 vs 2.82 / 3.08; round 1 measured 2, 3, 4, 8)
    const int ig = 5;
    const int64_t gcap = count / ig + nbins + 1;
    if (nbins + 1 > p->iseg_cap || gcap > p->igroup_cap) {
        dfree(p, p->d_iseg); dfree(p, p->d_igroups); dfree(p, p->d_ingroups);
        dfree(p, p->d_gcnt);
        p->d_iseg = dalloc<int64_t>(p, nbins + 1);
        p->d_gcnt = dalloc<int>(p, 2 * (nbins + 1));
        p->d_igroups = dalloc<int2>(p, gcap);
        p->d_ingroups = dalloc<int>(p, 1);
        p->iseg_cap = nbins + 1;
        p->igroup_cap = gcap;
    }
    p->ktic(2);
    ChargeKeyArgs ka{p->d_pos_cur, first, count, p->d_z, p->Nz, p->hx, p->hy, p->rad,
                     p->Nx, p->Ny, nbx, zb, p->d_keys, p->d_perm};
    charge_keys_kernel<<<(unsigned)((count + TB - 1) / TB), TB, 0, p->stream>>>(ka);
    SE_LAUNCHED(p);
    size_t bytes = p->cub_bytes;
    SE_CUDA(cub::DeviceRadixSort::SortPairs(p->d_cub, bytes, p->d_keys, p->d_keys2,
                                            p->d_perm, p->d_perm2, (int)count, 0, end_bit,
                                            p->stream));
    segment_offsets_kernel<<<(unsigned)((count + 1 + TB - 1) / TB), TB, 0, p->stream>>>(
        p->d_keys2, count, zb, nbins, p->d_iseg);
    SE_LAUNCHED(p);
    group_count_kernel<<<(nbins + 1 + TB - 1) / TB, TB, 0, p->stream>>>(p->d_iseg, nbins, ig,
                                                                       p->d_gcnt);
    SE_LAUNCHED(p);
    size_t sbytes = 0;
    SE_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, sbytes, p->d_gcnt, p->d_gcnt + nbins + 1,
                                          nbins + 1, p->stream));
    if (sbytes > p->gscan_bytes) {
        dfree(p, p->d_gscan);
        p->d_gscan = dalloc<char>(p, sbytes);
        p->gscan_bytes = sbytes;
    }
    sbytes = p->gscan_bytes;
    SE_CUDA(cub::DeviceScan::ExclusiveSum(p->d_gscan, sbytes, p->d_gcnt, p->d_gcnt + nbins + 1,
                                          nbins + 1, p->stream));
    group_fill_kernel<<<(nbins + 1 + TB - 1) / TB, TB, 0, p->stream>>>(
        p->d_iseg, p->d_gcnt + nbins + 1, nbins, ig, p->d_igroups, p->d_ingroups);
    SE_LAUNCHED(p);
    InterpArgs a{p->d_fields, p->d_pos_cur, p->d_z, p->d_wcc, p->d_scal, p->d_perm2,
                 p->d_igroups, p->d_ingroups, p->Nx, p->Ny, p->Nz, p->NXY, p->hx, p->hy,
                 p->rad, p->rad_keep, 1.0 / p->width, 1.0 / p->norm, p->mx, p->my, p->d_far, n};
    InterpArgsT<float> a32{p->d_fields32, p->d_pos_cur, p->d_z, p->d_wcc, p->d_scal, p->d_perm2,
                           p->d_igroups, p->d_ingroups, p->Nx, p->Ny, p->Nz, p->NXY, p->hx,
                           p->hy, p->rad, p->rad_keep, 1.0 / p->width, 1.0 / p->norm, p->mx,
                           p->my, p->d_far, n};
    // per warp: x / y / z weight tables in fp64 and (fp32 mode) the z table
    // again in fp32 for the inner loop
    const int smem = IWARPS * ig * ((2 * p->mx + 1 + 2 * p->my + 1 + IZC) * (int)sizeof(double) +
                                    IZC * (int)sizeof(float));
    if (smem > 200 * 1024) throw Error(SE_ERR_VALUE, "stencil too wide for the interpolation");
    auto go = [&](auto kern, const auto& args, int iw = IWARPS) {
        const unsigned blocks = (unsigned)((gcap + iw - 1) / iw);
        const int sm = smem / IWARPS * iw;
        SE_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
        kern<<<blocks, iw * 32, sm, p->stream>>>(args);
    };
    // fp32 mode: 3 CTAs / SM (80 registers, no spills; the per-charge data
    // lives in shared memory): 2.99 vs 3.62 ms at 2 CTAs (4-charge groups).
    // fp64: 4-warp CTAs at 125 registers, 16 warps / SM (4-charge groups:
    // 3.93 vs 4.01 ms with 8-warp CTAs; capped at 80 registers they spilled,
    // 4.28-4.38 ms).  z weight rows padded to 8 for 16-byte loads: 4.27 vs
    // 3.51 ms (130 registers, 12 warps / SM); 2-warp CTAs: 3.61 ms
    if (p->g32) {
        // 4-warp CTAs, 6 per SM: 2.66 vs 2.67 ms for 8-warp CTAs, 3 per SM
        if (forces) go(interp_kernel<4, 5, 6, 2, float, 4>, a32, 4);
        else go(interp_kernel<1, 5, 6, 2, float, 4>, a32, 4);
    } else if (forces) {
        go(interp_kernel<4, 5, 3, 2, double, 4>, a, 4);
    } else {
        go(interp_kernel<1, 5, 3, 2, double, 4>, a, 4);
    }
    p->ktoc(2);
    SE_LAUNCHED(p);
}

void interp_points(Plan* p, const double* d_pts, int64_t npts, double width,
                   double radius, double* d_out) {
    if (npts == 0) return;
    PointArgs a{};
    a.pts = d_pts; a.n = npts; a.fields = p->d_fields; a.znodes = p->d_z;
    a.fields32 = p->g32 ? p->d_fields32 : nullptr;
    a.wcc = p->d_wcc; a.scal = p->d_scal; a.Nx = p->Nx; a.Ny = p->Ny;
    a.Nz = p->Nz; a.NXY = p->NXY; a.hx = p->hx; a.hy = p->hy;
    a.width = width; a.rad = radius; a.rad_keep = radius + 1e-12 * radius;
    a.norm = std::sqrt(2.0 * M_PI * width * width);
    a.mx = (int)std::floor(radius / p->hx + 1e-12);
    a.my = (int)std::floor(radius / p->hy + 1e-12);
    a.out = d_out; a.flags = p->d_flags; a.z0 = p->P.z0; a.z1 = p->P.z1;
    if (npts <= 64) {
        point_interp_cta_kernel<<<(unsigned)npts, 256, 0, p->stream>>>(a);
    } else {
        const int64_t threads = npts * 32;
        point_interp_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, p->stream>>>(a);
    }
    SE_LAUNCHED(p);
}

}  // namespace se
