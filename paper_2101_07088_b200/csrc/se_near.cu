// Near-field pair sums, gauge, energy.
//
// Reference: NearField (slab.py:85-181) with the erf kernels of
// kernels.py:38-125; the gauge (slab.py:377-384), the energy
// (slab.py:387-391) and the wall-charge energy (slab.py:448-461).
//
// B200 design.  Sources (charges + one mirrored layer per jumping wall) are
// binned into a cell list with cells >= r_cut and sorted by cell (cub radix
// sort).  One thread per evaluation point, evaluation points sorted by cell
// so a warp walks the same neighbour cells in lockstep and source loads are
// warp-broadcast.  Candidates are screened with an fp32 distance test on
// wrapped coordinates (with a 1e-4 relative margin); survivors get the
// reference's exact fp64 test
//   d = p - s;  d_xy -= L * rint(d_xy / L);  r = sqrt((dx^2 + dy^2) + dz^2);
//   keep r <= r_query                                       (slab.py:143-148)
// evaluated without FMA contraction, so the pair set equals numpy's bit for
// bit.  Accepted pairs go to a per-thread queue; the warp drains the queues
// together (warp-synchronous) so the erf/exp kernel runs with all lanes
// busy instead of at the ~20 % hit rate of the raw candidate stream.
#include <cub/cub.cuh>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <type_traits>

#include "se_internal.cuh"
#include "se_erf_table.inc"

namespace se {

namespace {

constexpr double TWO_OVER_SQRTPI = 1.1283791670955126;   // 2/sqrt(pi)


// ---------------------------------------------------------------------------
// cell list
// ---------------------------------------------------------------------------
// xy columns of width >= r/hw (r = max query radius; hw neighbour columns
// each side), z bins of ~r/16
struct CellGeo {
    int ncx, ncy, ncz, hw;
    double csx, csy, csz, zlo, Lx, Ly;
};

__device__ __forceinline__ double wrap(double x, double L) {
    double w = x - L * floor(x / L);
    return (w >= L) ? 0.0 : w;
}

// cell = (xy column, z bin); a column's z bins are contiguous in the sort
__device__ __forceinline__ int cell_of(const CellGeo& g, double x, double y, double z,
                                       int* cx, int* cy, int* cz) {
    int ix = (int)(wrap(x, g.Lx) / g.csx); if (ix >= g.ncx) ix = g.ncx - 1;
    int iy = (int)(wrap(y, g.Ly) / g.csy); if (iy >= g.ncy) iy = g.ncy - 1;
    double fz = floor((z - g.zlo) / g.csz);
    int iz = fz < 0 ? 0 : (fz >= g.ncz ? g.ncz - 1 : (int)fz);
    *cx = ix; *cy = iy; *cz = iz;
    return (iy * g.ncx + ix) * g.ncz + iz;
}

struct SrcBuild {
    const double* pos; const double* q; int64_t n;
    double H, fb, ft; int nb, nt;        // mirrored layers present
    double4* out; int64_t ns;
};

__global__ void make_near_sources(SrcBuild a) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= a.n) return;
    double x = a.pos[3 * i], y = a.pos[3 * i + 1], z = a.pos[3 * i + 2], q = a.q[i];
    a.out[i] = make_double4(x, y, z, q);                        // slab.py:104-105
    int64_t off = a.n;
    if (a.nb) { a.out[off + i] = make_double4(x, y, -z, a.fb * q); off += a.n; }
    if (a.nt) a.out[off + i] = make_double4(x, y, __dsub_rn(2.0 * a.H, z), a.ft * q);
}

__global__ void zrange_kernel(const double4* s, int64_t ns, double* mm) {
    __shared__ double smin[256], smax[256];
    double lo = 1e300, hi = -1e300;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < ns;
         i += (int64_t)gridDim.x * blockDim.x) {
        double z = s[i].z;
        lo = fmin(lo, z); hi = fmax(hi, z);
    }
    smin[threadIdx.x] = lo; smax[threadIdx.x] = hi;
    __syncthreads();
    for (int w = 128; w > 0; w >>= 1) {
        if (threadIdx.x < w) {
            smin[threadIdx.x] = fmin(smin[threadIdx.x], smin[threadIdx.x + w]);
            smax[threadIdx.x] = fmax(smax[threadIdx.x], smax[threadIdx.x + w]);
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        mm[2 * blockIdx.x] = smin[0];
        mm[2 * blockIdx.x + 1] = smax[0];
    }
}

// the reference's tree z origin: min(source z) - r_cut - 1 (slab.py:120);
// zsrc (optional): the minimum over ALL sources when this cell list holds a
// rank's share of them (the cell-routed sharded near field)
__global__ void zmin_kernel(const double* mm, int nblk, double r_cut, const double* zsrc,
                            double* zmin) {
    double lo = 1e300;
    if (zsrc) lo = *zsrc;
    else for (int b = 0; b < nblk; ++b) lo = fmin(lo, mm[2 * b]);
    *zmin = __dsub_rn(__dsub_rn(lo, r_cut), 1.0);
}

__global__ void cell_keys_kernel(const double4* s, int64_t ns, CellGeo g,
                                 uint32_t* keys, int* perm) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= ns) return;
    double4 v = s[i];
    int cx, cy, cz;
    keys[i] = (uint32_t)cell_of(g, v.x, v.y, v.z, &cx, &cy, &cz);
    perm[i] = (int)i;
}

__global__ void cell_fill_kernel(const uint32_t* keys, const int* perm, int64_t ns,
                                 int ncell, const double4* src_in, CellGeo g,
                                 int* start, double4* src, float4* srcf, int* orig,
                                 int orig_off) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i > ns) return;
    int cur = (i < ns) ? (int)keys[i] : ncell;
    int prev = (i == 0) ? -1 : (int)keys[i - 1];
    for (int c = prev + 1; c <= cur; ++c) start[c] = (int)i;
    if (i == ns) return;
    int s = perm[i];
    double4 v = src_in[s];
    src[i] = v;
    srcf[i] = make_float4((float)wrap(v.x, g.Lx), (float)wrap(v.y, g.Ly),
                          (float)(v.z - g.zlo), (float)v.w);
    orig[i] = s + orig_off;
}

// ---------------------------------------------------------------------------
// pair evaluation
// ---------------------------------------------------------------------------
struct NearArgs {
    const double* eval; const int* order; int64_t ne;
    const int2* tasks; int64_t ntask; const int* ntask_dev; const int* pt_end;
    CellGeo g; const int* start; const double4* src; const float4* srcf;
    double r2max;                 // largest r2 with sqrt(r2) <= r_query
    // the reference's KD-tree pre-test (slab.py:120-135, scipy cKDTree on
    // (x mod Lx, y mod Ly, z - zmin), squared distance <= r*r) decides only
    // within a few ulps of the cutoff: pairs with r2 >= win_lo repeat it
    double rr, win_lo, lzbox; const double* zmin;
    int2* bnd; int* bnd_cnt; int bnd_cap; int* flags;   // deferred boundary pairs
    double c1, c2, ic1, ic2, inv4pie, self_value, point0;
    int kind, need_field;
    float r2f;                    // fp32 pre-test bound (with margin)
    float r2close;                // fp32 bound below which a pair may need the
                                  // general (close) path
    float Lxf, Lyf, iLxf, iLyf;
    double qLx, qLy;              // L / 4: |d| below it needs no minimum-image shift
    float zmarg;                  // fp32 z-window margin
    // SE_FP32 evaluation: single-precision displacements from the wrapped
    // fp32 coordinates; |r2_f32 - r2| is bounded, so pairs with r2_f32 <=
    // r2in_f are certainly inside the cutoff, > r2out_f certainly outside,
    // and only the thin band between takes the exact fp64 test
    float r2in_f, r2out_f, hLxf, hLyf;
    // far pairs: erfcx(x) on the far x range as one degree-FAR_DEG
    // polynomial in t = (x - pmid) * pinvh (coefficients in the kernel
    // parameter bank, so no table loads); use_poly = 0 falls back to the table
    int use_poly;
    double pmid, pinvh;
    double pc[19];
    double pc4[19], ic2sq, far_t1, far_t0, far_k;   // the fp64 far path (pair_terms)
    // fp32 mode: erfcx on the same x range as one degree-FAR_DEG32 polynomial
    int use_poly32;
    float pmid32, pinvh32, pc32[11];
    // close pairs: g(r) and coef(r) as CL_P piecewise degree-CL_D polynomials
    // in r on [0, CL_P cl_w) (table staged in shared memory by the close
    // launch); use_ctab = 0 evaluates the erf formulas
    const double* ctab; int use_ctab; double cl_w, cl_iw;
    double* out; int64_t out_stride;   // out[c * stride + i]
    int64_t* npairs;
    void* stats;
    int* list_far; int* list_close; int64_t cap_far, cap_close;
    int* cnt_far; int* cnt_close; int* overflow;   // overflow: count of ovl
    int* ovl;                                      // slots whose lists overflowed
    // SE_PAIR_HASH: per evaluation point, the wrap-around sum of mix64(source
    // index) over its accepted pairs ([0, ne)) and their count ([ne, 2 ne))
    const int* orig; unsigned long long* phash;
};

constexpr int NB_THREADS = 128;
// Pairs beyond FAR_SPLIT c1 take the erfc-only far kernel.  The reference
// switches at 6.5 c1 (kernels.py:96-113); between 5.9 c1 and 6.5 c1 its
// erf(r/c1) is 1 - erfc(r/c1) with erfc < 1.2e-16 and its exp(-(r/c1)^2)
// term below 8e-16, so the two formulas differ by < 1e-14 relative there --
// far inside the 1e-10 parity bar -- and the cheaper far kernel takes a
// quarter of the close pairs.
constexpr double FAR_SPLIT = 5.9;
constexpr int FAR_DEG = 18;
constexpr int FAR_DEG32 = 10;
// close-pair table: pieces, degree; the g and coef coefficients of a degree
// are interleaved so one 16-byte shared load serves both Horner steps (the
// close launch is bound by shared-memory wavefronts: 128 x 6 takes 7 vector
// loads per pair where 32 x 12 took 26 scalar ones)
constexpr int CL_P = 128, CL_D = 6;
constexpr int CL_TAB = 2 * CL_P * (CL_D + 1);

// 1/sqrt(x) for normal positive x: the hardware approximation (2^-20
// relative on sm_100a, tools/rsqrt_err.cu) + one third-order step
// y (1 + e/2 + 3e^2/8), e = 1 - x y^2 (error ~ e^3 < 2^-57): 5 FP64
// operations where two Newton steps take 7
__device__ __forceinline__ double rsqrt_pos(double x) {
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    const double e = fma(-x * y, y, 1.0);
    return fma(y * e, fma(e, 0.375, 0.5), y);
}

// erf / erfc / exp(-x^2) of one argument.  erfc = exp(-x^2) erfcx(x) with
// erfcx from the piecewise polynomial table (tools/gen_erfcx.py, ~2e-15
// relative); a Maclaurin series below 0.5.  One exp serves both the
// potential and the field.
__device__ __forceinline__ void erf_erfc(double x, const double* tab, double& erf_v,
                                         double& erfc_v, double& e) {
    e = exp_neg(fmin(x * x, 700.0));
    if (x < SE_ERFCX_X0) {
        const double u = x * x;
        // erf(x) = 2/sqrt(pi) sum_n (-1)^n x^(2n+1) / (n! (2n+1))
        double s = 1.0 / (479001600.0 * 25.0);
        s = fma(s, u, -1.0 / (39916800.0 * 23.0));
        s = fma(s, u, 1.0 / (3628800.0 * 21.0));
        s = fma(s, u, -1.0 / (362880.0 * 19.0));
        s = fma(s, u, 1.0 / (40320.0 * 17.0));
        s = fma(s, u, -1.0 / (5040.0 * 15.0));
        s = fma(s, u, 1.0 / (720.0 * 13.0));
        s = fma(s, u, -1.0 / (120.0 * 11.0));
        s = fma(s, u, 1.0 / (24.0 * 9.0));
        s = fma(s, u, -1.0 / (6.0 * 7.0));
        s = fma(s, u, 1.0 / (2.0 * 5.0));
        s = fma(s, u, -1.0 / 3.0);
        s = fma(s, u, 1.0);
        erf_v = TWO_OVER_SQRTPI * x * s;
        erfc_v = 1.0 - erf_v;
    } else if (x < SE_ERFCX_X0 + SE_ERFCX_NP * SE_ERFCX_W) {
        const int p = (int)((x - SE_ERFCX_X0) * (1.0 / SE_ERFCX_W));
        const double t = (x - (SE_ERFCX_X0 + (p + 0.5) * SE_ERFCX_W)) * (2.0 / SE_ERFCX_W);
        const double* c = tab + p * (SE_ERFCX_DEG + 1);
        double acc = c[SE_ERFCX_DEG];
#pragma unroll
        for (int j = SE_ERFCX_DEG - 1; j >= 0; --j) acc = fma(acc, t, c[j]);
        erfc_v = e * acc;
        erf_v = 1.0 - erfc_v;
    } else {
        erfc_v = 0.0;
        erf_v = 1.0;
    }
}

// Near kernel between two widths (erf(r/c1) - erf(r/c2)) / (4 pi eps r) and
// its radial derivative over r (kernels.py:38-113, slab.py:162-177).
// FAR: r > FAR_SPLIT c1 and r >= 0.01 c2, where erf(r/c1) is 1 in fp64 to
// within an ulp and the exp(-(r/c1)^2) terms are < 1e-14 of the kernel:
// erfc-only form.
// fp32 mode: the far kernel in single precision (__expf, an fp32 erfcx
// polynomial or erfcf); ~1e-6 relative per pair, far inside the Ewald
// tolerance
__device__ __forceinline__ void far_terms_f32(const NearArgs& a, float sr, float& g,
                                              float& coef) {
    const float ri = rsqrtf(sr);
    const float x = sr * ri * (float)a.ic2;
    const float e = __expf(-x * x);
    float C;
    if (a.use_poly32) {                          // erfc = exp(-x^2) erfcx(x)
        const float t = (x - a.pmid32) * a.pinvh32;
        float acc = a.pc32[FAR_DEG32];
#pragma unroll
        for (int j = FAR_DEG32 - 1; j >= 0; --j) acc = fmaf(acc, t, a.pc32[j]);
        C = e * acc;
    } else {
        C = erfcf(x);
    }
    const float i4 = (float)a.inv4pie;
    g = C * ri * i4;
    coef = a.need_field ? (C * ri + 1.1283792f * e * (float)a.ic2) * (ri * ri) * i4 : 0.f;
}

template <bool FAR, bool F32 = false>
__device__ __forceinline__ void pair_terms(const NearArgs& a, const double* tab,
                                           double r2, double& g, double& coef) {
    const bool nd = a.need_field;
    if (FAR && F32) {
        float gf, cf;
        far_terms_f32(a, (float)r2, gf, cf);
        g = (double)gf;
        coef = (double)cf;
        return;
    }
    if (!FAR && r2 == 0.0) {                     // slab.py:161-171,176
        g = (a.kind == 0) ? a.self_value : a.point0;
        coef = 0.0;
        return;
    }
    const double rinv = (FAR || r2 > 1e-280) ? rsqrt_pos(r2) : rsqrt(r2);
    const double r = r2 * rinv;
    if (!FAR && a.use_ctab) {
        const double* ct = tab + SE_ERFCX_NP * (SE_ERFCX_DEG + 1);
        int pc = (int)(r * a.cl_iw);
        pc = pc < CL_P - 1 ? pc : CL_P - 1;
        const double t = (r - (pc + 0.5) * a.cl_w) * (2.0 * a.cl_iw);
        const double2* cgc = reinterpret_cast<const double2*>(ct) + pc * (CL_D + 1);
        const double2 top = cgc[CL_D];
        double gv = top.x, cv = top.y;
#pragma unroll
        for (int j = CL_D - 1; j >= 0; --j) {
            const double2 cj = cgc[j];
            gv = fma(gv, t, cj.x); cv = fma(cv, t, cj.y);
        }
        g = gv;
        coef = nd ? cv : 0.0;
        return;
    }
    if (FAR && a.use_poly) {
        // erfc(x) / (4 pi eps r) = exp(-x^2) erfcx(x) / (4 pi eps r), x = r / c2,
        // with 1/(4 pi eps) folded into the erfcx coefficients (pc4) and the
        // derivative constant (far_k = 2/sqrt(pi) / c2 / (4 pi eps))
        const double e2 = exp_neg(r2 * a.ic2sq);
        const double t = fma(r, a.far_t1, a.far_t0);
        double acc = a.pc4[FAR_DEG];
#pragma unroll
        for (int j = FAR_DEG - 1; j >= 0; --j) acc = fma(acc, t, a.pc4[j]);
        g = (e2 * acc) * rinv;
        coef = nd ? fma(a.far_k, e2, g) * (rinv * rinv) : 0.0;
        return;
    }
    const double x2 = r * a.ic2;
    double E2, C2, e2;
    if (FAR && a.use_poly) {
        e2 = exp_neg(x2 * x2);
        const double t = (x2 - a.pmid) * a.pinvh;
        double acc = a.pc[FAR_DEG];
#pragma unroll
        for (int j = FAR_DEG - 1; j >= 0; --j) acc = fma(acc, t, a.pc[j]);
        C2 = e2 * acc;
        E2 = 1.0 - C2;
    } else {
        erf_erfc(x2, tab, E2, C2, e2);
    }
    if (FAR || (r > 6.5 * a.c1 && r >= 1e-2 * a.c2)) {
        g = C2 * rinv * a.inv4pie;
        coef = 0.0;
        if (nd) {
            const double dd = -(C2 * rinv + TWO_OVER_SQRTPI * e2 * a.ic2) * rinv;
            coef = -(dd * a.inv4pie) * rinv;
        }
        return;
    }
    double E1 = 1.0, C1 = 0.0, e1 = 0.0;
    const double x1 = r * a.ic1;
    if (r <= 6.5 * a.c1) erf_erfc(x1, tab, E1, C1, e1);
    const double v1 = (r < 1e-10 * a.c1) ? TWO_OVER_SQRTPI * a.ic1 : E1 * rinv;
    const double v2 = (r < 1e-10 * a.c2) ? TWO_OVER_SQRTPI * a.ic2 : E2 * rinv;
    g = (v1 - v2) * a.inv4pie;
    coef = 0.0;
    if (!nd) return;
    auto series = [](double x, double ic) {
        double u = x * x;
        return TWO_OVER_SQRTPI * (ic * ic) * x *
               (-2.0 / 3.0 + u * (2.0 / 5.0 + u * (-1.0 / 7.0 + u / 27.0)));
    };
    double d1, d2;
    if (r > 6.5 * a.c1) d1 = -rinv * rinv;
    else if (r < 1e-2 * a.c1) d1 = series(x1, a.ic1);
    else d1 = TWO_OVER_SQRTPI * e1 * a.ic1 * rinv - v1 * rinv;
    if (r < 1e-2 * a.c2) d2 = series(x2, a.ic2);
    else d2 = TWO_OVER_SQRTPI * e2 * a.ic2 * rinv - v2 * rinv;
    coef = -((d1 - d2) * a.inv4pie) * rinv;
}


// exact displacement and squared distance, reference operation order
//   d = p - s; d_xy -= L * round(d_xy / L); r2 = (dx^2 + dy^2) + dz^2
// round(d / L) is taken as rint(d * (1 / L)): the two differ only when d / L
// lies within ulps of a half-integer, i.e. for pairs whose minimum-image
// distance is ~L/2 > r_cut, which no list holds (r_cut < L/2 is enforced)
__device__ __forceinline__ double min_image(double d, double L) {
    if (fabs(d) <= 0.25 * L) return d;           // round(d/L) == 0 exactly
    return __dsub_rn(d, __dmul_rn(L, rint(d * (1.0 / L))));
}

// numpy's float remainder (npy_divmod): fmod, moved into [0, L) for L > 0
__device__ __forceinline__ double np_mod(double x, double L) {
    double m = fmod(x, L);
    if (m != 0.0) { if (m < 0.0) m = __dadd_rn(m, L); }
    else m = 0.0;
    return m;
}

__device__ __forceinline__ double box_wrap(double d, double L) {
    const double h = 0.5 * L;
    if (d > h) return __dsub_rn(d, L);
    if (d < -h) return __dadd_rn(d, L);
    return d;
}

// The reference's KD-tree test for one pair: coordinates shifted as in
// NearField._shift (slab.py:126-131), periodic differences, squared
// distance summed in dimension order, compared with fl(r*r).
__device__ __noinline__ bool tree_keep_s(double Lx, double Ly, double lz, double zm, double rr,
                                         double px, double py, double pz, double sx, double sy,
                                         double sz) {
    const double dx = box_wrap(__dsub_rn(np_mod(px, Lx), np_mod(sx, Lx)), Lx);
    const double dy = box_wrap(__dsub_rn(np_mod(py, Ly), np_mod(sy, Ly)), Ly);
    const double dz = box_wrap(__dsub_rn(__dsub_rn(pz, zm), __dsub_rn(sz, zm)), lz);
    const double s2 = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
    return s2 <= rr;
}
#define tree_keep(a, px, py, pz, sx, sy, sz) \
    tree_keep_s((a).g.Lx, (a).g.Ly, (a).lzbox, *(a).zmin, (a).rr, px, py, pz, sx, sy, sz)


// ---------------------------------------------------------------------------
// two-phase near field
//  scan: one warp per task (<= 32 evaluation points of ONE cell; lane = point).
//        The 27 neighbour cells are walked round-robin, 4 candidates per cell
//        per visit, with an fp32 pre-test; survivors are appended to the
//        point's far / close list in HBM (point-major, contiguous per lane).
//  eval: one thread per evaluation point walks its own lists: exact fp64
//        membership test and the erf kernels.  Lists have nearly equal
//        lengths across a warp (same cell), so the evaluation is dense.
// ---------------------------------------------------------------------------
constexpr int SCAN_STAGE = 128;             // staged candidates per warp

// Neighbour columns of a target column and the candidate range of one lane
// in one of them: columns whose xy distance to the target exceeds the query
// radius are skipped, and the z window is the chord sqrt(r^2 - d_xy^2).
struct ColumnWalk {
    int nxr, nyr;          // columns visited per axis (2 hw + 1, or all when fewer)
    bool allx, ally;
};

__device__ __forceinline__ ColumnWalk column_walk(const CellGeo& g) {
    ColumnWalk w;
    const int nw = 2 * g.hw + 1;
    w.allx = g.ncx < nw; w.ally = g.ncy < nw;
    w.nxr = w.allx ? g.ncx : nw; w.nyr = w.ally ? g.ncy : nw;
    return w;
}

// neighbour column (i) of target column c along one axis: wrapped index, the
// shift that brings its sources next to the target, and the fp32 distance
// from the target coordinate p to the column's interval
__device__ __forceinline__ void column_axis(int c, int i, bool all, int n, int hw, float cs,
                                           float L, float p, int* idx, float* shift,
                                           float* dist) {
    if (all) {                         // every column once, periodic distance
        *idx = i; *shift = 0.f;
        const float lo = i * cs, hi = lo + cs;
        float d = fmaxf(0.f, fmaxf(lo - p, p - hi));
        d = fminf(d, fmaxf(0.f, fmaxf(lo + L - p, p - (hi + L))));
        d = fminf(d, fmaxf(0.f, fmaxf(lo - L - p, p - (hi - L))));
        *dist = d;
        return;
    }
    const int u = c + i - hw;
    int w = u; float sh = 0.f;
    if (w < 0) { w += n; sh = -L; } else if (w >= n) { w -= n; sh = L; }
    *idx = w; *shift = sh;
    const float lo = u * cs, hi = lo + cs;
    *dist = fmaxf(0.f, fmaxf(lo - p, p - hi));
}

// SMALL: a box axis with fewer than 5 columns (every column visited once,
// periodic differences in the test); the common large-box case compiles
// without those branches
template <int SCAN_Q, int SU, int MINB, bool SMALL>
__global__ void __launch_bounds__(NB_THREADS, MINB) near_scan_kernel(NearArgs a) {
    constexpr int W = NB_THREADS / 32;
    __shared__ int qf[W][SCAN_Q + SU][32];
    __shared__ int qcl[W][SCAN_Q + SU][32];
    __shared__ float4 stage[W][SCAN_STAGE + SU];   // + SU: a step's reads never leave it
    const int tid = threadIdx.x, lane = tid & 31, wib = tid >> 5;
    const int64_t task = (blockIdx.x * (int64_t)blockDim.x + tid) >> 5;
    if (task >= a.ntask || task >= *a.ntask_dev) return;
    const int2 tk = a.tasks[task];
    const int col = tk.x;
    const int64_t slot = (int64_t)tk.y + lane;
    const bool live = slot < a.pt_end[col];
    const int64_t i = live ? a.order[slot] : 0;
    float pxf = 0.f, pyf = 0.f, pzf = 0.f;
    if (live) {
        pxf = (float)wrap(a.eval[3 * i], a.g.Lx);
        pyf = (float)wrap(a.eval[3 * i + 1], a.g.Ly);
        pzf = (float)(a.eval[3 * i + 2] - a.g.zlo);
    }
    const int cx = col % a.g.ncx, cy = col / a.g.ncx;
    ColumnWalk cw = column_walk(a.g);
    if (!SMALL) { cw.allx = cw.ally = false; cw.nxr = cw.nyr = 2 * a.g.hw + 1; }
    const float r2f = a.r2f, r2c = a.r2close;
    const float csxf = (float)a.g.csx, csyf = (float)a.g.csy, icsz = (float)(1.0 / a.g.csz);
    const int nzb = a.g.ncz;
    int* lfar = a.list_far + (int64_t)(slot < a.ne ? slot : 0) * a.cap_far;
    int* lcls = a.list_close + (int64_t)(slot < a.ne ? slot : 0) * a.cap_close;
    int nf = 0, nc = 0, qn = 0, qc = 0;
    bool overflow = false;
    // warp-wide flush of whole groups of 4 (16-byte stores, lists stay aligned)
    auto flush = [&](int (*q)[32], int& cnt, int& n, int* list, int cap, bool all) {
        const int m = all ? cnt : (cnt & ~3);
        if (n + m + 4 > cap) { overflow = true; cnt = 0; return; }   // point re-done by the fallback
        for (int e = 0; e < m; e += 4) {
            int4 v;
            v.x = q[e][lane];
            v.y = e + 1 < m ? q[e + 1][lane] : -1;
            v.z = e + 2 < m ? q[e + 2][lane] : -1;
            v.w = e + 3 < m ? q[e + 3][lane] : -1;
            *reinterpret_cast<int4*>(list + n + e) = v;
        }
        n += (m + 3) & ~3;
        for (int e = m; e < cnt; ++e) q[e - m][lane] = q[e][lane];
        cnt -= m;
    };
    for (int iy = 0; iy < cw.nyr; ++iy) {
        int yc; float sy, dyd;
        column_axis(cy, iy, cw.ally, a.g.ncy, a.g.hw, csyf, a.Lyf, pyf, &yc, &sy, &dyd);
        for (int ix = 0; ix < cw.nxr; ++ix) {
            int xc; float sx, dxd;
            column_axis(cx, ix, cw.allx, a.g.ncx, a.g.hw, csxf, a.Lxf, pxf, &xc, &sx, &dxd);
            const float d2 = fmaf(dxd, dxd, dyd * dyd);
            int j = 0, e = 0;
            if (live && d2 <= r2f) {
                const float hz = sqrtf(r2f - d2) * 1.0001f + a.zmarg;
                const int z0 = max(0, min(nzb - 1, (int)floorf((pzf - hz) * icsz)));
                const int z1 = max(0, min(nzb - 1, (int)floorf((pzf + hz) * icsz)));
                const int base = (yc * a.g.ncx + xc) * nzb;
                j = a.start[base + z0];
                e = a.start[base + z1 + 1];
            }
            if (!__any_sync(0xffffffffu, j < e)) continue;
            const float qx = pxf - sx, qy = pyf - sy;
            // the union of the lanes' windows is staged through shared memory
            // in coalesced chunks; each lane tests its own part from there
            int umin = (j < e) ? j : 0x7fffffff, umax = (j < e) ? e : 0;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                umin = min(umin, __shfl_xor_sync(0xffffffffu, umin, o));
                umax = max(umax, __shfl_xor_sync(0xffffffffu, umax, o));
            }
            for (int c0 = umin; c0 < umax; c0 += SCAN_STAGE) {
                const int c1 = min(umax, c0 + SCAN_STAGE);
                __syncwarp();
                for (int q = c0 + lane; q < c1; q += 32) stage[wib][q - c0] = a.srcf[q];
                __syncwarp();
                const int ee = min(e, c1);
                // jj stays within [c0, max(ee, c0)], so a step's reads
                // (jj .. jj + SU - 1) stay inside the padded stage
                const int eec = max(ee, c0);
                int jj = min(max(j, c0), eec);
                while (__any_sync(0xffffffffu, jj < ee)) {
                    // branch-free candidate tests: out-of-window slots read a
                    // stage entry past the window (padded) and are masked; a
                    // hit is pushed with one predicated shared store into the
                    // far or close queue
                    const float4* sp = &stage[wib][jj - c0];
                    int* const pf = &qf[wib][qn][lane];
                    int* const pc = &qcl[wib][qc][lane];
                    int nfh = 0, nch = 0;
#pragma unroll
                    for (int u = 0; u < SU; ++u) {
                        const int q = jj + u;
                        const float4 f = sp[u];
                        float dx = qx - f.x, dy = qy - f.y, dz = pzf - f.z;
                        if (SMALL && cw.allx) dx -= a.Lxf * rintf(dx * a.iLxf);
                        if (SMALL && cw.ally) dy -= a.Lyf * rintf(dy * a.iLyf);
                        const float r2 = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
                        const bool hit = q < ee && r2 <= r2f;
                        const bool far = r2 > r2c;
                        int* const dst = far ? pf + 32 * nfh : pc + 32 * nch;
                        if (hit) *dst = q;
                        nfh += (hit && far) ? 1 : 0;
                        nch += (hit && !far) ? 1 : 0;
                    }
                    qn += nfh;
                    qc += nch;
                    jj = min(jj + SU, eec);
                    if (__any_sync(0xffffffffu, qn >= SCAN_Q)) flush(qf[wib], qn, nf, lfar, a.cap_far, false);
                    if (__any_sync(0xffffffffu, qc >= SCAN_Q)) flush(qcl[wib], qc, nc, lcls, a.cap_close, false);
                }
            }
        }
    }
    flush(qf[wib], qn, nf, lfar, a.cap_far, true);
    flush(qcl[wib], qc, nc, lcls, a.cap_close, true);
    if (live) {
        a.cnt_far[slot] = overflow ? 0 : nf;
        a.cnt_close[slot] = overflow ? 0 : nc;
        if (overflow) a.ovl[atomicAdd(a.overflow, 1)] = (int)slot;
    }
}

// pairs within ulps of the cutoff need the reference's KD-tree test too:
// they are queued and settled by near_boundary_kernel (rare)
__device__ __forceinline__ void defer_pair(const NearArgs& a, int64_t i, int j) {
    const int slot = atomicAdd(a.bnd_cnt, 1);
    if (slot < a.bnd_cap) a.bnd[slot] = make_int2((int)i, j);
    else atomicOr(a.flags, FLAG_NEAR_BND);
}

__device__ __forceinline__ unsigned long long mix64(unsigned long long z);

template <bool FAR, bool F32 = false, bool HASH = false>
__device__ __forceinline__ void eval_list(const NearArgs& a, const double* tab, const int* list,
                                          int n, double px, double py, double pz, int64_t self_i,
                                          double& phi, double& ex, double& ey, double& ez,
                                          int& count, unsigned long long& hs) {
    const double Lx = a.g.Lx, Ly = a.g.Ly;
    const bool nd = a.need_field;
    // far lists: two 16-byte groups per step (one 32-byte sector of the
    // lane's list; 4.27 -> 4.22 ms); the close kernel keeps one (registers)
    constexpr int STEP = FAR ? 8 : 4;
    for (int k = 0; k < n; k += STEP) {
        const int4 j4 = *reinterpret_cast<const int4*>(list + k);
        const int4 j5 = (STEP == 8 && k + 4 < n) ? *reinterpret_cast<const int4*>(list + k + 4)
                                                 : make_int4(-1, -1, -1, -1);
        const int jj[8] = {j4.x, j4.y, j4.z, j4.w, j5.x, j5.y, j5.z, j5.w};
#pragma unroll
        for (int u = 0; u < STEP; ++u) {
            if (jj[u] >= 0) {
                const double4 sv = a.src[jj[u]];
                double dx = __dsub_rn(px, sv.x), dy = __dsub_rn(py, sv.y);
                // minimum image (min_image): |d| <= L/4 needs no shift, and
                // pairs across the periodic boundary are rare -- a warp-
                // uniform branch keeps the shift off the common path
                const bool wx = fabs(dx) > a.qLx, wy = fabs(dy) > a.qLy;
                if (__any_sync(__activemask(), wx || wy)) {
                    if (wx) dx = __dsub_rn(dx, __dmul_rn(Lx, rint(dx * (1.0 / Lx))));
                    if (wy) dy = __dsub_rn(dy, __dmul_rn(Ly, rint(dy * (1.0 / Ly))));
                }
                const double dz = __dsub_rn(pz, sv.z);
                const double r2 = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)),
                                            __dmul_rn(dz, dz));
                if (r2 >= a.win_lo && r2 <= a.r2max) {
                    defer_pair(a, self_i, jj[u]);      // decided by near_boundary_kernel
                } else if (r2 <= a.r2max) {            // == sqrt(r2) <= r_query
                    double g, coef;
                    pair_terms<FAR, F32>(a, tab, r2, g, coef);
                    phi = fma(sv.w, g, phi);
                    if (nd) {
                        const double cq = coef * sv.w;
                        ex = fma(cq, dx, ex); ey = fma(cq, dy, ey); ez = fma(cq, dz, ez);
                    }
                    ++count;
                    if (HASH) hs += mix64((unsigned long long)a.orig[jj[u]]);
                }
            }
        }
    }
}

// fp32 mode: the same list walk in single precision (float4 sources with
// the charge in w, fp32 minimum image), fp64 accumulation; membership is
// decided in fp32 away from the cutoff and by the exact fp64 test (with the
// boundary deferral) inside the thin band where fp32 cannot decide, so the
// pair set is still the reference's.
template <bool FAR, bool HASH>
__device__ __forceinline__ void eval_list_f32(const NearArgs& a, const double* tab, const int* list,
                                              int n, double px, double py, double pz,
                                              int64_t self_i, double& phi, double& ex,
                                              double& ey, double& ez, int& count,
                                              unsigned long long& hs) {
    const float pxf = (float)wrap(px, a.g.Lx), pyf = (float)wrap(py, a.g.Ly);
    const float pzf = (float)(pz - a.g.zlo);
    const bool nd = a.need_field;
    constexpr int STEP = FAR ? 8 : 4;     // far lists: two int4 groups per step
    for (int k = 0; k < n; k += STEP) {
        const int4 j4 = *reinterpret_cast<const int4*>(list + k);
        const int4 j5 = (STEP == 8 && k + 4 < n) ? *reinterpret_cast<const int4*>(list + k + 4)
                                                 : make_int4(-1, -1, -1, -1);
        const int jj[8] = {j4.x, j4.y, j4.z, j4.w, j5.x, j5.y, j5.z, j5.w};
        if (FAR) {
            // far pairs: the step's terms summed in fp32 (each term is an
            // fp32 evaluation already), one fp64 add per step and field
            float gphi = 0.f, gex = 0.f, gey = 0.f, gez = 0.f;
#pragma unroll
            for (int u = 0; u < STEP; ++u) {
                const int j = jj[u];
                if (j < 0) continue;
                const float4 f = a.srcf[j];
                float dx = pxf - f.x, dy = pyf - f.y;
                const float dz = pzf - f.z;
                dx = dx > a.hLxf ? dx - a.Lxf : (dx < -a.hLxf ? dx + a.Lxf : dx);
                dy = dy > a.hLyf ? dy - a.Lyf : (dy < -a.hLyf ? dy + a.Lyf : dy);
                const float r2f = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
                if (r2f > a.r2out_f) continue;
                if (r2f > a.r2in_f) {                // the band: exact fp64 decision
                    const double4 sv = a.src[j];
                    const double ddx = min_image(__dsub_rn(px, sv.x), a.g.Lx);
                    const double ddy = min_image(__dsub_rn(py, sv.y), a.g.Ly);
                    const double ddz = __dsub_rn(pz, sv.z);
                    const double r2 = __dadd_rn(__dadd_rn(__dmul_rn(ddx, ddx), __dmul_rn(ddy, ddy)),
                                                __dmul_rn(ddz, ddz));
                    if (r2 > a.r2max) continue;
                    if (r2 >= a.win_lo) { defer_pair(a, self_i, j); continue; }
                }
                float gf, cf;
                far_terms_f32(a, r2f, gf, cf);
                gphi = fmaf(f.w, gf, gphi);
                if (nd) {
                    const float cq = cf * f.w;
                    gex = fmaf(cq, dx, gex); gey = fmaf(cq, dy, gey); gez = fmaf(cq, dz, gez);
                }
                ++count;
                if (HASH) hs += mix64((unsigned long long)a.orig[j]);
            }
            phi += (double)gphi;
            if (nd) { ex += (double)gex; ey += (double)gey; ez += (double)gez; }
            continue;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int j = jj[u];
            if (j < 0) continue;
            const float4 f = a.srcf[j];
            float dx = pxf - f.x, dy = pyf - f.y;
            const float dz = pzf - f.z;
            dx = dx > a.hLxf ? dx - a.Lxf : (dx < -a.hLxf ? dx + a.Lxf : dx);
            dy = dy > a.hLyf ? dy - a.Lyf : (dy < -a.hLyf ? dy + a.Lyf : dy);
            const float r2f = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
            if (r2f > a.r2out_f) continue;
            double r2 = (double)r2f;
            if (r2f > a.r2in_f) {                    // the band: exact fp64 decision
                const double4 sv = a.src[j];
                const double ddx = min_image(__dsub_rn(px, sv.x), a.g.Lx);
                const double ddy = min_image(__dsub_rn(py, sv.y), a.g.Ly);
                const double ddz = __dsub_rn(pz, sv.z);
                r2 = __dadd_rn(__dadd_rn(__dmul_rn(ddx, ddx), __dmul_rn(ddy, ddy)),
                               __dmul_rn(ddz, ddz));
                if (r2 > a.r2max) continue;
                if (r2 >= a.win_lo) { defer_pair(a, self_i, j); continue; }
            }
            double g, coef;
            pair_terms<FAR, FAR>(a, tab, r2, g, coef);
            const double q = (double)f.w;
            phi = fma(q, g, phi);
            if (nd) {
                const double cq = coef * q;
                ex = fma(cq, (double)dx, ex); ey = fma(cq, (double)dy, ey);
                ez = fma(cq, (double)dz, ez);
            }
            ++count;
            if (HASH) hs += mix64((unsigned long long)a.orig[j]);
        }
    }
}

// Evaluation of one list kind per launch: the far lists (the bulk; erfc-only
// kernel, small register footprint, high occupancy) write the sums, the close
// lists (general kernel) add to them.
template <bool FAR, int MINB, bool F32 = false, bool HASH = false>
__global__ void __launch_bounds__(NB_THREADS, MINB) near_eval_kernel(NearArgs a) {
    // the close launch is persistent (grid = resident CTAs, warps stride
    // over the tasks) so its table staging is paid once per CTA, not per
    // 4 tasks; with the close table the erfcx table is not needed
    __shared__ __align__(16) double tab[SE_ERFCX_NP * (SE_ERFCX_DEG + 1) + (FAR ? 0 : CL_TAB)];
    const int tid = threadIdx.x, lane = tid & 31;
    if (!FAR || !a.use_poly) {
        if (FAR || !a.use_ctab)
            for (int e = tid; e < SE_ERFCX_NP * (SE_ERFCX_DEG + 1); e += blockDim.x)
                tab[e] = (&se_erfcx_tab[0][0])[e];
        if (!FAR && a.use_ctab)
            for (int e = tid; e < CL_TAB; e += blockDim.x)
                tab[SE_ERFCX_NP * (SE_ERFCX_DEG + 1) + e] = a.ctab[e];
        __syncthreads();
    }
    const int64_t ntask = min(a.ntask, (int64_t)*a.ntask_dev);
    const int64_t wstride = FAR ? ntask : (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t task = (blockIdx.x * (int64_t)blockDim.x + tid) >> 5; task < ntask;
         task += wstride) {
        const int2 tk = a.tasks[task];
        const int64_t slot = (int64_t)tk.y + lane;
        const bool live = slot < a.pt_end[tk.x];
        double phi = 0, ex = 0, ey = 0, ez = 0;
        int count = 0;
        unsigned long long hs = 0;
        int64_t i = 0;
        if (live) {
            i = a.order[slot];
            const double px = a.eval[3 * i], py = a.eval[3 * i + 1], pz = a.eval[3 * i + 2];
            if (F32)
                eval_list_f32<FAR, HASH>(a, tab,
                                         FAR ? a.list_far + slot * a.cap_far
                                             : a.list_close + slot * a.cap_close,
                                         FAR ? a.cnt_far[slot] : a.cnt_close[slot], px, py, pz,
                                         i, phi, ex, ey, ez, count, hs);
            else if (FAR)
                eval_list<true, false, HASH>(a, tab, a.list_far + slot * a.cap_far,
                                             a.cnt_far[slot], px, py, pz, i, phi, ex, ey, ez,
                                             count, hs);
            else
                eval_list<false, false, HASH>(a, tab, a.list_close + slot * a.cap_close,
                                              a.cnt_close[slot], px, py, pz, i, phi, ex, ey, ez,
                                              count, hs);
            if (HASH) {                             // overflowed points are re-done below
                if (FAR) { a.phash[i] = hs; a.phash[a.ne + i] = (unsigned long long)count; }
                else { a.phash[i] += hs; a.phash[a.ne + i] += (unsigned long long)count; }
            }
            if (FAR) {
                a.out[i] = phi;
                if (a.need_field) {
                    a.out[a.out_stride + i] = ex;
                    a.out[2 * a.out_stride + i] = ey;
                    a.out[3 * a.out_stride + i] = ez;
                }
            } else {
                a.out[i] += phi;
                if (a.need_field) {
                    a.out[a.out_stride + i] += ex;
                    a.out[2 * a.out_stride + i] += ey;
                    a.out[3 * a.out_stride + i] += ez;
                }
            }
        }
        unsigned long long cnt = (unsigned long long)count;
        for (int off = 16; off > 0; off >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, off);
        if (lane == 0 && a.npairs && cnt) atomicAdd((unsigned long long*)a.npairs, cnt);
    }
}

// splitmix64 finaliser: the per-pair term of the pair-set hash (SE_PAIR_HASH;
// the test side is tests/_golden.py pair_hash)
__device__ __forceinline__ unsigned long long mix64(unsigned long long z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

// One pair of an evaluation point (eval_list's body for one source).
template <bool FAR, bool F32, bool HASH = false>
__device__ __forceinline__ void eval_pair(const NearArgs& a, const double* tab, int j,
                                          double px, double py, double pz, int64_t self_i,
                                          double& phi, double& ex, double& ey, double& ez,
                                          int& count, unsigned long long* hsum = nullptr) {
    const double4 sv = a.src[j];
    const double dx = min_image(__dsub_rn(px, sv.x), a.g.Lx);
    const double dy = min_image(__dsub_rn(py, sv.y), a.g.Ly);
    const double dz = __dsub_rn(pz, sv.z);
    const double r2 = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
    if (r2 >= a.win_lo && r2 <= a.r2max) {
        defer_pair(a, self_i, j);                 // decided by near_boundary_kernel
    } else if (r2 <= a.r2max) {
        double g, coef;
        pair_terms<FAR, F32>(a, tab, r2, g, coef);
        phi = fma(sv.w, g, phi);
        if (a.need_field) {
            const double cq = coef * sv.w;
            ex = fma(cq, dx, ex); ey = fma(cq, dy, ey); ez = fma(cq, dz, ez);
        }
        ++count;
        if (HASH) *hsum += mix64((unsigned long long)a.orig[j]);
    }
}

// Fused near field: one warp per evaluation point (cell-sorted order, so
// neighbouring warps share their source windows in L1).  The lanes walk the
// point's chord windows 32 sources at a time with the fp32 pre-test; the
// hits are compacted (ballot) into a far and a close queue in shared memory
// and evaluated 32 at a time, so the pair kernels run on full warps and no
// pair list goes through HBM.
constexpr int FQ = 64;
constexpr int64_t NEAR_FUSED_MAX = 40000;       // evaluation points (measured crossover)

template <bool F32, int MINB, bool FROM_LIST = false, bool HASH = false>
__global__ void __launch_bounds__(NB_THREADS, MINB) near_fused_kernel(NearArgs a) {
    constexpr int W = NB_THREADS / 32;
    __shared__ __align__(16) double tab[SE_ERFCX_NP * (SE_ERFCX_DEG + 1) + CL_TAB];
    __shared__ int qf[W][FQ], qc[W][FQ];
    const int tid = threadIdx.x, lane = tid & 31, wib = tid >> 5;
    for (int e = tid; e < SE_ERFCX_NP * (SE_ERFCX_DEG + 1); e += blockDim.x)
        tab[e] = (&se_erfcx_tab[0][0])[e];
    if (a.use_ctab)
        for (int e = tid; e < CL_TAB; e += blockDim.x)
            tab[SE_ERFCX_NP * (SE_ERFCX_DEG + 1) + e] = a.ctab[e];
    __syncthreads();
    const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + tid) >> 5;
    // FROM_LIST: the points whose pair lists overflowed in the scan (device
    // count, grid-stride), evaluated here instead of rescanning
    const int64_t nw = FROM_LIST ? (int64_t)(*a.overflow) : a.ne;
    const int64_t wstep = FROM_LIST ? ((int64_t)gridDim.x * blockDim.x) >> 5 : nw;
    for (int64_t w = w0; w < nw; w += wstep) {
    const int64_t i = a.order[FROM_LIST ? a.ovl[w] : w];
    const double px = a.eval[3 * i], py = a.eval[3 * i + 1], pz = a.eval[3 * i + 2];
    int cx, cy, cz;
    cell_of(a.g, px, py, pz, &cx, &cy, &cz);
    const float pxf = (float)wrap(px, a.g.Lx), pyf = (float)wrap(py, a.g.Ly);
    const float pzf = (float)(pz - a.g.zlo);
    const ColumnWalk cw = column_walk(a.g);
    const float r2f = a.r2f, r2c = a.r2close;
    const float csxf = (float)a.g.csx, csyf = (float)a.g.csy, icsz = (float)(1.0 / a.g.csz);
    const int nzb = a.g.ncz;
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    int count = 0, nf = 0, nc = 0;
    unsigned long long hs = 0;
    const unsigned below = (1u << lane) - 1u;
    for (int iy = 0; iy < cw.nyr; ++iy) {
        int yc; float sy, dyd;
        column_axis(cy, iy, cw.ally, a.g.ncy, a.g.hw, csyf, a.Lyf, pyf, &yc, &sy, &dyd);
        for (int ix = 0; ix < cw.nxr; ++ix) {
            int xc; float sx, dxd;
            column_axis(cx, ix, cw.allx, a.g.ncx, a.g.hw, csxf, a.Lxf, pxf, &xc, &sx, &dxd);
            const float d2 = fmaf(dxd, dxd, dyd * dyd);
            if (d2 > r2f) continue;
            const float hz = sqrtf(r2f - d2) * 1.0001f + a.zmarg;
            const int z0 = max(0, min(nzb - 1, (int)floorf((pzf - hz) * icsz)));
            const int z1 = max(0, min(nzb - 1, (int)floorf((pzf + hz) * icsz)));
            const int base = (yc * a.g.ncx + xc) * nzb;
            const int j0 = a.start[base + z0], j1 = a.start[base + z1 + 1];
            const float qx = pxf - sx, qy = pyf - sy;
            for (int b = j0; b < j1; b += 32) {
                const int s = b + lane;
                bool far = false, close = false;
                if (s < j1) {
                    const float4 f = a.srcf[s];
                    float dx = qx - f.x, dy = qy - f.y, dz = pzf - f.z;
                    if (cw.allx) dx -= a.Lxf * rintf(dx * a.iLxf);
                    if (cw.ally) dy -= a.Lyf * rintf(dy * a.iLyf);
                    const float r2 = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
                    if (r2 <= r2f) { far = r2 > r2c; close = !far; }
                }
                const unsigned bf = __ballot_sync(0xffffffffu, far);
                const unsigned bc = __ballot_sync(0xffffffffu, close);
                if (far) qf[wib][nf + __popc(bf & below)] = s;
                if (close) qc[wib][nc + __popc(bc & below)] = s;
                nf += __popc(bf);
                nc += __popc(bc);
                __syncwarp();
                if (nf >= 32) {
                    eval_pair<true, F32, HASH>(a, tab, qf[wib][lane], px, py, pz, i, acc[0],
                                               acc[1], acc[2], acc[3], count, &hs);
                    __syncwarp();
                    if (lane < nf - 32) qf[wib][lane] = qf[wib][32 + lane];
                    nf -= 32;
                    __syncwarp();
                }
                if (nc >= 32) {
                    eval_pair<false, false, HASH>(a, tab, qc[wib][lane], px, py, pz, i, acc[0],
                                                  acc[1], acc[2], acc[3], count, &hs);
                    __syncwarp();
                    if (lane < nc - 32) qc[wib][lane] = qc[wib][32 + lane];
                    nc -= 32;
                    __syncwarp();
                }
            }
        }
    }
    if (lane < nf)
        eval_pair<true, F32, HASH>(a, tab, qf[wib][lane], px, py, pz, i, acc[0], acc[1], acc[2],
                                   acc[3], count, &hs);
    if (lane < nc)
        eval_pair<false, false, HASH>(a, tab, qc[wib][lane], px, py, pz, i, acc[0], acc[1],
                                      acc[2], acc[3], count, &hs);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[c] += __shfl_xor_sync(0xffffffffu, acc[c], o);
        count += __shfl_xor_sync(0xffffffffu, count, o);
        if (HASH) hs += __shfl_xor_sync(0xffffffffu, hs, o);
    }
    if (lane == 0) {
        if (HASH) { a.phash[i] = hs; a.phash[a.ne + i] = (unsigned long long)count; }
        a.out[i] = acc[0];
        if (a.need_field) {
            a.out[a.out_stride + i] = acc[1];
            a.out[2 * a.out_stride + i] = acc[2];
            a.out[3 * a.out_stride + i] = acc[3];
        }
        if (a.npairs && count) atomicAdd((unsigned long long*)a.npairs, (unsigned long long)count);
    }
    }
}

// A few evaluation points (the gauge origin): one CTA per point, the threads
// stride over the 27 neighbour cells' sources with the exact test and the
// general kernel, then a block reduction.  Avoids the sort / task / list
// machinery whose single-warp scan is latency-bound for one point.
constexpr int FEW_POINTS = 64;

__global__ void __launch_bounds__(256) near_few_kernel(NearArgs a) {
    __shared__ double tab[SE_ERFCX_NP * (SE_ERFCX_DEG + 1)];
    __shared__ double red[4][8];
    __shared__ unsigned long long redc[8];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int e = tid; e < SE_ERFCX_NP * (SE_ERFCX_DEG + 1); e += blockDim.x)
        tab[e] = (&se_erfcx_tab[0][0])[e];
    __syncthreads();
    const int64_t i = blockIdx.x;
    const double px = a.eval[3 * i], py = a.eval[3 * i + 1], pz = a.eval[3 * i + 2];
    int cx, cy, cz;
    cell_of(a.g, px, py, pz, &cx, &cy, &cz);
    const ColumnWalk cw = column_walk(a.g);
    const float pxf = (float)wrap(px, a.g.Lx), pyf = (float)wrap(py, a.g.Ly);
    const float pzf = (float)(pz - a.g.zlo);
    const float csxf = (float)a.g.csx, csyf = (float)a.g.csy, icsz = (float)(1.0 / a.g.csz);
    double phi = 0, ex = 0, ey = 0, ez = 0;
    unsigned long long count = 0, hs = 0;
    const double Lx = a.g.Lx, Ly = a.g.Ly;
    for (int iy = 0; iy < cw.nyr; ++iy) {
        int yc; float sy, dyd;
        column_axis(cy, iy, cw.ally, a.g.ncy, a.g.hw, csyf, a.Lyf, pyf, &yc, &sy, &dyd);
        for (int ix = 0; ix < cw.nxr; ++ix) {
            int xc; float sx, dxd;
            column_axis(cx, ix, cw.allx, a.g.ncx, a.g.hw, csxf, a.Lxf, pxf, &xc, &sx, &dxd);
            const float d2 = fmaf(dxd, dxd, dyd * dyd);
            if (d2 > a.r2f) continue;
            const float hz = sqrtf(a.r2f - d2) * 1.0001f + a.zmarg;
            const int z0 = max(0, min(a.g.ncz - 1, (int)floorf((pzf - hz) * icsz)));
            const int z1 = max(0, min(a.g.ncz - 1, (int)floorf((pzf + hz) * icsz)));
            const int base = (yc * a.g.ncx + xc) * a.g.ncz;
            for (int j = a.start[base + z0] + tid; j < a.start[base + z1 + 1]; j += blockDim.x) {
                const double4 sv = a.src[j];
                const double dx = min_image(__dsub_rn(px, sv.x), Lx);
                const double dy = min_image(__dsub_rn(py, sv.y), Ly);
                const double dz = __dsub_rn(pz, sv.z);
                const double r2 = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)),
                                            __dmul_rn(dz, dz));
                if (r2 >= a.win_lo && r2 <= a.r2max) {
                    defer_pair(a, i, j);
                } else if (r2 <= a.r2max) {
                    double g, coef;
                    pair_terms<false>(a, tab, r2, g, coef);
                    phi = fma(sv.w, g, phi);
                    if (a.need_field) {
                        const double cq = coef * sv.w;
                        ex = fma(cq, dx, ex); ey = fma(cq, dy, ey); ez = fma(cq, dz, ez);
                    }
                    ++count;
                    if (a.phash) hs += mix64((unsigned long long)a.orig[j]);
                }
            }
        }
    }
    for (int o = 16; o > 0; o >>= 1) {
        phi += __shfl_xor_sync(0xffffffffu, phi, o);
        ex += __shfl_xor_sync(0xffffffffu, ex, o);
        ey += __shfl_xor_sync(0xffffffffu, ey, o);
        ez += __shfl_xor_sync(0xffffffffu, ez, o);
        count += __shfl_xor_sync(0xffffffffu, count, o);
        hs += __shfl_xor_sync(0xffffffffu, hs, o);
    }
    if (lane == 0) {
        red[0][warp] = phi; red[1][warp] = ex; red[2][warp] = ey; red[3][warp] = ez;
        redc[warp] = count;
        if (a.phash) {                            // zeroed by the host
            atomicAdd(a.phash + i, hs);
            atomicAdd(a.phash + a.ne + i, count);
        }
    }
    __syncthreads();
    if (tid == 0) {
        double v[4] = {0, 0, 0, 0};
        unsigned long long cnt = 0;
        for (int w = 0; w < 8; ++w) {
            for (int c = 0; c < 4; ++c) v[c] += red[c][w];
            cnt += redc[w];
        }
        a.out[i] = v[0];
        if (a.need_field) {
            a.out[a.out_stride + i] = v[1];
            a.out[2 * a.out_stride + i] = v[2];
            a.out[3 * a.out_stride + i] = v[3];
        }
        if (a.npairs) atomicAdd((unsigned long long*)a.npairs, cnt);
    }
}

// Deferred boundary pairs: the reference's KD-tree test, then the general
// kernel; contributions added atomically (a handful of pairs per solve).
__global__ void near_boundary_kernel(NearArgs a) {
    __shared__ double tab[SE_ERFCX_NP * (SE_ERFCX_DEG + 1)];
    for (int e = threadIdx.x; e < SE_ERFCX_NP * (SE_ERFCX_DEG + 1); e += blockDim.x)
        tab[e] = (&se_erfcx_tab[0][0])[e];
    __syncthreads();
    const int n = min(*a.bnd_cnt, a.bnd_cap);
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n; e += gridDim.x * blockDim.x) {
        const int2 pr = a.bnd[e];
        const int64_t i = pr.x;
        const double px = a.eval[3 * i], py = a.eval[3 * i + 1], pz = a.eval[3 * i + 2];
        const double4 sv = a.src[pr.y];
        const double dx = min_image(__dsub_rn(px, sv.x), a.g.Lx);
        const double dy = min_image(__dsub_rn(py, sv.y), a.g.Ly);
        const double dz = __dsub_rn(pz, sv.z);
        const double r2 = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)),
                                    __dmul_rn(dz, dz));
        if (!tree_keep(a, px, py, pz, sv.x, sv.y, sv.z)) continue;
        double g, coef;
        pair_terms<false>(a, tab, r2, g, coef);
        atomicAdd(a.out + i, sv.w * g);
        if (a.need_field) {
            const double cq = coef * sv.w;
            atomicAdd(a.out + a.out_stride + i, cq * dx);
            atomicAdd(a.out + 2 * a.out_stride + i, cq * dy);
            atomicAdd(a.out + 3 * a.out_stride + i, cq * dz);
        }
        if (a.npairs) atomicAdd((unsigned long long*)a.npairs, 1ull);
        if (a.phash) {
            atomicAdd(a.phash + i, mix64((unsigned long long)a.orig[pr.y]));
            atomicAdd(a.phash + a.ne + i, 1ull);
        }
    }
}

__global__ void add_count_kernel(const int* src, int* acc) { *acc += *src; }

// point tasks: per xy column, ceil(count/32) warps (points sorted by z
// within the column, so a warp's z windows overlap)
__global__ void task_count_kernel(const int* pt_start, int ncol, int nzb, int* ntask) {
    int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= ncol) return;
    ntask[c] = (pt_start[(c + 1) * nzb] - pt_start[c * nzb] + 31) >> 5;
}

__global__ void task_fill_kernel(const int* pt_start, const int* toff, int ncol, int nzb,
                                 int2* tasks, int* pt_end) {
    int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= ncol) return;
    int b = pt_start[c * nzb], e = pt_start[(c + 1) * nzb];
    pt_end[c] = e;
    int o = toff[c];
    for (int f = b; f < e; f += 32) tasks[o++] = make_int2(c, f);
}

__global__ void point_starts_kernel(const uint32_t* keys, int64_t n, int ncell, int* start) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i > n) return;
    int cur = (i < n) ? (int)keys[i] : ncell;
    int prev = (i == 0) ? -1 : (int)keys[i - 1];
    for (int c = prev + 1; c <= cur; ++c) start[c] = (int)i;
}

__global__ void point_keys_kernel(const double* pts, int64_t n, CellGeo g, uint32_t* keys,
                                  int* perm) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    int cx, cy, cz;
    keys[i] = (uint32_t)cell_of(g, pts[3 * i], pts[3 * i + 1], pts[3 * i + 2], &cx, &cy, &cz);
    perm[i] = (int)i;
}

// ---------------------------------------------------------------------------
// final combination and energy                          slab.py:359-391
// ---------------------------------------------------------------------------
struct FinArgs {
    const double* far; const double* near; const double* q; int64_t n;
    int64_t first, nfar;          // own charges first..first+n; far has stride nfar
    double cell; int forces, potential, self_inf; double self_inf_value;
    const double* scal;           // scal[1] = B_i
    double* phi; double* E; double* partial;
};


__global__ void finalize_kernel(FinArgs a) {
    __shared__ double red[256];
    double acc = 0.0;
    double b_i = a.potential ? a.scal[1] : 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < a.n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t gi = a.first + i;
        double phi_near = a.near[i];
        if (a.self_inf) phi_near = phi_near + a.q[gi] * a.self_inf_value;
        double phi = (a.cell * a.far[gi] + phi_near) + b_i;
        a.phi[i] = phi;
        if (a.forces) {
            a.E[3 * i] = -(a.cell * a.far[a.nfar + gi]) + a.near[a.n + i];
            a.E[3 * i + 1] = -(a.cell * a.far[2 * a.nfar + gi]) + a.near[2 * a.n + i];
            a.E[3 * i + 2] = -(a.cell * a.far[3 * a.nfar + gi]) + a.near[3 * a.n + i];
        }
        acc += a.q[gi] * phi;
    }
    red[threadIdx.x] = acc;
    __syncthreads();
    for (int w = 128; w > 0; w >>= 1) {
        if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) a.partial[blockIdx.x] = red[0];
}

__global__ void sum_partials_kernel(const double* partial, int nb, double scale,
                                    double* dst) {
    __shared__ double red[256];
    double acc = 0.0;
    for (int i = threadIdx.x; i < nb; i += blockDim.x) acc += partial[i];
    red[threadIdx.x] = acc;
    __syncthreads();
    for (int w = 128; w > 0; w >>= 1) {
        if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) *dst = scale * red[0];
}

}  // namespace

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
static CellGeo cell_geo(const Plan* p, const CellList& cl) {
    CellGeo g;
    g.ncx = cl.ncx; g.ncy = cl.ncy; g.ncz = cl.ncz; g.hw = cl.hw;
    g.csx = cl.csx; g.csy = cl.csy; g.csz = cl.csz; g.zlo = cl.zlo;
    g.Lx = p->P.Lx; g.Ly = p->P.Ly;
    return g;
}

void build_cells(Plan* p, const double* d_pos, const double* d_q, int64_t n, bool in_domain,
                 const double* d_zsrc_min, CellList* clp, int parts) {
    NvtxRange nv("se.cell_list");
    const double eps = p->P.eps;
    const double fb = -(p->P.eps_b - eps) / (p->P.eps_b + eps);
    const double ft = -(p->P.eps_t - eps) / (p->P.eps_t + eps);
    const int nb = fb != 0.0, nt = ft != 0.0;
    const int64_t ns_all = n * (1 + nb + nt);
    // the list holds [off, off + ns) of the sources [charges; bottom; top]
    const int64_t off = (parts == CL_IMAGES) ? n : 0;
    const int64_t ns = (parts == CL_CHARGES) ? n : (parts == CL_IMAGES ? ns_all - n : ns_all);
    CellList& cl = clp ? *clp : p->cl;
    if (ns > cl.cap) {
        void* olds[] = {cl.src, cl.srcf, cl.orig};
        for (void* o : olds) dfree(p, o);
        const int64_t cap = ns < 64 ? 64 : ns;
        cl.src = dalloc<double4>(p, cap);
        cl.srcf = dalloc<float4>(p, cap);
        cl.orig = dalloc<int>(p, cap);
        cl.cap = cap;
    }
    if (ns_all > p->cl_cap) {
        void* olds[] = {p->d_ckeys, p->d_ckeys2,
                        p->d_cperm, p->d_cperm2, p->d_near_src, p->d_near_cub,
                        p->d_tgt, p->d_tkeys, p->d_tkeys2, p->d_tperm};
        for (void* o : olds) dfree(p, o);
        int64_t cap = ns_all < 64 ? 64 : ns_all;
        p->d_ckeys = dalloc<uint32_t>(p, cap);
        p->d_ckeys2 = dalloc<uint32_t>(p, cap);
        p->d_cperm = dalloc<int>(p, cap);
        p->d_cperm2 = dalloc<int>(p, cap);
        p->d_near_src = dalloc<double4>(p, cap);
        p->d_tgt = dalloc<int>(p, cap);
        p->d_tkeys = dalloc<uint32_t>(p, cap);
        p->d_tkeys2 = dalloc<uint32_t>(p, cap);
        p->d_tperm = dalloc<int>(p, cap);
        size_t bytes = 0;
        SE_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, (uint32_t*)nullptr,
                                                (uint32_t*)nullptr, (int*)nullptr,
                                                (int*)nullptr, (int)cap, 0, 32,
                                                p->stream));
        p->near_cub_bytes = bytes;
        p->d_near_cub = dalloc<char>(p, bytes);
        p->cl_cap = ns_all;
    }
    cl.n = ns;
    if (ns_all == 0) { cl.n = 0; return; }
    SrcBuild sb{d_pos, d_q, n, p->P.H, fb, ft, nb, nt, p->d_near_src, ns_all};
    make_near_sources<<<(unsigned)((n + 255) / 256), 256, 0, p->stream>>>(sb);
    SE_LAUNCHED(p);
    // device copy of the reference's KD-tree z origin (boundary pair tests),
    // over ALL sources whichever part this list holds
    if (!p->d_mm) p->d_mm = dalloc<double>(p, 256);
    zrange_kernel<<<64, 256, 0, p->stream>>>(p->d_near_src, ns_all, p->d_mm);
    SE_LAUNCHED(p);
    zmin_kernel<<<1, 1, 0, p->stream>>>(p->d_mm, 64, p->P.r_cut, d_zsrc_min, p->d_mm + 200);
    SE_LAUNCHED(p);
    double zmin = 1e300, zmax = -1e300;
    if (in_domain) {
        // charges lie in the extended domain [z0, z1] (checked by the spread),
        // the mirror layers in its reflections: no device round trip
        zmin = p->P.z0; zmax = p->P.z1;
        if (nb) zmin = std::min(zmin, -p->P.z1);
        if (nt) zmax = std::max(zmax, 2.0 * p->P.H - p->P.z0);
    } else {
        // z extent of the sources (one small device->host read)
        int nblk = 64;
        std::vector<double> mm(2 * nblk);
        SE_CUDA(cudaMemcpyAsync(mm.data(), p->d_mm, sizeof(double) * 2 * nblk,
                                cudaMemcpyDeviceToHost, p->stream));
        SE_CUDA(cudaStreamSynchronize(p->stream));
        for (int b = 0; b < nblk; ++b) { zmin = std::min(zmin, mm[2 * b]); zmax = std::max(zmax, mm[2 * b + 1]); }
    }
    const double rc = std::max(p->P.r_cut, p->P.r_nf);
    // xy columns of r_c / 2 (5 x 5 walk).  r_c / 3 (7 x 7): scan 2.59 ->
    // 2.44 ms but the evaluation 4.13 -> 4.25 ms (its lanes' list walks
    // drift apart, fewer shared source lines in L1); r_c / 4: 7.2 ms in all
    static const int cdiv = [] {
        const char* e = std::getenv("SE_CELL_XYDIV");
        return e ? std::max(2, std::atoi(e)) : 2;
    }();
    cl.hw = cdiv;
    cl.ncx = std::max(1, (int)std::floor(p->P.Lx / (rc / cdiv)));
    cl.ncy = std::max(1, (int)std::floor(p->P.Ly / (rc / cdiv)));
    cl.csx = p->P.Lx / cl.ncx;
    cl.csy = p->P.Ly / cl.ncy;
    cl.zlo = zmin - rc;
    double zspan = (zmax + rc) - cl.zlo;
    // z bins of r_c / 16 (C4 scan 2.64 -> 2.60 ms vs r_c / 8: tighter chord
    // windows; 24 / 32 no better), r_c / 8 if the cell grid would grow too large
    static const double zdiv = [] {
        const char* e = std::getenv("SE_CELL_ZDIV");
        return e ? std::atof(e) : 16.0;
    }();
    cl.ncz = std::max(1, (int)std::floor(zspan / (rc / zdiv)));
    if ((int64_t)cl.ncx * cl.ncy * cl.ncz > (1 << 26))
        cl.ncz = std::max(1, (int)std::floor(zspan / (0.125 * rc)));
    cl.csz = zspan / cl.ncz;
    int64_t ncell = (int64_t)cl.ncx * cl.ncy * cl.ncz;
    if (ncell > (1 << 26)) throw Error(SE_ERR_VALUE, "near-field cell grid too large");
    if (ncell + 1 > cl.cell_cap) {
        dfree(p, cl.start);
        cl.start = dalloc<int>(p, ncell + 1);
        cl.cell_cap = ncell + 1;
    }
    CellGeo g = cell_geo(p, cl);
    if (ns == 0) {
        SE_CUDA(cudaMemsetAsync(cl.start, 0, sizeof(int) * (ncell + 1), p->stream));
        return;
    }
    cell_keys_kernel<<<(unsigned)((ns + 255) / 256), 256, 0, p->stream>>>(
        p->d_near_src + off, ns, g, p->d_ckeys, p->d_cperm);
    SE_LAUNCHED(p);
    int end_bit = 1;
    while (end_bit < 32 && ((uint64_t)ncell >> end_bit) != 0) ++end_bit;
    size_t bytes = p->near_cub_bytes;
    SE_CUDA(cub::DeviceRadixSort::SortPairs(p->d_near_cub, bytes, p->d_ckeys, p->d_ckeys2,
                                            p->d_cperm, p->d_cperm2, (int)ns, 0, end_bit,
                                            p->stream));
    cell_fill_kernel<<<(unsigned)((ns + 1 + 255) / 256), 256, 0, p->stream>>>(
        p->d_ckeys2, p->d_cperm2, ns, (int)ncell, p->d_near_src + off, g, cl.start, cl.src,
        cl.srcf, cl.orig, (int)off);
    SE_LAUNCHED(p);
}

// erfcx on [xa, xb] as a degree-FAR_DEG polynomial in t = (x - mid) / half:
// Chebyshev interpolation, converted to the monomial basis; accepted when
// the relative error at 400 test points is below 1e-14.
static bool fit_far_poly(double xa, double xb, double* mid, double* inv_half, double* pc,
                         int deg = FAR_DEG, double tol = 1e-14) {
    const int n = deg + 1;
    const double m = 0.5 * (xa + xb), h = 0.5 * (xb - xa);
    if (!(h > 0) || xa < 0.25 || xb > 26.0) return false;
    auto erfcx = [](double x) { return std::erfc(x) * std::exp(x * x); };
    std::vector<double> f(n), c(n, 0.0);
    for (int k = 0; k < n; ++k) f[k] = erfcx(m + h * std::cos(M_PI * (k + 0.5) / n));
    for (int j = 0; j < n; ++j) {                    // Chebyshev coefficients
        double acc = 0;
        for (int k = 0; k < n; ++k) acc += f[k] * std::cos(M_PI * j * (k + 0.5) / n);
        c[j] = acc * (j == 0 ? 1.0 : 2.0) / n;
    }
    // monomial coefficients: sum_j c_j T_j(t), T_{j+1} = 2t T_j - T_{j-1}
    std::vector<double> tprev(n, 0.0), tcur(n, 0.0), tnext(n, 0.0), mono(n, 0.0);
    tprev[0] = 1.0;                                  // T_0
    tcur[1] = 1.0;                                   // T_1
    mono[0] += c[0];
    if (n > 1) mono[1] += c[1];
    for (int j = 2; j < n; ++j) {
        for (int i = 0; i < n; ++i) tnext[i] = (i > 0 ? 2.0 * tcur[i - 1] : 0.0) - tprev[i];
        for (int i = 0; i < n; ++i) mono[i] += c[j] * tnext[i];
        tprev = tcur; tcur = tnext;
    }
    double worst = 0;
    for (int k = 0; k <= 400; ++k) {
        const double t = -1.0 + 2.0 * k / 400.0, x = m + h * t;
        double acc = mono[n - 1];
        for (int j = n - 2; j >= 0; --j) acc = std::fma(acc, t, mono[j]);
        const double ref = erfcx(x);
        worst = std::max(worst, std::fabs(acc - ref) / ref);
    }
    if (!(worst < tol)) return false;
    *mid = m; *inv_half = 1.0 / h;
    for (int i = 0; i < n; ++i) pc[i] = mono[i];
    return true;
}

// The general near kernel on the host (same formulas as pair_terms<false>,
// libm erf / exp): g(r) and coef(r) = -g'(r)/r, r > 0.
static void kernel_host(const NearKernel& k, double r, double* g, double* coef) {
    const double ic1 = 1.0 / k.c1, ic2 = 1.0 / k.c2, ts = 2.0 / std::sqrt(M_PI);
    const double x1 = r * ic1, x2 = r * ic2;
    const double E1 = (r <= 6.5 * k.c1) ? std::erf(x1) : 1.0, E2 = std::erf(x2);
    const double e1 = std::exp(-x1 * x1), e2 = std::exp(-x2 * x2);
    const double v1 = (r < 1e-10 * k.c1) ? ts * ic1 : E1 / r;
    const double v2 = (r < 1e-10 * k.c2) ? ts * ic2 : E2 / r;
    *g = (v1 - v2) * k.inv4pie;
    auto series = [&](double x, double ic) {
        const double u = x * x;
        return ts * (ic * ic) * x * (-2.0 / 3.0 + u * (2.0 / 5.0 + u * (-1.0 / 7.0 + u / 27.0)));
    };
    double d1, d2;
    if (r > 6.5 * k.c1) d1 = -1.0 / (r * r);
    else if (r < 1e-2 * k.c1) d1 = series(x1, ic1);
    else d1 = ts * e1 * ic1 / r - v1 / r;
    if (r < 1e-2 * k.c2) d2 = series(x2, ic2);
    else d2 = ts * e2 * ic2 / r - v2 / r;
    *coef = -((d1 - d2) * k.inv4pie) / r;
}

// Piecewise Chebyshev fit of g and coef on [0, rhi]: CL_P pieces, degree
// CL_D, monomial in the local variable t in [-1, 1].  Accepted when the error
// at 33 points per piece is below 1e-13 (g) / 1e-11 (coef) of the largest
// value.
static bool fit_close_table(const NearKernel& k, double rhi, std::vector<double>& tab,
                            double* w_out) {
    const int n = CL_D + 1;
    const double w = rhi / CL_P;
    tab.assign(CL_TAB, 0.0);
    double gmax = 0, cmax = 0, gerr = 0, cerr = 0;
    std::vector<double> fg(n), fc(n), c(n), mono(n);
    for (int pc = 0; pc < CL_P; ++pc) {
        const double mid = (pc + 0.5) * w, h = 0.5 * w;
        for (int q = 0; q < n; ++q) {
            const double r = mid + h * std::cos(M_PI * (q + 0.5) / n);
            kernel_host(k, r, &fg[q], &fc[q]);
        }
        for (int f = 0; f < 2; ++f) {
            const std::vector<double>& fv = f ? fc : fg;
            for (int j = 0; j < n; ++j) {
                double acc = 0;
                for (int q = 0; q < n; ++q) acc += fv[q] * std::cos(M_PI * j * (q + 0.5) / n);
                c[j] = acc * (j == 0 ? 1.0 : 2.0) / n;
            }
            std::vector<double> tp(n, 0.0), tc(n, 0.0), tn(n, 0.0);
            std::fill(mono.begin(), mono.end(), 0.0);
            tp[0] = 1.0; mono[0] += c[0];
            if (n > 1) { tc[1] = 1.0; mono[1] += c[1]; }
            for (int j = 2; j < n; ++j) {
                for (int i2 = 0; i2 < n; ++i2) tn[i2] = (i2 > 0 ? 2.0 * tc[i2 - 1] : 0.0) - tp[i2];
                for (int i2 = 0; i2 < n; ++i2) mono[i2] += c[j] * tn[i2];
                tp = tc; tc = tn;
            }
            for (int i2 = 0; i2 < n; ++i2) tab[2 * (pc * n + i2) + f] = mono[i2];
        }
        for (int q = 0; q <= 32; ++q) {
            const double t = -1.0 + 2.0 * q / 32.0, r = mid + h * t;
            if (r <= 0) continue;
            double gx, cx;
            kernel_host(k, r, &gx, &cx);
            double ga = tab[2 * (pc * n + n - 1)], ca = tab[2 * (pc * n + n - 1) + 1];
            for (int j = n - 2; j >= 0; --j) {
                ga = std::fma(ga, t, tab[2 * (pc * n + j)]);
                ca = std::fma(ca, t, tab[2 * (pc * n + j) + 1]);
            }
            gmax = std::max(gmax, std::fabs(gx)); cmax = std::max(cmax, std::fabs(cx));
            gerr = std::max(gerr, std::fabs(ga - gx)); cerr = std::max(cerr, std::fabs(ca - cx));
        }
    }
    *w_out = w;
    // the formulas themselves carry ~1e-12 relative noise in coef where the
    // derivative switches from its series to the closed form (cancellation)
    return gerr <= 1e-13 * gmax && cerr <= 1e-11 * cmax;
}

static double r2_threshold(double radius) {
    // largest double t with sqrt(t) <= radius (IEEE sqrt on host == device)
    double t = radius * radius;
    while (std::sqrt(t) > radius) t = std::nextafter(t, -INFINITY);
    for (;;) {
        double u = std::nextafter(t, INFINITY);
        if (std::sqrt(u) <= radius) t = u; else break;
    }
    return t;
}

// kernel constants, cutoff tests, tables and buffers of one near-field
// evaluation over cell list `cl` (the boundary-pair buffer is bnd / bnd_cnt)
static NearArgs near_args(Plan* p, const CellList& cl, const double* d_eval, const int* d_order,
                          int64_t ne, const NearKernel& k, double* d_out4, int64_t* d_npairs,
                          int2*& bnd, int*& bnd_cnt, int64_t& bnd_cap, bool* close_ok_out) {
    bool close_ok = false;
    NearArgs a{};
    a.eval = d_eval; a.order = d_order; a.ne = ne;
    a.g = cell_geo(p, cl);
    a.start = cl.start; a.src = cl.src; a.srcf = cl.srcf;
    a.r2max = r2_threshold(k.radius);
    a.rr = k.radius * k.radius;
    a.win_lo = std::min(a.rr, a.r2max) * (1.0 - 1e-12);
    a.lzbox = 1e300;                 // pairs near the cutoff never wrap in z
    a.zmin = p->d_mm + 200;
    {
        const int64_t cap = std::max<int64_t>(4096, 8 * ne);
        if (cap > bnd_cap) {
            dfree(p, bnd); dfree(p, bnd_cnt);
            bnd = dalloc<int2>(p, cap);
            bnd_cnt = dalloc<int>(p, 1);
            bnd_cap = cap;
        }
        SE_CUDA(cudaMemsetAsync(bnd_cnt, 0, sizeof(int), p->stream));
        a.bnd = bnd; a.bnd_cnt = bnd_cnt;
        a.bnd_cap = (int)std::min<int64_t>(bnd_cap, INT32_MAX);
        a.flags = p->d_flags;
    }
    a.c1 = k.c1; a.c2 = k.c2; a.ic1 = 1.0 / k.c1; a.ic2 = 1.0 / k.c2;
    a.inv4pie = k.inv4pie;
    a.self_value = k.self_value; a.point0 = k.point0;
    a.kind = k.kind; a.need_field = k.need_field;
    double rr = k.radius * (1.0 + 1e-5) + 4e-7 * (p->P.Lx + p->P.Ly + p->P.H + std::fabs(cl.zlo));
    a.r2f = (float)(rr * rr);
    // close path needed below max(FAR_SPLIT c1, 0.01 c2) (+margin for fp32 error)
    double rcl = std::max(FAR_SPLIT * k.c1, 1e-2 * k.c2) * (1.0 + 1e-4) + 1e-6 * (p->P.Lx + p->P.Ly + p->P.H + std::fabs(cl.zlo));
    a.r2close = (float)(rcl * rcl);
    {
        // close-pair table, cached per kernel (rebuilt when the kernel changes)
        const double rhi = rcl * 1.001;
        CloseFit& cf = p->close_fit[k.kind ? 1 : 0];
        if (!cf.valid || cf.c1 != k.c1 || cf.c2 != k.c2 || cf.inv4pie != k.inv4pie ||
            cf.rhi != rhi) {
            std::vector<double> h;
            double w = 0;
            cf.ok = fit_close_table(k, rhi, h, &w);
            if (!cf.dev) cf.dev = dalloc<double>(p, CL_TAB);
            SE_CUDA(cudaMemcpy(cf.dev, h.data(), sizeof(double) * CL_TAB, cudaMemcpyHostToDevice));
            cf.c1 = k.c1; cf.c2 = k.c2; cf.inv4pie = k.inv4pie; cf.rhi = rhi; cf.w = w;
            cf.valid = true;
        }
        a.ctab = cf.dev; a.use_ctab = 0;          // enabled for the close launch only
        a.cl_w = cf.w; a.cl_iw = 1.0 / cf.w;
        close_ok = cf.ok;
    }
    {
        const double r_far = std::max(FAR_SPLIT * k.c1, 1e-2 * k.c2);
        const double xa = r_far / k.c2 * (1.0 - 1e-6), xb = k.radius / k.c2 * (1.0 + 1e-6);
        a.use_poly = fit_far_poly(xa, xb, &a.pmid, &a.pinvh, a.pc) ? 1 : 0;
        for (int j = 0; j <= FAR_DEG; ++j) a.pc4[j] = a.pc[j] * k.inv4pie;
        a.ic2sq = (1.0 / k.c2) * (1.0 / k.c2);
        a.far_t1 = (1.0 / k.c2) * a.pinvh;
        a.far_t0 = -a.pmid * a.pinvh;
        a.far_k = TWO_OVER_SQRTPI * (1.0 / k.c2) * k.inv4pie;
        double m32 = 0, ih32 = 0, c32[FAR_DEG32 + 1];
        a.use_poly32 = (k.fp32 && fit_far_poly(xa, xb, &m32, &ih32, c32, FAR_DEG32, 3e-7)) ? 1 : 0;
        a.pmid32 = (float)m32; a.pinvh32 = (float)ih32;
        for (int j = 0; j <= FAR_DEG32; ++j) a.pc32[j] = a.use_poly32 ? (float)c32[j] : 0.f;
    }
    {
        const double err = 2.0 * 4e-7 * (p->P.Lx + p->P.Ly + p->P.H + std::fabs(cl.zlo));
        const double rin = std::max(0.0, k.radius - err), rout = k.radius + err;
        a.r2in_f = std::nextafter((float)(rin * rin), 0.0f);
        a.r2out_f = std::nextafter((float)(rout * rout), INFINITY);
        a.hLxf = (float)(0.5 * p->P.Lx); a.hLyf = (float)(0.5 * p->P.Ly);
    }
    a.Lxf = (float)p->P.Lx; a.Lyf = (float)p->P.Ly;
    a.qLx = 0.25 * p->P.Lx; a.qLy = 0.25 * p->P.Ly;
    a.iLxf = (float)(1.0 / p->P.Lx); a.iLyf = (float)(1.0 / p->P.Ly);
    a.zmarg = (float)(1e-6 * (p->P.Lx + p->P.Ly + p->P.H + std::fabs(cl.zlo)));
    a.out = d_out4; a.out_stride = ne;
    a.npairs = d_npairs;
    a.orig = cl.orig;
    // the pair-set record belongs to the charges' evaluation (d_npairs set)
    a.phash = (d_npairs && p->pair_hash) ? p->d_phash : nullptr;
    const bool hash = a.phash != nullptr;
    if (close_ok_out) *close_ok_out = close_ok;
    return a;
}

void near_eval(Plan* p, const double* d_eval, const int* d_order, int64_t ne,
               const NearKernel& k, double* d_out4, int64_t* d_npairs, const CellList* clp,
               int part) {
    if (ne == 0) return;
    const bool do_scan = part != NEAR_LISTS, do_lists = part != NEAR_SCAN;
    NvtxRange nv("se.near_field");
    const CellList& cl = clp ? *clp : p->cl;
    bool close_ok = false;
    NearArgs a = near_args(p, cl, d_eval, d_order, ne, k, d_out4, d_npairs, p->d_bnd,
                           p->d_bnd_cnt, p->bnd_cap, &close_ok);
    const bool hash = a.phash != nullptr;
    if (cl.n == 0) {
        if (do_scan)
            SE_CUDA(cudaMemsetAsync(d_out4, 0, sizeof(double) * (k.need_field ? 4 : 1) * ne,
                                    p->stream));
        return;
    }
    // the few-point and fused paths run whole in the NEAR_SCAN half
    static const char* fenv = getenv("SE_NEAR_FUSED");
    const bool fused = fenv ? atoi(fenv) != 0 : ne <= NEAR_FUSED_MAX;
    if (!do_scan && (ne <= FEW_POINTS || fused)) return;
    if (ne <= FEW_POINTS) {
        near_few_kernel<<<(unsigned)ne, 256, 0, p->stream>>>(a);
        SE_LAUNCHED(p);
        near_boundary_kernel<<<4, 256, 0, p->stream>>>(a);
        SE_LAUNCHED(p);
        return;
    }
    // sort the evaluation points by cell and cut them into one-cell warp tasks
    const int ncell = cl.ncx * cl.ncy * cl.ncz;
    const int ncol = cl.ncx * cl.ncy;
    NearScratch& ns = p->ns;
    const int64_t tcap = ne / 32 + ncol + 1;
    if (ne > ns.pcap || ncell + 1 > ns.ccap || tcap > ns.tcap) {
        void* olds[] = {ns.keys, ns.keys2, ns.perm, ns.order, ns.pstart, ns.pend, ns.tcount,
                        ns.toff, ns.tasks, ns.cub};
        for (void* o : olds) dfree(p, o);
        ns.pcap = std::max<int64_t>(ne, ns.pcap);
        ns.ccap = std::max<int64_t>(ncell + 1, ns.ccap);
        ns.tcap = std::max<int64_t>(tcap, ns.tcap);
        ns.keys = dalloc<uint32_t>(p, ns.pcap);
        ns.keys2 = dalloc<uint32_t>(p, ns.pcap);
        ns.perm = dalloc<int>(p, ns.pcap);
        ns.order = dalloc<int>(p, ns.pcap);
        ns.pstart = dalloc<int>(p, ns.ccap + 1);
        ns.pend = dalloc<int>(p, ns.ccap);
        ns.tcount = dalloc<int>(p, ns.ccap + 1);
        ns.toff = dalloc<int>(p, ns.ccap + 1);
        ns.tasks = dalloc<int2>(p, ns.tcap);
        size_t b1 = 0, b2 = 0;
        SE_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, b1, (uint32_t*)nullptr, (uint32_t*)nullptr,
                                                (int*)nullptr, (int*)nullptr, (int)ns.pcap, 0, 32,
                                                p->stream));
        SE_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, b2, (int*)nullptr, (int*)nullptr,
                                              (int)ns.ccap + 1, p->stream));
        ns.cub_bytes = std::max(b1, b2);
        ns.cub = dalloc<char>(p, ns.cub_bytes);
    }
    CellGeo g = cell_geo(p, cl);
    size_t bytes = ns.cub_bytes;
    if (do_scan) {
        point_keys_kernel<<<(unsigned)((ne + 255) / 256), 256, 0, p->stream>>>(d_eval, ne, g,
                                                                                 ns.keys, ns.perm);
        SE_LAUNCHED(p);
        int end_bit = 1;
        while (end_bit < 32 && ((uint64_t)ncell >> end_bit) != 0) ++end_bit;
        SE_CUDA(cub::DeviceRadixSort::SortPairs(ns.cub, bytes, ns.keys, ns.keys2, ns.perm,
                                                ns.order, (int)ne, 0, end_bit, p->stream));
        point_starts_kernel<<<(unsigned)((ne + 1 + 255) / 256), 256, 0, p->stream>>>(
            ns.keys2, ne, ncell, ns.pstart);
        SE_LAUNCHED(p);
    }
    // Small problems (latency-bound: too few 32-point tasks to fill the GPU)
    // take the fused one-warp-per-point kernel, no pair lists and no host
    // sync; large ones the scan -> lists -> eval pipeline, which amortises
    // the chord-window set-up over the 32 points of a task.
    if (fused) {
        a.order = ns.order;
        const unsigned nblk = (unsigned)((ne * 32 + NB_THREADS - 1) / NB_THREADS);
        a.use_ctab = close_ok ? 1 : 0;
        if (d_npairs) { p->ktic(3); p->ktic(4); p->ktoc(4); p->ktic(5); }
        if (hash) {
            if (k.fp32) near_fused_kernel<true, 6, false, true><<<nblk, NB_THREADS, 0, p->stream>>>(a);
            else near_fused_kernel<false, 6, false, true><<<nblk, NB_THREADS, 0, p->stream>>>(a);
        } else if (k.fp32) near_fused_kernel<true, 6><<<nblk, NB_THREADS, 0, p->stream>>>(a);
        else near_fused_kernel<false, 6><<<nblk, NB_THREADS, 0, p->stream>>>(a);
        SE_LAUNCHED(p);
        near_boundary_kernel<<<4, 256, 0, p->stream>>>(a);
        if (d_npairs) { p->ktoc(5); p->ktoc(3); }
        SE_LAUNCHED(p);
        return;
    }
    const int nzb = cl.ncz;
    if (do_scan) {
        task_count_kernel<<<(ncol + 255) / 256, 256, 0, p->stream>>>(ns.pstart, ncol, nzb,
                                                                     ns.tcount);
        SE_LAUNCHED(p);
        SE_CUDA(cudaMemsetAsync(ns.tcount + ncol, 0, sizeof(int), p->stream));
        bytes = ns.cub_bytes;
        SE_CUDA(cub::DeviceScan::ExclusiveSum(ns.cub, bytes, ns.tcount, ns.toff, ncol + 1,
                                              p->stream));
        task_fill_kernel<<<(ncol + 255) / 256, 256, 0, p->stream>>>(ns.pstart, ns.toff, ncol,
                                                                    nzb, ns.tasks, ns.pend);
        SE_LAUNCHED(p);
    }
    a.order = ns.order;
    a.tasks = ns.tasks;
    a.pt_end = ns.pend;
    a.ntask_dev = ns.toff + ncol;
    a.ntask = tcap;
    const unsigned nblk = (unsigned)((tcap * 32 + NB_THREADS - 1) / NB_THREADS);
    // pair-list capacities from the expected neighbour count (+ margin);
    // an overflow doubles them and reruns the scan
    const double vol_cell = cl.csx * cl.csy * cl.csz;
    const double dens = (double)cl.n / ((double)ncell * vol_cell);
    const double ball = 4.0 / 3.0 * M_PI * std::pow(k.radius, 3.0);
    const double rclose = std::sqrt((double)a.r2close);
    const double ballc = 4.0 / 3.0 * M_PI * std::pow(std::min(rclose, k.radius), 3.0);
    NearLists& L = p->nl;
    int64_t want_far = (int64_t)(1.6 * dens * ball + 64), want_close = (int64_t)(2.0 * dens * ballc + 64);
    static const char* lsenv = getenv("SE_NEAR_LIST_SCALE");   // test hook: force overflows
    if (lsenv) {
        const double f = atof(lsenv);
        want_far = std::max<int64_t>(16, (int64_t)(want_far * f));
        want_close = std::max<int64_t>(16, (int64_t)(want_close * f));
    }
    want_far = (want_far + 15) & ~15LL;
    want_close = (want_close + 15) & ~15LL;
    // no host sync: points whose lists overflow are evaluated by the fused
    // kernel from a device list; the charges' overflow count accumulates in
    // a per-plan device counter that phase_results reads after its stream
    // sync and turns into a larger L.grow for the next solve
    want_far *= L.grow;
    want_close *= L.grow;
    if (ne * want_far > L.cap_far_total || ne * want_close > L.cap_close_total || ne > L.ncap) {
        void* olds[] = {L.far, L.close, L.cfar, L.cclose, L.ovf, L.ovl};
        for (void* o : olds) dfree(p, o);
        L.cap_far_total = std::max<int64_t>(ne * want_far, L.cap_far_total);
        L.cap_close_total = std::max<int64_t>(ne * want_close, L.cap_close_total);
        L.ncap = std::max<int64_t>(ne, L.ncap);
        L.far = dalloc<int>(p, L.cap_far_total);
        L.close = dalloc<int>(p, L.cap_close_total);
        L.cfar = dalloc<int>(p, L.ncap);
        L.cclose = dalloc<int>(p, L.ncap);
        L.ovf = dalloc<int>(p, 1);
        L.ovl = dalloc<int>(p, L.ncap);
    }
    a.list_far = L.far; a.list_close = L.close;
    a.cap_far = want_far; a.cap_close = want_close;
    a.cnt_far = L.cfar; a.cnt_close = L.cclose; a.overflow = L.ovf; a.ovl = L.ovl;
    if (do_scan) {
        SE_CUDA(cudaMemsetAsync(L.ovf, 0, sizeof(int), p->stream));
        if (d_npairs) { p->ktic(3); p->ktic(4); }
        // 16-deep queues, 4 candidates per step, 7 CTAs / SM (73 registers):
        // measured best of queue 8..24, step 4 / 8, 6..12 CTAs (3.17 vs 3.29 ms at 10)
        // (round 2, branch-free tests: queue 8 / 16 / 24, step 4 / 8, 6..8
        // CTAs all within 2.68-2.78 ms)
        if (cl.ncx < 2 * cl.hw + 1 || cl.ncy < 2 * cl.hw + 1)
            near_scan_kernel<16, 4, 7, true><<<nblk, NB_THREADS, 0, p->stream>>>(a);
        else
            near_scan_kernel<16, 4, 7, false><<<nblk, NB_THREADS, 0, p->stream>>>(a);
        if (d_npairs) p->ktoc(4);
        SE_LAUNCHED(p);
    }
    if (!do_lists) return;
    if (d_npairs) p->ktic(5);
    NearArgs ac = a;
    ac.use_ctab = close_ok ? 1 : 0;
    // the close launch: resident CTAs only (6 per SM), persistent over the tasks
    // (fp32 mode: 8 per SM, 3.10 -> 3.07 ms; fp64 8 / 10 per SM: 4.13 / 4.27
    // vs 4.12 ms)
    const unsigned nblk_c = std::min<unsigned>(nblk, (unsigned)((k.fp32 ? 8 : 6) * p->num_sms));
    if (hash) {
        if (k.fp32) near_eval_kernel<true, 10, true, true><<<nblk, NB_THREADS, 0, p->stream>>>(a);
        else near_eval_kernel<true, 8, false, true><<<nblk, NB_THREADS, 0, p->stream>>>(a);
        SE_LAUNCHED(p);
        if (k.fp32) near_eval_kernel<false, 8, true, true><<<nblk_c, NB_THREADS, 0, p->stream>>>(ac);
        else near_eval_kernel<false, 6, false, true><<<nblk_c, NB_THREADS, 0, p->stream>>>(ac);
        SE_LAUNCHED(p);
        if (k.fp32) near_fused_kernel<true, 6, true, true><<<148, NB_THREADS, 0, p->stream>>>(ac);
        else near_fused_kernel<false, 6, true, true><<<148, NB_THREADS, 0, p->stream>>>(ac);
    } else {
        // fp32 far pairs at 14 CTAs / SM (36 registers, small spills): 10 / 11 /
        // 12 / 14 / 16 measured 3.20 / 3.15 / 3.14 / 3.10 / 3.10 ms (round 1:
        // 10 vs 8, 3.33 vs 3.52 ms); fp64 at 8 CTAs / SM (64 registers): 7 / 9
        // / 10 measured 4.35 / 4.28 / 4.69 vs 4.27 ms
        if (k.fp32) near_eval_kernel<true, 14, true><<<nblk, NB_THREADS, 0, p->stream>>>(a);
        else near_eval_kernel<true, 8><<<nblk, NB_THREADS, 0, p->stream>>>(a);
        SE_LAUNCHED(p);
        if (k.fp32) near_eval_kernel<false, 8, true><<<nblk_c, NB_THREADS, 0, p->stream>>>(ac);
        else near_eval_kernel<false, 6><<<nblk_c, NB_THREADS, 0, p->stream>>>(ac);
        SE_LAUNCHED(p);
        if (k.fp32) near_fused_kernel<true, 6, true><<<148, NB_THREADS, 0, p->stream>>>(ac);
        else near_fused_kernel<false, 6, true><<<148, NB_THREADS, 0, p->stream>>>(ac);
    }
    SE_LAUNCHED(p);
    if (d_npairs) {                                  // the charges' evaluation
        add_count_kernel<<<1, 1, 0, p->stream>>>(L.ovf, p->d_ovf_acc);
        SE_LAUNCHED(p);
    }
    near_boundary_kernel<<<4, 256, 0, p->stream>>>(a);
    if (d_npairs) { p->ktoc(5); p->ktoc(3); }
    SE_LAUNCHED(p);
}

void finalize(Plan* p, int64_t first, int64_t count, uint32_t flags, double self_inf_value,
              double* d_phi, double* d_E) {
    const int nblk = 592;
    FinArgs a{};
    a.far = p->d_far; a.near = p->d_near; a.q = p->d_q; a.n = count;
    a.first = first; a.nfar = p->N;
    a.cell = p->hx * p->hy;
    a.forces = (flags & SE_NEED_FORCES) ? 1 : 0;
    a.potential = (flags & SE_NEED_POTENTIAL) && !(p->P.xi_is_inf != 0.0);
    a.self_inf = ((flags & SE_SUBTRACT_SELF) && p->P.xi_is_inf != 0.0) ? 1 : 0;
    a.self_inf_value = self_inf_value;
    a.scal = p->d_scal;
    a.phi = d_phi; a.E = d_E; a.partial = p->d_partial;
    finalize_kernel<<<nblk, 256, 0, p->stream>>>(a);
    SE_LAUNCHED(p);
    sum_partials_kernel<<<1, 256, 0, p->stream>>>(p->d_partial, nblk, 0.5, p->d_scal + 2);
    SE_LAUNCHED(p);
}

// wall-charge energy: 1/2 hx hy sum sigma (far + near + B_i) over the wall
// nodes of both walls                                       slab.py:448-461
__global__ void wall_points_kernel(int Nx, int Ny, double hx, double hy, double H,
                                   double* pts) {
    int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    int64_t nxy = (int64_t)Nx * Ny;
    if (e >= 2 * nxy) return;
    int64_t w = e / nxy, r = e % nxy;
    int ix = (int)(r / Ny), iy = (int)(r % Ny);
    pts[3 * e] = hx * ix;
    pts[3 * e + 1] = hy * iy;
    pts[3 * e + 2] = (w == 0) ? 0.0 : H;
}

__global__ void wall_energy_kernel(const double* far, const double* near,
                                   const double* sigb, const double* sigt,
                                   int64_t nxy, const double* scal, double* partial) {
    __shared__ double red[256];
    double acc = 0.0;
    const double b_i = scal[1];
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < 2 * nxy;
         e += (int64_t)gridDim.x * blockDim.x) {
        double sig = (e < nxy) ? sigb[e] : sigt[e - nxy];
        acc += sig * ((far[e] + near[e]) + b_i);
    }
    red[threadIdx.x] = acc;
    __syncthreads();
    for (int w = 128; w > 0; w >>= 1) {
        if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) partial[blockIdx.x] = red[0];
}

void wall_energy(Plan* p, const NearKernel& kpoint) {
    const int64_t nxy = p->NXY;
    if (!p->d_wall_pts) {
        p->d_wall_pts = dalloc<double>(p, 6 * (size_t)nxy);
        p->d_wall_far = dalloc<double>(p, 2 * (size_t)nxy);
        p->d_wall_near = dalloc<double>(p, 2 * (size_t)nxy);
    }
    wall_points_kernel<<<(unsigned)((2 * nxy + 255) / 256), 256, 0, p->stream>>>(
        p->Nx, p->Ny, p->hx, p->hy, p->P.H, p->d_wall_pts);
    SE_LAUNCHED(p);
    double w = 0.5 / p->P.xi;
    double rad = (p->P.H_E / p->P.g_t) * w;
    interp_points(p, p->d_wall_pts, 2 * nxy, w, rad, p->d_wall_far);
    near_eval(p, p->d_wall_pts, nullptr, 2 * nxy, kpoint, p->d_wall_near, nullptr);
    const int nblk = 256;
    wall_energy_kernel<<<nblk, 256, 0, p->stream>>>(p->d_wall_far, p->d_wall_near, p->d_sigb,
                                                    p->d_sigt, nxy, p->d_scal, p->d_partial);
    SE_LAUNCHED(p);
    sum_partials_kernel<<<1, 256, 0, p->stream>>>(p->d_partial, nblk, 0.5 * p->hx * p->hy,
                                                  p->d_scal + 3);
    SE_LAUNCHED(p);
}

}  // namespace se
