// Internal declarations of libslabewald_cuda.so (sm_100a).
//
// Data layout in HBM (z slowest, SURVEY.md section 7 "design decisions"):
//   rho    [Nz][2][Nx][Ny]        real spread grids, slot 0 = rho_over,
//                                 slot 1 = rho_in            (slab.py:282-289)
//   ext    [Nz][2][Nx][Ny/2+1]    complex: Chebyshev coefficients of the
//                                 xy half spectra (DCT-I along z, hand-written
//                                 FP64 tensor-core kernels, chebyshev.py:46-65)
//   spec4  [Nz][4][Nx][Ny/2+1]    psi, ikx psi, iky psi, dpsi/dz mode values
//   fields [Nz][4][Nx][Ny]        real field grids after the inverse xy FFT
// Sources for spreading are sorted by (xy bin, class, first z node) so one
// CTA finds every source touching its grid tile by binary search.
#pragma once

#include <cuda_runtime.h>
#include <cufft.h>
#include <nvtx3/nvToolsExt.h>

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/slabewald.h"

namespace se {

// NVTX range for the duration of a scope (stage names in nsys / ncu --nvtx)
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

// ----------------------------------------------------------------------------
// errors
// ----------------------------------------------------------------------------
struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define SE_CUDA(call)                                                        \
    do {                                                                     \
        cudaError_t e_ = (call);                                             \
        if (e_ != cudaSuccess && (cudaGetLastError(), true))                 \
            throw ::se::Error(e_ == cudaErrorMemoryAllocation ? SE_ERR_MEMORY \
                                                               : SE_ERR_CUDA, \
                              std::string(#call) + ": " +                    \
                                  cudaGetErrorString(e_));                   \
    } while (0)

#define SE_CUFFT(call)                                                       \
    do {                                                                     \
        cufftResult r_ = (call);                                             \
        if (r_ != CUFFT_SUCCESS)                                             \
            throw ::se::Error(SE_ERR_CUDA, std::string(#call) +              \
                                               ": cufft error " +            \
                                               std::to_string((int)r_));     \
    } while (0)

#define SE_LAUNCHED(plan)                                                    \
    do {                                                                     \
        (plan)->launches++;                                                  \
        cudaError_t e_ = cudaGetLastError();                                 \
        if (e_ != cudaSuccess)                                               \
            throw ::se::Error(SE_ERR_CUDA, std::string("launch: ") +         \
                                               cudaGetErrorString(e_));      \
    } while (0)

// device-side error flags (checked after the stream is synchronised)
enum : int {
    FLAG_Z_OUTSIDE = 1,      // gridops.py:87-88,119-120  ValueError
    FLAG_NONFINITE = 2,      // dpsolver.py:83-86        FloatingPointError
    FLAG_K0_FAIL = 4,        // dpsolver.py:208-211      FloatingPointError
    FLAG_K0_WARN = 8,        // dpsolver.py:212-213      warning
    FLAG_NEAR_BND = 16,      // boundary-pair buffer overflow (RuntimeError)
};

// ----------------------------------------------------------------------------
// spread / interpolation tiling
// ----------------------------------------------------------------------------
constexpr int TILE = 8;          // xy tile = 8 x 8 grid columns (one bin)
constexpr int INTERP_TZ = 16;    // z nodes per interp CTA (4 groups of 4)
constexpr int CHUNK = 64;        // sources staged in shared memory at a time
constexpr int MAX_M = 24;        // max xy stencil half width supported

// Per-source stencil tables, structure of arrays over the sorted sources.
struct Stencils {
    int64_t S = 0;               // number of sources (table stride)
    int mx = 0, my = 0;          // x / y half widths (gridops.py:20)
    int wz = 0;                  // z table width (max nodes per stencil)
    int* j0x = nullptr;          // floor(x / hx)
    int* j0y = nullptr;
    int* lo = nullptr;           // first z node
    int* hi = nullptr;           // one past the last z node
    double* q = nullptr;         // strength
    int rs = 0;                  // record stride (doubles)
    double* rec = nullptr;       // [S][rs]: wx[2mx+1] | wy[2my+1] | wz[wz]
    int* owner = nullptr;        // charge index of the source, -1 for images
};

// Sorted source set with segment offsets per (bin, class).
struct SourceSet {
    int64_t S = 0;
    int nbx = 0, nby = 0;        // bins along x, y
    int64_t* seg = nullptr;      // [nbx*nby*2 + 1] start offsets
    Stencils st;
};

// ----------------------------------------------------------------------------
// near field cell list
// ----------------------------------------------------------------------------
struct CellList {
    int ncx = 0, ncy = 0, ncz = 0, hw = 2;   // hw: neighbour columns each side
    double csx = 0, csy = 0, csz = 0, zlo = 0;
    int64_t n = 0;
    int* start = nullptr;        // [ncells + 1]
    double4* src = nullptr;      // sorted sources (x, y, z, q) original coords
    float4* srcf = nullptr;      // wrapped fp32 copy for the pre-test
    int* orig = nullptr;         // sorted -> original source index
    int64_t cap = 0, cell_cap = 0;   // allocated sources / cell starts
};

// which sources a cell list holds: the charges, their mirror layers, or both
enum : int { CL_CHARGES = 1, CL_IMAGES = 2, CL_ALL = 3 };

// ----------------------------------------------------------------------------
// the plan
// ----------------------------------------------------------------------------
struct Buf {
    void* p = nullptr;
    size_t bytes = 0;
};

// near-field pair lists (scan -> eval), point-major
struct NearLists {
    int64_t cap_far_total = 0, cap_close_total = 0, ncap = 0;
    int *far = nullptr, *close = nullptr, *cfar = nullptr, *cclose = nullptr, *ovf = nullptr;
    int* ovl = nullptr;        // slots whose lists overflowed (fallback list)
    int64_t grow = 1;          // capacity multiplier learned from overflows
};

// scratch of near_eval: evaluation points sorted by cell, one-cell warp tasks
// cached close-pair kernel table (se_near.cu)
struct CloseFit {
    bool valid = false, ok = false;
    double c1 = 0, c2 = 0, inv4pie = 0, rhi = 0, w = 0;
    double* dev = nullptr;
};

struct NearScratch {
    int64_t pcap = 0, ccap = 0, tcap = 0;
    uint32_t *keys = nullptr, *keys2 = nullptr;
    int *perm = nullptr, *order = nullptr, *pstart = nullptr, *pend = nullptr;
    int *tcount = nullptr, *toff = nullptr;
    int2* tasks = nullptr;
    void* cub = nullptr;
    size_t cub_bytes = 0;
};

// state of one solve between its phases (se_api.cu)
struct Solve {
    uint32_t flags = 0;
    // sharded solve with the near field routed by cell: the caller supplies
    // the near-field sums of this shard's charges (se_shard_near) and the
    // near part of the gauge (summed over ranks)
    bool near_external = false;
    const double* ext_near = nullptr;     // [4][count]
    const double* ext_near0 = nullptr;    // device scalar
    bool xi_inf = false, forces = false, potential = false, energy = false, corr = false,
         two = false, near_empty = true;
    int mode = 0;
    int64_t n_all = 0, first = 0, count = 0;
    cudaEvent_t ev[12] = {};
    int ne = 0;
    bool timed = false;
    int phase = 0;                // 0 idle, 1 spread done, 2 fields done
    // single-GPU solve: the charges' near field forked onto Plan::side after
    // the spread (0 off, 1 the whole near field, 2 its list scan only; 3 the
    // list scan stays on the solver's stream and the grid pipeline up to the
    // interpolation moves to the high-priority side stream)
    int near_fork = 0;
    bool near_forked = false;
};

// exp(-u) for |u| <= 700 without the special-case paths of libm exp:
// Cody-Waite reduction by ln2, a degree-10 polynomial on |r| <= ln2/2
// (Chebyshev interpolant in monomial form, 4.5e-16 relative including the
// Horner rounding), scaling by 2^n through the exponent bits.  n is rounded
// by the 1.5 x 2^52 shifter (its low word is n), so no FRND / F2I.F64, and
// the coefficients sit in constant memory, so each DFMA takes its operand
// from the constant bank (immediates cost two UMOVs per DFMA).
static __constant__ double kExpNegC[13] = {
    2.7626357241447223e-07, 2.764018079620985e-06, 2.4801504346997686e-05,
    1.9841170270440067e-04, 1.3888888932488599e-03, 8.333333385667782e-03,
    4.166666666657314e-02,  1.6666666666554406e-01, 5.000000000000006e-01,
    1.0000000000000067,     1.0,
    -6.93147180369123816490e-01, -1.90821492927058770002e-10};   // -ln2 hi, lo
__device__ __forceinline__ double exp_neg(double u) {
    const double v = -u;
    const double sh = fma(v, 1.4426950408889634, 6755399441055744.0);
    const double n = sh - 6755399441055744.0;
    double r = fma(n, kExpNegC[11], v);
    r = fma(n, kExpNegC[12], r);
    double p = kExpNegC[0];
#pragma unroll
    for (int j = 1; j < 11; ++j) p = fma(p, r, kExpNegC[j]);
    return p * __hiloint2double((1023 + __double2loint(sh)) << 20, 0);
}

// Gaussian stencil weight exp(-(d/w)^2 / 2) / norm with the reciprocals
// precomputed (within 2 ulp of the reference's exp(-0.5 (d/w)^2) / norm)
__device__ __forceinline__ double gauss_w(double d, double inv_width, double inv_norm) {
    const double u = d * inv_width;
    return exp_neg(0.5 * (u * u)) * inv_norm;
}

struct Plan {
    se_params P{};
    Solve solve;
    int dev = 0;
    int num_sms = 148;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    int64_t launches = 0;

    // grid
    int Nx = 0, Ny = 0, Nz = 0, Nyh = 0, N2 = 0;
    int64_t M = 0, NXY = 0, G = 0;
    double hx = 0, hy = 0;
    int mx = 0, my = 0;          // spread/interp stencil half widths
    int wz_max = 0;              // max z stencil width
    double rad = 0, rad_keep = 0, width = 0, norm = 0;   // spread kernel
    bool jumps = false, sigma_zero = true;

    // host copies of constants
    std::vector<double> z, wcc, tw0, twH, kx, ky;

    // device constants
    double *d_z = nullptr, *d_wcc = nullptr, *d_tw0 = nullptr, *d_twH = nullptr;
    double *d_kx = nullptr, *d_ky = nullptr;
    int* d_kidx = nullptr;                // mode -> unique |k| row (-1: k = 0)
    double* d_kmag = nullptr;             // |k| per half-spectrum mode
    unsigned char* d_sel = nullptr;       // correction mode mask (0 < k <= k_max)
    double* d_kuniq = nullptr;            // distinct |k| > 0
    double* d_maps = nullptr;             // integration maps + column sums [9][Nz]
    int win0 = 0, win1 = 0;               // correction node window [win0, win1)
    int n_uniq = 0;
    double* d_fac = nullptr;              // BVP factors [n_uniq][FAC_ROWS][Nz]
    double* d_sinv = nullptr;             // [n_uniq][4]
    double* d_kappa = nullptr;            // [n_uniq]
    cufftDoubleComplex *d_sbh = nullptr, *d_sth = nullptr;  // sigma hats
    double *d_sigb = nullptr, *d_sigt = nullptr;            // sigma samples
    double k0_scale = 0;
    double sigma_scale = 0;               // mean|sigma_b| + mean|sigma_t|

    // charges and per-solve buffers
    int64_t N = 0, q_cap = 0;
    double* d_q = nullptr;
    double* d_pos = nullptr;              // [N][3]
    double* d_phi = nullptr;              // [N]
    double* d_E = nullptr;                // [N][3]
    double* d_far = nullptr;              // [4][N] interp sums
    int64_t* d_iseg = nullptr;            // interp: sorted charges per 4x4 bin
    int2* d_igroups = nullptr;            // interp: (first sorted index, count)
    int* d_ingroups = nullptr;
    int* d_gcnt = nullptr;                // interp: groups per bin, offsets
    void* d_gscan = nullptr;              // interp: scan scratch
    size_t gscan_bytes = 0;
    int64_t iseg_cap = 0, igroup_cap = 0;
    const double* d_pos_cur = nullptr;    // positions of the solve in flight
    double* d_near = nullptr;             // [4][N] near sums
    double* d_scal = nullptr;             // device scalars (A_i, B_i, U, ...)
    int* d_flags = nullptr;
    double* d_k0 = nullptr;               // k=0 outputs [16]

    // sources
    double4* d_src = nullptr;             // unsorted spread sources
    int* d_src_cls = nullptr;             // class (0 over, 1 far/image)
    int* d_src_owner = nullptr;
    int64_t src_cap = 0;
    uint32_t* d_keys = nullptr;
    uint32_t* d_keys2 = nullptr;
    int* d_perm = nullptr;
    int* d_perm2 = nullptr;
    void* d_cub = nullptr;
    size_t cub_bytes = 0;
    SourceSet ss;

    // near field
    CellList cl;                          // charges + their mirror layers

    NearScratch ns;
    NearLists nl;
    CloseFit close_fit[2];
    int2* d_bnd = nullptr;                // near pairs within ulps of the cutoff
    int* d_bnd_cnt = nullptr;
    int64_t bnd_cap = 0;
    int64_t cl_cap = 0;
    uint32_t* d_ckeys = nullptr;
    uint32_t* d_ckeys2 = nullptr;
    int* d_cperm = nullptr;
    int* d_cperm2 = nullptr;
    int* d_tgt = nullptr;                 // charge targets in cell order
    uint32_t* d_tkeys = nullptr;
    uint32_t* d_tkeys2 = nullptr;
    int* d_tperm = nullptr;
    double4* d_near_src = nullptr;        // unsorted near-field sources
    void* d_near_cub = nullptr;
    size_t near_cub_bytes = 0;
    int64_t cell_cap = 0;
    double* d_mm = nullptr;               // z-range partials
    int64_t* d_count = nullptr;
    int* d_ovf_acc = nullptr;             // near-list overflows of the charges this solve
    // CUDA graph of a whole solve (SE_GRAPH): replayed while the device
    // buffers, size and flags repeat; invalidated when list capacities grow
    cudaGraphExec_t gexec = nullptr;
    cudaStream_t cap_stream = nullptr;
    cudaStream_t side = nullptr;          // near-field fork (Solve::near_fork), high priority
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    int fork_req = 0;                     // Solve::near_fork of the next solve_core solve
    cudaStream_t fork_main = nullptr;     // fork 3: the caller's stream while the grid
                                          // pipeline runs on `side`
    struct GraphKey {
        const void *pos = nullptr, *phi = nullptr, *E = nullptr;
        int64_t n = -1; uint32_t flags = 0;
        bool operator==(const GraphKey& o) const {
            return pos == o.pos && phi == o.phi && E == o.E && n == o.n && flags == o.flags;
        }
    } gkey, gwarm;
    bool pair_hash = false;               // SE_PAIR_HASH on the solve in flight
    bool last_overflow = false;           // the last solve's pair lists overflowed
    unsigned long long* d_phash = nullptr;   // [2][N] pair-set hash, count
    int64_t phash_cap = 0, phash_n = 0;
    double* d_partial = nullptr;          // reduction partials
    double* d_origin = nullptr;           // (0, 0, 0)
    double *d_wall_pts = nullptr, *d_wall_far = nullptr, *d_wall_near = nullptr;

    // grids
    double* d_rho = nullptr;              // [Nz][2][Nx][Ny]
    cufftDoubleComplex* d_ext = nullptr;  // [Nz][2][M] Chebyshev coefficients
    cufftDoubleComplex* d_hat = nullptr;  // [Nz][2][M] xy spectra / iDCT values
    double *d_dct_fwd = nullptr, *d_dct_inv = nullptr;   // [2][P8][P4] row-major
    int dct_p8 = 0, dct_p4 = 0;           // padded parity block (8-row tiles, k by 4)
    cufftDoubleComplex* d_spec = nullptr; // [Nz][4][M]
    double* d_fields = nullptr;           // [Nz][4][Nx][Ny]
    cufftDoubleComplex* d_scr = nullptr;  // BVP scratch [2][Nz][2][M] (y'', Thomas d / x)
    cufftDoubleComplex* d_bst = nullptr;  // split BVP column state [6][2][M]
    bool keep_stages = false;
    cufftDoubleComplex* d_keep = nullptr; // [Nz][2][M] psi coefficients (debug)
    cufftDoubleComplex* d_mom = nullptr;  // [M][2] correction moments / den
    cufftDoubleComplex* d_mism = nullptr; // [4][M] mismatch (debug)

    cufftHandle fft_fwd2 = 0, fft_fwd1 = 0, fft_z = 0, fft_inv4 = 0,
                fft_inv1 = 0, fft_sig = 0;

    // fp32 grid path (SE_FP32 on a single-GPU solve): spread grids, xy
    // spectra, spectral fields and field grids in single precision; the z
    // transforms, mode BVPs and correction stay fp64
    bool g32 = false;
    float* d_rho32 = nullptr;             // [Nz][2][Nx][Ny]
    cufftComplex* d_hat32 = nullptr;      // [Nz][2][M]
    cufftComplex* d_spec32 = nullptr;     // [Nz][4][M]
    float* d_fields32 = nullptr;          // [Nz][4][Nx][Ny]
    cufftHandle fft_fwd2_f = 0, fft_inv4_f = 0, fft_inv1_f = 0;

    // distributed grid pipeline (se_dist_*): rank `rank` of `nranks` owns the
    // z planes [rank zc, (rank+1) zc) for the xy FFTs and the half-spectrum
    // modes [rank mc, (rank+1) mc) for the z transforms and mode BVPs
    bool dist = false;
    int rank = 0, nranks = 1;
    int64_t zc = 0, mc = 0, Nz_pad = 0;
    double* d_rho_slab = nullptr;         // [zc][2][Nx][Ny]
    double* d_fields_slab = nullptr;      // [zc][4][Nx][Ny]
    cufftDoubleComplex* d_a2a_send = nullptr;   // [P][zc][4][mc]
    cufftDoubleComplex* d_a2a_recv = nullptr;
    double* d_dsc = nullptr;              // k = 0 / flag scalars summed over ranks
    cufftHandle fft_fwd_slab = 0, fft_inv4_slab = 0, fft_inv1_slab = 0;
    void* fft_work = nullptr;

    std::vector<Buf> owned;

    // per-kernel event timers (SE_TIMINGS): 0 spread, 1 bvp, 2 interp, 3 near,
    // 4 near scan, 5 near eval
    bool timing = false;
    cudaEvent_t kev[6][2] = {};
    void ktic(int k) { if (timing) cudaEventRecord(kev[k][0], stream); }
    void ktoc(int k) { if (timing) cudaEventRecord(kev[k][1], stream); }
};

// factor table rows per unique |k| (see se_spectral.cu)
constexpr int FAC_CP = 0, FAC_INV = 1, FAC_AINVB = 2, FAC_C0 = 3, FAC_C1 = 4;
constexpr int FAC_ROWS = 5;

void dfree(Plan* p, void* ptr);

// allocation helper (tracked, freed by the plan)
template <class T>
T* dalloc(Plan* p, size_t count) {
    void* ptr = nullptr;
    size_t bytes = count * sizeof(T);
    if (bytes == 0) bytes = 16;
    SE_CUDA(cudaMalloc(&ptr, bytes));
    p->owned.push_back({ptr, bytes});
    return static_cast<T*>(ptr);
}

// --- se_grid.cu ---
void build_sources(Plan* p, const double* d_pos, int64_t first, int64_t n, bool two_grids);
void partition_sources(Plan* p, const double* d_pos, int64_t n);
void spread(Plan* p, bool two_grids);
void interp_charges(Plan* p, int64_t n, int64_t first, int64_t count, bool forces);
void interp_points(Plan* p, const double* d_pts, int64_t npts, double width,
                   double radius, double* d_out);
void ensure_sources(Plan* p, int64_t cap);

// --- se_spectral.cu ---
// a contiguous range of (kx, ky) half-spectrum modes held with column stride M
struct ModeView {
    int64_t M;     // stride (columns per row)
    int64_t Mv;    // valid modes
    int64_t m0;    // global index of the first
};
void factor_bvp(Plan* p);
void z_forward(Plan* p, const ModeView& v);
void bvp_solve_view(Plan* p, bool two_grids, int mode, bool correction, const ModeView& v);
void z_inverse_assemble(Plan* p, bool forces, bool correction, const ModeView& v);
void forward_transforms(Plan* p, bool two_grids);
void ensure_grid32(Plan* p);
void ensure_grid64(Plan* p);
void bvp_solve(Plan* p, bool two_grids, int mode, bool correction);
void inverse_transforms(Plan* p, bool forces, bool correction);

// --- se_near.cu ---
struct NearKernel {
    double c1, c2, inv4pie, radius, self_value, point0;
    int kind;            // 0 avg, 1 point
    int need_field;
    int fp32;            // far pairs in single precision (SE_FP32)
};
void build_cells(Plan* p, const double* d_pos, const double* d_q, int64_t n, bool in_domain,
                 const double* d_zsrc_min = nullptr, CellList* cl = nullptr,
                 int parts = CL_ALL);
// part: NEAR_ALL, or the two halves of a split evaluation -- NEAR_SCAN (point
// sort, tasks, pair-list scan) and NEAR_LISTS (list evaluation, overflow
// fallback, boundary pairs), launched later with the same arguments
constexpr int NEAR_ALL = 0, NEAR_SCAN = 1, NEAR_LISTS = 2;
void near_eval(Plan* p, const double* d_eval, const int* d_eval_order,
               int64_t ne, const NearKernel& k, double* d_out4,
               int64_t* d_npairs, const CellList* cl = nullptr, int part = NEAR_ALL);

void finalize(Plan* p, int64_t first, int64_t count, uint32_t flags, double self_inf_value,
              double* d_phi, double* d_E);
void wall_energy(Plan* p, const NearKernel& kpoint);

// --- se_bd.cu ---
// persistent device scratch of the cell-list pair kernels (grown on demand)
struct PairScratch {
    int64_t ncap = 0, ccap = 0, bcap = 0;
    size_t tbytes = 0;
    uint32_t *k1 = nullptr, *k2 = nullptr;
    int *p1 = nullptr, *p2 = nullptr, *start = nullptr;
    double4* spos = nullptr;          // cell-sorted (x, y, z, q)
    void* tmp = nullptr;
    double* buf = nullptr;            // host-API staging: pos[3n] + out[3n]
    cudaStream_t stream = nullptr;    // host-API stream
    void reserve(int64_t n, int64_t ncell);
    void release();
    ~PairScratch() { release(); }
};
void steric_forces(int device, const double* pos, int64_t n, double Lx, double Ly, double Lz,
                   double a, double U0, double r_m, int p, double* out);
void steric_forces_device(int device, cudaStream_t st, const double* d_pos, int64_t n, double Lx,
                          double Ly, double Lz, double zlo, double zhi, double a, double U0,
                          double r_m, int p, double* d_out);
void bd_first_noise_device(int device, cudaStream_t st, int64_t n, uint64_t seed, double* d_prev);
void bd_step_device(int device, cudaStream_t st, double* d_pos, double* d_prev, const double* d_E,
                    const double* d_q, const double* d_fext, int64_t n, const se_bd_params& k,
                    uint64_t* draws, int64_t* rejections);
void tp_near_forces(const double* d_pos, const double* d_q, int64_t n, const double L[3],
                    double r_cut, double g_w, double xi, double eps, double* d_out,
                    cudaStream_t st, PairScratch& sc);

// --- se_tp.cu ---
struct TpPlan;
TpPlan* tp_create(int device, const double L[3], const int n[3], double eps);
void tp_destroy(TpPlan* p);
void tp_set_stream(TpPlan* p, cudaStream_t s);
void tp_set_graph(TpPlan* p, bool enable);
void tp_poisson(TpPlan* p, const double* rho, int with_field, double* phi, double* E);
void tp_forces(TpPlan* p, const double* pos, const double* q, int64_t n, double g_t,
               double radius, double g_w, double xi, double r_cut, double* forces);
void tp_forces_device(TpPlan* p, const double* d_pos, const double* d_q, int64_t n, double g_t,
                      double radius, double g_w, double xi, double r_cut, double* d_forces);

}  // namespace se
