// C-ABI of libslabewald_cuda.so: plan lifetime and the solve orchestration.
//
// Reference: SlabSolver.__init__ (slab.py:197-233) and SlabSolver.solve
// (slab.py:259-394); near_field_sum (slab.py:184-191); build_partition
// (slab.py:51-82).  See include/slabewald.h for the contract.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include "se_internal.cuh"

namespace se {

static thread_local std::string g_error;

void dfree(Plan* p, void* ptr) {
    if (!ptr) return;
    for (auto& b : p->owned)
        if (b.p == ptr) {
            cudaFree(ptr);
            b.p = nullptr;
            return;
        }
}

namespace {

__global__ void scale_complex(cufftDoubleComplex* a, int64_t n, double s) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) { a[i].x *= s; a[i].y *= s; }
}

// FP64 FMA throughput probe: 8 independent DFMA chains per thread
__global__ void dfma_probe_kernel(double* out, int iters, double a, double b) {
    double x0 = threadIdx.x * 1e-9, x1 = x0 + 1e-3, x2 = x0 + 2e-3, x3 = x0 + 3e-3;
    double x4 = x0 + 4e-3, x5 = x0 + 5e-3, x6 = x0 + 6e-3, x7 = x0 + 7e-3;
    for (int i = 0; i < iters; ++i) {
        x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
        x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
    double s = ((x0 + x1) + (x2 + x3)) + ((x4 + x5) + (x6 + x7));
    if (s == 12345.678) out[0] = s;       // keep the chains alive
}

__global__ void gauge_kernel(double* scal) {
    // B_i = -(far0 + near0)                                  slab.py:380-383
    scal[1] = -(scal[4] + scal[5]);
}

int fail(const Error& e) {
    g_error = e.what();
    return e.code;
}

void make_plan2d(cufftHandle* h, int nx, int ny, int nyh, cufftType type,
                 int64_t idist, int64_t odist, int batch, cudaStream_t s) {
    int real_embed[2] = {nx, ny};
    int cplx_embed[2] = {nx, nyh};
    const bool r2c = type == CUFFT_D2Z || type == CUFFT_R2C;
    int* in_e = r2c ? real_embed : cplx_embed;
    int* out_e = r2c ? cplx_embed : real_embed;
    SE_CUFFT(cufftCreate(h));
    size_t ws = 0;
    long long nn[2] = {nx, ny}, ie[2] = {in_e[0], in_e[1]}, oe[2] = {out_e[0], out_e[1]};
    SE_CUFFT(cufftMakePlanMany64(*h, 2, nn, ie, 1, idist, oe, 1, odist, type, batch, &ws));
    SE_CUFFT(cufftSetStream(*h, s));
}

}  // namespace

// buffers and cuFFT plans of the fp64 grid path, created on first use (a
// plan that only runs fp32 solves never holds them: C5 needs ~37 GB less)
void ensure_grid64(Plan* p) {
    const size_t nz = (size_t)p->Nz;
    if (!p->d_rho) {
        p->d_rho = dalloc<double>(p, 2 * (size_t)p->G);
        SE_CUDA(cudaMemsetAsync(p->d_rho, 0, 2 * (size_t)p->G * sizeof(double), p->stream));
    }
    if (!p->d_hat) p->d_hat = dalloc<cufftDoubleComplex>(p, nz * 2 * p->M);
    if (!p->d_spec) p->d_spec = dalloc<cufftDoubleComplex>(p, nz * 4 * p->M);
    if (!p->d_fields) p->d_fields = dalloc<double>(p, 4 * (size_t)p->G);
    if (!p->fft_fwd2)
        make_plan2d(&p->fft_fwd2, p->Nx, p->Ny, p->Nyh, CUFFT_D2Z, p->NXY, p->M, 2 * (int)nz,
                    p->stream);
    if (!p->fft_inv4)
        make_plan2d(&p->fft_inv4, p->Nx, p->Ny, p->Nyh, CUFFT_Z2D, p->M, p->NXY, 4 * (int)nz,
                    p->stream);
    if (!p->fft_inv1)
        make_plan2d(&p->fft_inv1, p->Nx, p->Ny, p->Nyh, CUFFT_Z2D, 4 * p->M, 4 * p->NXY,
                    (int)nz, p->stream);
}

// buffers and cuFFT plans of the fp32 grid path, created on first use
void ensure_grid32(Plan* p) {
    if (p->d_rho32) return;
    const size_t nz = (size_t)p->Nz;
    p->d_rho32 = dalloc<float>(p, 2 * (size_t)p->G);
    p->d_hat32 = dalloc<cufftComplex>(p, nz * 2 * p->M);
    p->d_spec32 = dalloc<cufftComplex>(p, nz * 4 * p->M);
    p->d_fields32 = dalloc<float>(p, 4 * (size_t)p->G);
    make_plan2d(&p->fft_fwd2_f, p->Nx, p->Ny, p->Nyh, CUFFT_R2C, p->NXY, p->M, 2 * (int)nz,
                p->stream);
    make_plan2d(&p->fft_inv4_f, p->Nx, p->Ny, p->Nyh, CUFFT_C2R, p->M, p->NXY, 4 * (int)nz,
                p->stream);
    make_plan2d(&p->fft_inv1_f, p->Nx, p->Ny, p->Nyh, CUFFT_C2R, 4 * p->M, 4 * p->NXY, (int)nz,
                p->stream);
}

namespace {

// ---------------------------------------------------------------------------
// the solve in three phases; the single-GPU solve runs them back to back and a
// sharded solve (charges split by index across ranks) runs them with a sum of
// the spread grids over ranks between phase 1 and phase 2.
// ---------------------------------------------------------------------------
// the solver's stream, cuFFT plans included
static void bind_stream(Plan* p, cudaStream_t st) {
    p->stream = st;
    cufftHandle hs[] = {p->fft_fwd2, p->fft_z, p->fft_inv4, p->fft_inv1, p->fft_sig,
                        p->fft_fwd_slab, p->fft_inv4_slab, p->fft_inv1_slab,
                        p->fft_fwd2_f, p->fft_inv4_f, p->fft_inv1_f};
    for (auto h : hs) if (h) SE_CUFFT(cufftSetStream(h, st));
}

static void mark(Plan* p, Solve& S) {
    if (S.timed) SE_CUDA(cudaEventRecord(S.ev[S.ne++], p->stream));
}

static Solve& current(Plan* p) { return p->solve; }

static void fork_near(Plan* p);

// SE_NEAR_FORK_AT: 1 (default) forks the near field before the spread, 0
// after it (C4 16.69 vs 16.83 ms fp64, 14.36 vs 14.38 ms fp32)
static bool fork_at_spread() {
    static const char* e = getenv("SE_NEAR_FORK_AT");
    return e ? atoi(e) == 1 : true;
}

void phase_spread(Plan* p, const double* d_pos, int64_t n_all, int64_t first, int64_t count,
                  uint32_t flags) {
    NvtxRange nv("se.spread_phase");
    p->launches = 0;
    if (n_all != p->N)
        throw Error(SE_ERR_VALUE, "positions and charges disagree on N");
    if (first < 0 || count < 0 || first + count > n_all)
        throw Error(SE_ERR_VALUE, "shard range outside the charge set");
    const se_params& P = p->P;
    Solve& S = current(p);
    S.phase = 0;
    S.flags = flags;
    S.near_external = false;
    S.near_fork = p->fork_req; S.near_forked = false;
    p->fork_req = 0;
    S.n_all = n_all; S.first = first; S.count = count;
    S.xi_inf = P.xi_is_inf != 0.0;
    S.forces = flags & SE_NEED_FORCES;
    S.potential = flags & SE_NEED_POTENTIAL;
    S.energy = flags & SE_NEED_ENERGY;
    S.corr = flags & SE_CORRECTION;
    const bool jumps = P.eps_b != P.eps || P.eps_t != P.eps || (flags & SE_FORCE_GENERAL);
    S.two = S.corr && jumps;
    S.mode = S.two ? 0 : (S.corr ? 1 : 2);
    S.near_empty = (n_all == 0) || S.xi_inf;
    if (!S.near_empty && P.r_cut >= 0.5 * std::min(P.Lx, P.Ly))
        throw Error(SE_ERR_VALUE, "near-field cutoff exceeds half the periodic box");
    cudaStream_t s = p->stream;
    SE_CUDA(cudaMemsetAsync(p->d_flags, 0, sizeof(int), s));
    SE_CUDA(cudaMemsetAsync(p->d_scal, 0, 8 * sizeof(double), s));
    SE_CUDA(cudaMemsetAsync(p->d_count, 0, sizeof(int64_t), s));
    SE_CUDA(cudaMemsetAsync(p->d_ovf_acc, 0, sizeof(int), s));
    S.timed = flags & SE_TIMINGS;
    S.ne = 0;
    if (S.timed) for (auto& e : S.ev) SE_CUDA(cudaEventCreate(&e));
    p->timing = S.timed;
    if (S.timed && !p->kev[0][0])
        for (auto& pr : p->kev) { SE_CUDA(cudaEventCreate(&pr[0])); SE_CUDA(cudaEventCreate(&pr[1])); }
    mark(p, S);
    p->d_pos_cur = d_pos;
    if (fork_at_spread()) fork_near(p);
    build_sources(p, d_pos, first, count, S.two);
    mark(p, S);
    spread(p, S.two);
    mark(p, S);
    S.phase = 1;
}

static void fork_near(Plan* p);

void phase_fields(Plan* p) {
    NvtxRange nv("se.field_phase");
    Solve& S = current(p);
    if (S.phase != 1) throw Error(SE_ERR_CUDA, "se_shard_fields before se_shard_spread");
    if (!S.near_forked) fork_near(p);
    forward_transforms(p, S.two);
    mark(p, S);
    bvp_solve(p, S.two, S.mode, S.corr);
    mark(p, S);
    inverse_transforms(p, S.forces, S.corr);
    mark(p, S);
    S.phase = 2;
}

static NearKernel kernel_of(const se_params& P, int kind, bool field, bool sub_unsplit) {
    const double eps = P.eps, inv4pie = 1.0 / (4.0 * M_PI * eps);
    const double two_sqrtpi = 2.0 / std::sqrt(M_PI);
    NearKernel k{};
    k.inv4pie = inv4pie;
    k.kind = kind;
    k.need_field = field ? 1 : 0;
    if (kind == 0) {                                        // kernels.py:90-125
        k.c1 = 2.0 * P.g_w;
        k.c2 = std::sqrt(4.0 * P.g_w * P.g_w + 1.0 / (P.xi * P.xi));
        k.radius = P.r_cut;
        k.self_value = sub_unsplit ? -two_sqrtpi / k.c2 / (4.0 * M_PI * eps)
                                   : two_sqrtpi * (0.5 / P.g_w - 1.0 / k.c2) / (4.0 * M_PI * eps);
    } else {                                                // kernels.py:83-87
        k.c1 = std::sqrt(2.0) * P.g_w;
        k.c2 = std::sqrt(2.0 * P.g_w * P.g_w + 1.0 / (P.xi * P.xi));
        k.radius = P.r_nf;
        k.point0 = (two_sqrtpi / k.c1 - two_sqrtpi / k.c2) / (4.0 * M_PI * eps);
    }
    return k;
}

// the charges' near-field kernel of the solve in flight
static NearKernel charge_kernel(const Plan* p, const Solve& S) {
    NearKernel k = kernel_of(p->P, 0, S.forces, S.flags & SE_SUBTRACT_SELF);
    k.fp32 = (S.flags & SE_FP32) ? 1 : 0;
    return k;
}

// the pair-set record (SE_PAIR_HASH) of this solve's charges, zeroed
static void prep_pair_hash(Plan* p, const Solve& S) {
    const int64_t count = S.count;
    p->pair_hash = (S.flags & SE_PAIR_HASH) != 0;
    if (!p->pair_hash) return;
    if (p->phash_cap < count) {
        dfree(p, p->d_phash);
        p->d_phash = dalloc<unsigned long long>(p, 2 * (size_t)std::max<int64_t>(count, 1));
        p->phash_cap = count;
    }
    SE_CUDA(cudaMemsetAsync(p->d_phash, 0, 16 * (size_t)std::max<int64_t>(count, 1), p->stream));
    p->phash_n = count;
}

// Solve::near_fork: the charges' near field depends only on the positions
// and charges, so it can run on a side stream while the grid pipeline
// (spread, transforms, mode BVPs, interpolation) runs on the solver's
// stream; the solver's stream joins it after the interpolation (fork 1: the whole near
// field; fork 2: the cell list and pair-list scan, the list evaluation then
// runs on the solver's stream after the join).  Captured into the solve's
// CUDA graph like the rest (the side stream joins the capture).
static void fork_near(Plan* p) {
    Solve& S = current(p);
    S.near_forked = false;
    if (!S.near_fork || S.near_external || S.near_empty || S.xi_inf || S.count <= 0) return;
    if (!p->side) {
        int lo = 0, hi = 0;
        SE_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
        SE_CUDA(cudaStreamCreateWithPriority(&p->side, cudaStreamNonBlocking, hi));
        SE_CUDA(cudaEventCreateWithFlags(&p->ev_fork, cudaEventDisableTiming));
        SE_CUDA(cudaEventCreateWithFlags(&p->ev_join, cudaEventDisableTiming));
    }
    SE_CUDA(cudaEventRecord(p->ev_fork, p->stream));
    SE_CUDA(cudaStreamWaitEvent(p->side, p->ev_fork, 0));
    if (S.near_fork == 3) {
        // the scan on the caller's stream, the grid pipeline on the side one
        prep_pair_hash(p, S);
        build_cells(p, p->d_pos_cur, p->d_q, S.n_all, true);
        near_eval(p, p->d_pos_cur + 3 * S.first, nullptr, S.count, charge_kernel(p, S),
                  p->d_near, p->d_count, nullptr, NEAR_SCAN);
        p->fork_main = p->stream;
        bind_stream(p, p->side);
        S.near_forked = true;
        return;
    }
    const cudaStream_t main = p->stream;
    p->stream = p->side;
    try {
        prep_pair_hash(p, S);
        const NearKernel kavg = charge_kernel(p, S);
        build_cells(p, p->d_pos_cur, p->d_q, S.n_all, true);
        near_eval(p, p->d_pos_cur + 3 * S.first, nullptr, S.count, kavg, p->d_near, p->d_count,
                  nullptr, S.near_fork == 1 ? NEAR_ALL : NEAR_SCAN);
        SE_CUDA(cudaEventRecord(p->ev_join, p->side));
    } catch (...) {
        p->stream = main;
        throw;
    }
    p->stream = main;
    S.near_forked = true;
}

void phase_charges(Plan* p, const double* d_pos, double* d_phi_out, double* d_E_out) {
    NvtxRange nv("se.charge_phase");
    Solve& S = current(p);
    if (S.phase != 2) throw Error(SE_ERR_CUDA, "se_shard_charges before se_shard_fields");
    if (d_pos != p->d_pos_cur) throw Error(SE_ERR_VALUE, "positions changed between phases");
    S.phase = 0;
    const se_params& P = p->P;
    cudaStream_t s = p->stream;
    const int64_t n = S.n_all, first = S.first, count = S.count;
    interp_charges(p, n, first, count, S.forces);
    mark(p, S);
    NearKernel kavg{}, kpt{};
    if (!S.xi_inf) {
        kavg = charge_kernel(p, S);
        kpt = kernel_of(P, 1, false, false);
    }
    if (S.near_forked && S.near_fork == 3) {
        SE_CUDA(cudaEventRecord(p->ev_join, p->stream));
        bind_stream(p, p->fork_main);
        p->fork_main = nullptr;
        s = p->stream;
    }
    if (S.near_forked) {
        SE_CUDA(cudaStreamWaitEvent(s, p->ev_join, 0));
        if (S.near_fork >= 2)
            near_eval(p, d_pos + 3 * first, nullptr, count, kavg, p->d_near, p->d_count, nullptr,
                      NEAR_LISTS);
    } else if (S.near_external) {
        prep_pair_hash(p, S);
        // routed by cell: the caller's sums for this shard (se_shard_near)
        if (count > 0)
            SE_CUDA(cudaMemcpyAsync(p->d_near, S.ext_near, sizeof(double) * 4 * (size_t)count,
                                    cudaMemcpyDeviceToDevice, s));
    } else if (!S.near_empty) {
        prep_pair_hash(p, S);
        build_cells(p, d_pos, p->d_q, n, true);           // sources: every charge
        near_eval(p, d_pos + 3 * first, nullptr, count, kavg, p->d_near, p->d_count);
    } else {
        prep_pair_hash(p, S);
        SE_CUDA(cudaMemsetAsync(p->d_near, 0, sizeof(double) * 4 * (size_t)std::max<int64_t>(count, 1), s));
    }
    mark(p, S);
    // gauge: pointwise potential vanishes at the origin      slab.py:377-384
    if (S.potential && !S.xi_inf) {
        const double w = 0.5 / P.xi;
        const double rad = (P.H_E / P.g_t) * w;
        interp_points(p, p->d_origin, 1, w, rad, p->d_scal + 4);
        if (S.near_external) {
            if (S.ext_near0)
                SE_CUDA(cudaMemcpyAsync(p->d_scal + 5, S.ext_near0, sizeof(double),
                                        cudaMemcpyDeviceToDevice, s));
            else
                SE_CUDA(cudaMemsetAsync(p->d_scal + 5, 0, sizeof(double), s));
        }
        else if (!S.near_empty)
            near_eval(p, p->d_origin, nullptr, 1, kpt, p->d_scal + 5, nullptr);
        gauge_kernel<<<1, 1, 0, s>>>(p->d_scal);
        SE_LAUNCHED(p);
    }
    const double two_sqrtpi = 2.0 / std::sqrt(M_PI);
    double self_inf = 0.0;
    if (S.xi_inf) self_inf = -two_sqrtpi / (2.0 * P.g_w) / (4.0 * M_PI * P.eps);
    if (count > 0) finalize(p, first, count, S.flags, self_inf, d_phi_out, d_E_out);
    // the wall-charge energy is global: the shard holding charge 0 adds it
    if (S.energy && !p->sigma_zero && first == 0) {
        if (S.near_external)
            throw Error(SE_ERR_VALUE, "the cell-routed near field needs a zero surface charge");
        if (S.xi_inf) throw Error(SE_ERR_VALUE, "wall-charge energy needs a finite xi");
        if (S.near_empty) p->cl.n = 0;
        wall_energy(p, kpt);
    }
    mark(p, S);
}

void phase_results(Plan* p, double* U, se_diag* diag) {
    NvtxRange nv("se.results");
    Solve& S = current(p);
    cudaStream_t s = p->stream;
    double scal[8], k0[16];
    int hflags = 0;
    int64_t npairs = 0;
    SE_CUDA(cudaMemcpyAsync(scal, p->d_scal, sizeof(scal), cudaMemcpyDeviceToHost, s));
    SE_CUDA(cudaMemcpyAsync(k0, p->d_k0, sizeof(k0), cudaMemcpyDeviceToHost, s));
    SE_CUDA(cudaMemcpyAsync(&hflags, p->d_flags, sizeof(int), cudaMemcpyDeviceToHost, s));
    SE_CUDA(cudaMemcpyAsync(&npairs, p->d_count, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    int ovf = 0;
    SE_CUDA(cudaMemcpyAsync(&ovf, p->d_ovf_acc, sizeof(int), cudaMemcpyDeviceToHost, s));
    SE_CUDA(cudaStreamSynchronize(s));
    p->last_overflow = ovf > 0;
    if (ovf > 0) {                  // lists overflowed: larger capacities next solve
        p->nl.grow *= 2;
        // the graph is stale and the next solve allocates: it runs eagerly
        // and a later one is captured
        if (p->gexec) { cudaGraphExecDestroy(p->gexec); p->gexec = nullptr; p->gkey = {}; }
        p->gwarm = {};
    }
    p->timing = false;
    if (hflags & FLAG_Z_OUTSIDE) throw Error(SE_ERR_VALUE, "point outside the extended z domain");
    if (hflags & FLAG_NONFINITE) throw Error(SE_ERR_FLOAT, "non-finite mismatch field");
    if (hflags & FLAG_NEAR_BND)
        throw Error(SE_ERR_CUDA, "too many near-field pairs at the exact cutoff distance");
    if (hflags & FLAG_K0_FAIL) {
        char buf[160];
        snprintf(buf, sizeof buf,
                 "k=0 coefficient mismatch %.2e: system not electroneutral or under-resolved",
                 k0[2]);
        throw Error(SE_ERR_FLOAT, buf);
    }
    const bool wall = !p->sigma_zero && S.first == 0;
    if (U) *U = S.energy ? (S.count > 0 ? scal[2] : 0.0) + (wall ? scal[3] : 0.0) : 0.0;
    if (diag) {
        diag->ai1 = k0[0]; diag->ai2 = k0[1]; diag->discrepancy = k0[2];
        diag->A_i = k0[3]; diag->A_b = k0[4]; diag->A_t = k0[5];
        diag->psi_i_bottom = k0[6]; diag->psi_i_top = k0[7];
        diag->psi_b_bottom = k0[8]; diag->psi_t_top = k0[9];
        diag->B_i = (S.potential && !S.xi_inf) ? scal[1] : 0.0;
        diag->U_wall = wall ? scal[3] : 0.0;
        diag->warn_discrepancy = (hflags & FLAG_K0_WARN) ? 1 : 0;
        diag->n_sources = (int32_t)p->ss.S;
        diag->n_pairs = npairs;
        diag->n_launches = p->launches;
        for (int i = 0; i < 16; ++i) diag->t_ms[i] = 0.0;
        if (S.timed) {
            for (int i = 0; i + 1 < S.ne && i < 8; ++i) {
                float ms = 0;
                SE_CUDA(cudaEventElapsedTime(&ms, S.ev[i], S.ev[i + 1]));
                diag->t_ms[i] = ms;
            }
            for (int k = 0; k < 6; ++k) {
                float ms = 0;
                if (cudaEventElapsedTime(&ms, p->kev[k][0], p->kev[k][1]) == cudaSuccess)
                    diag->t_ms[8 + k] = ms;
                else
                    cudaGetLastError();
            }
        }
    }
    if (S.timed) for (auto& e : S.ev) cudaEventDestroy(e);
    S.timed = false;
}

// ---------------------------------------------------------------------------
// distributed grid pipeline: spread grids summed by a
// reduce-scatter into z slabs -> xy FFT of the slab -> all-to-all to (kx,ky)
// pencils -> z DCT, mode BVPs, correction, inverse z DCT, assembly ->
// all-to-all back to slabs -> inverse xy FFT -> all-gather of the fields.
// The collectives are the caller's (NCCL through torch.distributed); the
// library packs and unpacks contiguous per-rank blocks.
// ---------------------------------------------------------------------------
namespace {

// hat slab [zc][2][M] -> send [P][zc][2][mc] (dest q: modes q mc ..)
__global__ void pack_modes_kernel(const double2* hat, int64_t M, int64_t zc, int64_t mc, int P,
                                  double2* send) {
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t per = zc * 2 * mc;
    if (e >= (int64_t)P * per) return;
    const int64_t q = e / per, r = e - q * per;
    const int64_t row = r / mc, l = r - row * mc;       // row = plane * 2 + grid
    const int64_t gm = q * mc + l;
    send[e] = gm < M ? hat[row * M + gm] : make_double2(0, 0);
}

// recv [P][zc][F][mc] (from s: planes s zc ..) -> pencil [Nz][F][mc]
__global__ void unpack_planes_kernel(const double2* recv, int64_t zc, int64_t mc, int F, int P,
                                     int Nz, double2* pen) {
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t per = zc * F * mc;
    if (e >= (int64_t)P * per) return;
    const int64_t s = e / per, r = e - s * per;
    const int64_t j = r / (F * mc), rest = r - j * F * mc;
    const int64_t z = s * zc + j;
    if (z < Nz) pen[z * F * mc + rest] = recv[e];
}

// pencil [Nz][4][mc] -> send [P][zc][4][mc] (dest q: planes q zc ..)
__global__ void pack_planes_kernel(const double2* pen, int64_t zc, int64_t mc, int P, int Nz,
                                   double2* send) {
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t per = zc * 4 * mc;
    if (e >= (int64_t)P * per) return;
    const int64_t q = e / per, r = e - q * per;
    const int64_t j = r / (4 * mc), rest = r - j * 4 * mc;
    const int64_t z = q * zc + j;
    send[e] = z < Nz ? pen[z * 4 * mc + rest] : make_double2(0, 0);
}

// recv [P][zc][4][mc] (from s: modes s mc ..) -> spec slab [zc][4][M]
__global__ void unpack_modes_kernel(const double2* recv, int64_t M, int64_t zc, int64_t mc, int P,
                                    double2* spec) {
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t per = zc * 4 * mc;
    if (e >= (int64_t)P * per) return;
    const int64_t s = e / per, r = e - s * per;
    const int64_t row = r / mc, l = r - row * mc;       // row = plane * 4 + field
    const int64_t gm = s * mc + l;
    if (gm < M) spec[row * M + gm] = recv[e];
}

// scalars of the mode stage to be summed over ranks: A_i, the k = 0
// diagnostics (owner of mode 0 only) and the flag bits as counts
__global__ void dsc_pack_kernel(const double* scal, const double* k0, const int* flags,
                                int owner, double* dsc) {
    for (int i = 0; i < 16; ++i) dsc[i] = 0.0;
    if (owner) {
        dsc[0] = scal[0];
        for (int i = 0; i < 10; ++i) dsc[1 + i] = k0[i];
        dsc[12] = (*flags & FLAG_K0_FAIL) ? 1.0 : 0.0;
        dsc[13] = (*flags & FLAG_K0_WARN) ? 1.0 : 0.0;
    }
    dsc[11] = (*flags & FLAG_NONFINITE) ? 1.0 : 0.0;
}

__global__ void dsc_apply_kernel(const double* dsc, double* scal, double* k0, int* flags) {
    scal[0] = dsc[0];
    for (int i = 0; i < 10; ++i) k0[i] = dsc[1 + i];
    int f = *flags;
    if (dsc[11] > 0) f |= FLAG_NONFINITE;
    if (dsc[12] > 0) f |= FLAG_K0_FAIL;
    if (dsc[13] > 0) f |= FLAG_K0_WARN;
    *flags = f;
}

}  // namespace

static ModeView my_modes(const Plan* p) {
    const int64_t m0 = (int64_t)p->rank * p->mc;
    const int64_t mv = std::max<int64_t>(0, std::min<int64_t>(p->mc, p->M - m0));
    return ModeView{p->mc, mv, m0};
}

void dist_setup(Plan* p, int rank, int nranks) {
    if (nranks < 1 || rank < 0 || rank >= nranks) throw Error(SE_ERR_VALUE, "bad rank / nranks");
    if (p->dist) throw Error(SE_ERR_VALUE, "plan already distributed");
    const int64_t P = nranks;
    p->rank = rank; p->nranks = nranks;
    p->zc = (p->Nz + P - 1) / P;
    p->mc = (p->M + P - 1) / P;
    p->Nz_pad = p->zc * P;
    // full grids padded to whole slabs (pad planes stay zero)
    ensure_grid64(p);
    dfree(p, p->d_rho); dfree(p, p->d_fields);
    p->d_rho = dalloc<double>(p, 2 * (size_t)p->Nz_pad * p->NXY);
    p->d_fields = dalloc<double>(p, 4 * (size_t)p->Nz_pad * p->NXY);
    SE_CUDA(cudaMemsetAsync(p->d_rho, 0, sizeof(double) * 2 * (size_t)p->Nz_pad * p->NXY, p->stream));
    SE_CUDA(cudaMemsetAsync(p->d_fields, 0, sizeof(double) * 4 * (size_t)p->Nz_pad * p->NXY, p->stream));
    p->d_rho_slab = dalloc<double>(p, 2 * (size_t)p->zc * p->NXY);
    p->d_fields_slab = dalloc<double>(p, 4 * (size_t)p->zc * p->NXY);
    const size_t a2a = (size_t)P * p->zc * 4 * p->mc;
    p->d_a2a_send = dalloc<cufftDoubleComplex>(p, a2a);
    p->d_a2a_recv = dalloc<cufftDoubleComplex>(p, a2a);
    p->d_dsc = dalloc<double>(p, 16);
    const int zc = (int)p->zc;
    make_plan2d(&p->fft_fwd_slab, p->Nx, p->Ny, p->Nyh, CUFFT_D2Z, p->NXY, p->M, 2 * zc, p->stream);
    make_plan2d(&p->fft_inv4_slab, p->Nx, p->Ny, p->Nyh, CUFFT_Z2D, p->M, p->NXY, 4 * zc, p->stream);
    make_plan2d(&p->fft_inv1_slab, p->Nx, p->Ny, p->Nyh, CUFFT_Z2D, 4 * p->M, 4 * p->NXY, zc,
                p->stream);
    p->dist = true;
}

// phase 2a: xy FFT of the summed slab, packed for the all-to-all to pencils
void dist_forward(Plan* p) {
    Solve& S = current(p);
    if (!p->dist) throw Error(SE_ERR_CUDA, "plan not distributed (se_dist_setup)");
    if (S.phase != 1) throw Error(SE_ERR_CUDA, "se_dist_forward before se_shard_spread");
    SE_CUFFT(cufftExecD2Z(p->fft_fwd_slab, p->d_rho_slab, p->d_hat));
    const int64_t total = (int64_t)p->nranks * p->zc * 2 * p->mc;
    pack_modes_kernel<<<(unsigned)((total + 255) / 256), 256, 0, p->stream>>>(
        reinterpret_cast<const double2*>(p->d_hat), p->M, p->zc, p->mc, p->nranks,
        reinterpret_cast<double2*>(p->d_a2a_send));
    SE_LAUNCHED(p);
    S.phase = 11;
}

// phase 2b: this rank's mode pencils: z DCT, BVPs, correction, inverse z DCT,
// assembly; packed for the all-to-all back; mode-stage scalars in d_dsc
void dist_modes(Plan* p) {
    Solve& S = current(p);
    if (S.phase != 11) throw Error(SE_ERR_CUDA, "se_dist_modes before se_dist_forward");
    const ModeView v = my_modes(p);
    const int64_t tot2 = (int64_t)p->nranks * p->zc * 2 * p->mc;
    unpack_planes_kernel<<<(unsigned)((tot2 + 255) / 256), 256, 0, p->stream>>>(
        reinterpret_cast<const double2*>(p->d_a2a_recv), p->zc, p->mc, 2, p->nranks, p->Nz,
        reinterpret_cast<double2*>(p->d_hat));
    SE_LAUNCHED(p);
    z_forward(p, v);
    mark(p, S);
    bvp_solve_view(p, S.two, S.mode, S.corr, v);
    mark(p, S);
    z_inverse_assemble(p, S.forces, S.corr, v);
    const int64_t tot4 = (int64_t)p->nranks * p->zc * 4 * p->mc;
    pack_planes_kernel<<<(unsigned)((tot4 + 255) / 256), 256, 0, p->stream>>>(
        reinterpret_cast<const double2*>(p->d_spec), p->zc, p->mc, p->nranks, p->Nz,
        reinterpret_cast<double2*>(p->d_a2a_send));
    SE_LAUNCHED(p);
    dsc_pack_kernel<<<1, 1, 0, p->stream>>>(p->d_scal, p->d_k0, p->d_flags, v.m0 == 0 ? 1 : 0,
                                            p->d_dsc);
    SE_LAUNCHED(p);
    S.phase = 12;
}

// phase 2c: summed scalars applied, spectra of this rank's planes unpacked,
// inverse xy FFT into the field slab (the caller all-gathers the slabs into
// the full field grid before se_shard_charges)
void dist_fields(Plan* p) {
    Solve& S = current(p);
    if (S.phase != 12) throw Error(SE_ERR_CUDA, "se_dist_fields before se_dist_modes");
    dsc_apply_kernel<<<1, 1, 0, p->stream>>>(p->d_dsc, p->d_scal, p->d_k0, p->d_flags);
    SE_LAUNCHED(p);
    const int64_t tot4 = (int64_t)p->nranks * p->zc * 4 * p->mc;
    unpack_modes_kernel<<<(unsigned)((tot4 + 255) / 256), 256, 0, p->stream>>>(
        reinterpret_cast<const double2*>(p->d_a2a_recv), p->M, p->zc, p->mc, p->nranks,
        reinterpret_cast<double2*>(p->d_spec));
    SE_LAUNCHED(p);
    if (S.forces) SE_CUFFT(cufftExecZ2D(p->fft_inv4_slab, p->d_spec, p->d_fields_slab));
    else SE_CUFFT(cufftExecZ2D(p->fft_inv1_slab, p->d_spec, p->d_fields_slab));
    mark(p, S);
    S.phase = 2;
}

// SE_NEAR_OVERLAP: Solve::near_fork of single-GPU solves, default 2 (the
// cell list and pair-list scan on the high-priority side stream): C4 fp64
// 17.69 -> 17.45 ms, the paper's configuration 1.08 -> 0.97 ms; 1 (the whole
// near field on the side stream) contends with the interpolation at C4
// (20.2 ms); 3 (the grid pipeline on the side stream instead) gains nothing
// A solve with the per-kernel event timers (SE_TIMINGS) runs serially, so
// each stage's events bracket its own kernels.
static int near_fork_mode(uint32_t flags) {
    static const char* e = getenv("SE_NEAR_OVERLAP");
    if (flags & SE_TIMINGS) return 0;
    return e ? atoi(e) : 2;
}

void solve_core(Plan* p, const double* d_pos, int64_t n, uint32_t flags,
                double* d_phi_out, double* d_E_out, double* U, se_diag* diag) {
    // fp32 mode of a whole (single-GPU) solve: the grid path in fp32 too
    if (p->fork_main) {                  // a fork-3 solve that threw midway
        bind_stream(p, p->fork_main);
        p->fork_main = nullptr;
    }
    p->g32 = (flags & SE_FP32) != 0;
    if (p->g32) ensure_grid32(p);
    else ensure_grid64(p);
    const bool graph = (flags & SE_GRAPH) && !(flags & (SE_TIMINGS | SE_PAIR_HASH));
    const Plan::GraphKey key{d_pos, d_phi_out, d_E_out, n, flags};
    if (graph && p->gexec && p->gkey == key) {
        // the host-side solve state is as the capture left it
        SE_CUDA(cudaGraphLaunch(p->gexec, p->stream));
        phase_results(p, U, diag);
        return;
    }
    if (graph && p->gwarm == key) {
        // capture (the warm solve sized every buffer and table) on a private
        // stream -- the caller's may be the legacy stream, which cannot be
        // captured -- then launch on the caller's
        if (p->gexec) { cudaGraphExecDestroy(p->gexec); p->gexec = nullptr; }
        if (!p->cap_stream) SE_CUDA(cudaStreamCreateWithFlags(&p->cap_stream, cudaStreamNonBlocking));
        const cudaStream_t run = p->stream;
        auto bind = [&](cudaStream_t st) { bind_stream(p, st); };
        SE_CUDA(cudaStreamSynchronize(run));
        bind(p->cap_stream);
        cudaGraph_t g = nullptr;
        cudaError_t ce = cudaStreamBeginCapture(p->cap_stream, cudaStreamCaptureModeThreadLocal);
        if (ce != cudaSuccess) { bind(run); SE_CUDA(ce); }
        try {
            p->fork_req = near_fork_mode(flags);
            phase_spread(p, d_pos, n, 0, n, flags);
            phase_fields(p);
            phase_charges(p, d_pos, d_phi_out, d_E_out);
        } catch (...) {
            cudaStreamEndCapture(p->cap_stream, &g);
            if (g) cudaGraphDestroy(g);
            cudaGetLastError();
            p->fork_main = nullptr;
            bind(run);
            p->gwarm = {};
            throw;
        }
        ce = cudaStreamEndCapture(p->cap_stream, &g);
        bind(run);
        SE_CUDA(ce);
        const cudaError_t ie = cudaGraphInstantiate(&p->gexec, g, 0);
        cudaGraphDestroy(g);
        SE_CUDA(ie);
        p->gkey = key;
        SE_CUDA(cudaGraphLaunch(p->gexec, p->stream));
        phase_results(p, U, diag);
        return;
    }
    p->fork_req = near_fork_mode(flags);
    phase_spread(p, d_pos, n, 0, n, flags);
    phase_fields(p);
    phase_charges(p, d_pos, d_phi_out, d_E_out);
    phase_results(p, U, diag);
    if (graph && !p->last_overflow) p->gwarm = key;
}

void ensure_charges(Plan* p, int64_t n) {
    if (n <= p->q_cap && p->d_q) return;
    void* olds[] = {p->d_q, p->d_pos, p->d_phi, p->d_E, p->d_far, p->d_near};
    for (void* o : olds) dfree(p, o);
    int64_t cap = std::max<int64_t>(n, 1);
    p->d_q = dalloc<double>(p, cap);
    p->d_pos = dalloc<double>(p, 3 * cap);
    p->d_phi = dalloc<double>(p, cap);
    p->d_E = dalloc<double>(p, 3 * cap);
    p->d_far = dalloc<double>(p, 4 * cap);
    p->d_near = dalloc<double>(p, 4 * cap);
    p->q_cap = cap;
}

}  // namespace
}  // namespace se

using namespace se;

extern "C" {

const char* se_last_error(void) { return g_error.c_str(); }

int se_fp64_peak(int device, double* tflops) {
    try {
        SE_CUDA(cudaSetDevice(device));
        int sms = 0;
        SE_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
        double* d = nullptr;
        SE_CUDA(cudaMalloc(&d, sizeof(double)));
        cudaEvent_t e0, e1;
        SE_CUDA(cudaEventCreate(&e0));
        SE_CUDA(cudaEventCreate(&e1));
        const int blocks = sms * 8, threads = 256, iters = 1 << 14;
        dfma_probe_kernel<<<blocks, threads>>>(d, 256, 0.999999, 1e-7);   // warm-up
        SE_CUDA(cudaEventRecord(e0));
        dfma_probe_kernel<<<blocks, threads>>>(d, iters, 0.999999, 1e-7);
        SE_CUDA(cudaEventRecord(e1));
        SE_CUDA(cudaEventSynchronize(e1));
        float ms = 0;
        SE_CUDA(cudaEventElapsedTime(&ms, e0, e1));
        *tflops = 2.0 * 8.0 * iters * (double)blocks * threads / (ms * 1e-3) / 1e12;
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        cudaFree(d);
        return SE_OK;
    } catch (const Error& e) {
        return fail(e);
    }
}
const char* se_version(void) { return "slabewald-b200 0.1.0 (sm_100a)"; }

int se_plan_create(const se_params* params, const double* z_nodes, const double* cc_w,
                   const double* t_wall0, const double* t_wallH, const double* kx,
                   const double* ky, const double* sigma_b, const double* sigma_t,
                   int device, se_plan** out) {
    Plan* p = nullptr;
    try {
        if (!params || !out) throw Error(SE_ERR_VALUE, "null argument");
        p = new Plan();
        p->P = *params;
        const se_params& P = p->P;
        if (P.Nx < 1 || P.Ny < 1 || P.Nz < 3)
            throw Error(SE_ERR_VALUE, "grid must have Nx, Ny >= 1 and Nz >= 3");
        p->dev = device;
        SE_CUDA(cudaSetDevice(device));
        SE_CUDA(cudaDeviceGetAttribute(&p->num_sms, cudaDevAttrMultiProcessorCount, device));
        SE_CUDA(cudaStreamCreateWithFlags(&p->stream, cudaStreamNonBlocking));
        p->own_stream = true;
        p->Nx = P.Nx; p->Ny = P.Ny; p->Nz = P.Nz;
        p->Nyh = P.Ny / 2 + 1;
        p->N2 = 2 * (P.Nz - 1);
        p->M = (int64_t)p->Nx * p->Nyh;
        p->NXY = (int64_t)p->Nx * p->Ny;
        p->G = p->NXY * p->Nz;
        p->hx = P.Lx / P.Nx;                   // gridops.py:54-55
        p->hy = P.Ly / P.Ny;
        p->rad = P.H_E;
        p->rad_keep = P.H_E + 1e-12 * P.H_E;    // gridops.py:25
        p->width = P.g_t;
        p->norm = std::sqrt(2.0 * M_PI * (P.g_t * P.g_t));
        p->mx = (int)std::floor(P.H_E / p->hx + 1e-12);
        p->my = (int)std::floor(P.H_E / p->hy + 1e-12);
        if (p->mx > MAX_M || p->my > MAX_M)
            throw Error(SE_ERR_VALUE, "Gaussian support wider than the tile kernels handle");
        const int nz = P.Nz;
        p->z.assign(z_nodes, z_nodes + nz);
        p->wcc.assign(cc_w, cc_w + nz);
        p->tw0.assign(t_wall0, t_wall0 + nz);
        p->twH.assign(t_wallH, t_wallH + nz);
        p->kx.assign(kx, kx + p->Nx);
        p->ky.assign(ky, ky + p->Ny);
        // widest z stencil: nodes within any window of length 2 H_E (+1 slack)
        int wz = 1;
        for (int i = 0, j = 0; i < nz; ++i) {
            while (j < nz && p->z[j] - p->z[i] <= 2.0 * P.H_E) ++j;
            wz = std::max(wz, j - i);
        }
        p->wz_max = std::min(wz + 1, nz);
        // correction window (dpsolver.py:106): z in [-H_E, H + H_E]
        const double zlo = -P.H_E, zhi = P.H + P.H_E;
        p->win0 = nz; p->win1 = 0;
        for (int j = 0; j < nz; ++j)
            if (p->z[j] >= zlo && p->z[j] <= zhi) { p->win0 = std::min(p->win0, j); p->win1 = j + 1; }
        if (p->win1 <= p->win0) p->win0 = p->win1 = 0;
        // per-mode |k| on the half spectrum, distinct values, selection
        std::vector<double> kmag(p->M);
        std::vector<unsigned char> sel(p->M);
        std::vector<double> uniq;
        for (int ix = 0; ix < p->Nx; ++ix)
            for (int iy = 0; iy < p->Nyh; ++iy) {
                double k = std::hypot(p->kx[ix], p->ky[iy]);   // dpsolver.py:38
                int64_t m = (int64_t)ix * p->Nyh + iy;
                kmag[m] = k;
                sel[m] = (k > 0.0 && k <= P.k_max) ? 1 : 0;     // dpsolver.py:105
                if (k > 0.0) uniq.push_back(k);
            }
        std::sort(uniq.begin(), uniq.end());
        uniq.erase(std::unique(uniq.begin(), uniq.end()), uniq.end());
        std::vector<int> kidx(p->M);
        for (int64_t m = 0; m < p->M; ++m)
            kidx[m] = kmag[m] > 0.0
                          ? (int)(std::lower_bound(uniq.begin(), uniq.end(), kmag[m]) - uniq.begin())
                          : -1;
        p->n_uniq = (int)uniq.size();
        auto up = [&](const std::vector<double>& h) {
            double* d = dalloc<double>(p, h.size());
            SE_CUDA(cudaMemcpy(d, h.data(), h.size() * sizeof(double), cudaMemcpyHostToDevice));
            return d;
        };
        p->d_z = up(p->z); p->d_wcc = up(p->wcc); p->d_tw0 = up(p->tw0); p->d_twH = up(p->twH);
        p->d_kx = up(p->kx); p->d_ky = up(p->ky); p->d_kmag = up(kmag);
        p->d_kuniq = up(uniq.empty() ? std::vector<double>{0.0} : uniq);
        p->d_kidx = dalloc<int>(p, p->M);
        SE_CUDA(cudaMemcpy(p->d_kidx, kidx.data(), p->M * sizeof(int), cudaMemcpyHostToDevice));
        p->d_sel = dalloc<unsigned char>(p, p->M);
        SE_CUDA(cudaMemcpy(p->d_sel, sel.data(), p->M, cudaMemcpyHostToDevice));
        factor_bvp(p);

        // buffers
        // the fp64 grids and their cuFFT plans come with the first fp64
        // solve (ensure_grid64), the fp32 ones with the first fp32 solve
        p->d_ext = dalloc<cufftDoubleComplex>(p, (size_t)nz * 2 * p->M);
        p->d_scr = dalloc<cufftDoubleComplex>(p, 4 * (size_t)nz * p->M);   // A, B columns
        p->d_bst = dalloc<cufftDoubleComplex>(p, 12 * (size_t)p->M);
        p->d_mom = dalloc<cufftDoubleComplex>(p, 2 * (size_t)p->M);
        p->d_mism = dalloc<cufftDoubleComplex>(p, 4 * (size_t)p->M);
        const char* keep = std::getenv("SE_KEEP_STAGES");
        p->keep_stages = keep && keep[0] == '1';
        if (p->keep_stages) p->d_keep = dalloc<cufftDoubleComplex>(p, (size_t)nz * 2 * p->M);
        p->d_k0 = dalloc<double>(p, 16);
        p->d_scal = dalloc<double>(p, 8);
        p->d_flags = dalloc<int>(p, 1);
        p->d_count = dalloc<int64_t>(p, 1);
        p->d_ovf_acc = dalloc<int>(p, 1);
        p->d_partial = dalloc<double>(p, 1024);
        p->d_mm = dalloc<double>(p, 256);
        p->d_origin = dalloc<double>(p, 3);
        SE_CUDA(cudaMemset(p->d_origin, 0, 3 * sizeof(double)));
        SE_CUDA(cudaMemset(p->d_k0, 0, 16 * sizeof(double)));

        // wall charge: samples and their normalised half spectra (slab.py:209-213)
        p->sigma_zero = (sigma_b == nullptr && sigma_t == nullptr);
        p->d_sigb = dalloc<double>(p, 2 * (size_t)p->NXY);
        p->d_sigt = p->d_sigb + p->NXY;
        p->d_sbh = dalloc<cufftDoubleComplex>(p, 2 * (size_t)p->M);
        p->d_sth = p->d_sbh + p->M;
        double sscale = 0.0;
        if (p->sigma_zero) {
            SE_CUDA(cudaMemset(p->d_sigb, 0, 2 * p->NXY * sizeof(double)));
            SE_CUDA(cudaMemset(p->d_sbh, 0, 2 * p->M * sizeof(cufftDoubleComplex)));
        } else {
            std::vector<double> zeros(p->NXY, 0.0);
            const double* sb = sigma_b ? sigma_b : zeros.data();
            const double* st = sigma_t ? sigma_t : zeros.data();
            SE_CUDA(cudaMemcpy(p->d_sigb, sb, p->NXY * sizeof(double), cudaMemcpyHostToDevice));
            SE_CUDA(cudaMemcpy(p->d_sigt, st, p->NXY * sizeof(double), cudaMemcpyHostToDevice));
            double ab = 0, at = 0;
            for (int64_t i = 0; i < p->NXY; ++i) { ab += std::fabs(sb[i]); at += std::fabs(st[i]); }
            sscale = ab / p->NXY + at / p->NXY;
            make_plan2d(&p->fft_sig, p->Nx, p->Ny, p->Nyh, CUFFT_D2Z, p->NXY, p->M, 2, p->stream);
            SE_CUFFT(cufftExecD2Z(p->fft_sig, p->d_sigb, p->d_sbh));
            scale_complex<<<(unsigned)((2 * p->M + 255) / 256), 256, 0, p->stream>>>(
                p->d_sbh, 2 * p->M, 1.0 / (double)p->NXY);
            SE_LAUNCHED(p);
        }
        p->sigma_scale = sscale;

        SE_CUDA(cudaStreamSynchronize(p->stream));
        *out = reinterpret_cast<se_plan*>(p);
        return SE_OK;
    } catch (const Error& e) {
        if (p) se_plan_destroy(reinterpret_cast<se_plan*>(p));
        return fail(e);
    } catch (const std::exception& e) {
        if (p) se_plan_destroy(reinterpret_cast<se_plan*>(p));
        return fail(Error(SE_ERR_CUDA, e.what()));
    }
}

void se_plan_destroy(se_plan* plan) {
    Plan* p = reinterpret_cast<Plan*>(plan);
    if (!p) return;
    cudaSetDevice(p->dev);
    if (p->stream) cudaStreamSynchronize(p->stream);
    cufftHandle hs[] = {p->fft_fwd2, p->fft_fwd1, p->fft_z, p->fft_inv4, p->fft_inv1, p->fft_sig,
                        p->fft_fwd_slab, p->fft_inv4_slab, p->fft_inv1_slab, p->fft_fwd2_f,
                        p->fft_inv4_f, p->fft_inv1_f};
    for (auto h : hs) if (h) cufftDestroy(h);
    for (auto& b : p->owned) if (b.p) cudaFree(b.p);
    if (p->gexec) cudaGraphExecDestroy(p->gexec);
    if (p->cap_stream) cudaStreamDestroy(p->cap_stream);
    if (p->side) cudaStreamDestroy(p->side);
    if (p->ev_fork) cudaEventDestroy(p->ev_fork);
    if (p->ev_join) cudaEventDestroy(p->ev_join);
    for (auto& pr : p->kev) { if (pr[0]) cudaEventDestroy(pr[0]); if (pr[1]) cudaEventDestroy(pr[1]); }
    if (p->stream && p->own_stream) cudaStreamDestroy(p->stream);
    delete p;
}

int se_plan_set_stream(se_plan* plan, void* stream) {
    Plan* p = reinterpret_cast<Plan*>(plan);
    try {
        if (!p) throw Error(SE_ERR_VALUE, "null plan");
        SE_CUDA(cudaSetDevice(p->dev));
        SE_CUDA(cudaStreamSynchronize(p->stream));
        if (p->own_stream && p->stream) { cudaStreamDestroy(p->stream); p->own_stream = false; }
        p->fork_main = nullptr;
        bind_stream(p, reinterpret_cast<cudaStream_t>(stream));
        return SE_OK;
    } catch (const Error& e) {
        return fail(e);
    }
}

int se_set_charges(se_plan* plan, const double* q, int64_t n) {
    Plan* p = reinterpret_cast<Plan*>(plan);
    try {
        if (!p) throw Error(SE_ERR_VALUE, "null plan");
        if (n < 0) throw Error(SE_ERR_VALUE, "negative charge count");
        SE_CUDA(cudaSetDevice(p->dev));
        ensure_charges(p, n);
        if (n > 0)
            SE_CUDA(cudaMemcpy(p->d_q, q, n * sizeof(double), cudaMemcpyHostToDevice));
        if (p->gexec) { cudaGraphExecDestroy(p->gexec); p->gexec = nullptr; }
        p->gkey = {}; p->gwarm = {};
        p->N = n;
        double aq = 0;
        for (int64_t i = 0; i < n; ++i) aq += std::fabs(q[i]);
        p->k0_scale = (aq / (p->P.Lx * p->P.Ly) + p->sigma_scale) / p->P.eps;   // slab.py:231-233
        return SE_OK;
    } catch (const Error& e) {
        return fail(e);
    }
}

int se_solve(se_plan* plan, const double* pos, int64_t n, uint32_t flags, double* phi_bar,
             double* E_bar, double* U, se_diag* diag) {
    Plan* p = reinterpret_cast<Plan*>(plan);
    try {
        if (!p) throw Error(SE_ERR_VALUE, "null plan");
        SE_CUDA(cudaSetDevice(p->dev));
        if (n != p->N) throw Error(SE_ERR_VALUE, "positions and charges disagree on N");
        if (n > 0)
            SE_CUDA(cudaMemcpyAsync(p->d_pos, pos, 3 * n * sizeof(double),
                                    cudaMemcpyHostToDevice, p->stream));
        solve_core(p, p->d_pos, n, flags, p->d_phi, p->d_E, U, diag);
        if (n > 0) {
            if (phi_bar)
                SE_CUDA(cudaMemcpyAsync(phi_bar, p->d_phi, n * sizeof(double),
                                        cudaMemcpyDeviceToHost, p->stream));
            if (E_bar && (flags & SE_NEED_FORCES))
                SE_CUDA(cudaMemcpyAsync(E_bar, p->d_E, 3 * n * sizeof(double),
                                        cudaMemcpyDeviceToHost, p->stream));
            SE_CUDA(cudaStreamSynchronize(p->stream));
        }
        return SE_OK;
    } catch (const Error& e) {
        return fail(e);
    }
}

int se_solve_device(se_plan* plan, const double* d_pos, int64_t n, uint32_t flags,
                    double* d_phi_bar, double* d_E_bar, double* U, se_diag* diag) {
    Plan* p = reinterpret_cast<Plan*>(plan);
    try {
        if (!p) throw Error(SE_ERR_VALUE, "null plan");
        SE_CUDA(cudaSetDevice(p->dev));
        solve_core(p, d_pos, n, flags, d_phi_bar ? d_phi_bar : p->d_phi,
                   d_E_bar ? d_E_bar : p->d_E, U, diag);
        return SE_OK;
    } catch (const Error& e) {
        return fail(e);
    }
}

// light-weight plan for the plan-free entry points (no grids, no FFTs)
static Plan* light_plan(const se_params* params, int device) {
    if (!params) throw Error(SE_ERR_VALUE, "null params");
    Plan* p = new Plan();
    p->P = *params;
    p->dev = device;
    SE_CUDA(cudaSetDevice(device));
    SE_CUDA(cudaDeviceGetAttribute(&p->num_sms, cudaDevAttrMultiProcessorCount, device));
    SE_CUDA(cudaStreamCreateWithFlags(&p->stream, cudaStreamNonBlocking));
    p->own_stream = true;
    p->d_flags = dalloc<int>(p, 1);
    SE_CUDA(cudaMemset(p->d_flags, 0, sizeof(int)));
    return p;
}

struct PlanGuard {
    Plan* p;
    ~PlanGuard() { if (p) se_plan_destroy(reinterpret_cast<se_plan*>(p)); }
};

int se_shard_spread(se_plan* plan, const double* d_pos_all, int64_t n_all, int64_t first,
                    int64_t count, uint32_t flags, double** d_rho, int64_t* rho_len) {
    Plan* p = reinterpret_cast<Plan*>(plan);
    try {
        if (!p) throw Error(SE_ERR_VALUE, "null plan");
        SE_CUDA(cudaSetDevice(p->dev));
        p->g32 = false;                 // the ranks sum fp64 grids
        ensure_grid64(p);
        phase_spread(p, d_pos_all, n_all, first, count, flags);
        if (d_rho) *d_rho = p->d_rho;
        if (rho_len) *rho_len = 2 * p->G;
        return SE_OK;
    } catch (const Error& e) {
        return fail(e);
    }
}

int se_shard_fields(se_plan* plan) {
    Plan* p = reinterpret_cast<Plan*>(plan);
    try {
        if (!p) throw Error(SE_ERR_VALUE, "null plan");
        SE_CUDA(cudaSetDevice(p->dev));
        phase_fields(p);
        return SE_OK;
    } catch (const Error& e) {
        return fail(e);
    }
}

int se_shard_charges(se_plan* plan, const double* d_pos_all, double* d_phi, double* d_E,
                     double* U_part, se_diag* diag) {
    Plan* p = reinterpret_cast<Plan*>(plan);
    try {
        if (!p) throw Error(SE_ERR_VALUE, "null plan");
        SE_CUDA(cudaSetDevice(p->dev));
        phase_charges(p, d_pos_all, d_phi, d_E);
        phase_results(p, U_part, diag);
        return SE_OK;
    } catch (const Error& e) {
        return fail(e);
    }
}

// ---- sharded solve with positions of the own shard only and the near field
// routed by cell.  The library indexes charges
// globally; the own-shard positions are addressed through a base pointer
// offset by -first rows, of which only rows [first, first + count) are read.
int se_shard_spread_own(se_plan* plan, const double* d_pos_own, int64_t n_all, int64_t first,
                        int64_t count, uint32_t flags, double** d_rho, int64_t* rho_len) {
    Plan* p = reinterpret_cast<Plan*>(plan);
    try {
        if (!p) throw Error(SE_ERR_VALUE, "null plan");
        SE_CUDA(cudaSetDevice(p->dev));
        p->g32 = false;
        ensure_grid64(p);
        const double* base = d_pos_own - 3 * first;
        phase_spread(p, base, n_all, first, count, flags);
        if (d_rho) *d_rho = p->d_rho;
        if (rho_len) *rho_len = 2 * p->G;
        return SE_OK;
    } catch (const Error& e) {
        return fail(e);
    }
}

int se_shard_near(se_plan* plan, void* stream, const double* d_src_pos, const double* d_src_q,
                  int64_t ns, int64_t nt, int gauge, const double* d_zsrc_min, double* d_out,
                  double* d_near0, int64_t* d_npairs) {
    Plan* p = reinterpret_cast<Plan*>(plan);
    cudaStream_t saved = p ? p->stream : nullptr;
    try {
        if (!p) throw Error(SE_ERR_VALUE, "null plan");
        if (nt < 0 || nt > ns) throw Error(SE_ERR_VALUE, "targets must be the first sources");
        SE_CUDA(cudaSetDevice(p->dev));
        const se_params& P = p->P;
        const Solve& S = p->solve;
        if (S.phase == 0) throw Error(SE_ERR_CUDA, "se_shard_near outside a sharded solve");
        if (S.xi_inf) throw Error(SE_ERR_VALUE, "no near field at xi = inf");
        p->stream = reinterpret_cast<cudaStream_t>(stream);
        const bool timing = p->timing;
        p->timing = false;
        p->pair_hash = false;
        if (d_npairs) SE_CUDA(cudaMemsetAsync(d_npairs, 0, sizeof(int64_t), p->stream));
        if (d_near0) SE_CUDA(cudaMemsetAsync(d_near0, 0, sizeof(double), p->stream));
        NearKernel kavg = kernel_of(P, 0, S.forces, S.flags & SE_SUBTRACT_SELF);
        kavg.fp32 = (S.flags & SE_FP32) ? 1 : 0;
        if (ns > 0) {
            build_cells(p, d_src_pos, d_src_q, ns, true, d_zsrc_min);
            near_eval(p, d_src_pos, nullptr, nt, kavg, d_out, d_npairs);
            if (gauge && d_near0)
                near_eval(p, p->d_origin, nullptr, 1, kernel_of(P, 1, false, false), d_near0,
                          nullptr);
        }
        p->timing = timing;
        p->stream = saved;
        return SE_OK;
    } catch (const Error& e) {
        if (p) p->stream = saved;
        return fail(e);
    }
}

int se_shard_charges_own(se_plan* plan, const double* d_pos_own, const double* d_near_own,
                         const double* d_near0, double* d_phi, double* d_E, double* U_part,
                         se_diag* diag) {
    Plan* p = reinterpret_cast<Plan*>(plan);
    try {
        if (!p) throw Error(SE_ERR_VALUE, "null plan");
        SE_CUDA(cudaSetDevice(p->dev));
        Solve& S = p->solve;
        S.near_external = true;
        S.ext_near = d_near_own;
        S.ext_near0 = d_near0;
        const double* base = d_pos_own - 3 * S.first;
        phase_charges(p, base, d_phi, d_E);
        phase_results(p, U_part, diag);
        S.near_external = false;
        return SE_OK;
    } catch (const Error& e) {
        p->solve.near_external = false;
        return fail(e);
    }
}

int se_dist_setup(se_plan* plan, int rank, int nranks, int64_t* sizes) {
    Plan* p = reinterpret_cast<Plan*>(plan);
    try {
        if (!p) throw Error(SE_ERR_VALUE, "null plan");
        SE_CUDA(cudaSetDevice(p->dev));
        dist_setup(p, rank, nranks);
        if (sizes) {
            sizes[0] = 2 * p->Nz_pad * p->NXY;        // full grids (doubles)
            sizes[1] = 2 * p->zc * p->NXY;            // grid slab
            sizes[2] = 2 * (int64_t)p->nranks * p->zc * 2 * p->mc;   // all-to-all forward
            sizes[3] = 2 * (int64_t)p->nranks * p->zc * 4 * p->mc;   // all-to-all back
            sizes[4] = 4 * p->zc * p->NXY;            // field slab
            sizes[5] = 4 * p->Nz_pad * p->NXY;        // full fields
            sizes[6] = 16;                            // summed scalars
        }
        return SE_OK;
    } catch (const Error& e) {
        return fail(e);
    }
}

int se_dist_buffers(se_plan* plan, void** ptrs) {
    Plan* p = reinterpret_cast<Plan*>(plan);
    try {
        if (!p || !p->dist) throw Error(SE_ERR_VALUE, "plan not distributed");
        ptrs[0] = p->d_rho; ptrs[1] = p->d_rho_slab; ptrs[2] = p->d_a2a_send;
        ptrs[3] = p->d_a2a_recv; ptrs[4] = p->d_fields_slab; ptrs[5] = p->d_fields;
        ptrs[6] = p->d_dsc;
        return SE_OK;
    } catch (const Error& e) {
        return fail(e);
    }
}

int se_dist_forward(se_plan* plan) {
    Plan* p = reinterpret_cast<Plan*>(plan);
    try {
        if (!p) throw Error(SE_ERR_VALUE, "null plan");
        SE_CUDA(cudaSetDevice(p->dev));
        dist_forward(p);
        return SE_OK;
    } catch (const Error& e) {
        return fail(e);
    }
}

int se_dist_modes(se_plan* plan) {
    Plan* p = reinterpret_cast<Plan*>(plan);
    try {
        if (!p) throw Error(SE_ERR_VALUE, "null plan");
        SE_CUDA(cudaSetDevice(p->dev));
        dist_modes(p);
        return SE_OK;
    } catch (const Error& e) {
        return fail(e);
    }
}

int se_dist_fields(se_plan* plan) {
    Plan* p = reinterpret_cast<Plan*>(plan);
    try {
        if (!p) throw Error(SE_ERR_VALUE, "null plan");
        SE_CUDA(cudaSetDevice(p->dev));
        dist_fields(p);
        return SE_OK;
    } catch (const Error& e) {
        return fail(e);
    }
}

int se_steric_forces(int device, const double* pos, int64_t n, double Lx, double Ly,
                     double Lz, double a, double U0, double r_m, int p, double* out) {
    try {
        steric_forces(device, pos, n, Lx, Ly, Lz, a, U0, r_m, p, out);
        return SE_OK;
    } catch (const Error& e) {
        return fail(e);
    }
}

int se_steric_forces_device(int device, void* stream, const double* d_pos, int64_t n, double Lx,
                            double Ly, double Lz, double zlo, double zhi, double a, double U0,
                            double r_m, int p, double* d_out) {
    try {
        steric_forces_device(device, static_cast<cudaStream_t>(stream), d_pos, n, Lx, Ly, Lz, zlo,
                             zhi, a, U0, r_m, p, d_out);
        return SE_OK;
    } catch (const Error& e) {
        return fail(e);
    }
}

int se_bd_first_noise_device(int device, void* stream, int64_t n, uint64_t seed, double* d_prev) {
    try {
        bd_first_noise_device(device, static_cast<cudaStream_t>(stream), n, seed, d_prev);
        return SE_OK;
    } catch (const Error& e) {
        return fail(e);
    }
}

int se_bd_step_device(int device, void* stream, double* d_pos, double* d_prev, const double* d_E,
                      const double* d_q, const double* d_fext, int64_t n,
                      const se_bd_params* params, uint64_t* draws, int64_t* rejections) {
    try {
        bd_step_device(device, static_cast<cudaStream_t>(stream), d_pos, d_prev, d_E, d_q, d_fext,
                       n, *params, draws, rejections);
        return SE_OK;
    } catch (const Error& e) {
        return fail(e);
    }
}

int se_tp_create(int device, double Lx, double Ly, double Lz, int nx, int ny, int nz,
                 double eps, se_tp** plan) {
    try {
        const double L[3] = {Lx, Ly, Lz};
        const int n[3] = {nx, ny, nz};
        *plan = reinterpret_cast<se_tp*>(tp_create(device, L, n, eps));
        return SE_OK;
    } catch (const Error& e) {
        *plan = nullptr;
        return fail(e);
    }
}

int se_tp_destroy(se_tp* plan) {
    tp_destroy(reinterpret_cast<TpPlan*>(plan));
    return SE_OK;
}

int se_tp_set_stream(se_tp* plan, void* stream) {
    try {
        tp_set_stream(reinterpret_cast<TpPlan*>(plan), static_cast<cudaStream_t>(stream));
        return SE_OK;
    } catch (const Error& e) {
        return fail(e);
    }
}

int se_tp_set_graph(se_tp* plan, int enable) {
    try {
        if (!plan) throw Error(SE_ERR_VALUE, "null plan");
        tp_set_graph(reinterpret_cast<TpPlan*>(plan), enable != 0);
        return SE_OK;
    } catch (const Error& e) {
        return fail(e);
    }
}

int se_tp_poisson(se_tp* plan, const double* rho, int with_field, double* phi, double* E) {
    try {
        tp_poisson(reinterpret_cast<TpPlan*>(plan), rho, with_field, phi, E);
        return SE_OK;
    } catch (const Error& e) {
        return fail(e);
    }
}

int se_tp_forces(se_tp* plan, const double* pos, const double* q, int64_t n, double g_t,
                 double radius, double g_w, double xi, double r_cut, double* forces) {
    try {
        tp_forces(reinterpret_cast<TpPlan*>(plan), pos, q, n, g_t, radius, g_w, xi, r_cut, forces);
        return SE_OK;
    } catch (const Error& e) {
        return fail(e);
    }
}

int se_tp_forces_device(se_tp* plan, const double* d_pos, const double* d_q, int64_t n,
                        double g_t, double radius, double g_w, double xi, double r_cut,
                        double* d_forces) {
    try {
        tp_forces_device(reinterpret_cast<TpPlan*>(plan), d_pos, d_q, n, g_t, radius, g_w, xi,
                         r_cut, d_forces);
        return SE_OK;
    } catch (const Error& e) {
        return fail(e);
    }
}

int se_near_field(const se_params* params, int device, const double* pos, const double* q,
                  int64_t n, const double* eval_pos, int64_t ne, int kind, int need_field,
                  int subtract_unsplit, double* phi, double* E) {
    try {
        Plan* p = light_plan(params, device);
        PlanGuard pg{p};
        const se_params& P = p->P;
        p->launches = 0;
        bool empty = n == 0 || P.xi_is_inf != 0.0;
        std::fill(phi, phi + ne, 0.0);
        if (E && need_field) std::fill(E, E + 3 * ne, 0.0);
        if (empty || ne == 0) return SE_OK;
        if (P.r_cut >= 0.5 * std::min(P.Lx, P.Ly))
            throw Error(SE_ERR_VALUE, "near-field cutoff exceeds half the periodic box");
        double *d_pos = nullptr, *d_q = nullptr, *d_ev = nullptr, *d_out = nullptr;
        SE_CUDA(cudaMalloc(&d_pos, 3 * n * sizeof(double)));
        SE_CUDA(cudaMalloc(&d_q, n * sizeof(double)));
        SE_CUDA(cudaMalloc(&d_ev, 3 * ne * sizeof(double)));
        SE_CUDA(cudaMalloc(&d_out, 4 * ne * sizeof(double)));
        struct Guard { void* a[4]; ~Guard() { for (void* x : a) cudaFree(x); } } g{{d_pos, d_q, d_ev, d_out}};
        SE_CUDA(cudaMemcpy(d_pos, pos, 3 * n * sizeof(double), cudaMemcpyHostToDevice));
        SE_CUDA(cudaMemcpy(d_q, q, n * sizeof(double), cudaMemcpyHostToDevice));
        SE_CUDA(cudaMemcpy(d_ev, eval_pos, 3 * ne * sizeof(double), cudaMemcpyHostToDevice));
        const double eps = P.eps, two_sqrtpi = 2.0 / std::sqrt(M_PI);
        NearKernel k{};
        k.inv4pie = 1.0 / (4.0 * M_PI * eps);
        k.kind = kind;
        k.need_field = need_field ? 1 : 0;
        if (kind == 0) {
            k.c1 = 2.0 * P.g_w;
            k.c2 = std::sqrt(4.0 * P.g_w * P.g_w + 1.0 / (P.xi * P.xi));
            k.radius = P.r_cut;
            k.self_value = subtract_unsplit ? -two_sqrtpi / k.c2 / (4.0 * M_PI * eps)
                                            : two_sqrtpi * (0.5 / P.g_w - 1.0 / k.c2) / (4.0 * M_PI * eps);
        } else {
            k.c1 = std::sqrt(2.0) * P.g_w;
            k.c2 = std::sqrt(2.0 * P.g_w * P.g_w + 1.0 / (P.xi * P.xi));
            k.radius = P.r_nf;
            k.point0 = (two_sqrtpi / k.c1 - two_sqrtpi / k.c2) / (4.0 * M_PI * eps);
        }
        build_cells(p, d_pos, d_q, n, false);
        near_eval(p, d_ev, nullptr, ne, k, d_out, nullptr);
        std::vector<double> h(4 * ne);
        int hflags = 0;
        SE_CUDA(cudaMemcpyAsync(h.data(), d_out, (need_field ? 4 : 1) * ne * sizeof(double),
                                cudaMemcpyDeviceToHost, p->stream));
        SE_CUDA(cudaMemcpyAsync(&hflags, p->d_flags, sizeof(int), cudaMemcpyDeviceToHost,
                                p->stream));
        SE_CUDA(cudaStreamSynchronize(p->stream));
        if (hflags & FLAG_NEAR_BND)
            throw Error(SE_ERR_CUDA, "too many near-field pairs at the exact cutoff distance");
        std::copy(h.begin(), h.begin() + ne, phi);
        if (E && need_field)
            for (int64_t i = 0; i < ne; ++i)
                for (int c = 0; c < 3; ++c) E[3 * i + c] = h[(c + 1) * ne + i];
        return SE_OK;
    } catch (const Error& e) {
        return fail(e);
    }
}

int se_build_partition(const se_params* params, int device, const double* pos,
                       const double* q, int64_t n, int64_t* n_over, int64_t* over,
                       int64_t* n_far, int64_t* far, int64_t* n_img, double* img_pos,
                       double* img_str, int64_t* img_src, int32_t* img_wall) {
    try {
        *n_over = *n_far = *n_img = 0;
        if (n == 0) return SE_OK;
        Plan* p = light_plan(params, device);
        PlanGuard pg{p};
        ensure_charges(p, n);
        SE_CUDA(cudaMemcpy(p->d_pos, pos, 3 * n * sizeof(double), cudaMemcpyHostToDevice));
        SE_CUDA(cudaMemcpy(p->d_q, q, n * sizeof(double), cudaMemcpyHostToDevice));
        partition_sources(p, p->d_pos, n);
        std::vector<int> cls(3 * n);
        std::vector<double4> src(3 * n);
        SE_CUDA(cudaMemcpyAsync(cls.data(), p->d_src_cls, 3 * n * sizeof(int),
                                cudaMemcpyDeviceToHost, p->stream));
        SE_CUDA(cudaMemcpyAsync(src.data(), p->d_src, 3 * n * sizeof(double4),
                                cudaMemcpyDeviceToHost, p->stream));
        SE_CUDA(cudaStreamSynchronize(p->stream));
        int64_t no = 0, nf = 0, ni = 0;
        for (int64_t i = 0; i < n; ++i) {
            if (cls[3 * i] == 0) over[no++] = i; else far[nf++] = i;
        }
        for (int64_t k = 0; k < no; ++k) {            // slab.py:66-78 loop order
            int64_t i = over[k];
            for (int w = 0; w < 2; ++w) {
                if (cls[3 * i + 1 + w] < 0) continue;
                double4 v = src[3 * i + 1 + w];
                img_pos[3 * ni] = v.x; img_pos[3 * ni + 1] = v.y; img_pos[3 * ni + 2] = v.z;
                img_str[ni] = v.w; img_src[ni] = i; img_wall[ni] = w;
                ++ni;
            }
        }
        *n_over = no; *n_far = nf; *n_img = ni;
        return SE_OK;
    } catch (const Error& e) {
        return fail(e);
    }
}

int64_t se_debug_fetch(se_plan* plan, int which, void* host, int64_t nbytes) {
    Plan* p = reinterpret_cast<Plan*>(plan);
    if (!p) return -1;
    const void* src = nullptr;
    int64_t size = 0;
    switch (which) {
        case 0: src = p->d_rho; size = p->d_rho ? 2 * p->G * sizeof(double) : 0; break;
        case 1: src = p->d_keep; size = p->keep_stages ? p->Nz * 2 * p->M * 16 : 0; break;
        case 2: src = p->d_fields; size = p->d_fields ? 4 * p->G * sizeof(double) : 0; break;
        case 3: src = p->d_mism; size = 4 * p->M * 16; break;
        case 4: src = p->d_far; size = 4 * p->N * sizeof(double); break;
        case 5: src = p->d_near; size = 4 * p->N * sizeof(double); break;
        case 6: src = p->d_phash; size = p->d_phash ? 2 * p->phash_n * 8 : 0; break;
        default: return -1;
    }
    if (!host) return size;
    if (nbytes < size || !src) return -1;
    cudaSetDevice(p->dev);
    if (cudaMemcpy(host, src, size, cudaMemcpyDeviceToHost) != cudaSuccess) return -1;
    return size;
}

}  // extern "C"
