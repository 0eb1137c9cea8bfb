// Triply periodic twin of the slab solver.
//
// References: solve_triply_periodic (dpsolver.py:221-249), PeriodicGrid3d
// spread / interpolate (gridops.py:136-192, stencils gridops.py:18-26,42-44)
// and TriplyPeriodicSolver.forces (bd.py:297-355): Gaussian spreading on a
// uniform periodic grid, FFT Poisson solve eps lap(phi) = -rho with the k = 0
// mode zeroed, E = -grad phi spectrally (unmatched Nyquist derivative
// dropped), interpolation of E at the charges, near-field pair forces under
// full minimum image (se_bd.cu), F = q (far + near).
//
// B200 design: grid [nx][ny][nz] (z fastest, numpy's C order) so one cuFFT
// 3-D D2Z / Z2D pair does the transforms (half spectrum; the real part of the
// reference's full inverse equals the C2R result for Hermitian spectra); one
// kernel forms phi_hat and the three field spectra in a single pass over the
// half spectrum with the 1/(nx ny nz) normalisation folded in.  Spreading is
// one warp per charge, lanes along z (coalesced fp64 RED to L2); the
// interpolation is one warp per charge with a warp reduction, no atomics.
#include <cufft.h>

#include <algorithm>
#include <cmath>

#include <cstdlib>

#include "se_internal.cuh"

namespace se {

namespace {

constexpr int TP_MAXS = 64;           // stencil nodes per axis
constexpr int TP_WARPS = 4;
constexpr int TP_K = 8;               // (oy, oz) pairs per lane (Sy Sz <= 256)

struct TpGrid {
    int n[3]; double h[3];
    int m[3];                         // stencil half widths (gridops.py:20)
    double radius, keep, inv_width, inv_norm;
    int64_t stride;                   // field plane stride (even: cuFFT alignment)
};

// per-warp stencil tables: weights and wrapped indices per axis
struct TpStencil {
    double w[3][TP_MAXS];
    int idx[3][TP_MAXS];
};

// gridops.py:18-26 and 42-44 for the three axes of one point
__device__ __forceinline__ void tp_stencil(const TpGrid& g, const double* p, TpStencil& s,
                                           int lane) {
#pragma unroll
    for (int ax = 0; ax < 3; ++ax) {
        const int S = 2 * g.m[ax] + 1;
        const long long j0 = (long long)floor(p[ax] / g.h[ax]);
        for (int o = lane; o < S; o += 32) {
            const long long j = j0 + o - g.m[ax];
            const double d = __dsub_rn(p[ax], __dmul_rn((double)j, g.h[ax]));
            long long r = j % g.n[ax];
            if (r < 0) r += g.n[ax];
            s.idx[ax][o] = (int)r;
            s.w[ax][o] = fabs(d) <= g.keep ? gauss_w(d, g.inv_width, g.inv_norm) : 0.0;
        }
    }
}

__global__ void __launch_bounds__(TP_WARPS * 32) tp_spread_kernel(TpGrid g, const double* pos,
                                                                  const double* q, int64_t n,
                                                                  double* rho) {
    __shared__ TpStencil sst[TP_WARPS];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int64_t i = blockIdx.x * (int64_t)TP_WARPS + wib;
    if (i >= n) return;
    TpStencil& s = sst[wib];
    const double p[3] = {pos[3 * i], pos[3 * i + 1], pos[3 * i + 2]};
    tp_stencil(g, p, s, lane);
    __syncwarp();
    const double qi = q[i];
    const int Sx = 2 * g.m[0] + 1, Sy = 2 * g.m[1] + 1, Sz = 2 * g.m[2] + 1;
    if (Sy * Sz <= 32 * TP_K) {
        // each lane owns up to TP_K (oy, oz) pairs (z fastest: consecutive
        // addresses per column), reused for every x offset
        int off[TP_K]; double wy[TP_K], wz[TP_K];
#pragma unroll
        for (int k = 0; k < TP_K; ++k) {
            const int e = lane + 32 * k;
            off[k] = 0; wy[k] = 0.0; wz[k] = 0.0;
            if (e < Sy * Sz) {
                const int oy = e / Sz, oz = e - oy * Sz;
                off[k] = s.idx[1][oy] * g.n[2] + s.idx[2][oz];
                wy[k] = s.w[1][oy]; wz[k] = s.w[2][oz];
            }
        }
        for (int ox = 0; ox < Sx; ++ox) {
            const double qwx = qi * s.w[0][ox];
            if (qwx == 0.0) continue;
            double* plane = rho + (int64_t)s.idx[0][ox] * g.n[1] * g.n[2];
#pragma unroll
            for (int k = 0; k < TP_K; ++k) {
                const double w = (qwx * wy[k]) * wz[k];                   // q wx wy wz
                if (w != 0.0) atomicAdd(plane + off[k], w);
            }
        }
        return;
    }
    for (int e = lane; e < Sx * Sy * Sz; e += 32) {
        const int oz = e % Sz, c = e / Sz, oy = c % Sy, ox = c / Sy;
        const double w = ((qi * s.w[0][ox]) * s.w[1][oy]) * s.w[2][oz];   // q wx wy wz
        if (w != 0.0)
            atomicAdd(rho + ((int64_t)s.idx[0][ox] * g.n[1] + s.idx[1][oy]) * g.n[2] + s.idx[2][oz], w);
    }
}

// phi_hat = rho_hat / (eps k^2), phi_hat(0) = 0; E_hat = -i k phi_hat with
// the unmatched Nyquist derivative dropped                dpsolver.py:229-249
struct TpPoissonArgs {
    const cufftDoubleComplex* rho_hat; int nx, ny, nz, nzh;
    double Lx, Ly, Lz, eps, scale;
    double fval[3];                  // numpy fftfreq's 1 / (n d), d = 1 / n
    cufftDoubleComplex* phi_hat;     // may be null
    cufftDoubleComplex* e_hat;       // [3][half], may be null
};

__device__ __forceinline__ double tp_wavenumber(int i, int n, double val, double L) {
    const int f = (i <= (n - 1) / 2) ? i : i - n;                 // fftfreq
    return 2.0 * M_PI * ((double)f * val) / L;
}

__global__ void tp_poisson_kernel(TpPoissonArgs a) {
    const int64_t half = (int64_t)a.nx * a.ny * a.nzh;
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= half) return;
    const int iz = (int)(e % a.nzh);
    const int iy = (int)((e / a.nzh) % a.ny);
    const int ix = (int)(e / ((int64_t)a.nzh * a.ny));
    const double kx = tp_wavenumber(ix, a.nx, a.fval[0], a.Lx);
    const double ky = tp_wavenumber(iy, a.ny, a.fval[1], a.Ly);
    const double kz = tp_wavenumber(iz, a.nz, a.fval[2], a.Lz);
    double k2 = (kx * kx + ky * ky) + kz * kz;
    const bool zero = (e == 0);
    if (zero) k2 = 1.0;
    const double d = a.eps * k2;
    const cufftDoubleComplex r = a.rho_hat[e];
    const double pr = zero ? 0.0 : r.x / d, pi = zero ? 0.0 : r.y / d;
    if (a.phi_hat) a.phi_hat[e] = make_cuDoubleComplex(pr * a.scale, pi * a.scale);
    if (a.e_hat) {
        // the most negative wavenumber of an even axis is the Nyquist one
        const double kv[3] = {(a.nx % 2 == 0 && ix == a.nx / 2) ? 0.0 : kx,
                              (a.ny % 2 == 0 && iy == a.ny / 2) ? 0.0 : ky,
                              (a.nz % 2 == 0 && iz == a.nz / 2) ? 0.0 : kz};
#pragma unroll
        for (int c = 0; c < 3; ++c)
            a.e_hat[c * half + e] = make_cuDoubleComplex(kv[c] * pi * a.scale,
                                                         -kv[c] * pr * a.scale);
    }
}

__global__ void __launch_bounds__(TP_WARPS * 32) tp_interp_kernel(TpGrid g, const double* pos,
                                                                  int64_t n, const double* f,
                                                                  double cell,
                                                                  double* out) {
    __shared__ TpStencil sst[TP_WARPS];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int64_t i = blockIdx.x * (int64_t)TP_WARPS + wib;
    if (i >= n) return;
    TpStencil& s = sst[wib];
    const double p[3] = {pos[3 * i], pos[3 * i + 1], pos[3 * i + 2]};
    tp_stencil(g, p, s, lane);
    __syncwarp();
    const int Sx = 2 * g.m[0] + 1, Sy = 2 * g.m[1] + 1, Sz = 2 * g.m[2] + 1;
    const int64_t G = g.stride;
    double a0 = 0.0, a1 = 0.0, a2 = 0.0;
    if (Sy * Sz <= 32 * TP_K) {
        int off[TP_K]; double wy[TP_K], wz[TP_K];
#pragma unroll
        for (int k = 0; k < TP_K; ++k) {
            const int e = lane + 32 * k;
            off[k] = 0; wy[k] = 0.0; wz[k] = 0.0;
            if (e < Sy * Sz) {
                const int oy = e / Sz, oz = e - oy * Sz;
                off[k] = s.idx[1][oy] * g.n[2] + s.idx[2][oz];
                wy[k] = s.w[1][oy]; wz[k] = s.w[2][oz];
            }
        }
        for (int ox = 0; ox < Sx; ++ox) {
            const double wx = s.w[0][ox];
            if (wx == 0.0) continue;
            const double* plane = f + (int64_t)s.idx[0][ox] * g.n[1] * g.n[2];
#pragma unroll
            for (int k = 0; k < TP_K; ++k) {
                const double w = (wx * wy[k]) * wz[k];                    // wx wy wz
                if (w != 0.0) {
                    a0 = fma(w, __ldg(plane + off[k]), a0);
                    a1 = fma(w, __ldg(plane + G + off[k]), a1);
                    a2 = fma(w, __ldg(plane + 2 * G + off[k]), a2);
                }
            }
        }
    } else
    for (int e = lane; e < Sx * Sy * Sz; e += 32) {
        const int oz = e % Sz, c = e / Sz, oy = c % Sy, ox = c / Sy;
        const double w = (s.w[0][ox] * s.w[1][oy]) * s.w[2][oz];         // wx wy wz
        if (w == 0.0) continue;
        const int64_t at = ((int64_t)s.idx[0][ox] * g.n[1] + s.idx[1][oy]) * g.n[2] + s.idx[2][oz];
        a0 = fma(w, __ldg(f + at), a0);
        a1 = fma(w, __ldg(f + G + at), a1);
        a2 = fma(w, __ldg(f + 2 * G + at), a2);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        a0 += __shfl_xor_sync(0xffffffffu, a0, o);
        a1 += __shfl_xor_sync(0xffffffffu, a1, o);
        a2 += __shfl_xor_sync(0xffffffffu, a2, o);
    }
    if (lane == 0) {
        out[i] = cell * a0;
        out[n + i] = cell * a1;
        out[2 * n + i] = cell * a2;
    }
}

// F = q (far + near)                                           bd.py:330
__global__ void tp_combine_kernel(const double* q, const double* far, const double* nearf,
                                  int64_t n, double* forces) {
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= 3 * n) return;
    const int64_t i = e / 3;
    const int c = (int)(e - 3 * i);
    forces[e] = q[i] * (far[c * n + i] + nearf[e]);
}

}  // namespace

struct TpPlan {
    int dev = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = true;
    int n[3]{}; double L[3]{}, h[3]{}, eps = 1.0;
    int64_t G = 0, Gs = 0, half = 0;   // grid size, plane stride (even), half spectrum
    cufftHandle fwd = 0, inv = 0;
    double* d_grid = nullptr;                  // [4][G]: rho / phi, Ex, Ey, Ez
    cufftDoubleComplex* d_hat = nullptr;       // [5][half]: rho_hat, phi_hat, E_hat x3
    int64_t cap = 0;
    double* d_pts = nullptr;                   // pos[3cap] q[cap] far[3cap] near[3cap] F[3cap]
    PairScratch pairs;                         // near-field cell list
    // CUDA graph of tp_forces_device (se_tp_set_graph): captured on the
    // second call with the same buffers and parameters, replayed after
    bool graph = false;
    cudaGraphExec_t gexec = nullptr;
    cudaStream_t cap_stream = nullptr;
    // the near field forked onto `side` next to the grid part (SE_TP_FORK)
    cudaStream_t side = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    struct Key {
        const void *pos = nullptr, *q = nullptr, *out = nullptr;
        int64_t n = -1; double g_t = 0, radius = 0, g_w = 0, xi = 0, r_cut = 0;
        bool operator==(const Key& o) const {
            return pos == o.pos && q == o.q && out == o.out && n == o.n && g_t == o.g_t &&
                   radius == o.radius && g_w == o.g_w && xi == o.xi && r_cut == o.r_cut;
        }
    } gkey, gwarm;
    ~TpPlan() {
        if (dev >= 0) cudaSetDevice(dev);
        if (gexec) cudaGraphExecDestroy(gexec);
        if (cap_stream) cudaStreamDestroy(cap_stream);
        if (side) cudaStreamDestroy(side);
        if (ev_fork) cudaEventDestroy(ev_fork);
        if (ev_join) cudaEventDestroy(ev_join);
        pairs.release();
        if (fwd) cufftDestroy(fwd);
        if (inv) cufftDestroy(inv);
        cudaFree(d_grid); cudaFree(d_hat); cudaFree(d_pts);
        if (own_stream && stream) cudaStreamDestroy(stream);
    }
};

TpPlan* tp_create(int device, const double L[3], const int n[3], double eps) {
    for (int ax = 0; ax < 3; ++ax) {
        if (n[ax] < 1) throw Error(SE_ERR_VALUE, "grid sizes must be positive");
        if (!(L[ax] > 0)) throw Error(SE_ERR_VALUE, "box lengths must be positive");
    }
    SE_CUDA(cudaSetDevice(device));
    TpPlan* p = new TpPlan();
    try {
        p->dev = device;
        p->eps = eps;
        for (int ax = 0; ax < 3; ++ax) { p->n[ax] = n[ax]; p->L[ax] = L[ax]; p->h[ax] = L[ax] / n[ax]; }
        p->G = (int64_t)n[0] * n[1] * n[2];
        p->Gs = (p->G + 1) & ~(int64_t)1;   // cuFFT wants 16-byte aligned real planes
        p->half = (int64_t)n[0] * n[1] * (n[2] / 2 + 1);
        SE_CUDA(cudaStreamCreateWithFlags(&p->stream, cudaStreamNonBlocking));
        SE_CUDA(cudaMalloc(&p->d_grid, 4 * p->Gs * sizeof(double)));
        SE_CUDA(cudaMalloc(&p->d_hat, 5 * p->half * sizeof(cufftDoubleComplex)));
        SE_CUFFT(cufftPlan3d(&p->fwd, n[0], n[1], n[2], CUFFT_D2Z));
        SE_CUFFT(cufftPlan3d(&p->inv, n[0], n[1], n[2], CUFFT_Z2D));
        SE_CUFFT(cufftSetStream(p->fwd, p->stream));
        SE_CUFFT(cufftSetStream(p->inv, p->stream));
    } catch (...) {
        delete p;
        throw;
    }
    return p;
}

void tp_destroy(TpPlan* p) { delete p; }

void tp_set_stream(TpPlan* p, cudaStream_t s) {
    SE_CUDA(cudaSetDevice(p->dev));
    if (p->own_stream && p->stream) cudaStreamDestroy(p->stream);
    p->stream = s;
    p->own_stream = false;
    SE_CUFFT(cufftSetStream(p->fwd, s));
    SE_CUFFT(cufftSetStream(p->inv, s));
}

// spectral solve of the grid in d_grid[0]; phi into d_grid[0] when asked,
// the field components into d_grid[1..3]                 dpsolver.py:221-249
static void tp_solve_grid(TpPlan* p, bool want_phi, bool want_field) {
    cufftDoubleComplex* rho_hat = p->d_hat;
    cufftDoubleComplex* phi_hat = p->d_hat + p->half;
    cufftDoubleComplex* e_hat = p->d_hat + 2 * p->half;
    SE_CUFFT(cufftExecD2Z(p->fwd, p->d_grid, rho_hat));
    TpPoissonArgs a{};
    a.rho_hat = rho_hat; a.nx = p->n[0]; a.ny = p->n[1]; a.nz = p->n[2]; a.nzh = p->n[2] / 2 + 1;
    a.Lx = p->L[0]; a.Ly = p->L[1]; a.Lz = p->L[2]; a.eps = p->eps;
    a.scale = 1.0 / (double)p->G;
    for (int ax = 0; ax < 3; ++ax) a.fval[ax] = 1.0 / (p->n[ax] * (1.0 / p->n[ax]));
    a.phi_hat = want_phi ? phi_hat : nullptr;
    a.e_hat = want_field ? e_hat : nullptr;
    tp_poisson_kernel<<<(unsigned)((p->half + 255) / 256), 256, 0, p->stream>>>(a);
    SE_CUDA(cudaGetLastError());
    if (want_phi) SE_CUFFT(cufftExecZ2D(p->inv, phi_hat, p->d_grid));
    if (want_field)
        for (int c = 0; c < 3; ++c)
            SE_CUFFT(cufftExecZ2D(p->inv, e_hat + c * p->half, p->d_grid + (1 + c) * p->Gs));
}

void tp_poisson(TpPlan* p, const double* rho, int with_field, double* phi, double* E) {
    SE_CUDA(cudaSetDevice(p->dev));
    SE_CUDA(cudaMemcpyAsync(p->d_grid, rho, p->G * sizeof(double), cudaMemcpyHostToDevice, p->stream));
    tp_solve_grid(p, true, with_field != 0);
    SE_CUDA(cudaMemcpyAsync(phi, p->d_grid, p->G * sizeof(double), cudaMemcpyDeviceToHost, p->stream));
    if (with_field && E)
        for (int c = 0; c < 3; ++c)
            SE_CUDA(cudaMemcpyAsync(E + c * p->G, p->d_grid + (1 + c) * p->Gs,
                                    p->G * sizeof(double), cudaMemcpyDeviceToHost, p->stream));
    SE_CUDA(cudaStreamSynchronize(p->stream));
}

static TpGrid tp_grid(const TpPlan* p, double width, double radius) {
    TpGrid g{};
    for (int ax = 0; ax < 3; ++ax) {
        g.n[ax] = p->n[ax];
        g.h[ax] = p->h[ax];
        g.m[ax] = (int)std::floor(radius / p->h[ax] + 1e-12);
        if (2 * g.m[ax] + 1 > TP_MAXS) throw Error(SE_ERR_VALUE, "stencil too wide for the periodic grid");
    }
    g.stride = p->Gs;
    g.radius = radius;
    g.keep = radius + 1e-12 * radius;
    g.inv_width = 1.0 / width;
    g.inv_norm = 1.0 / std::sqrt(2.0 * M_PI * (width * width));
    return g;
}

// plan scratch for n points: pos[3n] q[n] far[3n] near[3n] forces[3n]
static void tp_reserve(TpPlan* p, int64_t n) {
    if (n <= p->cap) return;
    cudaFree(p->d_pts);
    p->d_pts = nullptr;
    p->cap = 0;
    SE_CUDA(cudaMalloc(&p->d_pts, 13 * (size_t)n * sizeof(double)));
    p->cap = n;
}

static void tp_forces_eager(TpPlan* p, const double* d_pos, const double* d_q, int64_t n,
                            double g_t, double radius, double g_w, double xi, double r_cut,
                            double* d_forces);

void tp_set_graph(TpPlan* p, bool enable) {
    p->graph = enable;
    if (!enable && p->gexec) { cudaGraphExecDestroy(p->gexec); p->gexec = nullptr; }
    p->gkey = TpPlan::Key{};
    p->gwarm = TpPlan::Key{};
}

void tp_forces_device(TpPlan* p, const double* d_pos, const double* d_q, int64_t n, double g_t,
                      double radius, double g_w, double xi, double r_cut, double* d_forces) {
    SE_CUDA(cudaSetDevice(p->dev));
    if (!p->graph) {
        tp_forces_eager(p, d_pos, d_q, n, g_t, radius, g_w, xi, r_cut, d_forces);
        return;
    }
    TpPlan::Key key;
    key.pos = d_pos; key.q = d_q; key.out = d_forces; key.n = n;
    key.g_t = g_t; key.radius = radius; key.g_w = g_w; key.xi = xi; key.r_cut = r_cut;
    if (p->gexec && p->gkey == key) {
        SE_CUDA(cudaGraphLaunch(p->gexec, p->stream));
        return;
    }
    if (!(p->gwarm == key)) {                       // first call: eager, sizes every buffer
        tp_forces_eager(p, d_pos, d_q, n, g_t, radius, g_w, xi, r_cut, d_forces);
        p->gwarm = key;
        return;
    }
    // capture on a private stream (the caller's may be the legacy stream)
    if (p->gexec) { cudaGraphExecDestroy(p->gexec); p->gexec = nullptr; }
    if (!p->cap_stream) SE_CUDA(cudaStreamCreateWithFlags(&p->cap_stream, cudaStreamNonBlocking));
    const cudaStream_t run = p->stream;
    SE_CUDA(cudaStreamSynchronize(run));
    auto bind = [&](cudaStream_t st) {
        p->stream = st;
        cufftSetStream(p->fwd, st);
        cufftSetStream(p->inv, st);
    };
    bind(p->cap_stream);
    cudaGraph_t gr = nullptr;
    cudaError_t ce = cudaStreamBeginCapture(p->cap_stream, cudaStreamCaptureModeThreadLocal);
    if (ce != cudaSuccess) { bind(run); SE_CUDA(ce); }
    try {
        tp_forces_eager(p, d_pos, d_q, n, g_t, radius, g_w, xi, r_cut, d_forces);
    } catch (...) {
        cudaStreamEndCapture(p->cap_stream, &gr);
        if (gr) cudaGraphDestroy(gr);
        cudaGetLastError();
        bind(run);
        p->gwarm = TpPlan::Key{};
        throw;
    }
    ce = cudaStreamEndCapture(p->cap_stream, &gr);
    bind(run);
    SE_CUDA(ce);
    const cudaError_t ie = cudaGraphInstantiate(&p->gexec, gr, 0);
    cudaGraphDestroy(gr);
    SE_CUDA(ie);
    p->gkey = key;
    SE_CUDA(cudaGraphLaunch(p->gexec, p->stream));
}

static void tp_forces_eager(TpPlan* p, const double* d_pos, const double* d_q, int64_t n,
                            double g_t, double radius, double g_w, double xi, double r_cut,
                            double* d_forces) {
    tp_reserve(p, n);
    double* d_far = p->d_pts + 4 * p->cap;
    double* d_near = d_far + 3 * p->cap;
    const TpGrid g = tp_grid(p, g_t, radius);
    static const bool fork = [] {
        const char* e = std::getenv("SE_TP_FORK");
        return e ? std::atoi(e) != 0 : true;
    }();
    // the near field (pairs -> d_near) and the grid part (-> d_far) share
    // only the inputs: the pair pass runs on a high-priority side stream
    // next to the spread / FFTs / interpolation and joins before the sum
    const bool forked = fork && n > 0;
    if (forked) {
        if (!p->side) {
            int lo = 0, hi = 0;
            SE_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
            SE_CUDA(cudaStreamCreateWithPriority(&p->side, cudaStreamNonBlocking, hi));
            SE_CUDA(cudaEventCreateWithFlags(&p->ev_fork, cudaEventDisableTiming));
            SE_CUDA(cudaEventCreateWithFlags(&p->ev_join, cudaEventDisableTiming));
        }
        SE_CUDA(cudaEventRecord(p->ev_fork, p->stream));
        SE_CUDA(cudaStreamWaitEvent(p->side, p->ev_fork, 0));
        tp_near_forces(d_pos, d_q, n, p->L, r_cut, g_w, xi, p->eps, d_near, p->side, p->pairs);
        SE_CUDA(cudaEventRecord(p->ev_join, p->side));
    }
    SE_CUDA(cudaMemsetAsync(p->d_grid, 0, p->G * sizeof(double), p->stream));
    const unsigned nb = (unsigned)((n + TP_WARPS - 1) / TP_WARPS);
    if (n > 0) {
        tp_spread_kernel<<<nb, TP_WARPS * 32, 0, p->stream>>>(g, d_pos, d_q, n, p->d_grid);
        SE_CUDA(cudaGetLastError());
    }
    tp_solve_grid(p, false, true);
    if (n == 0) return;
    tp_interp_kernel<<<nb, TP_WARPS * 32, 0, p->stream>>>(g, d_pos, n, p->d_grid + p->Gs,
                                                          p->h[0] * p->h[1] * p->h[2], d_far);
    SE_CUDA(cudaGetLastError());
    if (forked) SE_CUDA(cudaStreamWaitEvent(p->stream, p->ev_join, 0));
    else tp_near_forces(d_pos, d_q, n, p->L, r_cut, g_w, xi, p->eps, d_near, p->stream, p->pairs);
    tp_combine_kernel<<<(unsigned)((3 * n + 255) / 256), 256, 0, p->stream>>>(d_q, d_far, d_near,
                                                                            n, d_forces);
    SE_CUDA(cudaGetLastError());
}

void tp_forces(TpPlan* p, const double* pos, const double* q, int64_t n, double g_t,
               double radius, double g_w, double xi, double r_cut, double* forces) {
    SE_CUDA(cudaSetDevice(p->dev));
    tp_reserve(p, n);
    double* d_pos = p->d_pts;
    double* d_q = d_pos + 3 * p->cap;
    double* d_f = p->d_pts + 10 * p->cap;
    if (n > 0) {
        SE_CUDA(cudaMemcpyAsync(d_pos, pos, 3 * n * sizeof(double), cudaMemcpyHostToDevice, p->stream));
        SE_CUDA(cudaMemcpyAsync(d_q, q, n * sizeof(double), cudaMemcpyHostToDevice, p->stream));
    }
    tp_forces_device(p, d_pos, d_q, n, g_t, radius, g_w, xi, r_cut, d_f);
    if (n > 0)
        SE_CUDA(cudaMemcpyAsync(forces, d_f, 3 * n * sizeof(double), cudaMemcpyDeviceToHost, p->stream));
    SE_CUDA(cudaStreamSynchronize(p->stream));
}

}  // namespace se
