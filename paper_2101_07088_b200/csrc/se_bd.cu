// Brownian-dynamics steric forces.
//
// Reference: steric_pair_forces / steric_force / lj_force (bd.py:46-63,
// 246-270): truncated, mollified Lennard-Jones repulsion between all pairs
// within the cutoff 2^(1/p) 2a, minimum image in x and y (periodic), open z;
// the reference sums the pair forces with np.bincount over a KD-tree pair
// list, here every particle gathers its own sum (same terms, its own order).
//
// B200 design: particles binned in cells >= the cutoff (x mod Lx, y mod Ly,
// z from the data), sorted by cell (cub), one thread per particle walking the
// 27 neighbour cells (all cells along an axis with fewer than 3), exact
// reference arithmetic for d, r and the force.
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <vector>

#include "se_internal.cuh"

namespace se {

namespace {

struct StericArgs {
    const double* pos; int64_t n;
    double Lx, Ly, zlo, csx, csy, csz; int ncx, ncy, ncz;
    double a, U0, r_m, cutoff; int p;
    const int* start; const int* order;
    double* out;
};

__device__ __forceinline__ int steric_cell(const StericArgs& s, double x, double y, double z,
                                           int* cx, int* cy, int* cz) {
    double wx = x - s.Lx * floor(x / s.Lx); if (wx >= s.Lx) wx = 0.0;
    double wy = y - s.Ly * floor(y / s.Ly); if (wy >= s.Ly) wy = 0.0;
    int ix = min(s.ncx - 1, (int)(wx / s.csx));
    int iy = min(s.ncy - 1, (int)(wy / s.csy));
    double fz = floor((z - s.zlo) / s.csz);
    int iz = fz < 0 ? 0 : (fz >= s.ncz ? s.ncz - 1 : (int)fz);
    *cx = ix; *cy = iy; *cz = iz;
    return (iz * s.ncy + iy) * s.ncx + ix;
}

__global__ void steric_keys_kernel(StericArgs s, uint32_t* keys, int* perm) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= s.n) return;
    int cx, cy, cz;
    keys[i] = (uint32_t)steric_cell(s, s.pos[3 * i], s.pos[3 * i + 1], s.pos[3 * i + 2],
                                    &cx, &cy, &cz);
    perm[i] = (int)i;
}

__global__ void steric_starts_kernel(const uint32_t* keys, int64_t n, int ncell, int* start) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i > n) return;
    const int cur = (i < n) ? (int)keys[i] : ncell;
    const int prev = (i == 0) ? -1 : (int)keys[i - 1];
    for (int c = prev + 1; c <= cur; ++c) start[c] = (int)i;
}

// the reference's lj_force (bd.py:46-49) and steric_force (bd.py:52-57)
__device__ __forceinline__ double steric_f(const StericArgs& s, double r) {
    if (r > s.cutoff) return 0.0;
    const double rs = s.r_m > 0 ? fmax(r, s.r_m) : fmax(r, 1e-12 * s.a);
    const double x = pow(2.0 * s.a / rs, (double)s.p);
    return 4.0 * s.U0 * s.p * x * (2.0 * x - 1.0) / rs;
}

__global__ void steric_force_kernel(StericArgs s) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= s.n) return;
    const double px = s.pos[3 * i], py = s.pos[3 * i + 1], pz = s.pos[3 * i + 2];
    int cx, cy, cz;
    steric_cell(s, px, py, pz, &cx, &cy, &cz);
    const bool allx = s.ncx < 3, ally = s.ncy < 3;
    const int nxr = allx ? s.ncx : 3, nyr = ally ? s.ncy : 3;
    double fx = 0.0, fy = 0.0, fz = 0.0;
    for (int dzc = -1; dzc <= 1; ++dzc) {
        const int zc = cz + dzc;
        if (zc < 0 || zc >= s.ncz) continue;
        for (int iy = 0; iy < nyr; ++iy) {
            int yc = ally ? iy : cy + iy - 1;
            if (yc < 0) yc += s.ncy; else if (yc >= s.ncy) yc -= s.ncy;
            for (int ix = 0; ix < nxr; ++ix) {
                int xc = allx ? ix : cx + ix - 1;
                if (xc < 0) xc += s.ncx; else if (xc >= s.ncx) xc -= s.ncx;
                const int c = (zc * s.ncy + yc) * s.ncx + xc;
                for (int q = s.start[c]; q < s.start[c + 1]; ++q) {
                    const int j = s.order[q];
                    if (j == i) continue;
                    // d = p_i - p_j; d_xy -= L round(d_xy / L)   (bd.py:263-265)
                    double dx = __dsub_rn(px, s.pos[3 * j]);
                    double dy = __dsub_rn(py, s.pos[3 * j + 1]);
                    const double dz = __dsub_rn(pz, s.pos[3 * j + 2]);
                    dx = __dsub_rn(dx, __dmul_rn(s.Lx, rint(dx / s.Lx)));
                    dy = __dsub_rn(dy, __dmul_rn(s.Ly, rint(dy / s.Ly)));
                    const double r = sqrt(__dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)),
                                                    __dmul_rn(dz, dz)));
                    if (r > s.cutoff) continue;
                    const double f = steric_f(s, r) / (r > 0 ? r : 1.0);
                    fx += f * dx; fy += f * dy; fz += f * dz;
                }
            }
        }
    }
    s.out[3 * i] = fx; s.out[3 * i + 1] = fy; s.out[3 * i + 2] = fz;
}

}  // namespace

void steric_forces(int device, const double* pos, int64_t n, double Lx, double Ly, double a,
                   double U0, double r_m, int p, double* out) {
    SE_CUDA(cudaSetDevice(device));
    std::fill(out, out + 3 * n, 0.0);
    if (n < 2) return;
    if (!(a > 0) || p < 1) throw Error(SE_ERR_VALUE, "steric parameters: a > 0, p >= 1");
    const double cutoff = std::pow(2.0, 1.0 / p) * 2.0 * a;
    double zmin = 1e300, zmax = -1e300;
    for (int64_t i = 0; i < n; ++i) { zmin = std::min(zmin, pos[3 * i + 2]); zmax = std::max(zmax, pos[3 * i + 2]); }
    StericArgs s{};
    s.n = n; s.Lx = Lx; s.Ly = Ly;
    s.ncx = std::max(1, (int)std::floor(Lx / cutoff));
    s.ncy = std::max(1, (int)std::floor(Ly / cutoff));
    s.csx = Lx / s.ncx; s.csy = Ly / s.ncy;
    s.zlo = zmin - cutoff;
    const double zspan = (zmax + cutoff) - s.zlo;
    s.ncz = std::max(1, (int)std::floor(zspan / cutoff));
    s.csz = zspan / s.ncz;
    const int64_t ncell = (int64_t)s.ncx * s.ncy * s.ncz;
    if (ncell > (1 << 28)) throw Error(SE_ERR_VALUE, "steric cell grid too large");
    s.a = a; s.U0 = U0; s.r_m = r_m; s.p = p; s.cutoff = cutoff;
    cudaStream_t st;
    SE_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    struct Guard {
        std::vector<void*> v; cudaStream_t s;
        ~Guard() { for (void* x : v) cudaFree(x); cudaStreamDestroy(s); }
    } g{{}, st};
    auto alloc = [&](size_t bytes) { void* ptr = nullptr; SE_CUDA(cudaMalloc(&ptr, bytes)); g.v.push_back(ptr); return ptr; };
    double* d_pos = (double*)alloc(3 * n * sizeof(double));
    double* d_out = (double*)alloc(3 * n * sizeof(double));
    uint32_t* k1 = (uint32_t*)alloc(n * sizeof(uint32_t));
    uint32_t* k2 = (uint32_t*)alloc(n * sizeof(uint32_t));
    int* p1 = (int*)alloc(n * sizeof(int));
    int* p2 = (int*)alloc(n * sizeof(int));
    int* start = (int*)alloc((ncell + 1) * sizeof(int));
    SE_CUDA(cudaMemcpyAsync(d_pos, pos, 3 * n * sizeof(double), cudaMemcpyHostToDevice, st));
    s.pos = d_pos; s.out = d_out;
    const unsigned nb = (unsigned)((n + 255) / 256);
    steric_keys_kernel<<<nb, 256, 0, st>>>(s, k1, p1);
    SE_CUDA(cudaGetLastError());
    int end_bit = 1;
    while (end_bit < 32 && ((uint64_t)ncell >> end_bit) != 0) ++end_bit;
    size_t bytes = 0;
    SE_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, k1, k2, p1, p2, (int)n, 0, end_bit, st));
    void* tmp = alloc(std::max<size_t>(bytes, 16));
    SE_CUDA(cub::DeviceRadixSort::SortPairs(tmp, bytes, k1, k2, p1, p2, (int)n, 0, end_bit, st));
    steric_starts_kernel<<<(unsigned)((n + 1 + 255) / 256), 256, 0, st>>>(k2, n, (int)ncell, start);
    SE_CUDA(cudaGetLastError());
    s.start = start; s.order = p2;
    steric_force_kernel<<<nb, 256, 0, st>>>(s);
    SE_CUDA(cudaGetLastError());
    SE_CUDA(cudaMemcpyAsync(out, d_out, 3 * n * sizeof(double), cudaMemcpyDeviceToHost, st));
    SE_CUDA(cudaStreamSynchronize(st));
}

}  // namespace se
