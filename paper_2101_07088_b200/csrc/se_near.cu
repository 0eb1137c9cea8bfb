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

#include "se_internal.cuh"

namespace se {

namespace {

constexpr double TWO_OVER_SQRTPI = 1.1283791670955126;   // 2/sqrt(pi)
constexpr int QN = 16;                                    // per-thread queue

__device__ __forceinline__ int pmod_i(int a, int n) { int r = a % n; return r < 0 ? r + n : r; }

// erf(r/c)/r and its r-derivative for one width c       kernels.py:38-72
struct ErfPair { double v, d; };

__device__ __forceinline__ ErfPair erf_terms(double r, double c, double inv_c,
                                             bool need_d) {
    ErfPair o;
    if (r < 1e-10 * c) o.v = TWO_OVER_SQRTPI / c;
    else o.v = erf(r / c) / r;
    o.d = 0.0;
    if (need_d) {
        if (r < 1e-2 * c) {
            double x = r / c, u = x * x;
            o.d = TWO_OVER_SQRTPI / (c * c) * x *
                  (-2.0 / 3.0 + u * (2.0 / 5.0 + u * (-1.0 / 7.0 + u / 27.0)));
        } else {
            double x = r / c;
            o.d = TWO_OVER_SQRTPI * exp(-x * x) / (c * r) - erf(x) / (r * r);
        }
    }
    (void)inv_c;
    return o;
}

// ---------------------------------------------------------------------------
// cell list
// ---------------------------------------------------------------------------
struct CellGeo {
    int ncx, ncy, ncz;
    double csx, csy, csz, zlo, Lx, Ly;
};

__device__ __forceinline__ double wrap(double x, double L) {
    double w = x - L * floor(x / L);
    return (w >= L) ? 0.0 : w;
}

__device__ __forceinline__ int cell_of(const CellGeo& g, double x, double y, double z,
                                       int* cx, int* cy, int* cz) {
    int ix = (int)(wrap(x, g.Lx) / g.csx); if (ix >= g.ncx) ix = g.ncx - 1;
    int iy = (int)(wrap(y, g.Ly) / g.csy); if (iy >= g.ncy) iy = g.ncy - 1;
    double fz = floor((z - g.zlo) / g.csz);
    int iz = fz < 0 ? 0 : (fz >= g.ncz ? g.ncz - 1 : (int)fz);
    *cx = ix; *cy = iy; *cz = iz;
    return (iz * g.ncy + iy) * g.ncx + ix;
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
                                 int* start, double4* src, float4* srcf, int* orig) {
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
                          (float)(v.z - g.zlo), 0.f);
    orig[i] = s;
}

// ---------------------------------------------------------------------------
// pair evaluation
// ---------------------------------------------------------------------------
struct NearArgs {
    const double* eval; const int* order; int64_t ne;
    CellGeo g; const int* start; const double4* src; const float4* srcf;
    double radius, c1, c2, inv4pie, self_value, point0;
    int kind, need_field;
    float r2f;                    // fp32 pre-test bound (with margin)
    float Lxf, Lyf, iLxf, iLyf;
    double* out; int64_t out_stride;   // out[c * stride + i]
    int64_t* npairs;
};

__device__ __forceinline__ void pair_terms(const NearArgs& a, double r,
                                           double& g, double& coef) {
    if (r == 0.0) {                              // slab.py:161-171,176
        g = (a.kind == 0) ? a.self_value : a.point0;
        coef = 0.0;
        return;
    }
    ErfPair t1 = erf_terms(r, a.c1, 0.0, a.need_field);
    ErfPair t2 = erf_terms(r, a.c2, 0.0, a.need_field);
    g = (t1.v - t2.v) * a.inv4pie;
    coef = a.need_field ? -((t1.d - t2.d) * a.inv4pie) / r : 0.0;
}

__global__ void __launch_bounds__(128) near_kernel(NearArgs a) {
    int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    bool live = t < a.ne;
    int64_t i = live ? (a.order ? a.order[t] : t) : 0;
    double px = 0, py = 0, pz = 0;
    if (live) { px = a.eval[3 * i]; py = a.eval[3 * i + 1]; pz = a.eval[3 * i + 2]; }
    int cx = 0, cy = 0, cz = 0;
    cell_of(a.g, px, py, pz, &cx, &cy, &cz);
    const float pxf = (float)wrap(px, a.g.Lx), pyf = (float)wrap(py, a.g.Ly);
    const float pzf = (float)(pz - a.g.zlo);
    const double Lx = a.g.Lx, Ly = a.g.Ly;

    double phi = 0, ex = 0, ey = 0, ez = 0;
    int64_t count = 0;
    int queue[QN];
    int qn = 0;

    auto drain = [&]() {
        for (int e = 0; e < qn; ++e) {
            double4 s = a.src[queue[e]];
            double dx = __dsub_rn(px, s.x), dy = __dsub_rn(py, s.y), dz = __dsub_rn(pz, s.z);
            dx = __dsub_rn(dx, __dmul_rn(Lx, rint(dx / Lx)));
            dy = __dsub_rn(dy, __dmul_rn(Ly, rint(dy / Ly)));
            double r = sqrt(__dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)),
                                      __dmul_rn(dz, dz)));
            double g, coef;
            pair_terms(a, r, g, coef);
            phi += s.w * g;
            if (a.need_field) {
                double cq = coef * s.w;
                ex += cq * dx; ey += cq * dy; ez += cq * dz;
            }
        }
        count += qn;
        qn = 0;
    };

    const int xs = (a.g.ncx >= 3) ? -1 : 0, xe = (a.g.ncx >= 3) ? 1 : a.g.ncx - 1;
    const int ys = (a.g.ncy >= 3) ? -1 : 0, ye = (a.g.ncy >= 3) ? 1 : a.g.ncy - 1;
    for (int dzc = -1; dzc <= 1; ++dzc) {
        int zc = cz + dzc;
        if (zc < 0 || zc >= a.g.ncz) continue;
        for (int dyc = ys; dyc <= ye; ++dyc) {
            int yc = (a.g.ncy >= 3) ? pmod_i(cy + dyc, a.g.ncy) : dyc;
            for (int dxc = xs; dxc <= xe; ++dxc) {
                int xc = (a.g.ncx >= 3) ? pmod_i(cx + dxc, a.g.ncx) : dxc;
                int c = (zc * a.g.ncy + yc) * a.g.ncx + xc;
                int b = a.start[c], e = a.start[c + 1];
                for (int j = b; j < e; ++j) {
                    bool hit = false;
                    if (live) {
                        float4 f = a.srcf[j];
                        float dx = pxf - f.x, dy = pyf - f.y, dz = pzf - f.z;
                        dx -= a.Lxf * rintf(dx * a.iLxf);
                        dy -= a.Lyf * rintf(dy * a.iLyf);
                        float r2 = dx * dx + dy * dy + dz * dz;
                        if (r2 <= a.r2f) {
                            double4 s = a.src[j];
                            double ddx = __dsub_rn(px, s.x), ddy = __dsub_rn(py, s.y);
                            double ddz = __dsub_rn(pz, s.z);
                            ddx = __dsub_rn(ddx, __dmul_rn(Lx, rint(ddx / Lx)));
                            ddy = __dsub_rn(ddy, __dmul_rn(Ly, rint(ddy / Ly)));
                            double r = sqrt(__dadd_rn(__dadd_rn(__dmul_rn(ddx, ddx),
                                                                __dmul_rn(ddy, ddy)),
                                                      __dmul_rn(ddz, ddz)));
                            hit = r <= a.radius;
                        }
                    }
                    if (hit) queue[qn++] = j;
                    if (__any_sync(__activemask(), qn == QN)) drain();
                }
            }
        }
    }
    drain();
    if (live) {
        a.out[i] = phi;
        if (a.need_field) {
            a.out[a.out_stride + i] = ex;
            a.out[2 * a.out_stride + i] = ey;
            a.out[3 * a.out_stride + i] = ez;
        }
    }
    // pair count (diagnostic)
    unsigned long long c = live ? (unsigned long long)count : 0ull;
    for (int off = 16; off > 0; off >>= 1) c += __shfl_xor_sync(__activemask(), c, off);
    if ((threadIdx.x & 31) == 0 && a.npairs) atomicAdd((unsigned long long*)a.npairs, c);
}

// ---------------------------------------------------------------------------
// final combination and energy                          slab.py:359-391
// ---------------------------------------------------------------------------
struct FinArgs {
    const double* far; const double* near; const double* q; int64_t n;
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
        double phi_near = a.near[i];
        if (a.self_inf) phi_near = phi_near + a.q[i] * a.self_inf_value;
        double phi = (a.cell * a.far[i] + phi_near) + b_i;
        a.phi[i] = phi;
        if (a.forces) {
            a.E[3 * i] = -(a.cell * a.far[a.n + i]) + a.near[a.n + i];
            a.E[3 * i + 1] = -(a.cell * a.far[2 * a.n + i]) + a.near[2 * a.n + i];
            a.E[3 * i + 2] = -(a.cell * a.far[3 * a.n + i]) + a.near[3 * a.n + i];
        }
        acc += a.q[i] * phi;
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
static CellGeo cell_geo(const Plan* p) {
    CellGeo g;
    g.ncx = p->cl.ncx; g.ncy = p->cl.ncy; g.ncz = p->cl.ncz;
    g.csx = p->cl.csx; g.csy = p->cl.csy; g.csz = p->cl.csz; g.zlo = p->cl.zlo;
    g.Lx = p->P.Lx; g.Ly = p->P.Ly;
    return g;
}

void build_cells(Plan* p, const double* d_pos, const double* d_q, int64_t n) {
    const double eps = p->P.eps;
    const double fb = -(p->P.eps_b - eps) / (p->P.eps_b + eps);
    const double ft = -(p->P.eps_t - eps) / (p->P.eps_t + eps);
    const int nb = fb != 0.0, nt = ft != 0.0;
    const int64_t ns = n * (1 + nb + nt);
    CellList& cl = p->cl;
    if (ns > p->cl_cap) {
        void* olds[] = {cl.src, cl.srcf, cl.orig, p->d_ckeys, p->d_ckeys2,
                        p->d_cperm, p->d_cperm2, p->d_near_src, p->d_near_cub,
                        p->d_tgt, p->d_tkeys, p->d_tkeys2, p->d_tperm};
        for (void* o : olds) dfree(p, o);
        int64_t cap = ns < 64 ? 64 : ns;
        cl.src = dalloc<double4>(p, cap);
        cl.srcf = dalloc<float4>(p, cap);
        cl.orig = dalloc<int>(p, cap);
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
        p->cl_cap = ns;
    }
    cl.n = ns;
    if (ns == 0) return;
    SrcBuild sb{d_pos, d_q, n, p->P.H, fb, ft, nb, nt, p->d_near_src, ns};
    make_near_sources<<<(unsigned)((n + 255) / 256), 256, 0, p->stream>>>(sb);
    SE_LAUNCHED(p);
    // z extent of the sources (one small device->host read)
    int nblk = 64;
    if (!p->d_mm) p->d_mm = dalloc<double>(p, 256);
    zrange_kernel<<<nblk, 256, 0, p->stream>>>(p->d_near_src, ns, p->d_mm);
    SE_LAUNCHED(p);
    std::vector<double> mm(2 * nblk);
    SE_CUDA(cudaMemcpyAsync(mm.data(), p->d_mm, sizeof(double) * 2 * nblk,
                            cudaMemcpyDeviceToHost, p->stream));
    SE_CUDA(cudaStreamSynchronize(p->stream));
    double zmin = 1e300, zmax = -1e300;
    for (int b = 0; b < nblk; ++b) { zmin = std::min(zmin, mm[2 * b]); zmax = std::max(zmax, mm[2 * b + 1]); }
    const double rc = std::max(p->P.r_cut, p->P.r_nf);
    cl.ncx = std::max(1, (int)std::floor(p->P.Lx / rc));
    cl.ncy = std::max(1, (int)std::floor(p->P.Ly / rc));
    cl.csx = p->P.Lx / cl.ncx;
    cl.csy = p->P.Ly / cl.ncy;
    cl.zlo = zmin - rc;
    double zspan = (zmax + rc) - cl.zlo;
    cl.ncz = std::max(1, (int)std::floor(zspan / rc));
    cl.csz = zspan / cl.ncz;
    int64_t ncell = (int64_t)cl.ncx * cl.ncy * cl.ncz;
    if (ncell > (1 << 26)) throw Error(SE_ERR_VALUE, "near-field cell grid too large");
    if (ncell + 1 > p->cell_cap) {
        dfree(p, cl.start);
        cl.start = dalloc<int>(p, ncell + 1);
        p->cell_cap = ncell + 1;
    }
    CellGeo g = cell_geo(p);
    cell_keys_kernel<<<(unsigned)((ns + 255) / 256), 256, 0, p->stream>>>(
        p->d_near_src, ns, g, p->d_ckeys, p->d_cperm);
    SE_LAUNCHED(p);
    int end_bit = 1;
    while (end_bit < 32 && ((uint64_t)ncell >> end_bit) != 0) ++end_bit;
    size_t bytes = p->near_cub_bytes;
    SE_CUDA(cub::DeviceRadixSort::SortPairs(p->d_near_cub, bytes, p->d_ckeys, p->d_ckeys2,
                                            p->d_cperm, p->d_cperm2, (int)ns, 0, end_bit,
                                            p->stream));
    cell_fill_kernel<<<(unsigned)((ns + 1 + 255) / 256), 256, 0, p->stream>>>(
        p->d_ckeys2, p->d_cperm2, ns, (int)ncell, p->d_near_src, g, cl.start, cl.src,
        cl.srcf, cl.orig);
    SE_LAUNCHED(p);
    // charge targets in cell order (coherent warps)
    cell_keys_kernel<<<(unsigned)((n + 255) / 256), 256, 0, p->stream>>>(
        p->d_near_src, n, g, p->d_tkeys, p->d_tperm);
    SE_LAUNCHED(p);
    bytes = p->near_cub_bytes;
    SE_CUDA(cub::DeviceRadixSort::SortPairs(p->d_near_cub, bytes, p->d_tkeys, p->d_tkeys2,
                                            p->d_tperm, p->d_tgt, (int)n, 0, end_bit,
                                            p->stream));
}

void near_eval(Plan* p, const double* d_eval, const int* d_order, int64_t ne,
               const NearKernel& k, double* d_out4, int64_t* d_npairs) {
    if (ne == 0) return;
    NearArgs a{};
    a.eval = d_eval; a.order = d_order; a.ne = ne;
    a.g = cell_geo(p);
    a.start = p->cl.start; a.src = p->cl.src; a.srcf = p->cl.srcf;
    a.radius = k.radius; a.c1 = k.c1; a.c2 = k.c2; a.inv4pie = k.inv4pie;
    a.self_value = k.self_value; a.point0 = k.point0;
    a.kind = k.kind; a.need_field = k.need_field;
    double rr = k.radius * (1.0 + 1e-4) + 1e-6 * (p->P.Lx + p->P.Ly + p->P.H);
    a.r2f = (float)(rr * rr);
    a.Lxf = (float)p->P.Lx; a.Lyf = (float)p->P.Ly;
    a.iLxf = (float)(1.0 / p->P.Lx); a.iLyf = (float)(1.0 / p->P.Ly);
    a.out = d_out4; a.out_stride = ne;
    a.npairs = d_npairs;
    if (p->cl.n == 0) {
        SE_CUDA(cudaMemsetAsync(d_out4, 0, sizeof(double) * (k.need_field ? 4 : 1) * ne,
                                p->stream));
        return;
    }
    near_kernel<<<(unsigned)((ne + 127) / 128), 128, 0, p->stream>>>(a);
    SE_LAUNCHED(p);
}

void finalize(Plan* p, int64_t n, uint32_t flags, double self_inf_value,
              double* d_phi, double* d_E) {
    const int nblk = 592;
    FinArgs a{};
    a.far = p->d_far; a.near = p->d_near; a.q = p->d_q; a.n = n;
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
