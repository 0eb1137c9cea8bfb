// Max relative error of the hardware rsqrt.approx.ftz.f64 (decides how many
// Newton steps rsqrt_pos needs).  nvcc -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cmath>
__global__ void k(double* out, int n) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    // log-uniform in [1e-8, 1e8]
    unsigned long long z = i * 0x9E3779B97F4A7C15ull; z ^= z >> 31; z *= 0xBF58476D1CE4E5B9ull; z ^= z >> 29;
    double u = (double)(z >> 11) * (1.0 / 9007199254740992.0);
    double x = exp((u - 0.5) * 36.8);
    double y; asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    double ref = 1.0 / sqrt(x);
    out[i] = fabs(y - ref) / ref;
}
int main() {
    int n = 1 << 24; double* d; cudaMalloc(&d, n * 8);
    k<<<n / 256, 256>>>(d, n);
    double* h = new double[n]; cudaMemcpy(h, d, n * 8, cudaMemcpyDeviceToHost);
    double m = 0; for (int i = 0; i < n; ++i) m = fmax(m, h[i]);
    printf("max rel err rsqrt.approx.ftz.f64: %.3e (2^%.2f)\n", m, log2(m));
}
