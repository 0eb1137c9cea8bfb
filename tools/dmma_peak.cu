// FP64 tensor-core (DMMA) throughput per mma.sync shape on this GPU:
// m8n8k4 (sm_80) vs the sm_90+ shapes m16n8k4 / m16n8k8 / m16n8k16.
// nvcc -gencode arch=compute_100a,code=sm_100a tools/dmma_peak.cu -o /tmp/dmma
#include <cstdio>
#define ITERS 4096
template <int S>
__global__ void k(double* out) {
    double a[8], b[4], c[4][4];
    for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
    for (int i = 0; i < 4; ++i) b[i] = threadIdx.x * 2e-3 + i;
    for (int t = 0; t < 4; ++t) for (int i = 0; i < 4; ++i) c[t][i] = 0;
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            if (S == 0)
                asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                             : "+d"(c[t][0]), "+d"(c[t][1]) : "d"(a[t]), "d"(b[t]));
            else if (S == 1)
                asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                             : "+d"(c[t][0]), "+d"(c[t][1]), "+d"(c[t][2]), "+d"(c[t][3])
                             : "d"(a[t]), "d"(a[t + 4]), "d"(b[t]));
            else if (S == 2)
                asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                             : "+d"(c[t][0]), "+d"(c[t][1]), "+d"(c[t][2]), "+d"(c[t][3])
                             : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[t]), "d"(b[(t + 1) & 3]));
            else
                asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
                             : "+d"(c[t][0]), "+d"(c[t][1]), "+d"(c[t][2]), "+d"(c[t][3])
                             : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                               "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
        }
    }
    double s = 0;
    for (int t = 0; t < 4; ++t) for (int i = 0; i < 4; ++i) s += c[t][i];
    if (s == 12345.0) out[0] = s;
}
template <int S>
void run(const char* name, double flop_per_mma) {
    double* d; cudaMalloc(&d, 8);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int wpb : {4, 8, 16}) {
        dim3 grid(sms * 2), block(32 * wpb);
        k<S><<<grid, block>>>(d);
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        cudaEventRecord(e0);
        k<S><<<grid, block>>>(d);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        double flops = (double)grid.x * wpb * ITERS * 4 * flop_per_mma;
        printf("%-8s warps/CTA %2d: %.1f TFLOP/s\n", name, wpb, flops / ms / 1e9);
    }
}
int main() {
    run<0>("m8n8k4", 2.0 * 8 * 8 * 4);
    run<1>("m16n8k4", 2.0 * 16 * 8 * 4);
    run<2>("m16n8k8", 2.0 * 16 * 8 * 8);
    run<3>("m16n8k16", 2.0 * 16 * 8 * 16);
}
