// Latency microbenchmarks (one warp, dependent chains, clock64): DADD, DFMA,
// FFMA, IMAD, LDS, F2F.F32.F64, MUFU.RSQ.  nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double *od, float *of, int *oi, long long *t, int n) {
    __shared__ int sm[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = (i * 7 + 1) & 1023;
    __syncthreads();
    double a = od[0], b = od[1];
    float x = of[0], y = of[1];
    int p = threadIdx.x & 1, q = oi[0];
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) a = __dadd_rn(a, b);
    long long t1 = clock64();
    for (int i = 0; i < n; ++i) a = fma(a, b, b);
    long long t2 = clock64();
    for (int i = 0; i < n; ++i) x = fmaf(x, y, y);
    long long t3 = clock64();
    for (int i = 0; i < n; ++i) q = q * 3 + 1;
    long long t4 = clock64();
    for (int i = 0; i < n; ++i) p = sm[p];
    long long t5 = clock64();
    for (int i = 0; i < n; ++i) { x = (float)a; a = (double)x + 1e-9; }
    long long t6 = clock64();
    for (int i = 0; i < n; ++i) { float r; asm volatile("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x)); x = r + 1.0f; }
    long long t7 = clock64();
    for (int i = 0; i < n; ++i) { double d = a; a = (p & 1) ? d : __dadd_rn(d, b); }
    long long t8 = clock64();
    od[2] = a; of[2] = x; oi[1] = q + p;
    if (threadIdx.x == 0) { t[0] = t1 - t0; t[1] = t2 - t1; t[2] = t3 - t2; t[3] = t4 - t3; t[4] = t5 - t4; t[5] = t6 - t5; t[6] = t7 - t6; t[7] = t8 - t7; }
}
int main() {
    double *od; float *of; int *oi; long long *t;
    cudaMallocManaged(&od, 64); cudaMallocManaged(&of, 64); cudaMallocManaged(&oi, 64); cudaMallocManaged(&t, 128);
    od[0] = 1.0; od[1] = 1e-7; of[0] = 1.0f; of[1] = 0.5f; oi[0] = 3;
    const int n = 4096;
    k<<<1, 32>>>(od, of, oi, t, n); cudaDeviceSynchronize();
    k<<<1, 32>>>(od, of, oi, t, n); cudaDeviceSynchronize();
    const char *names[] = {"DADD", "DFMA", "FFMA", "IMAD", "LDS (dep)", "F2F.F32.F64+F2F.F64.F32+DADD", "MUFU.RSQ+FADD", "FSEL/DADD select"};
    for (int i = 0; i < 8; ++i) printf("%-32s %.2f cycles/op\n", names[i], (double)t[i] / n);
    return 0;
}
