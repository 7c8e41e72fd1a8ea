// Dependent-chain latency and throughput of FP64 ops on this GPU (tools only).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void lat_dfma(double* out, long long* cyc, int n) {
    double a = threadIdx.x * 1e-3, b = 0.999999, c = 1e-7;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) { a = fma(a, b, c); a = fma(a, b, c); a = fma(a, b, c); a = fma(a, b, c); }
    long long t1 = clock64();
    out[threadIdx.x] = a; if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void lat_dadd(double* out, long long* cyc, int n) {
    double a = threadIdx.x * 1e-3, c = 1e-7;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) { a = a + c; a = a - c * 0.5; a = a + c; a = a - c * 0.25; }
    long long t1 = clock64();
    out[threadIdx.x] = a; if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void lat_clip(double* out, long long* cyc, int n) {
    double a = threadIdx.x * 1e-3, hi = 0.7;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
        a = a * 1.0000001 - 1e-9;
        a = (a > 0.0) ? a : 0.0; a = (a < hi) ? a : hi;
        a = a * 1.0000001 + 1e-9;
        a = (a > 0.0) ? a : 0.0; a = (a < hi) ? a : hi;
    }
    long long t1 = clock64();
    out[threadIdx.x] = a; if (threadIdx.x == 0) *cyc = t1 - t0;
}
__device__ __forceinline__ double iclip(double x, double hi) {
    long long xb = __double_as_longlong(x);
    const long long hb = __double_as_longlong(hi);
    xb = (xb < 0) ? 0 : xb;
    return __longlong_as_double(xb < hb ? xb : hb);
}
__global__ void lat_iclip(double* out, long long* cyc, int n) {
    double a = threadIdx.x * 1e-3, hi = 0.7 + threadIdx.x * 1e-9;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
        a = a * 1.0000001 - 1e-9;
        a = iclip(a, hi);
        a = a * 1.0000001 + 1e-9;
        a = iclip(a, hi);
    }
    long long t1 = clock64();
    out[threadIdx.x] = a; if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void lat_dsetp(double* out, long long* cyc, int n) {
    double a = threadIdx.x * 1e-3, hi = 0.7 + threadIdx.x * 1e-9;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
        a = a * 1.0000001 - 1e-9;
        a = (a < hi) ? a : hi;
        a = a * 1.0000001 + 1e-9;
        a = (a < hi) ? a : hi;
    }
    long long t1 = clock64();
    out[threadIdx.x] = a; if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void lat_ffma(float* out, long long* cyc, int n) {
    float a = threadIdx.x * 1e-3f, b = 0.999999f, c = 1e-7f;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) { a = fmaf(a, b, c); a = fmaf(a, b, c); a = fmaf(a, b, c); a = fmaf(a, b, c); }
    long long t1 = clock64();
    out[threadIdx.x] = a; if (threadIdx.x == 0) *cyc = t1 - t0;
}

int main() {
    double* d; float* f; long long* c; long long h;
    cudaMalloc(&d, 1024 * 8); cudaMalloc(&f, 1024 * 4); cudaMalloc(&c, 8);
    const int n = 4096;
    lat_dfma<<<1, 32>>>(d, c, n); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("DFMA dependent latency: %.2f cycles\n", (double)h / (4.0 * n));
    lat_dadd<<<1, 32>>>(d, c, n); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("DADD(+DMUL const) dependent chain: %.2f cycles per op-pair/2\n", (double)h / (4.0 * n));
    lat_clip<<<1, 32>>>(d, c, n); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("DFMA + clip(2 compares+selects) chain: %.2f cycles per (fma+clip)\n", (double)h / (2.0 * n));
    lat_iclip<<<1, 32>>>(d, c, n); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("DFMA + integer clip chain: %.2f cycles per (fma+clip)\n", (double)h / (2.0 * n));
    lat_dsetp<<<1, 32>>>(d, c, n); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("DFMA + one double min (DSETP+2 FSEL) chain: %.2f cycles\n", (double)h / (2.0 * n));
    lat_ffma<<<1, 32>>>(f, c, n); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("FFMA dependent latency: %.2f cycles\n", (double)h / (4.0 * n));
    return 0;
}
