// Register-file read bandwidth probe (tools only): is the Gram sweep bound by
// 32-bit register operand reads rather than by the FP64 pipe?
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ double sel(double a, double b, unsigned p) {
    double r;
    asm volatile("{.reg .pred q; setp.ne.b32 q, %3, 0; selp.f64 %0, %1, %2, q;}" : "=d"(r) : "d"(a), "d"(b), "r"(p));
    return r;
}

template <int KIND>
__global__ void probe(double* out, int n, double seed) {
    double a[8], b[8], c[8], r[8], s[8];
    for (int k = 0; k < 8; ++k) {
        a[k] = threadIdx.x * 1e-3 + k + seed;
        b[k] = 0.999999 - k * 1e-7 + seed;
        c[k] = 1e-7 * k + seed;
        r[k] = k * 0.5 + seed;
        s[k] = k * 0.25 + seed;
    }
    const double bb = 0.999999, cc = 1e-7;
    for (int i = 0; i < n; ++i) {
        const unsigned p = (i ^ threadIdx.x) & 1;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            if (KIND == 0) a[k] = fma(a[k], bb, cc);                 // 1 distinct 64-bit source
            if (KIND == 1) a[k] = fma(a[k], b[k], c[k]);             // 3 distinct sources
            if (KIND == 2) { const double o = r[k]; r[k] = sel(r[k], s[k], p); s[k] = sel(s[k], o, p); }  // 4 FSEL
            if (KIND == 3) { a[k] = fma(a[k], bb, cc); const double o = r[k]; r[k] = sel(r[k], s[k], p); s[k] = sel(s[k], o, p); }
            if (KIND == 4) { a[k] = fma(a[k], b[k], c[k]); const double o = r[k]; r[k] = sel(r[k], s[k], p); s[k] = sel(s[k], o, p); }
            if (KIND == 5) { r[k] = sel(r[k], 0.0, p); s[k] = sel(0.0, s[k], p); }  // 4 FSEL with RZ
            if (KIND == 6) { a[k] = fma(a[k], bb, cc); r[k] = sel(r[k], 0.0, p); s[k] = sel(0.0, s[k], p); }
            if (KIND == 7) { a[k] = fma(a[k], b[k], c[k]); b[k] = fma(b[k], c[k], a[k]); }  // 16 DFMA, 3 sources
            if (KIND == 8) { a[k] = fma(a[k], bb, cc); b[k] = fma(b[k], bb, cc); }          // 16 DFMA, 1 source
        }
    }
    double t = 0;
    for (int k = 0; k < 8; ++k) t += a[k] + b[k] + r[k] + s[k];
    if (t == -1.0) out[0] = t;
}

template <int KIND>
void run(const char* name, double* d) {
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int n = 4096, blocks = 148 * 6, threads = 128;
    float best = 1e30f;
    for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0);
        probe<KIND><<<blocks, threads>>>(d, n, 0.0);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        best = ms < best ? ms : best;
    }
    const double warp_iters = (double)blocks * threads / 32 * n / (148.0 * 4);
    int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    cudaFuncAttributes fa; cudaFuncGetAttributes(&fa, probe<KIND>);
    printf("%-44s regs %3d %6.2f cycles per iteration per SMSP\n", name, fa.numRegs, best * 1e-3 * clk * 1e3 / warp_iters);
}

int main() {
    double* d; cudaMalloc(&d, 8);
    run<0>("8 DFMA (1 varying source)", d);
    run<1>("8 DFMA (3 distinct sources)", d);
    run<8>("16 DFMA (1 varying source)", d);
    run<7>("16 DFMA (3 distinct sources)", d);
    run<2>("16 double selects (32 FSEL)", d);
    run<5>("16 selects vs 0 (32 FSEL)", d);
    run<3>("8 DFMA(1 src) + 32 FSEL", d);
    run<6>("8 DFMA(1 src) + 32 FSEL vs 0", d);
    run<4>("8 DFMA(3 src) + 32 FSEL", d);
    return 0;
}
