// Which instruction classes issue alongside the FP64 pipe on B200?  Per loop
// iteration: 8 independent DFMA chains (16 FP64-pipe cycles per warp on a
// 16-lane sub-partition) plus M independent instructions of one class; the
// cycles per iteration per SM sub-partition show whether the class overlaps
// (stays ~17) or serialises (16 + c*M).  Tools only.
#include <cstdio>
#include <cuda_runtime.h>

template <int M, int KIND>
__global__ void probe(double* out, int n, unsigned seed) {
    double a[8];
    unsigned y[16];
    float f[16];
    for (int k = 0; k < 8; ++k) a[k] = threadIdx.x * 1e-3 + k;
    for (int k = 0; k < 16; ++k) { y[k] = threadIdx.x * seed + k; f[k] = threadIdx.x * 1e-3f + k; }
    const double b = 0.999999, c = 1e-7;
    for (int i = 0; i < n; ++i) {
        const bool pr = ((y[0] >> 3) & 1u) != 0;  // one data-dependent predicate per iteration
#pragma unroll
        for (int k = 0; k < 8; ++k) a[k] = fma(a[k], b, c);
#pragma unroll
        for (int k = 0; k < M; ++k) {
            if (KIND == 0) asm volatile("add.u32 %0, %0, %1;" : "+r"(y[k]) : "r"(k + 1));
            if (KIND == 1) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(f[k]) : "f"(0.999f), "f"(1e-3f));
            if (KIND == 2) asm volatile("{.reg .pred p; setp.ne.u32 p, %2, 0; selp.b32 %0, %1, %0, p;}" : "+r"(y[k]) : "r"(y[(k + 1) & 15]), "r"((unsigned)pr));
            if (KIND == 3) { if (pr) y[k] = y[(k + 3) & 15]; }
            if (KIND == 4) asm volatile("max.s32 %0, %0, %1;" : "+r"(y[k]) : "r"(y[(k + 5) & 15]));
            if (KIND == 5) asm volatile("min.f32 %0, %0, %1;" : "+f"(f[k]) : "f"(f[(k + 5) & 15]));
            if (KIND == 6) asm volatile("{.reg .pred p; setp.lt.s32 p, %1, %2; @p add.u32 %0, %0, 1;}" : "+r"(y[k]) : "r"(y[(k + 1) & 15]), "r"(y[(k + 2) & 15]));
            if (KIND == 7) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(y[k]) : "r"(y[(k + 1) & 15]), "r"(y[(k + 2) & 15]));
            if (KIND == 8) asm volatile("{.reg .pred p; setp.ne.u32 p, %1, 0; @p mov.b32 %0, %2;}" : "+r"(y[k]) : "r"((unsigned)pr), "r"(y[(k + 1) & 15]));
            if (KIND == 9) asm volatile("{.reg .pred p; setp.ne.u32 p, %2, 0; selp.f32 %0, %1, %0, p;}" : "+f"(f[k]) : "f"(f[(k + 1) & 15]), "r"((unsigned)pr));
        }
    }
    double s = 0;
    for (int k = 0; k < 8; ++k) s += a[k];
    unsigned t = 0;
    float g = 0;
    for (int k = 0; k < 16; ++k) { t += y[k]; g += f[k]; }
    if (s == -1.0 || t == 7u || g == -1.f) out[0] = s + t + g;
}

template <int M, int KIND>
void run(const char* name, double* d) {
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int n = 4096, blocks = 148 * 8, threads = 256;
    for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        probe<M, KIND><<<blocks, threads>>>(d, n, 3u);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        const double warp_iters = (double)blocks * threads / 32 * n / (148.0 * 4);
        int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
        const double cycles = ms * 1e-3 * clk * 1e3;
        if (rep) printf("%-28s %6.2f cycles/iter/SMSP  (+%.2f per extra instruction)\n", name, cycles / warp_iters,
                        M ? (cycles / warp_iters - 17.2) / M : 0.0);
    }
}

int main() {
    double* d; cudaMalloc(&d, 8);
    run<0, 0>("8 DFMA", d);
    run<8, 0>("+ 8 IADD", d);
    run<8, 1>("+ 8 FFMA", d);
    run<8, 2>("+ 8 SEL (selp.b32)", d);
    run<8, 9>("+ 8 FSEL (selp.f32)", d);
    run<8, 3>("+ 8 C predicated assign", d);
    run<8, 8>("+ 8 @p mov.b32", d);
    run<16, 8>("+ 16 @p mov.b32", d);
    run<8, 4>("+ 8 IMNMX", d);
    run<8, 5>("+ 8 FMNMX", d);
    run<8, 6>("+ 8 (ISETP + @p IADD)", d);
    run<8, 7>("+ 8 LOP3", d);
    return 0;
}
