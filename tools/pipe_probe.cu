// Which pipe (and how many dispatch / pipe cycles) each instruction class of
// the iterative sweep costs on B200: 8 independent DFMA chains per thread plus
// 8 independent chains of the probed instruction per iteration.  IADD3 issues
// for free in the FP64 pipe's shadow (tools/dual_probe.cu), so it keeps
// predicates alive without adding cost.
#include <cstdio>
#include <cuda_runtime.h>

template <int KIND, int WITH_DFMA>
__global__ void probe(double* out, int n) {
    double a[8], x[8];
    unsigned y[8];
    float f[8];
    for (int k = 0; k < 8; ++k) {
        a[k] = threadIdx.x * 1e-3 + k;
        x[k] = threadIdx.x * 1e-4 + 0.5 * k;
        y[k] = threadIdx.x + k;
        f[k] = threadIdx.x * 1e-3f + k;
    }
    const double b = 0.999999, c = 1e-7;
    for (int i = 0; i < n; ++i) {
        if (WITH_DFMA) {
#pragma unroll
            for (int k = 0; k < 8; ++k) a[k] = fma(a[k], b, c);
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            if (KIND == 0) {}  // nothing
            if (KIND == 1) asm volatile("{.reg .pred p; setp.lt.f64 p, %1, %2; @p add.u32 %0, %0, 1;}" : "+r"(y[k]) : "d"(x[k]), "d"(b));
            if (KIND == 2) asm volatile("{.reg .pred p; setp.lt.u32 p, %0, 1000; @p add.u32 %0, %0, 3;}" : "+r"(y[k]));
            if (KIND == 3) asm volatile("{.reg .pred p; setp.ne.u32 p, %2, 0; selp.f32 %0, %0, %1, p;}" : "+f"(f[k]) : "f"(1.5f), "r"(i & 1));
            if (KIND == 4) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(y[k]) : "r"(k), "r"(i));
            if (KIND == 5) asm volatile("add.f64 %0, %0, %1;" : "+d"(x[k]) : "d"(c));
            if (KIND == 6) asm volatile("mad.lo.u32 %0, %0, 3, %1;" : "+r"(y[k]) : "r"(i));
            if (KIND == 7) asm volatile("{.reg .pred p; setp.ne.u32 p, %2, 0; selp.b32 %0, %0, %1, p;}" : "+r"(y[k]) : "r"(k), "r"(i & 1));
            if (KIND == 8) asm volatile("{.reg .pred p; .reg .b32 lo, hi; setp.ne.u32 p, %2, 0; mov.b64 {lo,hi}, %0; selp.b32 lo, lo, 0, p; selp.b32 hi, hi, 0, p; mov.b64 %0, {lo,hi};}" : "+d"(x[k]) : "r"(k), "r"(i & 1));
            if (KIND == 9) asm volatile("max.s32 %0, %0, %1;" : "+r"(y[k]) : "r"(i));
        }
    }
    double s = 0;
    unsigned t = 0;
    float g = 0;
    for (int k = 0; k < 8; ++k) { s += a[k] + x[k]; t += y[k]; g += f[k]; }
    if (s == -1.0 || t == 7u || g == -1.f) out[0] = s + t + g;
}

template <int KIND, int W>
void run(const char* name, double* d) {
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int n = 4096, blocks = 148 * 8, threads = 256;
    for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        probe<KIND, W><<<blocks, threads>>>(d, n);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        const double warp_iters = (double)blocks * threads / 32 * n / (148.0 * 4);
        int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
        if (rep) printf("%-34s %6.2f cycles per iteration per SMSP\n", name, ms * 1e-3 * clk * 1e3 / warp_iters);
    }
}

int main() {
    double* d; cudaMalloc(&d, 8);
    run<0, 1>("8 DFMA", d);
    run<1, 1>("8 DFMA + 8 DSETP(+@p IADD3)", d);
    run<1, 0>("8 DSETP(+@p IADD3)", d);
    run<2, 1>("8 DFMA + 8 ISETP(+@p IADD3)", d);
    run<2, 0>("8 ISETP(+@p IADD3)", d);
    run<3, 1>("8 DFMA + 8 (ISETP+FSEL)", d);
    run<4, 1>("8 DFMA + 8 LOP3", d);
    run<4, 0>("8 LOP3", d);
    run<5, 1>("8 DFMA + 8 DADD", d);
    run<6, 1>("8 DFMA + 8 IMAD", d);
    run<7, 1>("8 DFMA + 8 (ISETP+SEL)", d);
    run<7, 0>("8 (ISETP+SEL)", d);
    run<8, 1>("8 DFMA + 8 (ISETP+2 SEL)", d);
    run<9, 1>("8 DFMA + 8 IMNMX", d);
    run<9, 0>("8 IMNMX", d);
    return 0;
}
