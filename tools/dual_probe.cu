// Does an FP64 warp instruction block the SM sub-partition's dispatch for two
// cycles, or can integer / FP32 instructions issue in the second cycle?
// 8 independent DFMA chains per thread plus M independent integer (IADD3) or
// FP32 (FFMA) chains per iteration; cycles per iteration per warp-slot are
// compared against 2*8 (FP64 pipe bound) and 2*8 + M (serial dispatch).
#include <cstdio>
#include <cuda_runtime.h>

template <int M, int KIND>  // KIND 0: IADD3, 1: FFMA, 2: ISETP+SEL, 3: FSEL on a loop-invariant predicate, 4: predicated MOV
__global__ void probe(double* out, int n) {
    double a[8];
    unsigned y[16];
    float f[16];
    for (int k = 0; k < 8; ++k) a[k] = threadIdx.x * 1e-3 + k;
    for (int k = 0; k < 16; ++k) { y[k] = threadIdx.x + k; f[k] = threadIdx.x * 1e-3f + k; }
    const double b = 0.999999, c = 1e-7;
    for (int i = 0; i < n; ++i) {
        const bool pr = ((y[0] >> 3) & 1u) != 0;
#pragma unroll
        for (int k = 0; k < 8; ++k) a[k] = fma(a[k], b, c);
#pragma unroll
        for (int k = 0; k < M; ++k) {
            if (KIND == 0) asm volatile("add.u32 %0, %0, %1;" : "+r"(y[k]) : "r"(k + 1));
            if (KIND == 1) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(f[k]) : "f"(0.999f), "f"(1e-3f));
            if (KIND == 2) asm volatile("{.reg .pred p; setp.lt.u32 p, %0, 100; selp.b32 %0, %0, %1, p;}" : "+r"(y[k]) : "r"(k));
            // selects on a predicate computed once per iteration (one ISETP for all M)
            if (KIND == 3) y[k] = pr ? y[k] + 1u : y[(k + 1) & 15];
            if (KIND == 4) { if (pr) y[k] = y[(k + 3) & 15]; }
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
        probe<M, KIND><<<blocks, threads>>>(d, n);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        // warp-iterations per SM sub-partition
        const double warp_iters = (double)blocks * threads / 32 * n / (148.0 * 4);
        int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
        const double cycles = ms * 1e-3 * clk * 1e3;
        if (rep) printf("%-22s %6.2f cycles per iteration per SMSP (FP64-pipe bound 16; serial 16+M)\n", name,
                        cycles / warp_iters);
    }
}

int main() {
    double* d; cudaMalloc(&d, 8);
    run<0, 0>("8 DFMA", d);
    run<4, 0>("8 DFMA + 4 IADD", d);
    run<8, 0>("8 DFMA + 8 IADD", d);
    run<16, 0>("8 DFMA + 16 IADD", d);
    run<8, 1>("8 DFMA + 8 FFMA", d);
    run<16, 1>("8 DFMA + 16 FFMA", d);
    run<8, 2>("8 DFMA + 8 (ISETP+SEL)", d);
    run<8, 3>("8 DFMA + 8 SEL", d);
    run<16, 3>("8 DFMA + 16 SEL", d);
    run<8, 4>("8 DFMA + 8 pred MOV", d);
    run<16, 4>("8 DFMA + 16 pred MOV", d);
    run<0, 3>("(no DFMA check) 8 DFMA", d);
    return 0;
}
