// Cost of the sweep's clip building blocks next to a saturated FP64 pipe
// (tools only).  8 independent DFMA chains per iteration (16 FP64-pipe cycles
// per warp per SM sub-partition) plus M independent instances of one block;
// prints the extra cycles per block.
#include <cstdio>
#include <cuda_runtime.h>

template <int M, int KIND>
__global__ void probe(double* out, int n) {
    double a[8], x[8], h[8];
    for (int k = 0; k < 8; ++k) {
        a[k] = threadIdx.x * 1e-3 + k;
        x[k] = 0.25 + 1e-4 * threadIdx.x + 0.01 * k;
        h[k] = 0.5 - 1e-4 * k;
    }
    const double b = 0.999999, c = 1e-7;
    for (int i = 0; i < n; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) a[k] = fma(a[k], b, c);
#pragma unroll
        for (int k = 0; k < M; ++k) {
            double& v = x[k];
            const double w = h[k];
            if (KIND == 0) v = v + w;                                           // DADD
            if (KIND == 1) v = (v < w) ? v : w - 1e-9;                          // DSETP + 2 FSEL (+ DADD)
            if (KIND == 2) {                                                    // exact min of non-negative doubles on integers
                const long long vi = __double_as_longlong(v), wi = __double_as_longlong(w);
                v = __longlong_as_double(vi < wi ? vi : wi - 1);
            }
            if (KIND == 3) {                                                    // high-word compare + 2 selects
                const bool lt = __double2hiint(v) < __double2hiint(w);
                v = lt ? v : w - 1e-9;
            }
            if (KIND == 4) {                                                    // DSETP feeding predicated moves
                double r = w - 1e-9;
                if (v < w) r = v;
                v = r;
            }
        }
    }
    double s = 0;
    for (int k = 0; k < 8; ++k) s += a[k] + x[k];
    if (s == -1.0) out[0] = s;
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
        const double warp_iters = (double)blocks * threads / 32 * n / (148.0 * 4);
        int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
        const double cycles = ms * 1e-3 * clk * 1e3;
        if (rep) printf("%-34s %6.2f cycles/iter/SMSP  (+%.2f per block)\n", name, cycles / warp_iters,
                        M ? (cycles / warp_iters - 17.2) / M : 0.0);
    }
}

int main() {
    double* d; cudaMalloc(&d, 8);
    run<0, 0>("8 DFMA", d);
    run<4, 0>("+ 4 DADD", d);
    run<8, 0>("+ 8 DADD", d);
    run<4, 1>("+ 4 (DSETP, 2 FSEL, DADD)", d);
    run<8, 1>("+ 8 (DSETP, 2 FSEL, DADD)", d);
    run<4, 4>("+ 4 (DSETP, pred moves, DADD)", d);
    run<8, 4>("+ 8 (DSETP, pred moves, DADD)", d);
    run<4, 2>("+ 4 int64 min (ISETP.EX, SEL)", d);
    run<8, 2>("+ 8 int64 min (ISETP.EX, SEL)", d);
    run<4, 3>("+ 4 (hi-word ISETP, 2 FSEL, DADD)", d);
    run<8, 3>("+ 8 (hi-word ISETP, 2 FSEL, DADD)", d);
    return 0;
}
