// Throughput of FP64-pipe instruction kinds on this GPU (tools only):
// 8 independent chains per thread, 64 warps per SM.
#include <cstdio>
#include <cuda_runtime.h>

template <int KIND>
__global__ void thr(double* out, int n) {
    double a[8];
    for (int k = 0; k < 8; ++k) a[k] = threadIdx.x * 1e-3 + k;
    const double b = 0.999999, c = 1e-7;
    for (int i = 0; i < n; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            if (KIND == 0) a[k] = fma(a[k], b, c);
            if (KIND == 1) a[k] = a[k] + c;
            if (KIND == 2) a[k] = (a[k] < b) ? a[k] + c : a[k] - c;   // DSETP + DADD + selects
            if (KIND == 3) a[k] = a[k] * b;
        }
    }
    double s = 0;
    for (int k = 0; k < 8; ++k) s += a[k];
    if (s == -1.0) out[0] = s;
}

int main() {
    double* d; cudaMalloc(&d, 8);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int n = 4096, blocks = 148 * 8, threads = 256;
    const char* names[] = {"DFMA", "DADD", "DSETP+DADD+sel", "DMUL"};
    for (int kind = 0; kind < 4; ++kind) {
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(e0);
            if (kind == 0) thr<0><<<blocks, threads>>>(d, n);
            if (kind == 1) thr<1><<<blocks, threads>>>(d, n);
            if (kind == 2) thr<2><<<blocks, threads>>>(d, n);
            if (kind == 3) thr<3><<<blocks, threads>>>(d, n);
            cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            double ops = (double)blocks * threads * n * 8;
            if (rep) printf("%-16s %.2f G thread-ops/s  (%.1f per SM per cycle @1.965GHz)\n", names[kind], ops / ms / 1e6,
                            ops / (ms * 1e-3) / 148 / 1.965e9);
        }
    }
    return 0;
}
