// FP64-pipe use of the Gram-form iterative sweep alone (tools only): each
// thread runs NP independent pairs' sweeps from register state (no memory
// traffic in the loop), for several CTA sizes / register budgets, to separate
// the sweep's own dependency structure from the kernels' memory and queue
// effects.  Prints FP64 instructions per SM per cycle (peak 64).
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_2105_12415_b200/csrc/tc_pair.cuh"

using namespace tc;

template <int NP, int BS, int MINB>
__global__ void __launch_bounds__(BS, MINB) sweeps(double* out, int n_sweeps, double seed) {
    GramSolver<true, double> gs[NP];
    KP<double> kp;
    kp.c_factor = 1; kp.alpha_it = 10; kp.alpha_reg = 1e-4; kp.move_factor = 0.25; kp.start_coord = 1.0 / 3.0;
    kp.n_iterative = n_sweeps;
#pragma unroll
    for (int p = 0; p < NP; ++p) {
        double A[9], B[9];
        unsigned h = (blockIdx.x * BS + threadIdx.x) * 2654435761u + p * 97u;
#pragma unroll
        for (int k = 0; k < 9; ++k) {
            h = h * 1664525u + 1013904223u;
            A[k] = (h >> 8) * (1.0 / 16777216.0);
            h = h * 1664525u + 1013904223u;
            B[k] = (h >> 8) * (1.0 / 16777216.0) + seed;
        }
        gs[p].init(A, B, kp);
    }
#pragma unroll 1
    for (int it = 0; it < n_sweeps; ++it) {
#pragma unroll
        for (int p = 0; p < NP; ++p) gs[p].sweep();
    }
    double s = 0;
#pragma unroll
    for (int p = 0; p < NP; ++p) s += gs[p].x0 + gs[p].x1 + gs[p].x2 + gs[p].x3 + gs[p].g0;
    if (s == -1.0) out[0] = s;
}

template <int NP, int BS, int MINB>
void run(double* d, const char* name) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sweeps<NP, BS, MINB>, BS, 0);
    const int blocks = 148 * per_sm * 8, n = 256;
    float best = 1e30f;
    for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0);
        sweeps<NP, BS, MINB><<<blocks, BS>>>(d, n, 0.1);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, sweeps<NP, BS, MINB>);
    const double fp64_per_sweep = 54.0;  // SASS count of the BOX sweep (DFMA+DADD+DMUL+DSETP)
    const double ops = (double)blocks * BS * NP * n * fp64_per_sweep;
    printf("%-22s regs %3d  warps/SM %2d  %.1f FP64 instr per SM per cycle (%.0f%% of 64)  spill %zu B\n", name,
           fa.numRegs, per_sm * BS / 32, ops / (best * 1e-3) / 148 / 1.965e9,
           100.0 * ops / (best * 1e-3) / 148 / 1.965e9 / 64, fa.localSizeBytes);
}

int main() {
    double* d;
    cudaMalloc(&d, 8);
    run<1, 128, 4>(d, "1 pair, 128x4 CTAs");
    run<1, 256, 2>(d, "1 pair, 256x2 CTAs");
    run<1, 128, 5>(d, "1 pair, 128x5 CTAs");
    run<1, 128, 6>(d, "1 pair, 128x6 CTAs");
    run<1, 128, 8>(d, "1 pair, 128x8 CTAs");
    run<2, 128, 2>(d, "2 pairs, 128x2 CTAs");
    run<2, 128, 3>(d, "2 pairs, 128x3 CTAs");
    run<2, 128, 4>(d, "2 pairs, 128x4 CTAs");
    run<3, 128, 2>(d, "3 pairs, 128x2 CTAs");
    return 0;
}
