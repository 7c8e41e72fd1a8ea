// Cycles per Gram-form sweep (tools only) for several clip implementations:
// the iterative kernel's inner loop from registers, 4 x 128-thread CTAs per SM
// (the hybrid's occupancy), to find what bounds it (FP64 pipe: 46 DFMA/DADD/DMUL
// = 92 cycles per warp-sweep; dispatch: ~85 instructions).
#include <cstdio>
#include <cuda_runtime.h>

// CL: 0 current (ISETP sign + DSETP + 4 FSEL), 1 no clip at all (upper bound),
//     2 DSETP sign test, 3 hi-word IMNMX for the lower clip + DSETP/FSEL upper,
//     4 fmin/fmax, 5 current but slide clip via clip0_hi on x0 - t
template <int CL>
struct Sw {
    double G00, G01, G03, G04, G11, G13, G14, G33, G34, G44, SA0, SA1, SA3, SA4, SB0, SB1, SB3, SB4;
    double r0, r1, r2, r3, r3a, r3b, x0, x1, x2, x3, g0, g1, g3, g4;

    __device__ __forceinline__ static double c0hi(double x, double hi) {
        if (CL == 1) return x;
        if (CL == 0 || CL == 5) {
            const bool neg = __double2hiint(x) < 0;
            const double r = (x < hi) ? x : hi;
            return neg ? 0.0 : r;
        }
        if (CL == 2) {
            const bool neg = x < 0.0;
            const double r = (x < hi) ? x : hi;
            return neg ? 0.0 : r;
        }
        if (CL == 3) {
            const int h = max(__double2hiint(x), 0);
            const double m = __hiloint2double(h, __double2loint(x));
            return (m < hi) ? m : hi;
        }
        if (CL == 10) {
            double r = x;
            asm("{.reg .pred p, q; setp.lt.s32 q, %2, 0; setp.geu.f64 p, %1, %3; @p mov.b64 %0, %3; @q mov.b64 %0, 0d0000000000000000;}"
                : "+d"(r) : "d"(x), "r"(__double2hiint(x)), "d"(hi));
            return r;
        }
        if (CL == 11) {
            const int h = max(__double2hiint(x), 0);
            double r = __hiloint2double(h, __double2loint(x));
            asm("{.reg .pred p; setp.geu.f64 p, %0, %1; @p mov.b64 %0, %1;}" : "+d"(r) : "d"(hi));
            return r;
        }
        if (CL == 6) return (x < hi) ? x : hi;  // upper clip only (measures the lower clip)
        if (CL == 7) {
            // int64 pattern compare (exact for hi >= +0), then the sign-bit lower clip
            const long long xb = __double_as_longlong(x), hb = __double_as_longlong(hi);
            const double r = (xb < hb) ? x : hi;
            return (xb < 0) ? 0.0 : r;
        }
        if (CL == 8) {
            // hi-word IMNMX lower clip, int64 upper compare: no DSETP
            const int h = max(__double2hiint(x), 0);
            const long long mb = ((long long)h << 32) | (unsigned)__double2loint(x);
            const long long hb = __double_as_longlong(hi);
            return __longlong_as_double(mb < hb ? mb : hb);
        }
        if (CL == 9) {
            // clamp through a single compare against each bound, predicated moves
            double r = x;
            if (!(r < hi)) r = hi;
            if (__double2hiint(x) < 0) r = 0.0;
            return r;
        }
        return fmin(fmax(x, 0.0), hi);
    }
    __device__ __forceinline__ static double csym(double t, double xb, double xa) {
        if (CL == 1) return t;
        if (CL == 4) return fmax(fmin(t, xa), -xb);
        if (CL == 10 || CL == 11) {
            double r = t;
            const double lo = -xb;
            asm("{.reg .pred p, q; setp.le.f64 p, %0, %1; setp.ge.f64 q, %0, %2; @q mov.b64 %0, %2; @p mov.b64 %0, %1;}"
                : "+d"(r) : "d"(lo), "d"(xa));
            return r;
        }
        if (CL == 8) {
            // |t| clipped to the bound on t's side (int64 compare), sign restored
            const long long tb = __double_as_longlong(t);
            const long long mag = tb & 0x7FFFFFFFFFFFFFFFll;
            const long long lim = __double_as_longlong(tb < 0 ? xb : xa);
            const long long r = mag < lim ? mag : lim;
            return __longlong_as_double(r | (tb & (long long)0x8000000000000000ull));
        }
        const double lo = -xb;
        const bool below = !(t > lo), above = !(t < xa);
        return below ? lo : (above ? xa : t);
    }
    __device__ __forceinline__ static double sclip(double sr, double x, double hs) {
        // clamp(sr, -x, hs) with independent compares of the raw step
        const double lo = -x;
        const bool below = !(sr > lo), above = !(sr < hs);
        return below ? lo : (above ? hs : sr);
    }
    __device__ __forceinline__ void sweep_s() {
        double t, s;
        s = sclip(-g0 * r0, x0, (1.0 - x1) - x0); x0 += s;
        g0 += s * G00; g1 += s * G01; g3 += s * G03; g4 += s * G04;
        s = sclip(-g1 * r1, x1, (1.0 - x0) - x1); x1 += s;
        g0 += s * G01; g1 += s * G11; g3 += s * G13; g4 += s * G14;
        t = -(g1 - g0) * r3a;
        t = csym(t, x1, x0);
        x0 = x0 - t; x1 = x1 + t;
        g0 += t * SA0; g1 += t * SA1; g3 += t * SA3; g4 += t * SA4;
        s = sclip(-g3 * r2, x2, (1.0 - x3) - x2); x2 += s;
        g0 += s * G03; g1 += s * G13; g3 += s * G33; g4 += s * G34;
        s = sclip(-g4 * r3, x3, (1.0 - x2) - x3); x3 += s;
        g0 += s * G04; g1 += s * G14; g3 += s * G34; g4 += s * G44;
        t = -(g4 - g3) * r3b;
        t = csym(t, x3, x2);
        x2 = x2 - t; x3 = x3 + t;
        g0 += t * SB0; g1 += t * SB1; g3 += t * SB3; g4 += t * SB4;
    }
    __device__ __forceinline__ void sweep() {
        if (CL == 12) { sweep_s(); return; }
        double t, s;
        t = c0hi(x0 - g0 * r0, 1.0 - x1);
        s = t - x0; x0 = t;
        g0 += s * G00; g1 += s * G01; g3 += s * G03; g4 += s * G04;
        t = c0hi(x1 - g1 * r1, 1.0 - x0);
        s = t - x1; x1 = t;
        g0 += s * G01; g1 += s * G11; g3 += s * G13; g4 += s * G14;
        if (CL == 5) {
            const double S = x0 + x1;
            const double nx0 = c0hi(x0 + (g1 - g0) * r3a, S);
            t = x0 - nx0; x0 = nx0; x1 = S - nx0;
        } else {
            t = -(g1 - g0) * r3a;
            t = csym(t, x1, x0);
            x0 = x0 - t; x1 = x1 + t;
        }
        g0 += t * SA0; g1 += t * SA1; g3 += t * SA3; g4 += t * SA4;
        t = c0hi(x2 - g3 * r2, 1.0 - x3);
        s = t - x2; x2 = t;
        g0 += s * G03; g1 += s * G13; g3 += s * G33; g4 += s * G34;
        t = c0hi(x3 - g4 * r3, 1.0 - x2);
        s = t - x3; x3 = t;
        g0 += s * G04; g1 += s * G14; g3 += s * G34; g4 += s * G44;
        if (CL == 5) {
            const double S = x2 + x3;
            const double nx2 = c0hi(x2 + (g4 - g3) * r3b, S);
            t = x2 - nx2; x2 = nx2; x3 = S - nx2;
        } else {
            t = -(g4 - g3) * r3b;
            t = csym(t, x3, x2);
            x2 = x2 - t; x3 = x3 + t;
        }
        g0 += t * SB0; g1 += t * SB1; g3 += t * SB3; g4 += t * SB4;
    }
};

template <int CL, int BS, int MINB>
__global__ void __launch_bounds__(BS, MINB) sweeps(double* out, int n_sweeps, double seed) {
    Sw<CL> w;
    unsigned h = (blockIdx.x * BS + threadIdx.x) * 2654435761u;
    auto rnd = [&] { h = h * 1664525u + 1013904223u; return (h >> 8) * (1.0 / 16777216.0); };
    w.G00 = 1 + rnd(); w.G11 = 1 + rnd(); w.G33 = 1 + rnd(); w.G44 = 1 + rnd();
    w.G01 = 0.3 * rnd(); w.G03 = -0.2 * rnd(); w.G04 = 0.1 * rnd(); w.G13 = 0.2 * rnd(); w.G14 = -0.1 * rnd();
    w.G34 = 0.3 * rnd();
    w.SA0 = w.G01 - w.G00; w.SA1 = w.G11 - w.G01; w.SA3 = w.G13 - w.G03; w.SA4 = w.G14 - w.G04;
    w.SB0 = w.G04 - w.G03; w.SB1 = w.G14 - w.G13; w.SB3 = w.G34 - w.G33; w.SB4 = w.G44 - w.G34;
    w.r0 = 1 / w.G00; w.r1 = 1 / w.G11; w.r2 = 1 / w.G33; w.r3 = 1 / w.G44;
    w.r3a = 1 / (w.SA1 - w.SA0); w.r3b = 1 / (w.SB4 - w.SB3);
    w.x0 = w.x1 = w.x2 = w.x3 = 1.0 / 3.0;
    w.g0 = rnd() - 0.5 + seed; w.g1 = rnd() - 0.5; w.g3 = rnd() - 0.5; w.g4 = rnd() - 0.5;
#pragma unroll 1
    for (int it = 0; it < n_sweeps; ++it) w.sweep();
    const double s = w.x0 + w.x1 + w.x2 + w.x3 + w.g0;
    if (s == -1.0) out[0] = s;
}

template <int CL, int BS, int MINB>
void run_lat(double* d, const char* name) {
    // one CTA of BS threads per SM: BS/32 warps (<= 4: one per sub-partition)
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int blocks = 148, n = 4096;
    float best = 1e30f;
    for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0);
        sweeps<CL, BS, MINB><<<blocks, BS>>>(d, n, 0.1);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    printf("%-40s latency: %6.1f cycles per sweep (one warp per SMSP)\n", name, best * 1e-3 * clk * 1e3 / n);
}

template <int CL, int BS, int MINB>
void run(double* d, const char* name, size_t smem = 0) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    int per_sm = 0;
    if (smem > 48 * 1024) cudaFuncSetAttribute(sweeps<CL, BS, MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sweeps<CL, BS, MINB>, BS, smem);
    const int blocks = 148 * per_sm * 8, n = 512;
    float best = 1e30f;
    for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0);
        sweeps<CL, BS, MINB><<<blocks, BS, smem>>>(d, n, 0.1);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, sweeps<CL, BS, MINB>);
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const double warp_sweeps = (double)blocks * BS / 32 * n / (148.0 * 4);
    printf("%-40s regs %3d warps/SM %2d  %6.1f cycles per warp-sweep per SMSP\n", name, fa.numRegs,
           per_sm * BS / 32, best * 1e-3 * clk * 1e3 / warp_sweeps);
}

int main() {
    double* d;
    cudaMalloc(&d, 8);
    run<0, 128, 4>(d, "current clips, 16 w/SM (smem-capped)", 56 * 1024);
    run<0, 128, 4>(d, "current clips, 20 w/SM (smem-capped)", 44 * 1024);
    run<0, 128, 4>(d, "current clips, 12 w/SM (smem-capped)", 72 * 1024);
    run<0, 128, 4>(d, "current clips, 8 w/SM (smem-capped)", 110 * 1024);
    run<3, 128, 4>(d, "IMNMX, 16 w/SM (smem-capped)", 56 * 1024);
    run_lat<0, 128, 4>(d, "current clips");
    run_lat<1, 128, 4>(d, "no clips");
    run_lat<6, 128, 4>(d, "upper clip only");
    run_lat<8, 128, 4>(d, "all-integer clips");
    run<0, 128, 4>(d, "current clips, 24 warps/SM");
    run<0, 128, 1>(d, "current clips, 4 CTAs cap (1x128: regs free)");
    run<0, 128, 8>(d, "current clips, 32 warps/SM");
    run<1, 128, 4>(d, "no clips (bound), 24 w/SM");
    run<2, 128, 4>(d, "DSETP sign test, 24 w/SM");
    run<3, 128, 4>(d, "IMNMX hi-word lower clip, 24 w/SM");
    run<4, 128, 4>(d, "fmin/fmax, 24 w/SM");
    run<5, 128, 4>(d, "slide as clip0_hi(x0-t, x0+x1), 24 w/SM");
    run<5, 128, 8>(d, "slide as clip0_hi(x0-t, x0+x1), 32 w/SM");
    run<6, 128, 4>(d, "upper clip only, 24 w/SM");
    run<10, 128, 4>(d, "predicated PTX movs, 24 w/SM");
    run<12, 128, 4>(d, "step-form clips (s = clamp(-g r, -x, h - x)), 24 w/SM");
    run<12, 128, 8>(d, "step-form clips, 32 w/SM");
    run_lat<12, 128, 4>(d, "step-form clips");
    run<11, 128, 4>(d, "IMNMX lower + predicated mov, 24 w/SM");
    run_lat<10, 128, 4>(d, "predicated PTX movs");
    run<7, 128, 4>(d, "int64 upper compare + sign, 24 w/SM");
    run<8, 128, 4>(d, "all-integer clips, 24 w/SM");
    run<9, 128, 4>(d, "predicated-move clips, 24 w/SM");
    return 0;
}
