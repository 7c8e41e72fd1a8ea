// Host copy bandwidth (tools only): memcpy vs non-temporal (streaming-store)
// copies into a pinned-like destination, T threads.  The drop-in's staging
// is host-memcpy bound (tools/hostbw.py); NT stores skip the destination's
// read-for-ownership.
#include <immintrin.h>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

__attribute__((target("avx2"))) static void nt_copy_avx2(char* d, const char* s, size_t n) {
    size_t i = 0;
    for (; i < n && ((uintptr_t)(d + i) & 31); ++i) d[i] = s[i];
    for (; i + 128 <= n; i += 128) {
        __m256i a = _mm256_loadu_si256((const __m256i*)(s + i));
        __m256i b = _mm256_loadu_si256((const __m256i*)(s + i + 32));
        __m256i c = _mm256_loadu_si256((const __m256i*)(s + i + 64));
        __m256i e = _mm256_loadu_si256((const __m256i*)(s + i + 96));
        _mm256_stream_si256((__m256i*)(d + i), a);
        _mm256_stream_si256((__m256i*)(d + i + 32), b);
        _mm256_stream_si256((__m256i*)(d + i + 64), c);
        _mm256_stream_si256((__m256i*)(d + i + 96), e);
    }
    for (; i < n; ++i) d[i] = s[i];
    _mm_sfence();
}

template <class F>
static double run(F f, char* d, const char* s, size_t n, int T) {
    double best = 1e9;
    for (int r = 0; r < 3; ++r) {
        auto t0 = std::chrono::steady_clock::now();
        std::vector<std::thread> th;
        for (int t = 0; t < T; ++t) {
            size_t lo = n * t / T, hi = n * (t + 1) / T;
            th.emplace_back([=] { f(d + lo, s + lo, hi - lo); });
        }
        for (auto& x : th) x.join();
        double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        if (ms < best) best = ms;
    }
    return best;
}

int main() {
    const size_t n = size_t(1) << 30;
    char* s = (char*)aligned_alloc(4096, n);
    char* d = (char*)aligned_alloc(4096, n);
    memset(s, 1, n);
    memset(d, 2, n);
    printf("avx2 %d avx512f %d\n", __builtin_cpu_supports("avx2"), __builtin_cpu_supports("avx512f"));
    for (int T : {1, 4, 8, 16}) {
        double a = run([](char* x, const char* y, size_t m) { memcpy(x, y, m); }, d, s, n, T);
        double b = run(nt_copy_avx2, d, s, n, T);
        printf("T=%2d  memcpy %6.1f ms (%5.1f GB/s)   nt-copy %6.1f ms (%5.1f GB/s)\n", T, a, n / a / 1e6, b, n / b / 1e6);
    }
    return 0;
}
