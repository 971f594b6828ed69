/* Host DRAM ceilings on the GPU box (for the CPU-master path's roofline):
 * multi-threaded streaming read (AVX-512 loads), non-temporal write, and
 * read + 1/4-size NT write (the shape of the r = 1 host pack).
 *   gcc -O2 -mavx512f -pthread scripts/host_bw.c -o /tmp/host_bw && /tmp/host_bw */
#include <immintrin.h>
#include <pthread.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#define N (256L << 20) /* floats: 1 GiB */
static float *a, *b;
static int T, mode;
static double sink[64];

static void *work(void *p) {
    long t = (long)p, lo = N * t / T, hi = N * (t + 1) / T;
    __m512 acc = _mm512_setzero_ps();
    if (mode == 0) {
        for (long i = lo; i < hi; i += 16) acc = _mm512_add_ps(acc, _mm512_loadu_ps(a + i));
    } else if (mode == 1) {
        __m512 v = _mm512_set1_ps(1.0f);
        for (long i = lo; i < hi; i += 16) _mm512_stream_ps(b + i, v);
    } else {
        long wlo = lo / 4;
        for (long i = lo; i < hi; i += 64) {
            __m512 x = _mm512_add_ps(_mm512_add_ps(_mm512_loadu_ps(a + i), _mm512_loadu_ps(a + i + 16)),
                                     _mm512_add_ps(_mm512_loadu_ps(a + i + 32), _mm512_loadu_ps(a + i + 48)));
            _mm512_stream_ps(b + wlo + (i - lo) / 4, x);
            acc = _mm512_add_ps(acc, x);
        }
    }
    _mm_sfence();
    sink[t] = _mm512_reduce_add_ps(acc);
    return 0;
}

int main(void) {
    a = aligned_alloc(64, N * 4);
    b = aligned_alloc(64, N * 4);
    memset(a, 1, N * 4);
    memset(b, 1, N * 4);
    const char *names[3] = {"read", "NT write", "read + 1/4 NT write"};
    for (mode = 0; mode < 3; ++mode)
        for (T = 1; T <= 16; T *= 2) {
            pthread_t th[64];
            struct timespec s, e;
            double best = 1e9;
            for (int r = 0; r < 3; ++r) {
                clock_gettime(CLOCK_MONOTONIC, &s);
                for (long t = 0; t < T; t++) pthread_create(&th[t], 0, work, (void *)t);
                for (int t = 0; t < T; t++) pthread_join(th[t], 0);
                clock_gettime(CLOCK_MONOTONIC, &e);
                double dt = e.tv_sec - s.tv_sec + (e.tv_nsec - s.tv_nsec) * 1e-9;
                if (dt < best) best = dt;
            }
            double bytes = mode == 0 ? N * 4.0 : mode == 1 ? N * 4.0 : N * 5.0;
            printf("%-20s %2d threads: %6.1f GB/s\n", names[mode], T, bytes / best / 1e9);
        }
    return 0;
}
