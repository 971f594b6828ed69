// adt_host.cpp — the CPU half of the paper's CPU-master setting: Bitpack on the
// host cores, only the packed bytes cross PCIe, Bitunpack on the GPU.
//
// Paper (Fig. 2): the FP32 master weights
// live in host memory; before every host->GPU transfer the CPU keeps the top
// RoundTo bytes of every weight (OpenMP + AVX2 in the paper), the packed
// stream is copied to the GPU, and a CUDA kernel zero-fills the dropped bytes.
// The byte semantics are the reference codec's (codec.py:116-197: weight i ->
// payload bytes [i*r, (i+1)*r), most-significant byte first), and the layer's
// l2 norm (precision.py:25-28) is fused into the same read of the masters.
//
// B200-host design (16-core Emerald Rapids VM, AVX-512 VBMI):
//   * one pass over the masters: 64 words (256 B) per iteration — VPERMB /
//     VPERMT2B gather the kept bytes of 64 words into r full 64-byte vectors,
//     written with non-temporal stores when the destination is 64-B aligned
//     (no read-for-ownership of the pinned staging lines); the float64 sum of
//     squares rides along (VCVTPS2PD + VFMADD, four accumulators);
//   * work units of 64K weights (small sets: ~1/128 of the set; a function of
//     the set, so results never depend on the thread count), claimed in order
//     from an atomic counter by a persistent worker pool (spin, then sleep)
//     plus the calling thread;
//   * adt_host_to_device: the calling thread also issues cudaMemcpyAsync for
//     every run of finished units (>= min batch), so the DMA of unit k overlaps
//     the packing of unit k+16.., then queues the device unpack (adt_unpack).
// A scalar path (bswap, r-byte copies) serves hosts without AVX-512 VBMI.

#include <cuda_runtime.h>
#include <immintrin.h>
#include <stdint.h>
#include <string.h>

#include <atomic>
#include <condition_variable>
#include <cstdlib>
#include <functional>
#include <memory>
#include <mutex>
#include <thread>
#include <vector>

#include <sched.h>
#include <time.h>

#include "adt.h"

namespace {

constexpr uint64_t kUnitWeights = 1u << 16;   // weights per work unit at most (multiple of 64)
constexpr uint64_t kUnitMin = 1u << 12;       // ... and at least, for small sets
constexpr uint64_t kGroup = 64;               // weights per vector iteration

// ------------------------------------------------------------ scalar path
inline uint32_t bswap32(uint32_t w) { return __builtin_bswap32(w); }

double pack_scalar(const uint32_t *src, uint64_t n, int r, uint8_t *dst) {
    double acc = 0.0;
    for (uint64_t i = 0; i < n; ++i) {
        const uint32_t be = bswap32(src[i]);
        memcpy(dst + i * r, &be, static_cast<size_t>(r));
        float f;
        memcpy(&f, src + i, 4);
        acc += static_cast<double>(f) * static_cast<double>(f);
    }
    return acc;
}

// ------------------------------------------------------- AVX-512 VBMI path
// Byte-gather indices, built once. For r = 2, 3: output vector k of a 64-word
// group takes its bytes from the input vector pair (v[b], v[b+1]), b = 4k/r;
// byte j of the packed stream is byte 3 - (j % r) of word j / r.
struct PermTables {
    alignas(64) uint8_t r4[64];        // VPERMB: byte-swap each word of one vector
    alignas(64) uint8_t r2[2][64];     // VPERMT2B over (v[2k], v[2k+1])
    alignas(64) uint8_t r3[3][64];     // VPERMT2B over (v[k], v[k+1]), k = 0..2
    alignas(64) uint8_t r1lo[64];      // VPERMT2B over (v0, v1) -> bytes 0..31
    alignas(64) uint8_t r1hi[64];      // VPERMT2B over (v2, v3) -> bytes 32..63
    PermTables() {
        for (int j = 0; j < 64; ++j) r4[j] = static_cast<uint8_t>((j / 4) * 4 + 3 - j % 4);
        for (int k = 0; k < 2; ++k)
            for (int j = 0; j < 64; ++j) {
                const int g = 64 * k + j, w = g / 2, p = g % 2, base = 2 * k;
                r2[k][j] = static_cast<uint8_t>((w / 16 - base) * 64 + (w % 16) * 4 + 3 - p);
            }
        for (int k = 0; k < 3; ++k)
            for (int j = 0; j < 64; ++j) {
                const int g = 64 * k + j, w = g / 3, p = g % 3, base = k;
                r3[k][j] = static_cast<uint8_t>((w / 16 - base) * 64 + (w % 16) * 4 + 3 - p);
            }
        for (int j = 0; j < 64; ++j) {
            const int w = j;                                   // one byte per word
            r1lo[j] = static_cast<uint8_t>(j < 32 ? (w / 16) * 64 + (w % 16) * 4 + 3 : 0);
            const int w2 = j - 32;                             // words 32..63 from (v2, v3)
            r1hi[j] = static_cast<uint8_t>(j >= 32 ? (w2 / 16) * 64 + (w2 % 16) * 4 + 3 : 0);
        }
    }
};
const PermTables &perm() {
    static const PermTables t;
    return t;
}

#define ADT_AVX512 __attribute__((target("avx512f,avx512bw,avx512dq,avx512vbmi")))

ADT_AVX512 inline __m512d sq_acc(__m512d acc, __m256 h) {
    const __m512d d = _mm512_cvtps_pd(h);
    return _mm512_fmadd_pd(d, d, acc);
}

template <bool NT>
ADT_AVX512 inline void put(uint8_t *dst, __m512i v) {
    if (NT) _mm512_stream_si512(reinterpret_cast<__m512i *>(dst), v);
    else _mm512_storeu_si512(dst, v);
}

// Software prefetch of the masters ahead of the loads. The fused norm
// (VCVTPS2PD + FMA) lengthens each iteration, so the out-of-order window holds
// fewer loads in flight and one core's stream falls to a fraction of what the
// host DRAM delivers; prefetching into L2 several KB ahead restores the memory
// parallelism (ADT_HOST_PF = distance in bytes, 0 = off; ADT_HOST_PF_HINT =
// 0 for L1, 1 for L2 — scripts/host_pack_probe.py sweeps them).
int prefetch_bytes() {
    static const int v = [] {
        const char *e = getenv("ADT_HOST_PF");
        return e != nullptr ? atoi(e) : 8192;
    }();
    return v;
}
int prefetch_hint() {                 // 0 = L1 (T0), 1 = L2 (T1, default), 2 = non-temporal (NTA)
    static const int v = [] {
        const char *e = getenv("ADT_HOST_PF_HINT");
        return e != nullptr ? atoi(e) : 1;
    }();
    return v;
}

// Pack n words (n multiple of 64) into dst; returns the float64 sum of squares.
template <int R, bool NT>
ADT_AVX512 double pack_avx512(const uint32_t *src, uint64_t n, uint8_t *dst) {
    const PermTables &T = perm();
    const int pf = prefetch_bytes();
    const int hint = prefetch_hint();
    __m512d a0 = _mm512_setzero_pd(), a1 = _mm512_setzero_pd(), a2 = _mm512_setzero_pd(), a3 = _mm512_setzero_pd();
    const __m512i i4 = _mm512_load_si512(T.r4);
    const __m512i i2a = _mm512_load_si512(T.r2[0]), i2b = _mm512_load_si512(T.r2[1]);
    const __m512i i3a = _mm512_load_si512(T.r3[0]), i3b = _mm512_load_si512(T.r3[1]),
                  i3c = _mm512_load_si512(T.r3[2]);
    const __m512i i1l = _mm512_load_si512(T.r1lo), i1h = _mm512_load_si512(T.r1hi);
    for (uint64_t i = 0; i < n; i += kGroup) {
        if (pf > 0) {                 // may run past the unit's end: prefetches never fault
            const char *p = reinterpret_cast<const char *>(src + i) + pf;
            if (hint == 1) {
                _mm_prefetch(p, _MM_HINT_T1);
                _mm_prefetch(p + 64, _MM_HINT_T1);
                _mm_prefetch(p + 128, _MM_HINT_T1);
                _mm_prefetch(p + 192, _MM_HINT_T1);
            } else if (hint == 2) {
                _mm_prefetch(p, _MM_HINT_NTA);
                _mm_prefetch(p + 64, _MM_HINT_NTA);
                _mm_prefetch(p + 128, _MM_HINT_NTA);
                _mm_prefetch(p + 192, _MM_HINT_NTA);
            } else {
                _mm_prefetch(p, _MM_HINT_T0);
                _mm_prefetch(p + 64, _MM_HINT_T0);
                _mm_prefetch(p + 128, _MM_HINT_T0);
                _mm_prefetch(p + 192, _MM_HINT_T0);
            }
        }
        const __m512i v0 = _mm512_loadu_si512(src + i), v1 = _mm512_loadu_si512(src + i + 16),
                      v2 = _mm512_loadu_si512(src + i + 32), v3 = _mm512_loadu_si512(src + i + 48);
        uint8_t *o = dst + i * R;
        if (R == 4) {
            put<NT>(o, _mm512_permutexvar_epi8(i4, v0));
            put<NT>(o + 64, _mm512_permutexvar_epi8(i4, v1));
            put<NT>(o + 128, _mm512_permutexvar_epi8(i4, v2));
            put<NT>(o + 192, _mm512_permutexvar_epi8(i4, v3));
        } else if (R == 3) {
            put<NT>(o, _mm512_permutex2var_epi8(v0, i3a, v1));
            put<NT>(o + 64, _mm512_permutex2var_epi8(v1, i3b, v2));
            put<NT>(o + 128, _mm512_permutex2var_epi8(v2, i3c, v3));
        } else if (R == 2) {
            put<NT>(o, _mm512_permutex2var_epi8(v0, i2a, v1));
            put<NT>(o + 64, _mm512_permutex2var_epi8(v2, i2b, v3));
        } else {
            const __m512i lo = _mm512_permutex2var_epi8(v0, i1l, v1);
            const __m512i hi = _mm512_permutex2var_epi8(v2, i1h, v3);
            put<NT>(o, _mm512_mask_blend_epi8(0xFFFFFFFF00000000ull, lo, hi));
        }
        a0 = sq_acc(a0, _mm512_castps512_ps256(_mm512_castsi512_ps(v0)));
        a1 = sq_acc(a1, _mm256_castpd_ps(_mm512_extractf64x4_pd(_mm512_castsi512_pd(v0), 1)));
        a2 = sq_acc(a2, _mm512_castps512_ps256(_mm512_castsi512_ps(v1)));
        a3 = sq_acc(a3, _mm256_castpd_ps(_mm512_extractf64x4_pd(_mm512_castsi512_pd(v1), 1)));
        a0 = sq_acc(a0, _mm512_castps512_ps256(_mm512_castsi512_ps(v2)));
        a1 = sq_acc(a1, _mm256_castpd_ps(_mm512_extractf64x4_pd(_mm512_castsi512_pd(v2), 1)));
        a2 = sq_acc(a2, _mm512_castps512_ps256(_mm512_castsi512_ps(v3)));
        a3 = sq_acc(a3, _mm256_castpd_ps(_mm512_extractf64x4_pd(_mm512_castsi512_pd(v3), 1)));
    }
    if (NT) _mm_sfence();
    return _mm512_reduce_add_pd(_mm512_add_pd(_mm512_add_pd(a0, a1), _mm512_add_pd(a2, a3)));
}

// The same float64 sum of squares as pack_avx512 (same accumulators, same
// order: bit-identical), without the byte gather or any store — the norm of a
// layer that is not packed on the host (adt_host_to_device_ex direct layers).
ADT_AVX512 double sumsq_avx512(const uint32_t *src, uint64_t n) {
    const int pf = prefetch_bytes();
    __m512d a0 = _mm512_setzero_pd(), a1 = _mm512_setzero_pd(), a2 = _mm512_setzero_pd(), a3 = _mm512_setzero_pd();
    for (uint64_t i = 0; i < n; i += kGroup) {
        if (pf > 0) {
            const char *p = reinterpret_cast<const char *>(src + i) + pf;
            _mm_prefetch(p, _MM_HINT_T1);
            _mm_prefetch(p + 64, _MM_HINT_T1);
            _mm_prefetch(p + 128, _MM_HINT_T1);
            _mm_prefetch(p + 192, _MM_HINT_T1);
        }
        const __m512i v0 = _mm512_loadu_si512(src + i), v1 = _mm512_loadu_si512(src + i + 16),
                      v2 = _mm512_loadu_si512(src + i + 32), v3 = _mm512_loadu_si512(src + i + 48);
        a0 = sq_acc(a0, _mm512_castps512_ps256(_mm512_castsi512_ps(v0)));
        a1 = sq_acc(a1, _mm256_castpd_ps(_mm512_extractf64x4_pd(_mm512_castsi512_pd(v0), 1)));
        a2 = sq_acc(a2, _mm512_castps512_ps256(_mm512_castsi512_ps(v1)));
        a3 = sq_acc(a3, _mm256_castpd_ps(_mm512_extractf64x4_pd(_mm512_castsi512_pd(v1), 1)));
        a0 = sq_acc(a0, _mm512_castps512_ps256(_mm512_castsi512_ps(v2)));
        a1 = sq_acc(a1, _mm256_castpd_ps(_mm512_extractf64x4_pd(_mm512_castsi512_pd(v2), 1)));
        a2 = sq_acc(a2, _mm512_castps512_ps256(_mm512_castsi512_ps(v3)));
        a3 = sq_acc(a3, _mm256_castpd_ps(_mm512_extractf64x4_pd(_mm512_castsi512_pd(v3), 1)));
    }
    return _mm512_reduce_add_pd(_mm512_add_pd(_mm512_add_pd(a0, a1), _mm512_add_pd(a2, a3)));
}

double sumsq_scalar(const uint32_t *src, uint64_t n) {
    double acc = 0.0;
    for (uint64_t i = 0; i < n; ++i) {
        float f;
        memcpy(&f, src + i, 4);
        acc += static_cast<double>(f) * static_cast<double>(f);
    }
    return acc;
}

using PackFn = double (*)(const uint32_t *, uint64_t, uint8_t *);

ADT_AVX512 PackFn pick_avx512(int r, bool nt) {
    switch (r) {
        case 1: return nt ? pack_avx512<1, true> : pack_avx512<1, false>;
        case 2: return nt ? pack_avx512<2, true> : pack_avx512<2, false>;
        case 3: return nt ? pack_avx512<3, true> : pack_avx512<3, false>;
        default: return nt ? pack_avx512<4, true> : pack_avx512<4, false>;
    }
}

bool have_vbmi() {
    static const bool v = [] {
        __builtin_cpu_init();
        const char *e = getenv("ADT_HOST_SCALAR");          // A/B and test hook
        return !(e != nullptr && e[0] == '1') && __builtin_cpu_supports("avx512vbmi") &&
               __builtin_cpu_supports("avx512bw");
    }();
    return v;
}

bool use_nt() {
    static const bool v = [] {
        const char *e = getenv("ADT_HOST_NT");               // A/B: 0 = regular stores
        return !(e != nullptr && e[0] == '0');
    }();
    return v;
}

// One work unit: weights [lo, hi) of one layer, packed to `dst` (where weight
// lo's bytes go). Returns its sum of squares. nt: non-temporal stores allowed.
double pack_unit_to(const adt_segment &s, uint64_t lo, uint64_t hi, uint8_t *dst, bool nt) {
    const uint32_t *src = static_cast<const uint32_t *>(s.weights) + lo;
    const uint64_t n = hi - lo, body = have_vbmi() ? n / kGroup * kGroup : 0;
    double acc = 0.0;
    if (body) {
        nt = nt && use_nt() && (reinterpret_cast<uintptr_t>(dst) % 64 == 0);
        acc = pick_avx512(s.round_to, nt)(src, body, dst);
    }
    if (body < n) acc += pack_scalar(src + body, n - body, s.round_to, dst + body * s.round_to);
    return acc;
}

// pack_unit's sum of squares alone (same split into vector body + scalar tail)
double sumsq_unit(const adt_segment &s, uint64_t lo, uint64_t hi) {
    const uint32_t *src = static_cast<const uint32_t *>(s.weights) + lo;
    const uint64_t n = hi - lo, body = have_vbmi() ? n / kGroup * kGroup : 0;
    double acc = body ? sumsq_avx512(src, body) : 0.0;
    if (body < n) acc += sumsq_scalar(src + body, n - body);
    return acc;
}

// Host memory the DMA engine can read in place: [p, p + bytes) page-locked
// (cudaHostAlloc / cudaHostRegister; both ends checked).
bool page_locked(const void *p, uint64_t bytes) {
    cudaPointerAttributes a;
    const char *c = static_cast<const char *>(p);
    for (const char *q : {c, c + (bytes ? bytes - 1 : 0)}) {
        if (cudaPointerGetAttributes(&a, q) != cudaSuccess) {
            cudaGetLastError();
            return false;
        }
        if (a.type != cudaMemoryTypeHost) return false;
    }
    return true;
}

constexpr uint64_t kRunMergeGap = 64;     // inter-layer pad (< 64 B with 64-B aligned payloads) ships with its run

double pack_unit(const adt_segment &s, uint64_t lo, uint64_t hi, uint8_t *packed) {
    return pack_unit_to(s, lo, hi, packed + s.offset + lo * static_cast<uint64_t>(s.round_to), true);
}

// ------------------------------------------------------------ worker pool
// Persistent workers (affinity count - 1; the caller is the last worker).
// One job at a time: concurrent callers queue on `submit_mu`. A job is
// published as one atomic word (generation << 16 | participants), so a worker
// decides from a single load whether and for which generation it works. After
// a job, workers (and a caller waiting for them) spin for ADT_HOST_SPIN_US
// before sleeping on the condition variable: a futex wake of 15 threads costs
// tens of microseconds on the B200 host VM, more than a small layer set takes
// to pack (profiles/r02_small_host.md).
int spin_us() {
    static const int v = [] {
        const char *e = getenv("ADT_HOST_SPIN_US");
        return e != nullptr ? atoi(e) : 200;
    }();
    return v;
}

inline uint64_t now_ns() {
    timespec t;
    clock_gettime(CLOCK_MONOTONIC, &t);
    return static_cast<uint64_t>(t.tv_sec) * 1000000000ull + static_cast<uint64_t>(t.tv_nsec);
}

class Pool {
  public:
    static Pool &get() {
        static Pool *p = new Pool();   // never destroyed: workers may outlive static destructors
        return *p;
    }
    int workers() const { return static_cast<int>(threads_.size()); }

    // Run job(worker_index) on min(nthreads - 1, workers) pool threads; the
    // caller runs `caller()` concurrently and then waits for the pool threads.
    void run(int nthreads, const std::function<void(int)> &job, const std::function<void()> &caller) {
        std::lock_guard<std::mutex> serial(submit_mu_);
        const int use = std::max(0, std::min(nthreads - 1, workers()));
        if (use == 0) {
            caller();
            return;
        }
        job_ = &job;
        active_.store(use, std::memory_order_relaxed);
        {
            std::lock_guard<std::mutex> g(mu_);
            ++gen_;
            word_.store((gen_ << 16) | static_cast<uint64_t>(use), std::memory_order_release);
        }
        if (sleepers_.load(std::memory_order_acquire) > 0) cv_.notify_all();
        caller();
        const uint64_t t0 = now_ns(), budget = static_cast<uint64_t>(spin_us()) * 1000u;
        for (unsigned k = 0; active_.load(std::memory_order_acquire) != 0; ++k) {
            if ((k & 63) == 0 && now_ns() - t0 > budget) {
                std::unique_lock<std::mutex> g(mu_);
                done_cv_.wait(g, [&] { return active_.load(std::memory_order_acquire) == 0; });
                break;
            }
            _mm_pause();
        }
        job_ = nullptr;
    }

  private:
    Pool() {
        cpu_set_t set;
        int n = 1;
        if (sched_getaffinity(0, sizeof(set), &set) == 0) n = CPU_COUNT(&set);
        for (int i = 0; i + 1 < n; ++i) threads_.emplace_back([this, i] { loop(i); });
        for (auto &t : threads_) t.detach();
    }
    void loop(int idx) {
        uint64_t seen = 0;                     // generation last looked at
        for (;;) {
            uint64_t w = word_.load(std::memory_order_acquire);
            if ((w >> 16) == seen) {           // no new job: spin, then sleep
                const uint64_t t0 = now_ns(), budget = static_cast<uint64_t>(spin_us()) * 1000u;
                for (unsigned k = 0; ((w = word_.load(std::memory_order_acquire)) >> 16) == seen; ++k) {
                    if ((k & 63) == 0 && now_ns() - t0 > budget) {
                        std::unique_lock<std::mutex> g(mu_);
                        sleepers_.fetch_add(1, std::memory_order_acq_rel);
                        cv_.wait(g, [&] { return (word_.load(std::memory_order_acquire) >> 16) != seen; });
                        sleepers_.fetch_sub(1, std::memory_order_acq_rel);
                        w = word_.load(std::memory_order_acquire);
                        break;
                    }
                    _mm_pause();
                }
            }
            seen = w >> 16;
            if (idx >= static_cast<int>(w & 0xFFFF)) continue;   // not a participant of this generation
            (*job_)(idx);                      // job_ stays valid until every participant is done
            if (active_.fetch_sub(1, std::memory_order_acq_rel) == 1) {
                std::lock_guard<std::mutex> g(mu_);
                done_cv_.notify_all();
            }
        }
    }
    std::vector<std::thread> threads_;
    std::mutex mu_, submit_mu_;
    std::condition_variable cv_, done_cv_;
    const std::function<void(int)> *job_ = nullptr;
    uint64_t gen_ = 0;                         // guarded by mu_ (writers) / submit_mu_
    std::atomic<uint64_t> word_{0};            // gen << 16 | participants
    std::atomic<int> active_{0}, sleepers_{0};
};

struct Unit {
    int seg;
    uint64_t lo, hi;
};

int validate_host(const adt_segment *segs, int nseg, const uint8_t *packed) {
    if (nseg < 0 || (nseg > 0 && segs == nullptr)) return ADT_ERR_ARG;
    bool any = false;
    for (int i = 0; i < nseg; ++i) {
        const adt_segment &g = segs[i];
        if (g.round_to < 1 || g.round_to > 4) return ADT_ERR_ROUND_TO;
        if (g.reserved != 0) return ADT_ERR_ARG;
        if (g.count == 0) continue;
        any = true;
        if (g.weights == nullptr) return ADT_ERR_ARG;
        if (reinterpret_cast<uintptr_t>(g.weights) % 4) return ADT_ERR_ALIGN;
        if (g.count > (UINT64_MAX - g.offset) / 4) return ADT_ERR_ARG;
    }
    if (any && packed == nullptr) return ADT_ERR_ARG;
    return ADT_OK;
}

// Weights per work unit for a set: 64K, or for a small set about 1/128 of
// its weights (>= 4K, multiple of 64) so that its units spread over every
// host thread (LeNet, 430K weights: 106 units instead of 10). A function of
// the set alone, never of the thread count: the per-layer sums (summed unit
// by unit in a fixed order) are the same on every host. ADT_HOST_UNIT pins it.
uint64_t unit_weights(const adt_segment *segs, int nseg) {
    static const uint64_t pinned = [] {
        const char *e = getenv("ADT_HOST_UNIT");
        const uint64_t v = e != nullptr ? strtoull(e, nullptr, 10) : 0;
        return std::min(kUnitWeights, v / kGroup * kGroup);
    }();
    if (pinned) return pinned;
    uint64_t total = 0;
    for (int s = 0; s < nseg; ++s) total += segs[s].count;
    const uint64_t u = (total / 128 + kGroup - 1) / kGroup * kGroup;
    return std::max(kUnitMin, std::min(kUnitWeights, u));
}

void add_units(std::vector<Unit> &u, const adt_segment *segs, int s, uint64_t unit) {
    for (uint64_t lo = 0; lo < segs[s].count; lo += unit) u.push_back({s, lo, std::min(segs[s].count, lo + unit)});
}

std::vector<Unit> make_units(const adt_segment *segs, int nseg) {
    const uint64_t unit = unit_weights(segs, nseg);
    std::vector<Unit> u;
    for (int s = 0; s < nseg; ++s) add_units(u, segs, s, unit);
    return u;
}

// Pack every unit on `threads` threads; `on_progress(ready_prefix)` is called
// by the caller thread between its own units with the count of leading units
// that are complete (for the DMA pipeline). Per-unit sums go to unit_ss.
void pack_units(const adt_segment *segs, const std::vector<Unit> &units, size_t nnorm, uint8_t *packed, int threads,
                std::vector<double> &unit_ss, const std::function<void(size_t)> &on_progress,
                bool caller_packs = true) {
    const size_t nu = units.size();
    std::unique_ptr<std::atomic<uint8_t>[]> done(new std::atomic<uint8_t>[nu == 0 ? 1 : nu]);
    for (size_t i = 0; i < nu; ++i) done[i].store(0, std::memory_order_relaxed);
    std::atomic<size_t> next{0};
    auto work_one = [&](size_t k) {
        const Unit &u = units[k];
        unit_ss[k] = k < nnorm ? sumsq_unit(segs[u.seg], u.lo, u.hi) : pack_unit(segs[u.seg], u.lo, u.hi, packed);
        done[k].store(1, std::memory_order_release);
    };
    const std::function<void(int)> job = [&](int) {
        for (size_t k; (k = next.fetch_add(1, std::memory_order_relaxed)) < nu;) work_one(k);
    };
    size_t prefix = 0;
    auto advance = [&] {
        while (prefix < nu && done[prefix].load(std::memory_order_acquire)) ++prefix;
        on_progress(prefix);
    };
    const std::function<void()> caller = [&] {
        for (size_t k; caller_packs && (k = next.fetch_add(1, std::memory_order_relaxed)) < nu;) {
            work_one(k);
            advance();
        }
        while (prefix < nu) {                 // the pool finishes the last units
            advance();
            if (prefix < nu) _mm_pause();
        }
    };
    // caller_packs = false: `threads` pool workers pack, the caller only follows
    // the completed prefix (issuing the DMA of each finished run at once)
    Pool::get().run(caller_packs ? threads : threads + 1, job, caller);
    on_progress(nu);
}

bool caller_packs_h2d() {            // A/B: ADT_H2D_CALLER_PACKS=0 -> the calling thread only issues copies
    static const bool v = [] {
        const char *e = getenv("ADT_H2D_CALLER_PACKS");
        return !(e != nullptr && e[0] == '0');
    }();
    return v;
}

void finish_sums(const std::vector<Unit> &units, const std::vector<double> &unit_ss, int nseg, double *seg_sumsq) {
    if (seg_sumsq == nullptr) return;
    for (int s = 0; s < nseg; ++s) seg_sumsq[s] = 0.0;
    for (size_t k = 0; k < units.size(); ++k) seg_sumsq[units[k].seg] += unit_ss[k];   // fixed unit order
}

int resolve_threads(int threads) {
    const int avail = Pool::get().workers() + 1;
    return threads <= 0 ? avail : std::min(threads, avail);
}

}  // namespace

extern "C" {

int adt_host_threads(int *n) {
    if (n == nullptr) return ADT_ERR_ARG;
    *n = Pool::get().workers() + 1;
    return ADT_OK;
}

int adt_host_simd(void) { return have_vbmi() ? 512 : 0; }

int adt_pack_host(const adt_segment *segs, int nseg, uint8_t *packed, double *seg_sumsq, int threads) {
    const int v = validate_host(segs, nseg, packed);
    if (v != ADT_OK) return v;
    const std::vector<Unit> units = make_units(segs, nseg);
    std::vector<double> ss(units.size(), 0.0);
    pack_units(segs, units, 0, packed, resolve_threads(threads), ss, [](size_t) {});
    finish_sums(units, ss, nseg, seg_sumsq);
    return ADT_OK;
}

int adt_host_to_device(const adt_segment *host_segs, const adt_segment *dev_segs, int nseg, uint8_t *host_packed,
                       uint8_t *dev_packed, uint64_t packed_bytes, double *seg_sumsq, int threads,
                       uint64_t min_copy_bytes, void *stream) {
    return adt_host_to_device_ex(host_segs, dev_segs, nseg, host_packed, dev_packed, packed_bytes, seg_sumsq, threads,
                                 min_copy_bytes, 0u, nullptr, stream);
}

int adt_host_to_device_ex(const adt_segment *host_segs, const adt_segment *dev_segs, int nseg, uint8_t *host_packed,
                          uint8_t *dev_packed, uint64_t packed_bytes, double *seg_sumsq, int threads,
                          uint64_t min_copy_bytes, uint32_t flags, uint8_t *direct_out, void *stream) {
    int v = validate_host(host_segs, nseg, host_packed);
    if (v != ADT_OK) return v;
    if (nseg > 0 && dev_packed == nullptr) return ADT_ERR_ARG;
    if ((flags & ~static_cast<uint32_t>(ADT_H2D_DIRECT_FULL | ADT_H2D_SKIP_DIRECT_NORMS | ADT_H2D_ZERO_COPY)) != 0)
        return ADT_ERR_ARG;
    if ((flags & ADT_H2D_DIRECT_FULL) && dev_segs == nullptr) return ADT_ERR_ARG;   // direct copies land in the replicas
    // ZERO_COPY: no staging copies; the unpack reads the packed stream from the
    // page-locked staging buffer over the link (device-mapped host memory).
    const bool zero_copy = (flags & ADT_H2D_ZERO_COPY) != 0;
    const uint8_t *mapped = nullptr;
    if (zero_copy) {
        if (dev_segs == nullptr || !page_locked(host_packed, packed_bytes)) return ADT_ERR_ARG;
        void *d = nullptr;
        if (packed_bytes > 0 && cudaHostGetDevicePointer(&d, host_packed, 0) != cudaSuccess) {
            cudaGetLastError();
            return ADT_ERR_ARG;
        }
        mapped = static_cast<const uint8_t *>(d);
    }
    uint64_t end_prev = 0;                    // payloads in increasing, non-overlapping order (the DMA
    for (int i = 0; i < nseg; ++i) {          // ships the stream front to back as units complete)
        const adt_segment &h = host_segs[i];
        if (dev_segs != nullptr) {
            const adt_segment &d = dev_segs[i];
            if (h.count != d.count || h.offset != d.offset || h.round_to != d.round_to) return ADT_ERR_ARG;
        }
        if (h.count == 0) continue;
        const uint64_t end = h.offset + h.count * static_cast<uint64_t>(h.round_to);
        if (h.offset < end_prev || end > packed_bytes) return ADT_ERR_ARG;
        end_prev = end;
    }
    // Full-width layers (round_to 4: the replica is the master word for word)
    // whose host words are page-locked skip the packer: the DMA reads them
    // straight from the masters into the replicas (4n bytes on the link either
    // way), so host DRAM carries their 4n once instead of read 4n + write 4n +
    // DMA-read 4n; the device skips their unpack. Their norms still come from
    // the host (a read-only pass). The packed stream keeps their (unused) span.
    std::vector<uint8_t> direct(static_cast<size_t>(nseg > 0 ? nseg : 1), 0);
    if (flags & ADT_H2D_DIRECT_FULL)
        for (int i = 0; i < nseg; ++i)
            direct[i] = host_segs[i].count > 0 && host_segs[i].round_to == 4 &&
                        page_locked(host_segs[i].weights, host_segs[i].count * 4) &&
                        reinterpret_cast<uintptr_t>(dev_segs[i].weights) % 16 == 0;
    if (direct_out != nullptr)
        for (int i = 0; i < nseg; ++i) direct_out[i] = direct[i];
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    cudaError_t err = cudaSuccess;
    // The direct copies go first (the DMA has work from t = 0 while the first
    // units are packed); ADT_H2D_DIRECT_LAST=1 queues them after the packed
    // stream instead (A/B: the packed runs then ship while the host packs, the
    // direct layers once the host is idle).
    static const bool direct_last = [] {
        const char *e = getenv("ADT_H2D_DIRECT_LAST");
        return e != nullptr && e[0] == '1';
    }();
    auto ship_direct = [&] {
        for (int i = 0; i < nseg && err == cudaSuccess; ++i)
            if (direct[i])
                err = cudaMemcpyAsync(dev_segs[i].weights, host_segs[i].weights, host_segs[i].count * 4,
                                      cudaMemcpyHostToDevice, st);
    };
    if (!direct_last) ship_direct();
    // byte runs of the stream the DMA must carry: the packed layers' payloads,
    // neighbours merged when only the inter-layer pad separates them
    struct Run { uint64_t a, b; };
    std::vector<Run> runs;
    for (int i = 0; i < nseg && !zero_copy; ++i) {
        const adt_segment &h = host_segs[i];
        if (h.count == 0 || direct[i]) continue;
        const uint64_t a = h.offset, b = h.offset + h.count * static_cast<uint64_t>(h.round_to);
        if (!runs.empty() && a - runs.back().b < kRunMergeGap) runs.back().b = b;
        else runs.push_back({a, b});
    }
    // units: the direct layers' norm-only units first (while the DMA reads the
    // same words), then the packed layers' units in stream order
    std::vector<Unit> units;
    const bool skip_direct_norms = (flags & ADT_H2D_SKIP_DIRECT_NORMS) != 0;
    const uint64_t unit = unit_weights(host_segs, nseg);
    if (seg_sumsq != nullptr && !skip_direct_norms)
        for (int s = 0; s < nseg; ++s)
            if (direct[s]) add_units(units, host_segs, s, unit);
    const size_t nnorm = units.size();
    for (int s = 0; s < nseg; ++s)
        if (!direct[s]) add_units(units, host_segs, s, unit);
    std::vector<double> ss(units.size(), 0.0);
    // byte range of the packed stream that is final once units [0, k) are done:
    // [0, start of unit k) — nothing while the norm-only units run
    auto ready_bytes = [&](size_t k) -> uint64_t {
        if (k >= units.size()) return packed_bytes;
        if (k < nnorm) return 0;
        const adt_segment &s = host_segs[units[k].seg];
        return s.offset + units[k].lo * static_cast<uint64_t>(s.round_to);
    };
    size_t run = 0;
    auto ship = [&](uint64_t a, uint64_t b) {      // copy the runs' bytes inside [a, b)
        while (run < runs.size() && err == cudaSuccess) {
            const uint64_t lo = std::max(a, runs[run].a), hi = std::min(b, runs[run].b);
            if (lo < hi)
                err = cudaMemcpyAsync(dev_packed + lo, host_packed + lo, hi - lo, cudaMemcpyHostToDevice, st);
            if (runs[run].b > b) break;            // the rest of this run ships with a later range
            ++run;
        }
    };
    uint64_t sent = 0;
    // 0 = automatic: 1 MiB copies, or for a small stream quarters of it (>= 64 KiB)
    // so its DMA starts before the last unit is packed
    const uint64_t batch = min_copy_bytes != 0 ? min_copy_bytes
                                               : std::min<uint64_t>(1u << 20, std::max<uint64_t>(64u << 10, packed_bytes / 4));
    pack_units(host_segs, units, nnorm, host_packed, resolve_threads(threads), ss, [&](size_t prefix) {
        const uint64_t end = ready_bytes(prefix);
        if (err != cudaSuccess || end <= sent) return;
        if (end - sent < batch && prefix < units.size()) return;
        ship(sent, end);
        sent = end;
    }, caller_packs_h2d());
    if (direct_last) ship_direct();
    finish_sums(units, ss, nseg, seg_sumsq);
    if (seg_sumsq != nullptr && skip_direct_norms)
        for (int i = 0; i < nseg; ++i)
            if (direct[i]) seg_sumsq[i] = __builtin_nan("");     // the caller's to fill (device pass)
    if (err != cudaSuccess) return ADT_ERR_CUDA_BASE - static_cast<int>(err);
    if (dev_segs == nullptr) return ADT_OK;
    bool any_direct = false;
    for (int i = 0; i < nseg; ++i) any_direct = any_direct || direct[i];
    const uint8_t *src = zero_copy ? mapped : dev_packed;
    if (!any_direct) return adt_unpack(dev_segs, nseg, src, stream);
    std::vector<adt_segment> rest(dev_segs, dev_segs + nseg);     // the direct layers are complete already
    for (int i = 0; i < nseg; ++i)
        if (direct[i]) rest[i].count = 0;
    return adt_unpack(rest.data(), nseg, src, stream);
}

int adt_host_to_device_ring(const adt_segment *host_segs, const adt_segment *dev_segs, int nseg, uint8_t *ring,
                            uint64_t ring_bytes, uint64_t slot_bytes, uint8_t *dev_packed, uint64_t packed_bytes,
                            double *seg_sumsq, int threads, void *stream) {
    int v = validate_host(host_segs, nseg, ring);
    if (v != ADT_OK) return v;
    if (nseg > 0 && dev_packed == nullptr) return ADT_ERR_ARG;
    if (ring == nullptr || reinterpret_cast<uintptr_t>(ring) % 64 || slot_bytes % 64 ||
        slot_bytes < kUnitWeights * 4 + 64 || ring_bytes < 2 * slot_bytes)   // a slot holds any one unit + pad
        return ADT_ERR_ARG;
    uint64_t end_prev = 0;
    for (int i = 0; i < nseg; ++i) {
        const adt_segment &h = host_segs[i];
        if (dev_segs != nullptr) {
            const adt_segment &d = dev_segs[i];
            if (h.count != d.count || h.offset != d.offset || h.round_to != d.round_to) return ADT_ERR_ARG;
        }
        if (h.count == 0) continue;
        const uint64_t end = h.offset + h.count * static_cast<uint64_t>(h.round_to);
        if (h.offset < end_prev || end > packed_bytes) return ADT_ERR_ARG;
        end_prev = end;
    }
    const std::vector<Unit> units = make_units(host_segs, nseg);
    std::vector<double> ss(units.size(), 0.0);
    auto start_of = [&](size_t k) -> uint64_t {
        if (k >= units.size()) return packed_bytes;
        const adt_segment &s = host_segs[units[k].seg];
        return s.offset + units[k].lo * static_cast<uint64_t>(s.round_to);
    };
    // chunks: runs of consecutive units whose stream span [a, b) (b = the next
    // chunk's start: inter-layer pad included) fits one ring slot
    struct Chunk { uint64_t a, b; size_t u0, u1; };
    std::vector<Chunk> chunks;
    for (size_t k = 0; k < units.size();) {
        const uint64_t a = start_of(k);
        size_t e = k + 1;
        while (e < units.size() && start_of(e + 1) - a <= slot_bytes) ++e;
        chunks.push_back({a, start_of(e), k, e});
        k = e;
    }
    const size_t nc = chunks.size();
    const int nslots = static_cast<int>(std::min<uint64_t>(ring_bytes / slot_bytes, 1024));
    const int nthreads = resolve_threads(threads);
    if (nslots <= nthreads) return ADT_ERR_ARG;      // every in-flight chunk needs its own slot
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    std::vector<cudaEvent_t> ev(nslots, nullptr);
    for (auto &e : ev)
        if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) e = nullptr;
    std::unique_ptr<std::atomic<uint8_t>[]> done(new std::atomic<uint8_t>[nc == 0 ? 1 : nc]);
    std::unique_ptr<std::atomic<int64_t>[]> issued(new std::atomic<int64_t>[nslots]);
    for (size_t i = 0; i < nc; ++i) done[i].store(0, std::memory_order_relaxed);
    for (int i = 0; i < nslots; ++i) issued[i].store(-1, std::memory_order_relaxed);
    std::atomic<size_t> next{0};
    std::atomic<int> failed{0};
    const bool nt = getenv("ADT_RING_NT") != nullptr && getenv("ADT_RING_NT")[0] == '1';
    // packers: chunk c -> slot c % nslots, after the copy of chunk c - nslots has left it
    const std::function<void(int)> job = [&](int) {
        for (size_t c; (c = next.fetch_add(1, std::memory_order_relaxed)) < nc;) {
            const int slot = static_cast<int>(c % nslots);
            if (c >= static_cast<size_t>(nslots)) {
                const int64_t prev = static_cast<int64_t>(c) - nslots;
                while (issued[slot].load(std::memory_order_acquire) < prev && !failed.load()) _mm_pause();
                if (ev[slot] != nullptr) cudaEventSynchronize(ev[slot]);
            }
            uint8_t *base = ring + static_cast<uint64_t>(slot) * slot_bytes;
            const Chunk &ch = chunks[c];
            for (size_t k = ch.u0; k < ch.u1; ++k) {
                const Unit &u = units[k];
                ss[k] = pack_unit_to(host_segs[u.seg], u.lo, u.hi, base + (start_of(k) - ch.a), nt);
            }
            done[c].store(1, std::memory_order_release);
        }
    };
    cudaError_t err = cudaSuccess;
    // the caller: issues each chunk's copy (in order) as soon as it is packed
    const std::function<void()> caller = [&] {
        for (size_t c = 0; c < nc; ++c) {
            while (!done[c].load(std::memory_order_acquire)) _mm_pause();
            const int slot = static_cast<int>(c % nslots);
            if (err == cudaSuccess)
                err = cudaMemcpyAsync(dev_packed + chunks[c].a, ring + static_cast<uint64_t>(slot) * slot_bytes,
                                      chunks[c].b - chunks[c].a, cudaMemcpyHostToDevice, st);
            if (err == cudaSuccess && ev[slot] != nullptr) err = cudaEventRecord(ev[slot], st);
            if (err != cudaSuccess) failed.store(1);
            issued[slot].store(static_cast<int64_t>(c), std::memory_order_release);
        }
    };
    // the caller only issues copies: nthreads - 1 pool threads pack (plus one extra when available)
    Pool::get().run(nthreads + 1, job, caller);
    for (auto &e : ev)
        if (e != nullptr) cudaEventDestroy(e);
    finish_sums(units, ss, nseg, seg_sumsq);
    if (err != cudaSuccess) return ADT_ERR_CUDA_BASE - static_cast<int>(err);
    return dev_segs == nullptr ? ADT_OK : adt_unpack(dev_segs, nseg, dev_packed, stream);
}

}  // extern "C"
