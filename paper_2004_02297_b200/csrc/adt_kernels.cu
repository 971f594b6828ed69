// adt_kernels.cu — sm_100a kernels and the C ABI (include/adt.h) of the ADT codec.
//
// What the reference computes (pure NumPy, /root/reference/pkg/src/weightpack):
//   pack    codec.py:116-180  keep the top r bytes of every FP32 word, MSB first
//   unpack  codec.py:183-197  kept bytes -> word MSBs, low bytes zero
//   norm    precision.py:25-28 float64 l2-norm of a layer's master weights
//
// B200 design: the path is pure byte movement, HBM-bound
// (pack reads 4n and writes r*n bytes; unpack the reverse), so the kernels are
// built around coalesced 128-bit traffic, not tensor cores:
//   * multi-tensor: one launch walks a per-layer descriptor table passed by
//     value in kernel parameter space (__grid_constant__, up to 256 layers per
//     launch); each CTA owns one 4096-weight tile of one layer and finds its
//     layer from a coarse tile->layer hint table in the same parameter block;
//   * byte compaction with PRMT (__byte_perm): r = 1, 2, 4 are warp-coalesced
//     32/64/128-bit stores straight from registers; r = 3 (12 bytes per 4
//     weights) and ragged tiles are staged per warp in shared memory and leave
//     as one bulk async copy (cp.async.bulk);
//   * the layer's float64 sum of squares is fused into the pack pass (every
//     weight is read once): one partial per warp slice, plain stores, summed
//     in a fixed order by a small finalize kernel, so norms are run-to-run
//     bit-identical (no floating-point atomics).
//
// One translation unit: this file (tables, tile helpers, pack / unpack /
// finalize kernels, host launch code, C ABI) includes adt_sgd.cuh (fused
// optimizer step + pack), adt_peer.cuh (peer-memory barrier and copies),
// adt_awp.cuh (device-resident AWP) and adt_tma.cuh (the TMA A/B family).

#include <cuda_runtime.h>
#include <stdint.h>
#include <limits.h>
#include <stdlib.h>
#include <string.h>
#include <dlfcn.h>

#include "adt.h"
#include <math_constants.h>

namespace {

constexpr int kThreads = 256;                      // 8 warps per CTA
constexpr int kVec = 4;                            // float4 groups per thread per tile
constexpr int kTile = kThreads * kVec * 4;         // weights per tile
static_assert(kTile == ADT_TILE_WEIGHTS, "tile size is part of the ABI");

template <int MAXSEG>
struct Table {
    const uint8_t *srcs[ADT_MAX_SOURCES];  // unpack sources (device, peer-mapped or pinned host)
    uint8_t *packed_out;        // pack destination
    double *seg_sumsq;          // per-layer result (chunk-relative)
    double *partials;           // per-tile scratch (chunk-relative)
    int nseg;
    uint32_t tile_begin[MAXSEG + 1];
    uint64_t count[MAXSEG];
    uint64_t offset[MAXSEG];
    uintptr_t weights[MAXSEG];
    uint8_t round_to[MAXSEG];
    uint8_t src_idx[MAXSEG];    // which srcs[] a layer's payload is read from (adt_unpack_multi)
    // Coarse tile -> layer map: seg_hint[k] = the layer holding tile k << hint_shift
    // (<= kHints buckets). A CTA starts its layer search there and steps forward
    // over the few layer boundaries inside its bucket, instead of a per-warp
    // binary search over the whole table (~70 warp instructions for 161 layers).
    uint32_t hint_shift;
    uint8_t seg_hint[1024];
    // Device-resident AWP (adt_pack_dyn / adt_unpack_dyn): per-layer widths read
    // from device memory (chunk-relative) instead of round_to[], so a width
    // change decided on the device needs no new launch table. nullptr = round_to[].
    const uint8_t *dyn_r;
    uint32_t tile_rot;           // unpack: the tile walk starts rotated by this many tiles (< ntiles)
    // Peer-abort guard (p2p transport): the peer barrier's timeout word. When
    // it is nonzero at kernel start the kernel does no work, so a stalled or
    // dead peer never lets stale / half-written peer bytes reach a replica or
    // a master (the host raises at its next poll). nullptr = unguarded.
    const uint32_t *abort;
};
constexpr int kHints = 1024;

__device__ __forceinline__ bool aborted(const uint32_t *word) {
    return word != nullptr && *reinterpret_cast<const volatile uint32_t *>(word) != 0u;
}

template <int MAXSEG>
__device__ __forceinline__ int width_of(const Table<MAXSEG> &T, int s) {
    return T.dyn_r != nullptr ? static_cast<int>(T.dyn_r[s]) : static_cast<int>(T.round_to[s]);
}

// ----------------------------------------------------------- byte compaction
// Word w of the layer is little-endian in memory (byte 3 = MSB). The payload
// wants the MSBs first: for 4 consecutive words a,b,c,d and r kept bytes the
// payload is a3..a(4-r) b3.. c3.. d3.. — r 32-bit payload words per 4 weights.
__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
    return __byte_perm(a, b, sel);
}

__device__ __forceinline__ void pack_r1(const uint4 &v, uint32_t *o) {
    o[0] = prmt(prmt(v.x, v.y, 0x0073), prmt(v.z, v.w, 0x0073), 0x5410);
}
__device__ __forceinline__ void pack_r2(const uint4 &v, uint32_t *o) {
    o[0] = prmt(v.x, v.y, 0x6723);
    o[1] = prmt(v.z, v.w, 0x6723);
}
__device__ __forceinline__ void pack_r3(const uint4 &v, uint32_t *o) {
    o[0] = prmt(v.x, v.y, 0x7123);
    o[1] = prmt(v.y, v.z, 0x6712);
    o[2] = prmt(v.z, v.w, 0x5671);
}
__device__ __forceinline__ void pack_r4(const uint4 &v, uint32_t *o) {
    o[0] = prmt(v.x, 0, 0x0123);
    o[1] = prmt(v.y, 0, 0x0123);
    o[2] = prmt(v.z, 0, 0x0123);
    o[3] = prmt(v.w, 0, 0x0123);
}
__device__ __forceinline__ void pack_any(int r, const uint4 &v, uint32_t *o) {
    switch (r) {
        case 1: pack_r1(v, o); break;
        case 2: pack_r2(v, o); break;
        case 3: pack_r3(v, o); break;
        default: pack_r4(v, o); break;
    }
}

__device__ __forceinline__ uint4 unpack_r1(uint32_t p) {
    return make_uint4(prmt(p, 0, 0x0444), prmt(p, 0, 0x1444), prmt(p, 0, 0x2444), prmt(p, 0, 0x3444));
}
__device__ __forceinline__ uint4 unpack_r2(uint32_t p, uint32_t q) {
    return make_uint4(prmt(p, 0, 0x0144), prmt(p, 0, 0x2344), prmt(q, 0, 0x0144), prmt(q, 0, 0x2344));
}
__device__ __forceinline__ uint4 unpack_r3(uint32_t p, uint32_t q, uint32_t s) {
    return make_uint4(prmt(p, 0, 0x0124), prmt(p, q, 0x3450) & 0xFFFFFF00u,
                      prmt(q, s, 0x2340) & 0xFFFFFF00u, prmt(s, 0, 0x1234));
}
__device__ __forceinline__ uint4 unpack_r4(const uint4 &p) {
    return make_uint4(prmt(p.x, 0, 0x0123), prmt(p.y, 0, 0x0123), prmt(p.z, 0, 0x0123), prmt(p.w, 0, 0x0123));
}
__device__ __forceinline__ uint4 unpack_words(int r, const uint32_t *w) {
    switch (r) {
        case 1: return unpack_r1(w[0]);
        case 2: return unpack_r2(w[0], w[1]);
        case 3: return unpack_r3(w[0], w[1], w[2]);
        default: return unpack_r4(make_uint4(w[0], w[1], w[2], w[3]));
    }
}

// ------------------------------------------------------------------ helpers
template <int MAXSEG>
__device__ __forceinline__ int find_segment(const Table<MAXSEG> &T, uint32_t tile) {
    // last s with tile_begin[s] <= tile (zero-tile layers are never selected;
    // tile_begin[nseg] = the tile count stops the walk)
    int s = T.seg_hint[tile >> T.hint_shift];
    while (T.tile_begin[s + 1] <= tile) ++s;
    return s;
}

// Host: fill hint_shift / seg_hint for a table whose tile_begin[0..nseg] is set.
template <typename Tab>
void fill_hints(Tab &T, int nseg, uint32_t ntiles) {
    uint32_t shift = 0;
    while ((static_cast<uint64_t>(ntiles) >> shift) >= static_cast<uint64_t>(kHints)) ++shift;
    T.hint_shift = shift;
    int seg = 0;
    const uint32_t nb = ntiles == 0 ? 0 : ((ntiles - 1) >> shift) + 1;
    for (uint32_t k = 0; k < static_cast<uint32_t>(kHints); ++k) {
        const uint32_t tile = k < nb ? (k << shift) : 0;
        if (k < nb)
            while (seg + 1 < nseg && T.tile_begin[seg + 1] <= tile) ++seg;
        T.seg_hint[k] = static_cast<uint8_t>(k < nb ? seg : 0);
    }
}

// float32 -> float64 widening on the integer pipe. cvt.f64.f32 (F2F) issues on
// the XU pipe, which ncu showed as the pack+norm bottleneck (58.6% XU, see
// profiles/r01_v1_*); rebuilding the double from the float's bits is exact for
// normal numbers, and zeros / subnormals / inf / NaN (rare) fall back to F2F.
__device__ __forceinline__ double widen(uint32_t w) {
    const uint32_t a = w & 0x7FFFFFFFu;           // |x| (the square ignores the sign)
    if (a - 0x00800000u < 0x7F000000u) {          // 0 < exponent < 255
        return __hiloint2double(static_cast<int>((a >> 3) + (896u << 20)), static_cast<int>(a << 29));
    }
    return a == 0u ? 0.0 : static_cast<double>(__uint_as_float(a));
}

__device__ __forceinline__ double sq_acc(double acc, uint32_t w) {
    const double d = widen(w);  // exact
    return fma(d, d, acc);      // exact square, rounded add
}

// Norm partials: ONE float64 per warp per tile (kWarpsPerTile per tile), a
// fixed-order shuffle reduction and one plain store by lane 0 — no CTA barrier,
// fence or atomic on the pack path (an earlier per-CTA fence + L2 atomic kept
// every CTA resident ~1 us longer, profiles/r01_v1_*). adt_norm_finalize_kernel
// sums a layer's partials in (tile, warp) order.
constexpr int kWarpsPerTile = kThreads / 32;
__device__ __forceinline__ void warp_partial(double *partials, uint32_t tile, double acc,
                                             int warp = static_cast<int>(threadIdx.x >> 5)) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xFFFFFFFFu, acc, o);
    if ((threadIdx.x & 31) == 0) partials[tile * kWarpsPerTile + warp] = acc;
}

// Per layer (one CTA each): fixed-order sum of its partials -> seg_sumsq.
// Launched behind the pack pass (programmatic dependent launch) or on a side
// stream by the caller (adt_norm_finalize). Thread t sums partials t, t+1024,
// t+2048, ... (coalesced; 8 loads in flight), then a fixed shuffle/CTA tree.
// (A contiguous-run-per-thread version was uncoalesced: 28 us for AlexNet.)
// The order depends only on the layer's partial count: bit-identical results.
#ifndef ADT_FIN_THREADS
#define ADT_FIN_THREADS 1024
#endif
constexpr int kFinThreads = ADT_FIN_THREADS;
template <int MAXSEG>
__global__ void __launch_bounds__(kFinThreads)
adt_norm_finalize_kernel(const __grid_constant__ Table<MAXSEG> T) {
#if __CUDA_ARCH__ >= 900
    asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
    __shared__ double red[kFinThreads / 32];
    const int s = blockIdx.x;
    const uint32_t lo = T.tile_begin[s] * kWarpsPerTile;
    const uint32_t n = (T.tile_begin[s + 1] - T.tile_begin[s]) * kWarpsPerTile;
    const double *p = T.partials + lo;
    double a = 0.0;
    uint32_t i = threadIdx.x;
    for (; i + 7 * kFinThreads < n; i += 8 * kFinThreads) {
        double x[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) x[j] = p[i + j * kFinThreads];
#pragma unroll
        for (int j = 0; j < 8; ++j) a += x[j];
    }
    for (; i < n; i += kFinThreads) a += p[i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) a += __shfl_down_sync(0xFFFFFFFFu, a, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = a;
    __syncthreads();
    if (threadIdx.x == 0) {
        double tot = 0.0;
#pragma unroll
        for (int w = 0; w < kFinThreads / 32; ++w) tot += red[w];
        T.seg_sumsq[s] = tot;  // 0.0 for empty layers
    }
}

// ---------------------------------------------------------------- pack pass
// Mapping: warp w owns the tile's float4 groups [128w, 128w+128) (512 weights),
// lane l handles groups 128w + 32j + l (j = 0..3): every load and every
// direct store instruction of a warp is one contiguous, coalesced span.
// r = 3 (12 bytes per group) and ragged last tiles go through a per-warp
// shared-memory staging area and leave as 16-byte vectors; only __syncwarp is
// needed, so no warp ever waits for another (no CTA barriers in the pack).
constexpr int kWarpGroups = kTile / 4 / kWarpsPerTile;       // 128
constexpr int kWarpStageWords = kWarpGroups * 4;              // <= r words per group, r <= 4

// Float64 sum of squares of the 16 words a thread holds. Fast path (all
// normal numbers, checked with two unsigned min/max per word): rebuild each
// double from the float's bits on the integer pipe, no per-word branch.
// Otherwise (zero / subnormal / inf / NaN present): per-word widen().
__device__ __forceinline__ double sumsq16(const uint4 (&v)[kVec]) {
    uint32_t lo = 0xFFFFFFFFu, hi = 0u;
#pragma unroll
    for (int k = 0; k < kVec; ++k) {
        const uint32_t w[4] = {v[k].x, v[k].y, v[k].z, v[k].w};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const uint32_t a = w[j] & 0x7FFFFFFFu;
            lo = min(lo, a);
            hi = max(hi, a);
        }
    }
    double acc = 0.0;
    if (lo >= 0x00800000u && hi < 0x7F800000u) {
#pragma unroll
        for (int k = 0; k < kVec; ++k) {
            const uint32_t w[4] = {v[k].x, v[k].y, v[k].z, v[k].w};
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const uint32_t a = w[j] & 0x7FFFFFFFu;
                const double d = __hiloint2double(static_cast<int>((a >> 3) + (896u << 20)),
                                                  static_cast<int>(w[j] << 29));
                acc = fma(d, d, acc);
            }
        }
    } else {
#pragma unroll
        for (int k = 0; k < kVec; ++k) {
            acc = sq_acc(acc, v[k].x);
            acc = sq_acc(acc, v[k].y);
            acc = sq_acc(acc, v[k].z);
            acc = sq_acc(acc, v[k].w);
        }
    }
    return acc;
}

// Copy `nbytes` from a warp's staging words to global, 16-byte vectors first.
__device__ __forceinline__ void warp_store_bytes(const uint32_t *ws, uint8_t *dst, uint32_t nbytes, int lane) {
    const uint32_t n16 = nbytes / 16;
    const uint4 *s4 = reinterpret_cast<const uint4 *>(ws);
    uint4 *d4 = reinterpret_cast<uint4 *>(dst);
    for (uint32_t i = lane; i < n16; i += 32) d4[i] = s4[i];
    const uint8_t *s1 = reinterpret_cast<const uint8_t *>(ws);
    for (uint32_t i = n16 * 16 + lane; i < nbytes; i += 32) dst[i] = s1[i];
}

#ifndef ADT_PACK_STAGE_ALL
#define ADT_PACK_STAGE_ALL 0    // A/B: route r = 1/2/4 full tiles through the staged (bulk-store) path too
#endif
#ifndef ADT_PACK_BULK_STORE
#define ADT_PACK_BULK_STORE 1   // A/B (profiles/r01_ab_bulk_store.md): 1B r=3 step 2308 -> 2183 us
#endif
// Write a tile's packed bytes (the r top bytes of each of the thread's 16 words).
// r = 1/2/4 full tiles: coalesced 32/64/128-bit stores straight from registers;
// r = 3 and ragged tiles: the warp's span via its staging words, 16-B vectors.
#ifndef ADT_PACK_EVICT_LAST
#define ADT_PACK_EVICT_LAST 0   // A/B: packed-stream stores with an L2 evict_last policy
#endif
__device__ __forceinline__ uint64_t l2_keep_policy() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ void st_keep(uint32_t *a, uint32_t x, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.b32 [%0], %1, %2;" ::"l"(a), "r"(x), "l"(pol) : "memory");
}
__device__ __forceinline__ void st_keep(uint2 *a, uint2 x, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.v2.b32 [%0], {%1, %2}, %3;" ::"l"(a), "r"(x.x), "r"(x.y), "l"(pol) : "memory");
}
__device__ __forceinline__ void st_keep(uint4 *a, uint4 x, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.v4.b32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(a), "r"(x.x), "r"(x.y), "r"(x.z),
                 "r"(x.w), "l"(pol) : "memory");
}
template <typename V>
__device__ __forceinline__ void st_packed(V *a, V x) {
    if (ADT_PACK_EVICT_LAST) st_keep(a, x, l2_keep_policy());
    else *a = x;
}

template <bool BULK = (ADT_PACK_BULK_STORE != 0)>
__device__ __forceinline__ void store_packed(uint8_t *dst, const uint4 (&v)[kVec], uint32_t m, int r, int warp,
                                             int lane, uint32_t g0, uint32_t *ws) {
    if (!ADT_PACK_STAGE_ALL && m == kTile && r != 3) {
        if (r == 1) {
            uint32_t *d = reinterpret_cast<uint32_t *>(dst);
#pragma unroll
            for (int k = 0; k < kVec; ++k) { uint32_t o[1]; pack_r1(v[k], o); st_packed(d + g0 + 32 * k, o[0]); }
        } else if (r == 2) {
            uint2 *d = reinterpret_cast<uint2 *>(dst);
#pragma unroll
            for (int k = 0; k < kVec; ++k) { uint32_t o[2]; pack_r2(v[k], o); st_packed(d + g0 + 32 * k, make_uint2(o[0], o[1])); }
        } else {
            uint4 *d = reinterpret_cast<uint4 *>(dst);
#pragma unroll
            for (int k = 0; k < kVec; ++k) {
                uint32_t o[4];
                pack_r4(v[k], o);
                st_packed(d + g0 + 32 * k, make_uint4(o[0], o[1], o[2], o[3]));
            }
        }
        return;
    }
    if (r == 3) {
#pragma unroll
        for (int k = 0; k < kVec; ++k) {
            uint32_t o[3];
            pack_r3(v[k], o);
            uint32_t *p = ws + (lane + 32 * k) * 3;   // stride 3: conflict-free
            p[0] = o[0]; p[1] = o[1]; p[2] = o[2];
        }
    } else {
#pragma unroll
        for (int k = 0; k < kVec; ++k) {
            uint32_t o[4];
            pack_any(r, v[k], o);
            uint32_t *p = ws + (lane + 32 * k) * r;
            p[0] = o[0];
            if (r > 1) p[1] = o[1];
            if (r > 2) p[2] = o[2];
            if (r > 3) p[3] = o[3];
        }
    }
    const uint32_t span = kWarpGroups * 4 * r;            // the warp's packed bytes
    const uint32_t lo = warp * span, nbytes = m * r;
    if (!BULK) {                                          // plain generic-proxy stores (adt_roundtrip)
        __syncwarp();
        if (lo < nbytes) warp_store_bytes(ws, dst + lo, min(span, nbytes - lo), lane);
        __syncwarp();
        return;
    }
#if ADT_PACK_BULK_STORE
    // The warp's 16-B-multiple part leaves shared memory as ONE bulk async copy
    // (cp.async.bulk shared->global, SASS UBLKCP) issued by lane 0; the ragged
    // (< 16 B) tail of a layer goes out with plain stores.
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // STS -> async proxy
    __syncwarp();
    if (lo < nbytes) {
        const uint32_t mine = min(span, nbytes - lo), n16 = mine & ~15u;
        if (lane == 0 && n16) {
            if (ADT_PACK_EVICT_LAST) {
                asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;\n\t"
                             "cp.async.bulk.commit_group;\n\t"
                             "cp.async.bulk.wait_group.read 0;" ::"l"(dst + lo),
                             "r"(static_cast<uint32_t>(__cvta_generic_to_shared(ws))), "r"(n16), "l"(l2_keep_policy())
                             : "memory");
            } else {
                asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n\t"
                             "cp.async.bulk.commit_group;\n\t"
                             "cp.async.bulk.wait_group.read 0;" ::"l"(dst + lo),
                             "r"(static_cast<uint32_t>(__cvta_generic_to_shared(ws))), "r"(n16) : "memory");
            }
        }
        const uint8_t *s1 = reinterpret_cast<const uint8_t *>(ws);
        for (uint32_t i = n16 + lane; i < mine; i += 32) dst[lo + i] = s1[i];
    }
#else
    __syncwarp();
    if (lo < nbytes) warp_store_bytes(ws, dst + lo, min(span, nbytes - lo), lane);
#endif
    (void)warp_store_bytes;
    __syncwarp();
}

#ifndef ADT_PDL
// 1: pack triggers its dependents early and the unpack launches as a
// programmatic dependent. Measured (profiles/r02_ab_pdl.md): ResNet-50 step
// -0.6 us, but AlexNet +4.2 us and VGG-16 +12 us — the early-resident unpack
// CTAs keep the side-stream finalize off the SMs and slow the unpack itself.
// Off; with 1 the runtime switch ADT_PDL=0 disables the launch attribute.
#define ADT_PDL 0
#endif
// WRITE=false is the norm-only pass (adt_sumsq).
#ifndef ADT_PACK_MIN_BLOCKS
#define ADT_PACK_MIN_BLOCKS 6   // resident CTAs/SM the register budget must allow (A/B: profiles/r01_ab_occupancy.md)
#endif
// ADT_PERSISTENT = 1: grid = resident CTAs, each CTA walks tiles blockIdx.x,
// blockIdx.x + gridDim.x, ... and tracks its layer incrementally, instead of
// one CTA per tile with a per-warp binary search over the layer table (the
// search was ~25 % of the pack's and ~50 % of the unpack's instructions on
// ResNet-50's 161 layers, profiles/r01d). Results do not depend on it.
#ifndef ADT_PERSISTENT
#define ADT_PERSISTENT 0
#endif

template <int MAXSEG, bool NORM, bool WRITE, bool BULK = (ADT_PACK_BULK_STORE != 0)>
__device__ __forceinline__ void pack_tile(const Table<MAXSEG> &T, uint32_t tile, int s, uint32_t *ws,
                                          int warp = static_cast<int>(threadIdx.x >> 5)) {
    const uint64_t e0 = static_cast<uint64_t>(tile - T.tile_begin[s]) * kTile;
    const uint32_t m = static_cast<uint32_t>(min(static_cast<uint64_t>(kTile), T.count[s] - e0));
    const int r = width_of(T, s);
    const int lane = threadIdx.x & 31;
    const uint32_t g0 = warp * kWarpGroups + lane;                 // group of j = 0
    const uint4 *src = reinterpret_cast<const uint4 *>(T.weights[s]) + e0 / 4;

    uint4 v[kVec];
    if (m == kTile) {
#pragma unroll
        for (int k = 0; k < kVec; ++k) v[k] = __ldcs(src + g0 + 32 * k);
    } else {
        const uint32_t *src1 = reinterpret_cast<const uint32_t *>(src);
#pragma unroll
        for (int k = 0; k < kVec; ++k) {
            const uint32_t g = g0 + 32 * k, i = g * 4;
            if (i + 4 <= m) {
                v[k] = __ldcs(src + g);
            } else {
                uint32_t w[4];
#pragma unroll
                for (int j = 0; j < 4; ++j) w[j] = (i + j < m) ? src1[i + j] : 0u;
                v[k] = make_uint4(w[0], w[1], w[2], w[3]);
            }
        }
    }

    if (WRITE) store_packed<BULK>(T.packed_out + T.offset[s] + e0 * r, v, m, r, warp, lane, g0, ws);

    if (NORM) warp_partial(T.partials, tile, sumsq16(v), warp);
}

// Split CTAs (ADT_CTA_WARPS = 4 or 2): a CTA of kCtaWarps warps runs warps
// [sub*kCtaWarps, (sub+1)*kCtaWarps) of tile blockIdx.x / kSplit — the same
// per-warp slices, bytes and norm partials as one 8-warp CTA per tile, in
// shorter-lived CTAs (a smaller drain tail at the end of the grid). A/B.
#ifndef ADT_CTA_WARPS
#define ADT_CTA_WARPS 8
#endif
constexpr int kCtaWarps = ADT_CTA_WARPS;
constexpr int kCtaThreads = 32 * kCtaWarps;
constexpr int kSplit = kWarpsPerTile / kCtaWarps;
static_assert(kSplit * kCtaWarps == kWarpsPerTile, "CTA warps must divide the tile's warps");

template <int MAXSEG, bool NORM, bool WRITE>
__global__ void __launch_bounds__(kCtaThreads, ADT_PACK_MIN_BLOCKS * kSplit)
adt_pack_kernel(const __grid_constant__ Table<MAXSEG> T, uint32_t ntiles) {
    __shared__ __align__(16) uint32_t stage[kCtaWarps][kWarpStageWords];
    uint32_t *ws = stage[threadIdx.x >> 5];
#if ADT_PDL && __CUDA_ARCH__ >= 900
    // Let a programmatic dependent (finalize, unpack) be scheduled as soon as
    // every pack CTA has started: its launch and CTA rasterisation overlap the
    // pack's last wave; it still reads nothing before griddepcontrol.wait,
    // which waits for this whole grid and its memory operations.
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
    if (!ADT_PERSISTENT) {
        const uint32_t tile = blockIdx.x / kSplit;
        const int warp = static_cast<int>(blockIdx.x % kSplit) * kCtaWarps + static_cast<int>(threadIdx.x >> 5);
        pack_tile<MAXSEG, NORM, WRITE>(T, tile, find_segment(T, tile), ws, warp);
        return;
    }
    int s = find_segment(T, blockIdx.x);
    for (uint32_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        while (T.tile_begin[s + 1] <= tile) ++s;                   // tile_begin[nseg] = ntiles stops it
        pack_tile<MAXSEG, NORM, WRITE>(T, tile, s, ws);
    }
}

// -------------------------------------------------------------- unpack pass
#ifndef ADT_UNPACK_MIN_BLOCKS
#define ADT_UNPACK_MIN_BLOCKS 5
#endif
#ifndef ADT_FIXUP_CTAS_PER_SM
#define ADT_FIXUP_CTAS_PER_SM 4   // adt_awp_fixup grid (its CTAs exit after one load when nothing escalated)
#endif
#ifndef ADT_UNPACK_STCS
#define ADT_UNPACK_STCS 2      // replica stores evict-first, direct (1) and staged (2) paths (profiles/r01_ab_layer_hint.md)
#endif
#ifndef ADT_UNPACK_REVERSE
#define ADT_UNPACK_REVERSE 1   // A/B: AlexNet step 132.7 -> 127.2 us (profiles/r01_ab_unpack_order.md)
#endif
template <int MAXSEG>
__device__ __forceinline__ void unpack_tile(const Table<MAXSEG> &T, uint32_t tile, int s, uint32_t *ws,
                                            int warp = static_cast<int>(threadIdx.x >> 5)) {
    const uint64_t e0 = static_cast<uint64_t>(tile - T.tile_begin[s]) * kTile;
    const uint32_t m = static_cast<uint32_t>(min(static_cast<uint64_t>(kTile), T.count[s] - e0));
    const int r = width_of(T, s);
    const int lane = threadIdx.x & 31;
    const uint32_t g0 = warp * kWarpGroups + lane;
    const uint8_t *src = T.srcs[T.src_idx[s]] + T.offset[s] + e0 * r;
    uint4 *dst = reinterpret_cast<uint4 *>(T.weights[s]) + e0 / 4;

    if (m == kTile && r != 3) {
        uint4 out[kVec];
        if (r == 1) {
            const uint32_t *p = reinterpret_cast<const uint32_t *>(src);
            uint32_t w[kVec];
#pragma unroll
            for (int k = 0; k < kVec; ++k) w[k] = __ldcs(p + g0 + 32 * k);
#pragma unroll
            for (int k = 0; k < kVec; ++k) out[k] = unpack_r1(w[k]);
        } else if (r == 2) {
            const uint2 *p = reinterpret_cast<const uint2 *>(src);
            uint2 w[kVec];
#pragma unroll
            for (int k = 0; k < kVec; ++k) w[k] = __ldcs(p + g0 + 32 * k);
#pragma unroll
            for (int k = 0; k < kVec; ++k) out[k] = unpack_r2(w[k].x, w[k].y);
        } else {
            const uint4 *p = reinterpret_cast<const uint4 *>(src);
            uint4 w[kVec];
#pragma unroll
            for (int k = 0; k < kVec; ++k) w[k] = __ldcs(p + g0 + 32 * k);
#pragma unroll
            for (int k = 0; k < kVec; ++k) out[k] = unpack_r4(w[k]);
        }
#pragma unroll
        for (int k = 0; k < kVec; ++k) {
            if (ADT_UNPACK_STCS) __stcs(dst + g0 + 32 * k, out[k]);   // evict-first: keep the packed stream in L2
            else dst[g0 + 32 * k] = out[k];
        }
        return;
    }

    // staged per warp: r = 3 tiles and every layer's ragged last tile
    const uint32_t span = kWarpGroups * 4 * r, lo = warp * span, nbytes = m * r;
    if (lo >= nbytes) return;
    const uint32_t mine = min(span, nbytes - lo), n16 = mine / 16;
    const uint4 *s4 = reinterpret_cast<const uint4 *>(src + lo);
    uint4 *w4 = reinterpret_cast<uint4 *>(ws);
    for (uint32_t i = lane; i < n16; i += 32) w4[i] = __ldcs(s4 + i);
    uint8_t *w1 = reinterpret_cast<uint8_t *>(ws);
    for (uint32_t i = n16 * 16 + lane; i < mine; i += 32) w1[i] = src[lo + i];
    __syncwarp();
    uint32_t *dst1 = reinterpret_cast<uint32_t *>(dst);
#pragma unroll
    for (int k = 0; k < kVec; ++k) {
        const uint32_t gl = lane + 32 * k, g = g0 + 32 * k;   // local / tile group
        if (g * 4 >= m) break;
        const uint4 o = unpack_words(r, ws + gl * r);
        if (g * 4 + 4 <= m) {
            if (ADT_UNPACK_STCS >= 2) __stcs(dst + g, o);
            else dst[g] = o;
        } else {
            if (g * 4 + 0 < m) dst1[g * 4 + 0] = o.x;
            if (g * 4 + 1 < m) dst1[g * 4 + 1] = o.y;
            if (g * 4 + 2 < m) dst1[g * 4 + 2] = o.z;
        }
    }
    __syncwarp();   // the staging words are reused by this warp's next tile (persistent walk)
}

template <int MAXSEG>
__global__ void __launch_bounds__(kCtaThreads, ADT_UNPACK_MIN_BLOCKS * kSplit)
adt_unpack_kernel(const __grid_constant__ Table<MAXSEG> T, uint32_t ntiles) {
    __shared__ __align__(16) uint32_t stage[kCtaWarps][kWarpStageWords];
    uint32_t *ws = stage[threadIdx.x >> 5];
#if ADT_PDL && __CUDA_ARCH__ >= 900
    // Launched as a programmatic dependent (launch_unpack): before touching the
    // packed stream, the replicas or the abort word, wait for the preceding
    // grid (the pack, a barrier, ...) to complete and flush. A no-op when the
    // launch was an ordinary one.
    asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
    if (aborted(T.abort)) return;
    // Newest-first (ADT_UNPACK_REVERSE): CTAs are dispatched roughly in
    // blockIdx order, so walking the tiles backwards reads the payload the
    // pack pass wrote last — the part still resident in the 126 MB L2 —
    // before it is evicted.
    if (!ADT_PERSISTENT) {
        // Rotated walk (adt_unpack_multi_ex): each rank starts right before its
        // own pieces, so at any moment the ranks pull from different peers
        // instead of all draining the same owner's NVLink port in lockstep.
        const uint32_t b = blockIdx.x / kSplit;
        const int warp = static_cast<int>(blockIdx.x % kSplit) * kCtaWarps + static_cast<int>(threadIdx.x >> 5);
        uint32_t tile = (ADT_UNPACK_REVERSE ? ntiles - 1 - b : b) + T.tile_rot;
        if (tile >= ntiles) tile -= ntiles;
        unpack_tile<MAXSEG>(T, tile, find_segment(T, tile), ws, warp);
        return;
    }
    if (ADT_UNPACK_REVERSE) {
        int s = find_segment(T, ntiles - 1 - blockIdx.x);
        for (uint32_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
            const uint32_t tile = ntiles - 1 - t;
            while (T.tile_begin[s] > tile) --s;
            unpack_tile<MAXSEG>(T, tile, s, ws);
        }
    } else {
        int s = find_segment(T, blockIdx.x);
        for (uint32_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
            while (T.tile_begin[s + 1] <= tile) ++s;
            unpack_tile<MAXSEG>(T, tile, s, ws);
        }
    }
}


// ---------------------------------------------- small sets: one launch per step
// Sets of at most one tile per SM (LeNet: 106 tiles) are latency-bound: three
// dependent launches (pack, finalize, unpack) cost more than their bytes. One
// cooperative launch does the whole step: every CTA packs one tile (norm
// partials fused, plain stores), a grid barrier, then every CTA unpacks the
// tile packed by CTA ntiles-1-b (reading another CTA's bytes back from global
// memory: the same round trip as the two-kernel step), and CTA l < nseg sums
// layer l's partials in the fixed (tile, warp) order of adt_norm_finalize.
template <int MAXSEG>
struct RoundTable {
    Table<MAXSEG> P;          // masters -> packed stream (P.weights = masters, P.packed_out, partials, seg_sumsq)
    Table<MAXSEG> U;          // packed stream -> replicas (U.weights = replicas, U.srcs[0] = packed)
    uint32_t *barrier;        // [2]: arrivals, generation (zero-initialised, caller-owned)
};

__device__ __forceinline__ void grid_barrier(uint32_t *bar) {
    __syncthreads();
    if (threadIdx.x == 0) {
        volatile uint32_t *gen = bar + 1;
        const uint32_t g = *gen;
        __threadfence();                                   // this CTA's packed bytes and partials
        if (atomicAdd(bar, 1u) == gridDim.x - 1) {
            atomicExch(bar, 0u);
            __threadfence();
            atomicAdd(bar + 1, 1u);                        // release the generation
        } else {
            while (*gen == g) __nanosleep(20);
        }
        __threadfence();
    }
    __syncthreads();
}

template <int MAXSEG>
__global__ void __launch_bounds__(kThreads)
adt_roundtrip_kernel(const __grid_constant__ RoundTable<MAXSEG> R, uint32_t ntiles) {
    __shared__ __align__(16) uint32_t stage[kWarpsPerTile][kWarpStageWords];
    __shared__ double red[kFinThreads / 32];
    uint32_t *ws = stage[threadIdx.x >> 5];
    const uint32_t tile = blockIdx.x;
    pack_tile<MAXSEG, true, true, false>(R.P, tile, find_segment(R.P, tile), ws);
    grid_barrier(R.barrier);
    const uint32_t ut = ntiles - 1 - tile;
    unpack_tile<MAXSEG>(R.U, ut, find_segment(R.U, ut), ws);
    if (static_cast<int>(blockIdx.x) < R.P.nseg && R.P.seg_sumsq != nullptr) {
        // adt_norm_finalize_kernel's exact order (kFinThreads virtual threads,
        // each summing p[v], p[v + kFinThreads], ...; the same shuffle tree per
        // virtual warp; warp sums added in order) so both step forms agree bit for bit
        constexpr int kVirt = kFinThreads / kThreads;
        const int s = blockIdx.x;
        const uint32_t lo = R.P.tile_begin[s] * kWarpsPerTile;
        const uint32_t n = (R.P.tile_begin[s + 1] - R.P.tile_begin[s]) * kWarpsPerTile;
        const double *p = R.P.partials + lo;
#pragma unroll
        for (int k = 0; k < kVirt; ++k) {
            double a = 0.0;
            for (uint32_t i = threadIdx.x + k * kThreads; i < n; i += kFinThreads) a += p[i];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) a += __shfl_down_sync(0xFFFFFFFFu, a, o);
            if ((threadIdx.x & 31) == 0) red[(threadIdx.x >> 5) + k * kWarpsPerTile] = a;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            double t = 0.0;
#pragma unroll
            for (int w = 0; w < kFinThreads / 32; ++w) t += red[w];
            R.P.seg_sumsq[s] = t;
        }
    }
}

#include "adt_sgd.cuh"

}  // namespace

#include "adt_tma.cuh"

namespace {

#include "adt_peer.cuh"
#include "adt_awp.cuh"
#include "adt_f64.cuh"

// ----------------------------------------------------------------- host side
enum class Pass { Pack, PackNorm, Norm, Unpack, Finalize };

int cuda_status(cudaError_t e) { return e == cudaSuccess ? ADT_OK : ADT_ERR_CUDA_BASE - static_cast<int>(e); }

// Kernel family: one-tile-per-CTA register kernels (default; measured fastest,
// profiles/r01_*) or the persistent TMA bulk-copy pipeline (ADT_KERNEL=tma),
// kept for A/B measurements.
bool use_tma_kernels() {
    static const int v = [] {
        const char *e = getenv("ADT_KERNEL");
        return (e != nullptr && e[0] == 't') ? 1 : 0;
    }();
    return v != 0;
}

int sm_count_cached(int *out) {
    static int cache[64] = {0};
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return ADT_ERR_NO_DEVICE;
    if (dev >= 0 && dev < 64 && cache[dev] > 0) { *out = cache[dev]; return ADT_OK; }
    int v = 0;
    e = cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    if (e != cudaSuccess) return cuda_status(e);
    if (dev >= 0 && dev < 64) cache[dev] = v;
    *out = v;
    return ADT_OK;
}

template <typename K>
cudaError_t allow_smem(K kernel, size_t bytes) {
    return cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes));
}

template <int MAXSEG>
cudaError_t launch_tma(Pass pass, const Table<MAXSEG> &T, uint32_t ntiles, cudaStream_t stream) {
    int sms = 0;
    if (sm_count_cached(&sms) != ADT_OK) return cudaErrorNoDevice;
    const uint32_t grid = min(ntiles, static_cast<uint32_t>(tma::kCtasPerSm * sms));
    const size_t smem = sizeof(tma::Smem);
    cudaError_t e = cudaSuccess;
    switch (pass) {
        case Pass::Pack: {
            auto k = tma::adt_pack_tma_kernel<MAXSEG, false, true>;
            if ((e = allow_smem(k, smem)) == cudaSuccess) k<<<grid, tma::kBlock, smem, stream>>>(T, ntiles);
        } break;
        case Pass::PackNorm: {
            auto k = tma::adt_pack_tma_kernel<MAXSEG, true, true>;
            if ((e = allow_smem(k, smem)) == cudaSuccess) k<<<grid, tma::kBlock, smem, stream>>>(T, ntiles);
        } break;
        case Pass::Norm: {
            auto k = tma::adt_pack_tma_kernel<MAXSEG, true, false>;
            if ((e = allow_smem(k, smem)) == cudaSuccess) k<<<grid, tma::kBlock, smem, stream>>>(T, ntiles);
        } break;
        case Pass::Unpack: {
            auto k = tma::adt_unpack_tma_kernel<MAXSEG>;
            if ((e = allow_smem(k, smem)) == cudaSuccess) k<<<grid, tma::kBlock, smem, stream>>>(T, ntiles);
        } break;
        case Pass::Finalize: break;
    }
    return e;
}

// Finalize launched as a programmatic dependent of the pack pass: its launch
// is processed while the pack drains; griddepcontrol.wait in the kernel
// orders its reads after the pack's partial stores.
template <int MAXSEG>
cudaError_t launch_finalize(const Table<MAXSEG> &T, bool pdl, cudaStream_t stream) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(T.nseg);
    cfg.blockDim = dim3(kFinThreads);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, adt_norm_finalize_kernel<MAXSEG>, T);
}

// The unpack as a programmatic dependent of whatever precedes it on the
// stream (the kernel's griddepcontrol.wait keeps it ordered after that grid):
// behind the pack pass its launch overlaps the pack's last wave. Runtime A/B:
// ADT_PDL=0 launches it as an ordinary kernel.
bool pdl_unpack() {
    static const bool v = [] {
        const char *e = getenv("ADT_PDL");
        return ADT_PDL && !(e != nullptr && e[0] == '0');
    }();
    return v;
}

template <int MAXSEG>
cudaError_t launch_unpack(const Table<MAXSEG> &T, dim3 grid, uint32_t ntiles, cudaStream_t stream) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(ADT_PERSISTENT ? kThreads : kCtaThreads);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_unpack() ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, adt_unpack_kernel<MAXSEG>, T, ntiles);
}

// nsrc == 0: `reserved` must be 0 (single packed buffer); otherwise it names
// the source buffer (adt_unpack_multi) and must be < nsrc.
int validate(const adt_segment *segs, int nseg, const void *packed, bool need_packed, int nsrc = 0) {
    if (nseg < 0 || (nseg > 0 && segs == nullptr)) return ADT_ERR_ARG;
    bool any = false;
    for (int i = 0; i < nseg; ++i) {
        const adt_segment &g = segs[i];
        if (g.round_to < 1 || g.round_to > 4) return ADT_ERR_ROUND_TO;
        if (nsrc == 0 ? g.reserved != 0 : (g.reserved < 0 || g.reserved >= nsrc)) return ADT_ERR_ARG;
        if (g.count == 0) continue;
        any = true;
        if (g.weights == nullptr) return ADT_ERR_ARG;
        if (reinterpret_cast<uintptr_t>(g.weights) % 16 || g.offset % 16) return ADT_ERR_ALIGN;
        if (g.count > (UINT64_MAX - g.offset) / 4) return ADT_ERR_ARG;
        if ((g.count + kTile - 1) / kTile > static_cast<uint64_t>(INT_MAX)) return ADT_ERR_ARG;
    }
    if (any && need_packed) {
        if (packed == nullptr) return ADT_ERR_ARG;
        if (reinterpret_cast<uintptr_t>(packed) % 16) return ADT_ERR_ALIGN;
    }
    return ADT_OK;
}

template <int MAXSEG>
int launch_chunk(Pass pass, const adt_segment *segs, int nseg, const uint8_t *const *srcs, int nsrc,
                 uint8_t *pout, double *seg_sumsq, double *partials, uint32_t ntiles, bool finalize,
                 cudaStream_t stream, const uint8_t *dyn_r = nullptr, int start_seg = -1,
                 const uint32_t *abort = nullptr) {
    Table<MAXSEG> T;
    T.dyn_r = dyn_r;
    T.tile_rot = 0;
    T.abort = abort;
    for (int i = 0; i < ADT_MAX_SOURCES; ++i) T.srcs[i] = (srcs != nullptr && i < nsrc) ? srcs[i] : nullptr;
    T.packed_out = pout;
    T.seg_sumsq = seg_sumsq;
    T.partials = partials;
    T.nseg = nseg;
    uint32_t acc = 0;
    for (int i = 0; i < nseg; ++i) {
        T.tile_begin[i] = acc;
        acc += static_cast<uint32_t>((segs[i].count + kTile - 1) / kTile);
        T.count[i] = segs[i].count;
        T.offset[i] = segs[i].offset;
        T.weights[i] = reinterpret_cast<uintptr_t>(segs[i].weights);
        T.round_to[i] = static_cast<uint8_t>(segs[i].round_to);
        T.src_idx[i] = static_cast<uint8_t>(pass == Pass::Unpack ? segs[i].reserved : 0);
    }
    T.tile_begin[nseg] = acc;
    fill_hints(T, nseg, acc);
    if (start_seg >= 0 && start_seg < nseg && T.tile_begin[start_seg] < acc) T.tile_rot = T.tile_begin[start_seg];
    cudaError_t e = cudaSuccess;
    if (ntiles > 0 && pass != Pass::Finalize) {
        if (use_tma_kernels() && dyn_r == nullptr) {
            e = launch_tma<MAXSEG>(pass, T, ntiles, stream);
        } else {
            const bool split = !ADT_PERSISTENT && (pass == Pass::Pack || pass == Pass::PackNorm ||
                                                   pass == Pass::Norm || pass == Pass::Unpack);
            const dim3 block(split ? kCtaThreads : kThreads);
            uint32_t g = split ? ntiles * kSplit : ntiles;
            if (ADT_PERSISTENT) {
                int sms = 0;
                if (sm_count_cached(&sms) != ADT_OK) return ADT_ERR_NO_DEVICE;
                const int per_sm = pass == Pass::Unpack ? ADT_UNPACK_MIN_BLOCKS : ADT_PACK_MIN_BLOCKS;
                g = min(ntiles, static_cast<uint32_t>(sms * per_sm));
            }
            const dim3 grid(g);
            switch (pass) {
                case Pass::Pack: adt_pack_kernel<MAXSEG, false, true><<<grid, block, 0, stream>>>(T, ntiles); break;
                case Pass::PackNorm: adt_pack_kernel<MAXSEG, true, true><<<grid, block, 0, stream>>>(T, ntiles); break;
                case Pass::Norm: adt_pack_kernel<MAXSEG, true, false><<<grid, block, 0, stream>>>(T, ntiles); break;
                case Pass::Unpack: e = launch_unpack<MAXSEG>(T, grid, ntiles, stream); break;
                case Pass::Finalize: break;
            }
            if (e == cudaSuccess) e = cudaGetLastError();
        }
    }
    // PDL only directly behind this call's own pack pass; a standalone
    // adt_norm_finalize (often on another stream) is an ordinary launch.
    if (e == cudaSuccess && finalize && nseg > 0) e = launch_finalize<MAXSEG>(T, pass != Pass::Finalize, stream);
    return cuda_status(e);
}

constexpr int kSmallSeg = 16;
constexpr int kLargeSeg = 256;

// Greedy chunking (<= kLargeSeg layers, < 2^31 tiles per launch); the partial
// offsets of a chunk depend only on `segs`, so a separate finalize call
// (adt_norm_finalize) walks exactly the chunks the pack pass wrote.
int run(Pass pass, const adt_segment *segs, int nseg, const uint8_t *const *srcs, int nsrc, uint8_t *pout,
        double *seg_sumsq, double *partials, bool finalize, void *stream_v, const uint8_t *dyn_r = nullptr,
        int start_seg = -1, const uint32_t *abort = nullptr) {
    cudaStream_t stream = static_cast<cudaStream_t>(stream_v);
    uint64_t partial_base = 0;
    int base = 0;
    while (base < nseg) {
        int cnt = 0;
        uint64_t tiles = 0;
        while (base + cnt < nseg && cnt < kLargeSeg) {
            const uint64_t t = (segs[base + cnt].count + kTile - 1) / kTile;
            if (cnt > 0 && tiles + t > static_cast<uint64_t>(INT_MAX / kSplit)) break;
            tiles += t;
            ++cnt;
        }
        double *ss = seg_sumsq ? seg_sumsq + base : nullptr;
        double *pp = partials ? partials + partial_base : nullptr;
        const int st = cnt <= kSmallSeg
            ? launch_chunk<kSmallSeg>(pass, segs + base, cnt, srcs, nsrc, pout, ss, pp, static_cast<uint32_t>(tiles),
                                      finalize, stream, dyn_r ? dyn_r + base : nullptr, start_seg - base, abort)
            : launch_chunk<kLargeSeg>(pass, segs + base, cnt, srcs, nsrc, pout, ss, pp, static_cast<uint32_t>(tiles),
                                      finalize, stream, dyn_r ? dyn_r + base : nullptr, start_seg - base, abort);
        if (st != ADT_OK) return st;
        partial_base += tiles * kWarpsPerTile;
        base += cnt;
    }
    return ADT_OK;
}


// Per-call SGD parameters shared by every chunk.
struct SgdArgs {
    const uint8_t *srcs[ADT_MAX_SOURCES];  // gradient buffers (NC >= 1)
    float scale[ADT_MAX_SOURCES];
    float total, lr, mu, wd;
    int nc;                                 // 0 = one pre-averaged gradient per segment
    const uint8_t *widths;                  // device-resident widths (global layer index) or nullptr
    const uint32_t *abort;                  // peer-abort guard word or nullptr
};

template <int MAXSEG, int NC>
cudaError_t launch_sgd_kernel(const SgdTable<MAXSEG> &T, uint32_t ntiles, cudaStream_t stream) {
    adt_sgd_pack_kernel<MAXSEG, NC><<<ntiles, kThreads, 0, stream>>>(T);
    return cudaGetLastError();
}

template <int MAXSEG>
cudaError_t launch_sgd_nc(const SgdTable<MAXSEG> &T, int nc, uint32_t ntiles, cudaStream_t stream) {
    switch (nc) {
        case 0: return launch_sgd_kernel<MAXSEG, 0>(T, ntiles, stream);
        case 1: return launch_sgd_kernel<MAXSEG, 1>(T, ntiles, stream);
        case 2: return launch_sgd_kernel<MAXSEG, 2>(T, ntiles, stream);
        case 3: return launch_sgd_kernel<MAXSEG, 3>(T, ntiles, stream);
        case 4: return launch_sgd_kernel<MAXSEG, 4>(T, ntiles, stream);
        case 5: return launch_sgd_kernel<MAXSEG, 5>(T, ntiles, stream);
        case 6: return launch_sgd_kernel<MAXSEG, 6>(T, ntiles, stream);
        case 7: return launch_sgd_kernel<MAXSEG, 7>(T, ntiles, stream);
        case 8: return launch_sgd_kernel<MAXSEG, 8>(T, ntiles, stream);
        case 9: return launch_sgd_kernel<MAXSEG, 9>(T, ntiles, stream);
        case 10: return launch_sgd_kernel<MAXSEG, 10>(T, ntiles, stream);
        case 11: return launch_sgd_kernel<MAXSEG, 11>(T, ntiles, stream);
        case 12: return launch_sgd_kernel<MAXSEG, 12>(T, ntiles, stream);
        case 13: return launch_sgd_kernel<MAXSEG, 13>(T, ntiles, stream);
        case 14: return launch_sgd_kernel<MAXSEG, 14>(T, ntiles, stream);
        case 15: return launch_sgd_kernel<MAXSEG, 15>(T, ntiles, stream);
        case 16: return launch_sgd_kernel<MAXSEG, 16>(T, ntiles, stream);
        default: return cudaErrorInvalidValue;
    }
}

// One chunk of <= MAXSEG segments. Segment i: weights/velocity/count/offset/
// round_to from the caller's arrays; gradient = grad[i] (an address for nc = 0,
// a byte offset into every gradient buffer otherwise).
template <int MAXSEG>
int launch_sgd_chunk(const adt_sgd_segment *segs, const adt_grad_segment *gsegs, int nseg, const SgdArgs &A,
                     uint8_t *pout, double *seg_sumsq, double *partials, uint32_t ntiles, cudaStream_t stream,
                     int base) {
    SgdTable<MAXSEG> T;
    T.dyn_r = A.widths != nullptr ? A.widths + base : nullptr;
    T.tile_rot = 0;
    T.abort = A.abort;
    for (int i = 0; i < ADT_MAX_SOURCES; ++i) {
        T.srcs[i] = A.srcs[i];
        T.scale[i] = A.scale[i];
    }
    T.packed_out = pout;
    T.seg_sumsq = seg_sumsq;
    T.partials = partials;
    T.nseg = nseg;
    T.total = A.total;
    T.lr = A.lr;
    T.momentum = A.mu;
    T.weight_decay = A.wd;
    uint32_t acc = 0;
    for (int i = 0; i < nseg; ++i) {
        const uint64_t count = segs ? segs[i].count : gsegs[i].count;
        T.tile_begin[i] = acc;
        acc += static_cast<uint32_t>((count + kTile - 1) / kTile);
        T.count[i] = count;
        if (segs) {
            T.offset[i] = segs[i].offset;
            T.weights[i] = reinterpret_cast<uintptr_t>(segs[i].weights);
            T.velocity[i] = reinterpret_cast<uintptr_t>(segs[i].velocity);
            T.grad[i] = reinterpret_cast<uintptr_t>(segs[i].grad);
            T.round_to[i] = static_cast<uint8_t>(segs[i].round_to);
        } else {
            T.offset[i] = gsegs[i].offset;
            T.weights[i] = reinterpret_cast<uintptr_t>(gsegs[i].weights);
            T.velocity[i] = reinterpret_cast<uintptr_t>(gsegs[i].velocity);
            T.grad[i] = static_cast<uintptr_t>(gsegs[i].grad_offset);
            T.round_to[i] = static_cast<uint8_t>(gsegs[i].round_to);
        }
        T.src_idx[i] = 0;
    }
    T.tile_begin[nseg] = acc;
    fill_hints(T, nseg, acc);
    cudaError_t e = cudaSuccess;
    if (ntiles > 0) e = launch_sgd_nc<MAXSEG>(T, A.nc, ntiles, stream);
    if (e == cudaSuccess && seg_sumsq != nullptr && nseg > 0)
        e = launch_finalize<MAXSEG>(static_cast<const Table<MAXSEG> &>(T), true, stream);
    return cuda_status(e);
}

int run_sgd(const adt_sgd_segment *segs, const adt_grad_segment *gsegs, int nseg, const SgdArgs &A, uint8_t *pout,
            double *seg_sumsq, double *partials, cudaStream_t stream) {
    uint64_t partial_base = 0;
    int base = 0;
    auto count_of = [&](int i) { return segs ? segs[i].count : gsegs[i].count; };
    while (base < nseg) {
        int cnt = 0;
        uint64_t tiles = 0;
        while (base + cnt < nseg && cnt < kLargeSeg) {
            const uint64_t t = (count_of(base + cnt) + kTile - 1) / kTile;
            if (cnt > 0 && tiles + t > static_cast<uint64_t>(INT_MAX)) break;
            tiles += t;
            ++cnt;
        }
        double *ss = seg_sumsq ? seg_sumsq + base : nullptr;
        double *pp = partials ? partials + partial_base : nullptr;
        const adt_sgd_segment *sb = segs ? segs + base : nullptr;
        const adt_grad_segment *gb = gsegs ? gsegs + base : nullptr;
        const int st = cnt <= kSmallSeg
            ? launch_sgd_chunk<kSmallSeg>(sb, gb, cnt, A, pout, ss, pp, static_cast<uint32_t>(tiles), stream, base)
            : launch_sgd_chunk<kLargeSeg>(sb, gb, cnt, A, pout, ss, pp, static_cast<uint32_t>(tiles), stream, base);
        if (st != ADT_OK) return st;
        partial_base += tiles * kWarpsPerTile;
        base += cnt;
    }
    return ADT_OK;
}

}  // namespace

// -------------------------------------------------------------------- C ABI
extern "C" {

int adt_abi_version(void) { return ADT_ABI_VERSION; }

const char *adt_strerror(int status) {
    switch (status) {
        case ADT_OK: return "ok";
        case ADT_ERR_ROUND_TO: return "round_to must be an integer in [1, 4]";
        case ADT_ERR_ALIGN: return "weights, packed buffer and layer offsets must be 16-byte aligned";
        case ADT_ERR_ARG: return "invalid argument (null pointer, negative count or size overflow)";
        case ADT_ERR_NO_DEVICE: return "no CUDA device available";
        default:
            if (status <= ADT_ERR_CUDA_BASE)
                return cudaGetErrorString(static_cast<cudaError_t>(ADT_ERR_CUDA_BASE - status));
            return "unknown adt status";
    }
}

int adt_partials_count(const adt_segment *segs, int nseg, uint64_t *npartials) {
    if (npartials == nullptr || nseg < 0 || (nseg > 0 && segs == nullptr)) return ADT_ERR_ARG;
    uint64_t t = 0;
    for (int i = 0; i < nseg; ++i) t += (segs[i].count + kTile - 1) / kTile;
    *npartials = t * kWarpsPerTile;
    return ADT_OK;
}

int adt_pack(const adt_segment *segs, int nseg, uint8_t *packed, double *seg_sumsq,
             double *partials, void *stream) {
    const int v = validate(segs, nseg, packed, true);
    if (v != ADT_OK) return v;
    if (nseg > 0 && seg_sumsq != nullptr && partials == nullptr) return ADT_ERR_ARG;
    return run(partials ? Pass::PackNorm : Pass::Pack, segs, nseg, nullptr, 0, packed, seg_sumsq, partials,
               seg_sumsq != nullptr, stream);
}

int adt_norm_finalize(const adt_segment *segs, int nseg, double *partials, double *seg_sumsq, void *stream) {
    if (nseg < 0 || (nseg > 0 && (segs == nullptr || partials == nullptr || seg_sumsq == nullptr))) return ADT_ERR_ARG;
    return run(Pass::Finalize, segs, nseg, nullptr, 0, nullptr, seg_sumsq, partials, true, stream);
}

int adt_unpack(const adt_segment *segs, int nseg, const uint8_t *packed, void *stream) {
    const int v = validate(segs, nseg, packed, true);
    if (v != ADT_OK) return v;
    const uint8_t *srcs[1] = {packed};
    return run(Pass::Unpack, segs, nseg, srcs, 1, nullptr, nullptr, nullptr, false, stream);
}

int adt_unpack_multi(const adt_segment *segs, int nseg, const uint8_t *const *sources, int nsrc, void *stream) {
    if (nsrc < 1 || nsrc > ADT_MAX_SOURCES || sources == nullptr) return ADT_ERR_ARG;
    for (int i = 0; i < nsrc; ++i)
        if (reinterpret_cast<uintptr_t>(sources[i]) % 16) return ADT_ERR_ALIGN;
    const int v = validate(segs, nseg, sources[0], false, nsrc);
    if (v != ADT_OK) return v;
    for (int i = 0; i < nseg; ++i)
        if (segs[i].count > 0 && sources[segs[i].reserved] == nullptr) return ADT_ERR_ARG;
    return run(Pass::Unpack, segs, nseg, sources, nsrc, nullptr, nullptr, nullptr, false, stream);
}

int adt_copy_multi(uint8_t *dst, const uint8_t *const *sources, int nsrc, uint64_t offset, uint64_t bytes,
                   const uint32_t *abort, void *stream) {
    if (nsrc < 1 || nsrc > ADT_MAX_SOURCES || sources == nullptr || dst == nullptr) return ADT_ERR_ARG;
    SrcList S;
    for (int i = 0; i < ADT_MAX_SOURCES; ++i) S.p[i] = i < nsrc ? sources[i] : nullptr;
    for (int i = 0; i < nsrc; ++i)
        if (S.p[i] == nullptr) return ADT_ERR_ARG;
    if (bytes == 0) return ADT_OK;
    adt_copy_multi_param_kernel<<<nsrc, 128, 0, static_cast<cudaStream_t>(stream)>>>(dst, S, offset, bytes, abort);
    return cuda_status(cudaGetLastError());
}

int adt_peer_barrier(uint32_t *const *flags, int nranks, int rank, uint32_t *state, uint64_t timeout_ns,
                     void *stream) {
    if (flags == nullptr || state == nullptr || nranks < 1 || nranks > ADT_MAX_SOURCES || rank < 0 ||
        rank >= nranks || timeout_ns == 0)
        return ADT_ERR_ARG;
    FlagList F;
    for (int i = 0; i < ADT_MAX_SOURCES; ++i) F.p[i] = i < nranks ? flags[i] : nullptr;
    for (int i = 0; i < nranks; ++i) {
        if (F.p[i] == nullptr) return ADT_ERR_ARG;
        if (reinterpret_cast<uintptr_t>(F.p[i]) % 4) return ADT_ERR_ALIGN;
    }
    adt_peer_barrier_kernel<<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(F, nranks, rank, state, timeout_ns);
    return cuda_status(cudaGetLastError());
}

int adt_ipc_handle_bytes(void) { return static_cast<int>(sizeof(cudaIpcMemHandle_t)); }

int adt_ipc_get_handle(void *dev_ptr, void *handle_out, uint64_t *offset_out) {
    if (dev_ptr == nullptr || handle_out == nullptr || offset_out == nullptr) return ADT_ERR_ARG;
    // The handle names the whole cudaMalloc allocation (a caching allocator may
    // have carved dev_ptr out of a larger segment): report dev_ptr's offset in it.
    // The allocation base comes from the driver (cuPointerGetAttribute, resolved
    // with dlsym so the library still loads on machines without a driver).
    using GetAttr = int (*)(void *, int, unsigned long long);
    static GetAttr get_attr = [] {
        void *h = dlopen("libcuda.so.1", RTLD_NOW | RTLD_GLOBAL);
        return h ? reinterpret_cast<GetAttr>(dlsym(h, "cuPointerGetAttribute")) : nullptr;
    }();
    if (get_attr == nullptr) return ADT_ERR_NO_DEVICE;
    unsigned long long base = 0;
    const int kRangeStart = 11;  // CU_POINTER_ATTRIBUTE_RANGE_START_ADDR
    if (get_attr(&base, kRangeStart, reinterpret_cast<unsigned long long>(dev_ptr)) != 0 || base == 0)
        return ADT_ERR_ARG;
    cudaIpcMemHandle_t h;
    const cudaError_t e = cudaIpcGetMemHandle(&h, dev_ptr);
    if (e != cudaSuccess) return cuda_status(e);
    memcpy(handle_out, &h, sizeof(h));
    *offset_out = reinterpret_cast<unsigned long long>(dev_ptr) - base;
    return ADT_OK;
}

int adt_ipc_open(const void *handle, void **dev_ptr_out) {
    if (handle == nullptr || dev_ptr_out == nullptr) return ADT_ERR_ARG;
    cudaIpcMemHandle_t h;
    memcpy(&h, handle, sizeof(h));
    return cuda_status(cudaIpcOpenMemHandle(dev_ptr_out, h, cudaIpcMemLazyEnablePeerAccess));
}

int adt_ipc_close(void *dev_ptr) {
    if (dev_ptr == nullptr) return ADT_ERR_ARG;
    return cuda_status(cudaIpcCloseMemHandle(dev_ptr));
}

int adt_sumsq(const adt_segment *segs, int nseg, double *seg_sumsq, double *partials, void *stream) {
    const int v = validate(segs, nseg, nullptr, false);
    if (v != ADT_OK) return v;
    if (nseg > 0 && (seg_sumsq == nullptr || partials == nullptr)) return ADT_ERR_ARG;
    return run(Pass::Norm, segs, nseg, nullptr, 0, nullptr, seg_sumsq, partials, true, stream);
}

}  // extern "C"

namespace {
int sgd_pack_impl(const adt_sgd_segment *segs, int nseg, float lr, float momentum, float weight_decay,
                  uint8_t *packed, double *seg_sumsq, double *partials, const uint8_t *widths, void *stream) {
    if (nseg < 0 || (nseg > 0 && segs == nullptr)) return ADT_ERR_ARG;
    if (nseg > 0 && seg_sumsq != nullptr && partials == nullptr) return ADT_ERR_ARG;
    bool any = false;
    for (int i = 0; i < nseg; ++i) {
        const adt_sgd_segment &g = segs[i];
        if (g.round_to < 1 || g.round_to > 4) return ADT_ERR_ROUND_TO;
        if (g.reserved != 0) return ADT_ERR_ARG;
        if (g.count == 0) continue;
        any = true;
        if (!g.weights || !g.velocity || !g.grad) return ADT_ERR_ARG;
        if (reinterpret_cast<uintptr_t>(g.weights) % 16 || reinterpret_cast<uintptr_t>(g.velocity) % 16 ||
            reinterpret_cast<uintptr_t>(g.grad) % 16 || g.offset % 16)
            return ADT_ERR_ALIGN;
        if (g.count > (UINT64_MAX - g.offset) / 4) return ADT_ERR_ARG;
        if ((g.count + kTile - 1) / kTile > static_cast<uint64_t>(INT_MAX)) return ADT_ERR_ARG;
    }
    if (any && (packed == nullptr)) return ADT_ERR_ARG;
    if (any && reinterpret_cast<uintptr_t>(packed) % 16) return ADT_ERR_ALIGN;
    SgdArgs A = {};
    A.lr = lr;
    A.mu = momentum;
    A.wd = weight_decay;
    A.nc = 0;
    A.widths = widths;
    return run_sgd(segs, nullptr, nseg, A, packed, seg_sumsq, partials, static_cast<cudaStream_t>(stream));
}

int reduce_sgd_pack_impl(const adt_grad_segment *segs, int nseg, const float *const *grads,
                         const int64_t *sample_counts, int ncontrib, float lr, float momentum, float weight_decay,
                         uint8_t *packed, double *seg_sumsq, double *partials, const uint8_t *widths,
                         const uint32_t *abort, void *stream) {
    if (nseg < 0 || (nseg > 0 && segs == nullptr)) return ADT_ERR_ARG;
    if (ncontrib < 1 || ncontrib > ADT_MAX_SOURCES || grads == nullptr || sample_counts == nullptr)
        return ADT_ERR_ARG;
    if (nseg > 0 && seg_sumsq != nullptr && partials == nullptr) return ADT_ERR_ARG;
    SgdArgs A = {};
    int64_t total = 0;
    for (int c = 0; c < ncontrib; ++c) {
        if (grads[c] == nullptr) return ADT_ERR_ARG;
        if (reinterpret_cast<uintptr_t>(grads[c]) % 16) return ADT_ERR_ALIGN;
        A.srcs[c] = reinterpret_cast<const uint8_t *>(grads[c]);
        A.scale[c] = static_cast<float>(sample_counts[c]);   // dtype.type(c.sample_count), net.py:230
        total += sample_counts[c];
    }
    A.total = static_cast<float>(total);                      // dtype.type(total), net.py:231
    A.lr = lr;
    A.mu = momentum;
    A.wd = weight_decay;
    A.nc = ncontrib;
    A.widths = widths;
    A.abort = abort;
    bool any = false;
    for (int i = 0; i < nseg; ++i) {
        const adt_grad_segment &g = segs[i];
        if (g.round_to < 1 || g.round_to > 4) return ADT_ERR_ROUND_TO;
        if (g.reserved != 0) return ADT_ERR_ARG;
        if (g.count == 0) continue;
        any = true;
        if (!g.weights || !g.velocity) return ADT_ERR_ARG;
        if (reinterpret_cast<uintptr_t>(g.weights) % 16 || reinterpret_cast<uintptr_t>(g.velocity) % 16 ||
            g.grad_offset % 16 || g.offset % 16)
            return ADT_ERR_ALIGN;
        if (g.count > (UINT64_MAX - g.offset) / 4 || g.count > (UINT64_MAX - g.grad_offset) / 4) return ADT_ERR_ARG;
        if ((g.count + kTile - 1) / kTile > static_cast<uint64_t>(INT_MAX)) return ADT_ERR_ARG;
    }
    if (any && (packed == nullptr)) return ADT_ERR_ARG;
    if (any && reinterpret_cast<uintptr_t>(packed) % 16) return ADT_ERR_ALIGN;
    return run_sgd(nullptr, segs, nseg, A, packed, seg_sumsq, partials, static_cast<cudaStream_t>(stream));
}
}  // namespace

extern "C" {

int adt_sgd_pack(const adt_sgd_segment *segs, int nseg, float lr, float momentum, float weight_decay,
                 uint8_t *packed, double *seg_sumsq, double *partials, void *stream) {
    return sgd_pack_impl(segs, nseg, lr, momentum, weight_decay, packed, seg_sumsq, partials, nullptr, stream);
}

int adt_reduce_sgd_pack(const adt_grad_segment *segs, int nseg, const float *const *grads,
                        const int64_t *sample_counts, int ncontrib, float lr, float momentum, float weight_decay,
                        uint8_t *packed, double *seg_sumsq, double *partials, const uint32_t *abort, void *stream) {
    return reduce_sgd_pack_impl(segs, nseg, grads, sample_counts, ncontrib, lr, momentum, weight_decay, packed,
                                seg_sumsq, partials, nullptr, abort, stream);
}

int adt_sgd_pack_dyn(const adt_sgd_segment *segs, int nseg, float lr, float momentum, float weight_decay,
                     uint8_t *packed, double *partials, const uint8_t *widths, void *stream) {
    if (nseg > 0 && (segs == nullptr || widths == nullptr)) return ADT_ERR_ARG;
    for (int i = 0; i < nseg; ++i)
        if (segs[i].round_to != 4) return ADT_ERR_ARG;   // capacity layout
    return sgd_pack_impl(segs, nseg, lr, momentum, weight_decay, packed, nullptr, partials, widths, stream);
}

int adt_reduce_sgd_pack_dyn(const adt_grad_segment *segs, int nseg, const float *const *grads,
                            const int64_t *sample_counts, int ncontrib, float lr, float momentum,
                            float weight_decay, uint8_t *packed, double *partials, const uint8_t *widths,
                            const uint32_t *abort, void *stream) {
    if (nseg > 0 && (segs == nullptr || widths == nullptr)) return ADT_ERR_ARG;
    for (int i = 0; i < nseg; ++i)
        if (segs[i].round_to != 4) return ADT_ERR_ARG;
    return reduce_sgd_pack_impl(segs, nseg, grads, sample_counts, ncontrib, lr, momentum, weight_decay, packed,
                                nullptr, partials, widths, abort, stream);
}

int adt_pack_dyn(const adt_segment *segs, int nseg, uint8_t *packed, double *partials, const uint8_t *widths,
                 void *stream) {
    const int v = validate(segs, nseg, packed, true);
    if (v != ADT_OK) return v;
    if (nseg > 0 && widths == nullptr) return ADT_ERR_ARG;
    for (int i = 0; i < nseg; ++i)
        if (segs[i].round_to != 4) return ADT_ERR_ARG;   // capacity layout
    return run(partials ? Pass::PackNorm : Pass::Pack, segs, nseg, nullptr, 0, packed, nullptr, partials, false,
               stream, widths);
}

int adt_unpack_dyn(const adt_segment *segs, int nseg, const uint8_t *packed, const uint8_t *widths, void *stream) {
    const int v = validate(segs, nseg, packed, true);
    if (v != ADT_OK) return v;
    if (nseg > 0 && widths == nullptr) return ADT_ERR_ARG;
    for (int i = 0; i < nseg; ++i)
        if (segs[i].round_to != 4) return ADT_ERR_ARG;
    const uint8_t *srcs[1] = {packed};
    return run(Pass::Unpack, segs, nseg, srcs, 1, nullptr, nullptr, nullptr, false, stream, widths);
}

int adt_awp_observe(const double *seg_sumsq, const adt_awp_device *dev, const adt_awp_config *cfg,
                    const uint32_t *abort, void *stream) {
    if (seg_sumsq == nullptr || dev == nullptr || cfg == nullptr) return ADT_ERR_ARG;
    const adt_awp_device &D = *dev;
    if (D.nlayers < 1 || D.ngroups < 1 || D.ngroups > D.nlayers || D.ring_steps < 1 || D.reserved != 0) return ADT_ERR_ARG;
    if (!D.groups || !D.members || !D.member_start || !D.widths_in || !D.widths_out || !D.escalated || !D.ring ||
        !D.counter)
        return ADT_ERR_ARG;
    if (cfg->interval < 1 || cfg->step_bits < 1 || cfg->max_bits < 1 || cfg->max_bits > 32) return ADT_ERR_ARG;
    adt_awp_observe_kernel<<<1, kAwpThreads, 0, static_cast<cudaStream_t>(stream)>>>(seg_sumsq, D, *cfg, abort);
    return cuda_status(cudaGetLastError());
}

extern "C++" {
namespace {
// masters == nullptr: gather mode (re-unpack from `sources`, segment l's
// payload in sources[replicas[l].reserved]); seg_layer == nullptr: segment i
// is layer base + i.
template <int MAXSEG>
int launch_fixup_chunk(const adt_segment *masters, const adt_segment *replicas, int nseg, uint8_t *packed,
                       const uint8_t *const *sources, int nsrc, const int32_t *seg_layer, const int32_t *escalated,
                       const uint8_t *widths_new, int base, cudaStream_t stream, const uint32_t *abort = nullptr) {
    FixupTable<MAXSEG> F;
    Table<MAXSEG> &T = F.T;
    T.abort = abort;
    for (int i = 0; i < ADT_MAX_SOURCES; ++i) T.srcs[i] = (sources != nullptr && i < nsrc) ? sources[i] : nullptr;
    T.packed_out = packed;
    T.seg_sumsq = nullptr;
    T.partials = nullptr;
    T.dyn_r = masters == nullptr ? widths_new : nullptr;
    T.tile_rot = 0;
    T.nseg = nseg;
    uint32_t acc = 0;
    for (int i = 0; i < nseg; ++i) {
        T.tile_begin[i] = acc;
        acc += static_cast<uint32_t>((replicas[i].count + kTile - 1) / kTile);
        T.count[i] = replicas[i].count;
        T.offset[i] = replicas[i].offset;
        T.weights[i] = reinterpret_cast<uintptr_t>(replicas[i].weights);
        T.round_to[i] = 4;
        T.src_idx[i] = static_cast<uint8_t>(masters == nullptr ? replicas[i].reserved : 0);
        F.masters[i] = masters != nullptr ? reinterpret_cast<uintptr_t>(masters[i].weights) : 0;
        F.layer_of[i] = seg_layer != nullptr ? seg_layer[i] : base + i;
    }
    T.tile_begin[nseg] = acc;
    fill_hints(T, nseg, acc);
    F.escalated = escalated;
    F.widths_new = widths_new;
    F.gather = masters == nullptr ? 1 : 0;
    int sms = 0;
    if (sm_count_cached(&sms) != ADT_OK) return ADT_ERR_NO_DEVICE;
    const uint32_t grid = max(1u, min(acc, static_cast<uint32_t>(ADT_FIXUP_CTAS_PER_SM * sms)));
    adt_awp_fixup_kernel<MAXSEG><<<grid, kThreads, 0, stream>>>(F);
    return cuda_status(cudaGetLastError());
}
}  // namespace
}  // extern "C++"

int adt_awp_fixup(const adt_segment *masters, const adt_segment *replicas, int nseg, uint8_t *packed,
                  const int32_t *escalated, const uint8_t *widths_new, void *stream) {
    int v = validate(replicas, nseg, packed, true);
    if (v != ADT_OK) return v;
    if ((v = validate(masters, nseg, packed, true)) != ADT_OK) return v;
    if (nseg > 0 && (escalated == nullptr || widths_new == nullptr)) return ADT_ERR_ARG;
    for (int i = 0; i < nseg; ++i)
        if (replicas[i].round_to != 4 || masters[i].count != replicas[i].count ||
            masters[i].offset != replicas[i].offset)
            return ADT_ERR_ARG;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    for (int base = 0; base < nseg; base += kLargeSeg) {
        const int cnt = min(kLargeSeg, nseg - base);
        const int st = cnt <= kSmallSeg
            ? launch_fixup_chunk<kSmallSeg>(masters + base, replicas + base, cnt, packed, nullptr, 0, nullptr,
                                            escalated, widths_new + base, base, s)
            : launch_fixup_chunk<kLargeSeg>(masters + base, replicas + base, cnt, packed, nullptr, 0, nullptr,
                                            escalated, widths_new + base, base, s);
        if (st != ADT_OK) return st;
    }
    return ADT_OK;
}

int adt_awp_fixup_pieces(const adt_segment *masters, const adt_segment *replicas, int nseg, const int32_t *seg_layer,
                         uint8_t *packed, const int32_t *escalated, const uint8_t *widths_new, const uint32_t *abort,
                         void *stream) {
    int v = validate(replicas, nseg, packed, true);
    if (v != ADT_OK) return v;
    if ((v = validate(masters, nseg, packed, true)) != ADT_OK) return v;
    if (nseg > 0 && (escalated == nullptr || widths_new == nullptr || seg_layer == nullptr)) return ADT_ERR_ARG;
    for (int i = 0; i < nseg; ++i)
        if (replicas[i].round_to != 4 || masters[i].count != replicas[i].count ||
            masters[i].offset != replicas[i].offset || seg_layer[i] < 0)
            return ADT_ERR_ARG;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    for (int base = 0; base < nseg; base += kLargeSeg) {
        const int cnt = min(kLargeSeg, nseg - base);
        const int st = cnt <= kSmallSeg
            ? launch_fixup_chunk<kSmallSeg>(masters + base, replicas + base, cnt, packed, nullptr, 0, seg_layer + base,
                                            escalated, widths_new + base, base, s, abort)
            : launch_fixup_chunk<kLargeSeg>(masters + base, replicas + base, cnt, packed, nullptr, 0, seg_layer + base,
                                            escalated, widths_new + base, base, s, abort);
        if (st != ADT_OK) return st;
    }
    return ADT_OK;
}

int adt_awp_fixup_gather(const adt_segment *replicas, int nseg, const int32_t *seg_layer,
                         const uint8_t *const *sources, int nsrc, const int32_t *escalated,
                         const uint8_t *widths_new, const uint32_t *abort, void *stream) {
    if (nsrc < 1 || nsrc > ADT_MAX_SOURCES || sources == nullptr) return ADT_ERR_ARG;
    const int v = validate(replicas, nseg, sources[0], false, nsrc);
    if (v != ADT_OK) return v;
    if (nseg > 0 && (escalated == nullptr || widths_new == nullptr || seg_layer == nullptr)) return ADT_ERR_ARG;
    for (int i = 0; i < nseg; ++i)
        if (replicas[i].round_to != 4 || seg_layer[i] < 0 || sources[replicas[i].reserved] == nullptr)
            return ADT_ERR_ARG;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    for (int base = 0; base < nseg; base += kLargeSeg) {
        const int cnt = min(kLargeSeg, nseg - base);
        const int st = cnt <= kSmallSeg
            ? launch_fixup_chunk<kSmallSeg>(nullptr, replicas + base, cnt, nullptr, sources, nsrc, seg_layer + base,
                                            escalated, widths_new + base, base, s, abort)
            : launch_fixup_chunk<kLargeSeg>(nullptr, replicas + base, cnt, nullptr, sources, nsrc, seg_layer + base,
                                            escalated, widths_new + base, base, s, abort);
        if (st != ADT_OK) return st;
    }
    return ADT_OK;
}

int adt_unpack_multi_ex(const adt_segment *segs, int nseg, const uint8_t *const *sources, int nsrc,
                        const uint8_t *widths, int start_seg, const uint32_t *abort, void *stream) {
    if (nsrc < 1 || nsrc > ADT_MAX_SOURCES || sources == nullptr) return ADT_ERR_ARG;
    for (int i = 0; i < nsrc; ++i)
        if (reinterpret_cast<uintptr_t>(sources[i]) % 16) return ADT_ERR_ALIGN;
    const int v = validate(segs, nseg, sources[0], false, nsrc);
    if (v != ADT_OK) return v;
    for (int i = 0; i < nseg; ++i) {
        if (segs[i].count > 0 && sources[segs[i].reserved] == nullptr) return ADT_ERR_ARG;
        if (widths != nullptr && segs[i].round_to != 4) return ADT_ERR_ARG;   // capacity layout
    }
    return run(Pass::Unpack, segs, nseg, sources, nsrc, nullptr, nullptr, nullptr, false, stream, widths,
               start_seg < nseg ? start_seg : -1, abort);
}

int adt_unpack_multi_dyn(const adt_segment *segs, int nseg, const uint8_t *const *sources, int nsrc,
                         const uint8_t *widths, const uint32_t *abort, void *stream) {
    if (nsrc < 1 || nsrc > ADT_MAX_SOURCES || sources == nullptr) return ADT_ERR_ARG;
    for (int i = 0; i < nsrc; ++i)
        if (reinterpret_cast<uintptr_t>(sources[i]) % 16) return ADT_ERR_ALIGN;
    const int v = validate(segs, nseg, sources[0], false, nsrc);
    if (v != ADT_OK) return v;
    if (nseg > 0 && widths == nullptr) return ADT_ERR_ARG;
    for (int i = 0; i < nseg; ++i)
        if (segs[i].round_to != 4 || (segs[i].count > 0 && sources[segs[i].reserved] == nullptr)) return ADT_ERR_ARG;
    return run(Pass::Unpack, segs, nseg, sources, nsrc, nullptr, nullptr, nullptr, false, stream, widths, -1, abort);
}

int adt_awp_combine(const double *tails, int npieces_total, const int32_t *piece_layer, int nlayers,
                    double *seg_sumsq, const uint32_t *abort, void *stream) {
    if (tails == nullptr || piece_layer == nullptr || seg_sumsq == nullptr || npieces_total < 0 || nlayers < 1)
        return ADT_ERR_ARG;
    adt_awp_combine_kernel<<<(nlayers + 255) / 256, 256, 0, static_cast<cudaStream_t>(stream)>>>(
        tails, npieces_total, piece_layer, nlayers, seg_sumsq, abort);
    return cuda_status(cudaGetLastError());
}

int adt_sumsq_f64_partials(uint64_t n, uint64_t *npartials) {
    if (npartials == nullptr) return ADT_ERR_ARG;
    *npartials = static_cast<uint64_t>(f64_ctas(n));
    return ADT_OK;
}

int adt_sumsq_f64(const double *x, uint64_t n, double *partials, double *out, void *stream) {
    if (out == nullptr || partials == nullptr || (n > 0 && x == nullptr)) return ADT_ERR_ARG;
    if (reinterpret_cast<uintptr_t>(x) % 8) return ADT_ERR_ALIGN;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int ctas = f64_ctas(n);
    if (n > 0) {
        adt_sumsq_f64_kernel<<<ctas, kF64Threads, 0, s>>>(x, n, partials);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return cuda_status(e);
        adt_sumsq_f64_finalize<<<1, 32, 0, s>>>(partials, ctas, out);
    } else {
        cudaError_t e = cudaMemsetAsync(out, 0, sizeof(double), s);
        if (e != cudaSuccess) return cuda_status(e);
    }
    return cuda_status(cudaGetLastError());
}

}  // extern "C"

namespace {
// Fill a Table<16> from segments (adt_roundtrip): tile map, hints, widths.
uint32_t fill_small_table(Table<kSmallSeg> &T, const adt_segment *segs, int nseg) {
    memset(&T, 0, sizeof(T));
    T.nseg = nseg;
    uint32_t acc = 0;
    for (int i = 0; i < nseg; ++i) {
        T.tile_begin[i] = acc;
        acc += static_cast<uint32_t>((segs[i].count + kTile - 1) / kTile);
        T.count[i] = segs[i].count;
        T.offset[i] = segs[i].offset;
        T.weights[i] = reinterpret_cast<uintptr_t>(segs[i].weights);
        T.round_to[i] = static_cast<uint8_t>(segs[i].round_to);
    }
    T.tile_begin[nseg] = acc;
    fill_hints(T, nseg, acc);
    return acc;
}
}  // namespace

extern "C" {

int adt_roundtrip_max_tiles(int *tiles) {
    if (tiles == nullptr) return ADT_ERR_ARG;
    int sms = 0;
    const int st = sm_count_cached(&sms);
    if (st != ADT_OK) return st;
    *tiles = sms;                                  // one resident CTA per SM: co-residency by construction
    return ADT_OK;
}

int adt_roundtrip(const adt_segment *masters, const adt_segment *replicas, int nseg, uint8_t *packed,
                  double *seg_sumsq, double *partials, uint32_t *barrier, void *stream) {
    int v = validate(masters, nseg, packed, true);
    if (v != ADT_OK) return v;
    if ((v = validate(replicas, nseg, packed, true)) != ADT_OK) return v;
    if (nseg < 1 || nseg > kSmallSeg || partials == nullptr || barrier == nullptr) return ADT_ERR_ARG;
    for (int i = 0; i < nseg; ++i)
        if (masters[i].count != replicas[i].count || masters[i].offset != replicas[i].offset ||
            masters[i].round_to != replicas[i].round_to)
            return ADT_ERR_ARG;
    RoundTable<kSmallSeg> R;
    const uint32_t ntiles = fill_small_table(R.P, masters, nseg);
    fill_small_table(R.U, replicas, nseg);
    int cap = 0;
    if ((v = adt_roundtrip_max_tiles(&cap)) != ADT_OK) return v;
    if (ntiles == 0 || ntiles > static_cast<uint32_t>(cap)) return ADT_ERR_ARG;
    R.P.packed_out = packed;
    R.P.partials = partials;
    R.P.seg_sumsq = seg_sumsq;
    R.U.srcs[0] = packed;
    R.barrier = barrier;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(ntiles);
    cfg.blockDim = dim3(kThreads);
    cfg.stream = static_cast<cudaStream_t>(stream);
    static const bool coop = [] {                  // A/B hook: ADT_RT_COOP=0 launches it as a plain grid
        const char *e = getenv("ADT_RT_COOP");
        return !(e != nullptr && e[0] == '0');
    }();
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;   // all CTAs co-resident (the grid barrier)
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = coop ? 1 : 0;
    return cuda_status(cudaLaunchKernelEx(&cfg, adt_roundtrip_kernel<kSmallSeg>, R, ntiles));
}

int adt_device_sm_count(int *sm_count) {
    if (sm_count == nullptr) return ADT_ERR_ARG;
    return sm_count_cached(sm_count);
}

}  // extern "C"
