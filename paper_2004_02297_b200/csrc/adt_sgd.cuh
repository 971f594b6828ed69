// adt_sgd.cuh — fused momentum-SGD (+ gradient combine) + pack + norm kernels.
// Included by adt_kernels.cu inside its anonymous namespace (one translation
// unit: the kernels share the tile helpers, tables and store paths defined there).

// ------------------------------------------------- fused SGD update + pack
// the momentum-SGD step right before the path
// (net.py:203-246, weight half of gather_and_update) fused with the pack and
// the norm: one pass reads W, v and the gradient(s) and writes W', v' and W''s
// packed bytes + norm partials, so the updated master is never re-read.
//
// NC = 0 (adt_sgd_pack): one pre-averaged gradient g.
// NC >= 1 (adt_reduce_sgd_pack, the gradient return path): NC worker
//   contributions g_c, read from NC source buffers (local, or peer ranks'
//   gradient buckets mapped over NVLink — the reduce-scatter is this kernel's
//   load stage), combined exactly as net.py:229-231:
//     g = pairwise_sum(g_c * f32(count_c)) / f32(total)
//   with pairwise_sum's association tree (net.py:186-200).
// Then per weight, float32 with the reference's rounding at every operation
// (no FMA contraction):
//   g' = g + wd*W   (only when wd != 0)   v' = v*mu + g'   W' = W - lr*v'
template <int MAXSEG>
struct SgdTable : Table<MAXSEG> {
    uintptr_t velocity[MAXSEG];
    uintptr_t grad[MAXSEG];        // NC = 0: gradient address; NC >= 1: byte offset inside every srcs[c]
    float scale[ADT_MAX_SOURCES];  // f32(sample_count_c)
    float total;                   // f32(sum of sample counts)
    float lr, momentum, weight_decay;
};

// net.py:186-200 on registers: adjacent pairs, level by level, an odd
// leftover carried up unchanged. x[] is fully unrolled (constant indices).
template <int LEN>
struct Pairwise {
    static __device__ __forceinline__ float run(float *x) {
#pragma unroll
        for (int i = 0; i < LEN / 2; ++i) x[i] = __fadd_rn(x[2 * i], x[2 * i + 1]);
        if (LEN % 2) x[LEN / 2] = x[LEN - 1];
        return Pairwise<(LEN + 1) / 2>::run(x);
    }
};
template <>
struct Pairwise<1> {
    static __device__ __forceinline__ float run(float *x) { return x[0]; }
};

template <int NC, int MAXSEG>
__device__ __forceinline__ uint32_t combine(const uint32_t *g, const SgdTable<MAXSEG> &T) {
    if constexpr (NC == 0) {
        return g[0];
    } else {
        float x[NC];
#pragma unroll
        for (int c = 0; c < NC; ++c) x[c] = __fmul_rn(__uint_as_float(g[c]), T.scale[c]);
        return __float_as_uint(__fdiv_rn(Pairwise<NC>::run(x), T.total));
    }
}

__device__ __forceinline__ uint32_t sgd1(uint32_t wb, uint32_t &vb, uint32_t gb, float lr, float mu, float wd) {
    const float w = __uint_as_float(wb);
    float g = __uint_as_float(gb);
    if (wd != 0.0f) g = __fadd_rn(g, __fmul_rn(wd, w));
    const float v = __fadd_rn(__fmul_rn(__uint_as_float(vb), mu), g);
    vb = __float_as_uint(v);
    return __float_as_uint(__fsub_rn(w, __fmul_rn(lr, v)));
}

#ifndef ADT_SGD_HOIST_MAX_NC
#define ADT_SGD_HOIST_MAX_NC 4      // whole-tile gradient prefetch up to this many contributions
#endif
#ifndef ADT_SGD_HOIST2_MAX_NC
#define ADT_SGD_HOIST2_MAX_NC 7     // two k-steps ahead up to this many (8: spills, no gain)
#endif
#ifndef ADT_SGD_HOIST_NC0
#define ADT_SGD_HOIST_NC0 1         // pre-averaged gradient: k-steps of g loads ahead
#endif
__host__ __device__ constexpr int sgd_hoist(int nc) {
    return nc == 0 ? ADT_SGD_HOIST_NC0
                   : (nc <= ADT_SGD_HOIST_MAX_NC) ? kVec : (nc <= ADT_SGD_HOIST2_MAX_NC) ? 2 : 1;
}
#ifndef ADT_SGD_MIN_BLOCKS
#define ADT_SGD_MIN_BLOCKS 3          // pre-averaged gradient: 3 CTAs/SM (213 us vs 217 us at 4 on AlexNet, r01_ab_reduce_prefetch.md)
#endif
#ifndef ADT_SGD_NC2_MIN_BLOCKS
#define ADT_SGD_NC2_MIN_BLOCKS 2
#endif
constexpr int sgd_min_blocks(int nc) {
    return nc == 0 ? ADT_SGD_MIN_BLOCKS : nc == 1 ? 3 : nc == 2 ? ADT_SGD_NC2_MIN_BLOCKS : 2;
}

template <int MAXSEG, int NC>
__global__ void __launch_bounds__(kThreads, sgd_min_blocks(NC))
adt_sgd_pack_kernel(const __grid_constant__ SgdTable<MAXSEG> T) {
    constexpr int NG = NC > 0 ? NC : 1;
    __shared__ __align__(16) uint32_t stage[kWarpsPerTile][kWarpStageWords];
    if (aborted(T.abort)) return;      // a peer barrier timed out: never step with stale gradients
    const uint32_t tile = blockIdx.x;
    const int s = find_segment(T, tile);
    const uint64_t e0 = static_cast<uint64_t>(tile - T.tile_begin[s]) * kTile;
    const uint32_t m = static_cast<uint32_t>(min(static_cast<uint64_t>(kTile), T.count[s] - e0));
    const int r = width_of(T, s);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t g0 = warp * kWarpGroups + lane;
    uint4 *wp = reinterpret_cast<uint4 *>(T.weights[s]) + e0 / 4;
    uint4 *vp = reinterpret_cast<uint4 *>(T.velocity[s]) + e0 / 4;
    const uint4 *gp[NG];
#pragma unroll
    for (int c = 0; c < NG; ++c)
        gp[c] = reinterpret_cast<const uint4 *>((NC == 0 ? static_cast<uintptr_t>(0)
                                                         : reinterpret_cast<uintptr_t>(T.srcs[c])) + T.grad[s]) + e0 / 4;
    const float lr = T.lr, mu = T.momentum, wd = T.weight_decay;

    uint4 w[kVec], v[kVec];
    if (m == kTile) {
#pragma unroll
        for (int k = 0; k < kVec; ++k) {
            w[k] = __ldcs(wp + g0 + 32 * k);
            v[k] = __ldcs(vp + g0 + 32 * k);
        }
        // Gradient loads are issued kH k-steps at a time ahead of their combines
        // (the IEEE division's slow-path call keeps the compiler from hoisting
        // the next k's loads above it on its own): the whole tile for few
        // contributions, two k-steps for a few more, one beyond (NC loads per
        // k-step are already in flight), within the register budget.
        constexpr int kH = sgd_hoist(NC);
        // many contributions: address each load from the table's source base
        // (a constant-bank operand) + one shared offset instead of keeping NC
        // 64-bit pointers live (they pushed NC >= 14 past 128 registers: spills)
        constexpr bool kLeanPtrs = NC > ADT_SGD_HOIST2_MAX_NC;
        const uintptr_t goff = kLeanPtrs ? T.grad[s] + e0 * 4 : 0;
#pragma unroll
        for (int kb = 0; kb < kVec; kb += kH) {
            uint4 g[kH][NG];
            uintptr_t go = goff;
            if (kLeanPtrs) asm volatile("" : "+l"(go));   // opaque per k-step: the NC addresses are not kept live
#pragma unroll
            for (int h = 0; h < kH; ++h)
#pragma unroll
                for (int c = 0; c < NG; ++c)
                    g[h][c] = __ldcs((kLeanPtrs ? reinterpret_cast<const uint4 *>(reinterpret_cast<uintptr_t>(T.srcs[c]) + go)
                                                : gp[c]) + g0 + 32 * (kb + h));
#pragma unroll
            for (int h = 0; h < kH; ++h) {
                const int k = kb + h;
                uint32_t gx[NG], gy[NG], gz[NG], gw[NG];
#pragma unroll
                for (int c = 0; c < NG; ++c) { gx[c] = g[h][c].x; gy[c] = g[h][c].y; gz[c] = g[h][c].z; gw[c] = g[h][c].w; }
                w[k].x = sgd1(w[k].x, v[k].x, combine<NC>(gx, T), lr, mu, wd);
                w[k].y = sgd1(w[k].y, v[k].y, combine<NC>(gy, T), lr, mu, wd);
                w[k].z = sgd1(w[k].z, v[k].z, combine<NC>(gz, T), lr, mu, wd);
                w[k].w = sgd1(w[k].w, v[k].w, combine<NC>(gw, T), lr, mu, wd);
            }
        }
        // stores after every load: no load is ordered behind a possibly-aliasing store
#pragma unroll
        for (int k = 0; k < kVec; ++k) {
            wp[g0 + 32 * k] = w[k];
            vp[g0 + 32 * k] = v[k];
        }
    } else {
        uint32_t *w1 = reinterpret_cast<uint32_t *>(wp), *v1 = reinterpret_cast<uint32_t *>(vp);
#pragma unroll
        for (int k = 0; k < kVec; ++k) {
            const uint32_t i = (g0 + 32 * k) * 4;
            uint32_t ww[4], vv[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                ww[j] = 0u;
                vv[j] = 0u;
                if (i + j < m) {
                    uint32_t gg[NG];
#pragma unroll
                    for (int c = 0; c < NG; ++c) gg[c] = reinterpret_cast<const uint32_t *>(gp[c])[i + j];
                    vv[j] = v1[i + j];
                    ww[j] = sgd1(w1[i + j], vv[j], combine<NC>(gg, T), lr, mu, wd);
                    w1[i + j] = ww[j];
                    v1[i + j] = vv[j];
                }
            }
            w[k] = make_uint4(ww[0], ww[1], ww[2], ww[3]);
        }
    }
    store_packed(T.packed_out + T.offset[s] + e0 * r, w, m, r, warp, lane, g0, stage[warp]);
    if (T.partials != nullptr) warp_partial(T.partials, tile, sumsq16(w));
}
