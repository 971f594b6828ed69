// adt_tma.cuh — persistent, TMA-pipelined pack / unpack kernels (sm_100a).
//
// Each CTA = 8 consumer warps + 1 producer warp. The producer's elected lane
// streams the CTA's tiles (tile = blockIdx.x + k*gridDim.x) into a 4-stage
// shared-memory ring with bulk async copies (cp.async.bulk, SASS UBLKCP),
// each stage guarded by a full/empty mbarrier pair; consumers compact bytes
// from shared memory with PRMT and write coalesced 32/64/128-bit stores. The
// bytes in flight per SM (2 CTAs x 3-4 stages x 16 KB) no longer depend on
// registers, which is what limited the one-tile-per-CTA kernels.
//
// Consumer mapping: warp w owns the tile's float4 groups [128w, 128w+128);
// lane l handles groups 128w + l + 32j, j = 0..3 (coalesced at every width).
// r = 3 (12 bytes per group) and ragged tails go through a per-warp staging
// buffer so global stores stay 16-byte vectors, synchronised by __syncwarp
// only. The fused float64 norm stores one partial per warp per tile (summed by
// adt_norm_finalize_kernel).
#pragma once

namespace tma {

constexpr int kConsumerWarps = 8;
constexpr int kConsumers = kConsumerWarps * 32;
constexpr int kBlock = kConsumers + 32;
#ifndef ADT_TMA_STAGES
#define ADT_TMA_STAGES 4
#endif
#ifndef ADT_TMA_CTAS
#define ADT_TMA_CTAS 2
#endif
constexpr int kStages = ADT_TMA_STAGES;   // ring depth per CTA
constexpr int kCtasPerSm = ADT_TMA_CTAS;   // persistent CTAs per SM
constexpr int kGroups = kTile / 4;                       // float4 groups per tile (1024)
constexpr int kWarpGroups = kGroups / kConsumerWarps;    // 128
constexpr int kStageBytes = kTile * 4;                   // one FP32 tile (>= any packed tile)

struct Smem {
    uint4 stage[kStages][kStageBytes / 16];
    uint32_t wstage[kConsumerWarps][kWarpGroups * 4];    // per-warp output staging (<= 2 KB)
    unsigned long long full[kStages];
    unsigned long long empty[kStages];
    double red[2][kConsumerWarps];
};

__device__ __forceinline__ uint32_t saddr(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long *b, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(saddr(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long *b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(saddr(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long *b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(saddr(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long *b, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(saddr(b)), "r"(parity) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, unsigned long long *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
        ::"r"(saddr(dst)), "l"(src), "r"(bytes), "r"(saddr(bar)) : "memory");
}
__device__ __forceinline__ void consumer_sync(int id) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(kConsumers) : "memory");
}

struct TileInfo {
    int s;
    uint64_t e0;
    uint32_t m;
    int r;
};

template <int MAXSEG>
__device__ __forceinline__ TileInfo tile_info(const Table<MAXSEG> &T, uint32_t tile) {
    TileInfo ti;
    ti.s = find_segment(T, tile);
    ti.e0 = static_cast<uint64_t>(tile - T.tile_begin[ti.s]) * kTile;
    ti.m = static_cast<uint32_t>(min(static_cast<uint64_t>(kTile), T.count[ti.s] - ti.e0));
    ti.r = T.round_to[ti.s];
    return ti;
}

// Per-warp norm partial, indexed (tile, warp) like the register kernels'
// (warp w here covers the tile's contiguous groups [128w, 128w+128)).
__device__ __forceinline__ void norm_tile(double *partials, uint32_t tile, double acc) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xFFFFFFFFu, acc, o);
    if ((threadIdx.x & 31) == 0) partials[tile * kConsumerWarps + (threadIdx.x >> 5)] = acc;
}

// Copy `nbytes` (clipped to the warp's span) from the warp's staging buffer.
__device__ __forceinline__ void warp_copy_out(const uint32_t *ws, uint8_t *dst, uint32_t nbytes, int lane) {
    const uint32_t n16 = nbytes / 16;
    const uint4 *s4 = reinterpret_cast<const uint4 *>(ws);
    uint4 *d4 = reinterpret_cast<uint4 *>(dst);
    for (uint32_t i = lane; i < n16; i += 32) d4[i] = s4[i];
    const uint8_t *s1 = reinterpret_cast<const uint8_t *>(ws);
    for (uint32_t i = n16 * 16 + lane; i < nbytes; i += 32) dst[i] = s1[i];
}

template <int MAXSEG, bool NORM, bool WRITE>
__global__ void __launch_bounds__(kBlock, kCtasPerSm)
adt_pack_tma_kernel(const __grid_constant__ Table<MAXSEG> T, uint32_t ntiles) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    Smem &S = *reinterpret_cast<Smem *>(smem_raw);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int i = 0; i < kStages; ++i) {
            mbar_init(&S.full[i], 1);
            mbar_init(&S.empty[i], kConsumerWarps);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    if (warp == kConsumerWarps) {  // ---------------- producer
        if (lane == 0) {
            int k = 0;
            for (uint32_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++k) {
                const int st = k % kStages;
                if (k >= kStages) mbar_wait(&S.empty[st], ((k / kStages) - 1) & 1);
                const TileInfo ti = tile_info(T, tile);
                const uint32_t bytes = (ti.m / 4) * 16;
                if (bytes) {
                    mbar_expect_tx(&S.full[st], bytes);
                    bulk_g2s(S.stage[st], reinterpret_cast<const uint8_t *>(T.weights[ti.s]) + ti.e0 * 4, bytes,
                             &S.full[st]);
                } else {
                    mbar_arrive(&S.full[st]);
                }
            }
        }
        return;
    }

    // -------------------------------------------------- consumers
    uint32_t *ws = S.wstage[warp];
    int k = 0;
    for (uint32_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++k) {
        const int st = k % kStages;
        mbar_wait(&S.full[st], (k / kStages) & 1);
        const TileInfo ti = tile_info(T, tile);
        const uint4 *stg = S.stage[st];
        uint4 v[4];
        if (ti.m == kTile) {
#pragma unroll
            for (int j = 0; j < 4; ++j) v[j] = stg[warp * kWarpGroups + lane + 32 * j];
        } else {
            const uint32_t *src1 = reinterpret_cast<const uint32_t *>(T.weights[ti.s]) + ti.e0;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const uint32_t g = warp * kWarpGroups + lane + 32 * j;
                if (g * 4 + 4 <= ti.m) {
                    v[j] = stg[g];
                } else {
                    uint32_t w[4];
#pragma unroll
                    for (int q = 0; q < 4; ++q) w[q] = (g * 4 + q < ti.m) ? src1[g * 4 + q] : 0u;
                    v[j] = make_uint4(w[0], w[1], w[2], w[3]);
                }
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&S.empty[st]);  // stage free: data is in registers

        double acc = 0.0;
        if (NORM) {
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                acc = sq_acc(acc, v[j].x);
                acc = sq_acc(acc, v[j].y);
                acc = sq_acc(acc, v[j].z);
                acc = sq_acc(acc, v[j].w);
            }
        }
        if (WRITE) {
            const int r = ti.r;
            uint8_t *dst = T.packed_out + T.offset[ti.s] + ti.e0 * r;
            const uint32_t g0 = warp * kWarpGroups + lane;
            if (ti.m == kTile && r != 3) {
                if (r == 1) {
                    uint32_t *d = reinterpret_cast<uint32_t *>(dst);
#pragma unroll
                    for (int j = 0; j < 4; ++j) { uint32_t o[1]; pack_r1(v[j], o); d[g0 + 32 * j] = o[0]; }
                } else if (r == 2) {
                    uint2 *d = reinterpret_cast<uint2 *>(dst);
#pragma unroll
                    for (int j = 0; j < 4; ++j) { uint32_t o[2]; pack_r2(v[j], o); d[g0 + 32 * j] = make_uint2(o[0], o[1]); }
                } else {
                    uint4 *d = reinterpret_cast<uint4 *>(dst);
#pragma unroll
                    for (int j = 0; j < 4; ++j) { uint32_t o[4]; pack_r4(v[j], o); d[g0 + 32 * j] = make_uint4(o[0], o[1], o[2], o[3]); }
                }
            } else {
                // per-warp staging: r words per group, then 16-byte stores of the warp's span
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    uint32_t o[4];
                    pack_any(r, v[j], o);
                    uint32_t *p = ws + (lane + 32 * j) * r;
                    p[0] = o[0];
                    if (r > 1) p[1] = o[1];
                    if (r > 2) p[2] = o[2];
                    if (r > 3) p[3] = o[3];
                }
                __syncwarp();
                const uint32_t span = kWarpGroups * 4 * r;          // bytes per warp span
                const uint32_t lo = warp * span;
                const uint32_t nbytes = ti.m * r;
                if (lo < nbytes) warp_copy_out(ws, dst + lo, min(span, nbytes - lo), lane);
                __syncwarp();
            }
        }
        if (NORM) norm_tile(T.partials, tile, acc);
    }
}

template <int MAXSEG>
__global__ void __launch_bounds__(kBlock, kCtasPerSm)
adt_unpack_tma_kernel(const __grid_constant__ Table<MAXSEG> T, uint32_t ntiles) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    if (aborted(T.abort)) return;
    Smem &S = *reinterpret_cast<Smem *>(smem_raw);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int i = 0; i < kStages; ++i) {
            mbar_init(&S.full[i], 1);
            mbar_init(&S.empty[i], kConsumerWarps);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    if (warp == kConsumerWarps) {  // ---------------- producer
        if (lane == 0) {
            int k = 0;
            for (uint32_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++k) {
                const int st = k % kStages;
                if (k >= kStages) mbar_wait(&S.empty[st], ((k / kStages) - 1) & 1);
                const TileInfo ti = tile_info(T, tile);
                const uint32_t bytes = (ti.m * ti.r / 16) * 16;
                if (bytes) {
                    mbar_expect_tx(&S.full[st], bytes);
                    bulk_g2s(S.stage[st], T.srcs[T.src_idx[ti.s]] + T.offset[ti.s] + ti.e0 * ti.r, bytes, &S.full[st]);
                } else {
                    mbar_arrive(&S.full[st]);
                }
            }
        }
        return;
    }

    int k = 0;
    for (uint32_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++k) {
        const int st = k % kStages;
        mbar_wait(&S.full[st], (k / kStages) & 1);
        const TileInfo ti = tile_info(T, tile);
        const int r = ti.r;
        uint4 *stg = S.stage[st];
        if (ti.m < kTile) {
            // ragged tail: the last (< 16) payload bytes come straight from global
            const uint32_t nbytes = ti.m * r, done = (nbytes / 16) * 16;
            const uint8_t *src = T.srcs[T.src_idx[ti.s]] + T.offset[ti.s] + ti.e0 * r;
            uint8_t *s1 = reinterpret_cast<uint8_t *>(stg);
            if (threadIdx.x < nbytes - done) s1[done + threadIdx.x] = src[done + threadIdx.x];
            consumer_sync(2);
        }
        uint4 out[4];
        const uint32_t *s32 = reinterpret_cast<const uint32_t *>(stg);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const uint32_t g = warp * kWarpGroups + lane + 32 * j;
            switch (r) {
                case 1: out[j] = unpack_r1(s32[g]); break;
                case 2: { const uint2 p = reinterpret_cast<const uint2 *>(stg)[g]; out[j] = unpack_r2(p.x, p.y); } break;
                case 3: out[j] = unpack_r3(s32[3 * g], s32[3 * g + 1], s32[3 * g + 2]); break;
                default: out[j] = unpack_r4(stg[g]); break;
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&S.empty[st]);
        uint4 *dst = reinterpret_cast<uint4 *>(T.weights[ti.s]) + ti.e0 / 4;
        if (ti.m == kTile) {
#pragma unroll
            for (int j = 0; j < 4; ++j) dst[warp * kWarpGroups + lane + 32 * j] = out[j];
        } else {
            uint32_t *dst1 = reinterpret_cast<uint32_t *>(dst);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const uint32_t g = warp * kWarpGroups + lane + 32 * j;
                if (g * 4 + 4 <= ti.m) {
                    dst[g] = out[j];
                } else if (g * 4 < ti.m) {
                    const uint32_t ow[4] = {out[j].x, out[j].y, out[j].z, out[j].w};
                    for (uint32_t q = 0; g * 4 + q < ti.m; ++q) dst1[g * 4 + q] = ow[q];
                }
            }
        }
    }
}

}  // namespace tma
