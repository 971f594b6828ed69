// adt_awp.cuh — device-resident AWP: decision, re-pack of escalated layers, rank combine.
// Included by adt_kernels.cu inside its anonymous namespace (one translation
// unit: the kernels share the tile helpers, tables and store paths defined there).

// ------------------------------------------------ device-resident AWP step
// Algorithm 1 (precision.py:125-141) on the device, so the
// width decision of a step needs no host round trip and the whole step
// (pack -> [finalize -> observe] || unpack -> fixup) replays as one graph.
// One CTA; thread g walks group g's layers in layer order (groups share one
// state, observed sequentially as in the reference; independent groups run
// in parallel). float64 arithmetic in the reference's operation order:
// norm = sqrt(sum of squares) (IEEE, as math.sqrt), delta = (n - prev) / prev.
constexpr int kAwpThreads = 256;
__global__ void __launch_bounds__(kAwpThreads)
adt_awp_observe_kernel(const double *__restrict__ seg_sumsq, const __grid_constant__ adt_awp_device D,
                       const __grid_constant__ adt_awp_config C, const uint32_t *abort) {
    __shared__ int64_t slot_batch[2];
    __shared__ int32_t n_esc;
    if (aborted(abort)) return;        // inputs came from a failed exchange: the AWP state does not advance
    if (threadIdx.x == 0) {
        slot_batch[0] = D.counter[0] % D.ring_steps;
        slot_batch[1] = D.counter[1];
        n_esc = 0;
    }
    __syncthreads();
    adt_awp_row *rows = D.ring + slot_batch[0] * D.nlayers;
    const int32_t batch = static_cast<int32_t>(slot_batch[1]);
    for (int g = threadIdx.x; g < D.ngroups; g += blockDim.x) {
        adt_awp_group st = D.groups[g];
        const int32_t lo = D.member_start[g], hi = D.member_start[g + 1];
        for (int32_t k = lo; k < hi; ++k) {
            const int32_t l = D.members[k];
            const double n = sqrt(seg_sumsq[l]);
            if (st.has_prev) {
                double delta;
                if (st.prev_norm > 0.0) delta = __ddiv_rn(__dsub_rn(n, st.prev_norm), st.prev_norm);
                else delta = (n == 0.0) ? 0.0 : CUDART_INF;
                st.last_delta = delta;
                st.has_delta = 1;
                if (delta < C.threshold) st.counter += 1;        // NaN never counts
                else if (C.consecutive) st.counter = 0;
            } else {
                st.has_delta = 0;
            }
            if (st.counter == C.interval) {                      // also on the first observation
                st.bits = min(st.bits + C.step_bits, C.max_bits);
                st.counter = 0;
            }
            st.prev_norm = n;
            st.has_prev = 1;
            adt_awp_row row;
            row.norm = n;
            row.delta = st.has_delta ? st.last_delta : 0.0;
            row.batch = batch;
            row.layer = l;
            row.counter = st.counter;
            row.bits = st.bits;
            row.has_delta = st.has_delta;
            row.pad = 0;
            rows[l] = row;
        }
        D.groups[g] = st;
        const uint8_t w = static_cast<uint8_t>((st.bits + 7) / 8);   // bits_to_round_to
        for (int32_t k = lo; k < hi; ++k) {
            const int32_t l = D.members[k];
            D.widths_out[l] = w;
            if (w != D.widths_in[l]) D.escalated[1 + atomicAdd(&n_esc, 1)] = l;
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        D.escalated[0] = n_esc;
        D.counter[0] += 1;
        D.counter[1] += 1;
    }
}

// Re-pack of the layers whose width the observation just raised: their
// payload was written (and speculatively unpacked) at the old width; read the
// master tile again, store its top widths_new bytes into the packed buffer
// and the matching replica words (the reference re-packs at the new widths
// and unpacks that, training.py:209-225). CTAs stride over the tiles of the
// escalated layers only; with no escalation every CTA scans the widths and exits.
template <int MAXSEG>
struct FixupTable {
    Table<MAXSEG> T;                 // replicas (weights[]), offsets, tile map; packed_out = the packed buffer
    uintptr_t masters[MAXSEG];
    int32_t layer_of[MAXSEG];        // global layer id of each segment (a layer piece)
    const int32_t *escalated;        // count, then global layer ids
    const uint8_t *widths_new;       // per segment (chunk-relative)
    int32_t gather;                  // 0: re-pack from masters + write replicas; 1: re-unpack from T.srcs
};

template <int MAXSEG>
__global__ void __launch_bounds__(kThreads)
adt_awp_fixup_kernel(const __grid_constant__ FixupTable<MAXSEG> F) {
    __shared__ __align__(16) uint32_t stage[kWarpsPerTile][kWarpStageWords];
    const Table<MAXSEG> &T = F.T;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint32_t *ws = stage[warp];
    if (aborted(T.abort)) return;
    const int32_t n_esc = F.escalated[0];                // usually 0: one load and out
    uint32_t vt = blockIdx.x;                            // virtual tile index over the escalated segments
    for (int32_t e = 0; e < n_esc; ++e) {
        const int32_t layer = F.escalated[1 + e];
        for (int s = 0; s < T.nseg; ++s) {
            if (F.layer_of[s] != layer) continue;        // segments of other layers / chunks
            const int r = F.widths_new[s];
            const uint32_t nt = T.tile_begin[s + 1] - T.tile_begin[s];
            if (nt == 0) continue;
            for (; vt < nt; vt += gridDim.x) {
                if (F.gather) {                           // the owner re-packed it: read it again
                    unpack_tile<MAXSEG>(T, T.tile_begin[s] + vt, s, ws);
                    continue;
                }
                const uint64_t e0 = static_cast<uint64_t>(vt) * kTile;
                const uint32_t m = static_cast<uint32_t>(min(static_cast<uint64_t>(kTile), T.count[s] - e0));
                const uint32_t g0 = warp * kWarpGroups + lane;
                const uint4 *src = reinterpret_cast<const uint4 *>(F.masters[s]) + e0 / 4;
                const uint32_t *src1 = reinterpret_cast<const uint32_t *>(src);
                const uint32_t keep = 0xFFFFFFFFu << (8 * (4 - r));
                uint4 v[kVec];
#pragma unroll
                for (int k = 0; k < kVec; ++k) {
                    const uint32_t g = g0 + 32 * k, i = g * 4;
                    if (i + 4 <= m) {
                        v[k] = src[g];
                    } else {
                        uint32_t w[4];
#pragma unroll
                        for (int j = 0; j < 4; ++j) w[j] = (i + j < m) ? src1[i + j] : 0u;
                        v[k] = make_uint4(w[0], w[1], w[2], w[3]);
                    }
                }
                store_packed(T.packed_out + T.offset[s] + e0 * r, v, m, r, warp, lane, g0, ws);
                uint4 *dst = reinterpret_cast<uint4 *>(T.weights[s]) + e0 / 4;
                uint32_t *dst1 = reinterpret_cast<uint32_t *>(dst);
#pragma unroll
                for (int k = 0; k < kVec; ++k) {
                    const uint32_t g = g0 + 32 * k, i = g * 4;
                    const uint4 o = make_uint4(v[k].x & keep, v[k].y & keep, v[k].z & keep, v[k].w & keep);
                    if (i + 4 <= m) {
                        dst[g] = o;
                    } else {
                        if (i + 0 < m) dst1[i + 0] = o.x;
                        if (i + 1 < m) dst1[i + 1] = o.y;
                        if (i + 2 < m) dst1[i + 2] = o.z;
                    }
                }
            }
            vt -= nt;                                    // continue the stride in the next escalated segment
        }
    }
}

// Per-layer sums of squares from the ranks' per-piece sums (the norm tails
// gathered from every rank), added in fixed (rank, piece) order — the same
// order as sharded.ShardPlan.combine_sumsq, so every rank gets the same bits.
__global__ void __launch_bounds__(256)
adt_awp_combine_kernel(const double *__restrict__ tails, int npieces_total, const int32_t *__restrict__ piece_layer,
                       int nlayers, double *__restrict__ seg_sumsq, const uint32_t *abort) {
    if (aborted(abort)) return;
    for (int l = blockIdx.x * blockDim.x + threadIdx.x; l < nlayers; l += gridDim.x * blockDim.x) {
        double acc = 0.0;
        for (int k = 0; k < npieces_total; ++k)
            if (piece_layer[k] == l) acc += tails[k];
        seg_sumsq[l] = acc;
    }
}
