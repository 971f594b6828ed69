// adt_peer.cuh — small peer-memory kernels: norm-tail gather, stream-ordered barrier.
// Included by adt_kernels.cu inside its anonymous namespace (one translation
// unit: the kernels share the tile helpers, tables and store paths defined there).

// ------------------------------------------------------- small peer copies
// dst[q*bytes + i] = srcs[q][offset + i]: gathers each rank's norm tail (a few
// dozen bytes) out of its peer-mapped send buffer.
struct SrcList {
    const uint8_t *p[ADT_MAX_SOURCES];
};
__global__ void adt_copy_multi_param_kernel(uint8_t *dst, const __grid_constant__ SrcList S, uint64_t offset,
                                            uint64_t bytes, const uint32_t *abort) {
    if (aborted(abort)) return;
    const uint8_t *src = S.p[blockIdx.x] + offset;
    for (uint64_t i = threadIdx.x; i < bytes; i += blockDim.x) dst[blockIdx.x * bytes + i] = src[i];
}

// ------------------------------------------------ stream-ordered peer barrier
// One warp. Lane q publishes this rank's new epoch into rank q's flag array
// (peer memory over NVLink, release at system scope after a system fence, so
// every write of the kernels before it on this stream is visible to the peers
// first), then waits until every rank's epoch has arrived in the local array
// (acquire at system scope: the kernels after it on this stream see the
// peers' writes). The epoch comes from a device counter, so the barrier is
// CUDA-graph capturable. The wait is bounded in time (%globaltimer): on
// timeout the epoch is written to state[1] — the abort word every guarded
// kernel behind it checks (Table::abort), so the step's peer reads, the AWP
// observation and the optimizer step are skipped instead of consuming stale
// bytes — and the kernel exits (no hung GPU; the host raises at its next
// poll). Once state[1] is set, later barriers return at once (fail fast).
struct FlagList {
    uint32_t *p[ADT_MAX_SOURCES];
};
__device__ __forceinline__ uint64_t global_ns() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__global__ void __launch_bounds__(32) adt_peer_barrier_kernel(const __grid_constant__ FlagList F, int nranks,
                                                              int rank, uint32_t *state, uint64_t timeout_ns) {
    const int lane = threadIdx.x;
    uint32_t epoch = 0, failed = 0;
    if (lane == 0) {
        epoch = state[0] + 1u;
        failed = *reinterpret_cast<volatile uint32_t *>(state + 1);
    }
    epoch = __shfl_sync(0xFFFFFFFFu, epoch, 0);
    if (__shfl_sync(0xFFFFFFFFu, failed, 0) != 0u) {
        if (lane == 0) state[0] = epoch;
        return;
    }
    __threadfence_system();
    if (lane < nranks) {
        uint32_t *dst = F.p[lane] + rank;
        asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(dst), "r"(epoch) : "memory");
    }
    const uint32_t *mine = F.p[rank];
    bool done = false;
    const uint64_t t0 = global_ns();
    for (uint32_t it = 0;; ++it) {
        uint32_t v = epoch;
        if (lane < nranks) asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(mine + lane) : "memory");
        done = __all_sync(0xFFFFFFFFu, static_cast<int32_t>(v - epoch) >= 0);
        if (done) break;
        if ((it & 63u) == 63u) {   // lane 0's clock decides for the whole warp (no divergent exit)
            const int late = lane == 0 ? static_cast<int>(global_ns() - t0 > timeout_ns) : 0;
            if (__shfl_sync(0xFFFFFFFFu, late, 0)) break;
        }
        __nanosleep(64);
    }
    if (lane == 0) {
        state[0] = epoch;
        if (!done) {
            state[1] = epoch;
            __threadfence();
        }
    }
}
