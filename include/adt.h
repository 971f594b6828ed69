/*
 * adt.h — C ABI of the B200 ADT codec (Approximate Data Transfer, arXiv:2004.02297).
 *
 * The reference (`weightpack`, pure Python) has no native boundary; its drop-in
 * surface is the Python API re-exported at /root/reference/pkg/src/weightpack/__init__.py:5-25.
 * Each entry point below replaces the reference function cited beside it; the
 * Python package `paper_2004_02297_b200` binds them through ctypes (see
 * INTEGRATION.md for the binding a maintainer would add to `weightpack`).
 *
 * Rules of the boundary:
 *   - plain pointers and sizes only; all buffers are caller-allocated device
 *     memory (or mapped pinned host memory where stated); the library never
 *     allocates;
 *   - every call is stream-ordered on `stream` (a cudaStream_t passed as void*;
 *     NULL = legacy default stream) and returns an int status: 0 = ADT_OK,
 *     negative = error (see adt_strerror); the library never aborts;
 *   - thread-safe: no mutable globals besides a per-device attribute cache
 *     (and the host packer's worker pool, see adt_pack_host);
 *   - peer-abort guard: entry points that read other ranks' memory take
 *     `const uint32_t *abort` (device memory, or NULL = unguarded). It is the
 *     `state + 1` word of adt_peer_barrier: when it is nonzero at kernel start
 *     the kernel does no work, so after a barrier timeout no stale or
 *     half-written peer bytes reach a replica, a master or the AWP state.
 *
 * Packed layout (codec.py:76-107): layer l's payload is
 * count_l * round_to_l bytes at byte `offset` of the packed buffer; weight i of
 * the layer occupies payload bytes [i*r, (i+1)*r), most-significant byte first
 * (the top r bytes of the IEEE-754 word, big-endian). Offsets must be 16-byte
 * aligned (pad between layers is not part of any payload).
 */
#ifndef ADT_H
#define ADT_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ADT_ABI_VERSION 11

/* status codes */
#define ADT_OK 0
#define ADT_ERR_ROUND_TO (-1)   /* round_to outside [1, 4]            -> ValueError (codec.py:52-57) */
#define ADT_ERR_ALIGN (-2)      /* weights/packed/offset not 16-B aligned */
#define ADT_ERR_ARG (-3)        /* NULL pointer with nonzero count, nseg < 0, overflow */
#define ADT_ERR_NO_DEVICE (-4)  /* no CUDA device / driver */
#define ADT_ERR_CUDA_BASE (-1000) /* -(1000 + cudaError_t) for CUDA runtime errors */

/* Weights per tile: the unit of work of one CTA. */
#define ADT_TILE_WEIGHTS 4096
/* float64 norm partials per tile (one per 512-weight warp slice). */
#define ADT_PARTIALS_PER_TILE 8
/* Source buffers one adt_unpack_multi call may read (ranks of a node). */
#define ADT_MAX_SOURCES 16

/* One layer (a "segment" of the packed stream). */
typedef struct adt_segment {
    void *weights;      /* FP32 words of the layer, 16-B aligned. pack: read; unpack: written */
    uint64_t count;     /* number of weights (may be 0) */
    uint64_t offset;    /* byte offset of this layer's payload in the packed buffer, 16-B aligned */
    int32_t round_to;   /* bytes kept per weight, 1..4 (codec.py:52-57; bits_to_round_to codec.py:60-67) */
    int32_t reserved;   /* 0; for adt_unpack_multi: index of the source buffer holding this payload */
} adt_segment;

/* One layer of the fused SGD step + pack (adt_sgd_pack). */
typedef struct adt_sgd_segment {
    void *weights;      /* FP32 master W, updated in place (16-B aligned) */
    void *velocity;     /* FP32 momentum buffer v, updated in place */
    const void *grad;   /* FP32 averaged gradient g */
    uint64_t count;
    uint64_t offset;    /* payload offset of the packed W' in the packed buffer (16-B aligned) */
    int32_t round_to;
    int32_t reserved;   /* must be 0 */
} adt_sgd_segment;

/* One layer piece of the fused gradient-reduce + SGD step + pack
 * (adt_reduce_sgd_pack). Its gradient contributions live at the SAME byte
 * offset `grad_offset` inside every contribution's gradient buffer (a flat
 * per-worker gradient bucket, or a rank's received shard). */
typedef struct adt_grad_segment {
    void *weights;         /* FP32 master W (this rank's shard piece), updated in place, 16-B aligned */
    void *velocity;        /* FP32 momentum buffer v, updated in place */
    uint64_t count;
    uint64_t offset;       /* payload offset of the packed W' in the packed buffer (16-B aligned) */
    uint64_t grad_offset;  /* byte offset of this piece's gradients in every grads[c] (16-B aligned) */
    int32_t round_to;
    int32_t reserved;      /* must be 0 */
} adt_grad_segment;

/* ABI version (ADT_ABI_VERSION). */
int adt_abi_version(void);

/* Human-readable text for a status code (static storage). */
const char *adt_strerror(int status);

/* Number of float64 norm partials a pack/sumsq over `segs` writes
 * (ADT_PARTIALS_PER_TILE per 4096-weight tile); size `partials` to at least
 * this. Host-only, no device work. */
int adt_partials_count(const adt_segment *segs, int nseg, uint64_t *npartials);

/*
 * Multi-tensor pack.  Replaces codec.pack / pack_vectorized / pack_parallel
 * (codec.py:116-180) applied to every layer, and fuses precision.l2_norm
 * (precision.py:25-28) into the same read of the weights:
 *   partials  != NULL: the pass also stores float64 sums of squares, one per
 *                      512-weight warp slice (adt_partials_count doubles);
 *   seg_sumsq != NULL: (needs partials) a small finalize kernel is launched
 *                      behind the pass (programmatic dependent launch) and
 *                      writes seg_sumsq[l] = layer l's sum of squares, summed
 *                      in a fixed (tile, warp) order: bit-identical run to run.
 * Callers that want the finalize off the critical path pass seg_sumsq = NULL
 * and call adt_norm_finalize on another stream (see sync.WeightSync).
 */
int adt_pack(const adt_segment *segs, int nseg, uint8_t *packed,
             double *seg_sumsq, double *partials, void *stream);

/* seg_sumsq[l] = fixed-order sum of layer l's partials written by adt_pack /
 * adt_sumsq over the same `segs`. */
int adt_norm_finalize(const adt_segment *segs, int nseg, double *partials,
                      double *seg_sumsq, void *stream);

/*
 * Multi-tensor unpack.  Replaces codec.unpack (codec.py:183-197) applied to
 * every layer: writes count_l FP32 words to segs[l].weights, the kept bytes in
 * the high bytes and zeros below.  `packed` may be device memory or mapped
 * (pinned, cudaHostAlloc) host memory — the latter is the zero-copy
 * host->device path (packed weights crossing from CPU master
 * weights to the GPU).
 */
int adt_unpack(const adt_segment *segs, int nseg, const uint8_t *packed, void *stream);

/*
 * Gather-unpack: like adt_unpack, but layer l's payload is read from
 * sources[segs[l].reserved] + segs[l].offset. The sources are the ranks' packed
 * send buffers mapped into this process — peer device memory opened with
 * adt_ipc_open (read over NVLink inside the kernel: the all-gather and the
 * unpack are one pass) or local device/pinned buffers. nsrc <= ADT_MAX_SOURCES.
 * Replaces the per-worker loop of training.py:214-225 (send_weights + unpack).
 */
int adt_unpack_multi(const adt_segment *segs, int nseg, const uint8_t *const *sources, int nsrc,
                     void *stream);

/* adt_unpack_multi with two options: widths != NULL reads each segment's width
 * from device memory (capacity layout, round_to 4, as adt_unpack_multi_dyn);
 * start_seg >= 0 rotates the tile walk to begin just before segment start_seg
 * (the caller's own first piece), so that ranks reading each other's buffers
 * at the same moment pull from different peers rather than all draining one
 * owner's NVLink port in lockstep. Results do not depend on either option's
 * scheduling. */
int adt_unpack_multi_ex(const adt_segment *segs, int nseg, const uint8_t *const *sources, int nsrc,
                        const uint8_t *widths, int start_seg, const uint32_t *abort, void *stream);

/* dst[q*bytes .. (q+1)*bytes) = sources[q][offset .. offset+bytes) for q < nsrc
 * (small peer reads, e.g. every rank's norm tail). */
int adt_copy_multi(uint8_t *dst, const uint8_t *const *sources, int nsrc, uint64_t offset, uint64_t bytes,
                   const uint32_t *abort, void *stream);

/*
 * Stream-ordered barrier over peer memory (replaces the NCCL all-reduce of a
 * flag the p2p transport would otherwise use between "my pack is written" and
 * "peers read it"; the reference's in-process workers need none,
 * training.py:214-225). flags[q] = rank q's array of nranks uint32 epochs,
 * mapped into this process (adt_ipc_open) — flags[rank] is local; all start
 * at 0. state = 2 local uint32: [0] this rank's epoch counter (start 0),
 * [1] 0, or the epoch whose wait timed out after timeout_ns nanoseconds of
 * device time (the kernel then returns instead of hanging). state + 1 is the
 * abort word of the guarded entry points queued behind the barrier; once it
 * is set, later barriers return at once. Callers poll it (e.g. a D2H copy
 * after every step) and raise. Every rank must issue the same sequence of
 * barriers. Graph-capturable.
 */
int adt_peer_barrier(uint32_t *const *flags, int nranks, int rank, uint32_t *state, uint64_t timeout_ns,
                     void *stream);

/* CUDA IPC plumbing for adt_unpack_multi (thin wrappers over cudaIpc*):
 * handle size in bytes; export the allocation holding dev_ptr (*offset_out =
 * dev_ptr's byte offset inside it); map a peer's allocation (peer access
 * enabled lazily; add the exporter's offset); unmap it. */
int adt_ipc_handle_bytes(void);
int adt_ipc_get_handle(void *dev_ptr, void *handle_out, uint64_t *offset_out);
int adt_ipc_open(const void *handle, void **dev_ptr_out);
int adt_ipc_close(void *dev_ptr);

/*
 * Norm-only pass (no packed output): seg_sumsq[l] = float64 sum of squares of
 * layer l.  Replaces precision.l2_norm (precision.py:25-28) for the batch whose
 * norm is not fused into a pack (the last observation of a run, training.py:246-254).
 */
int adt_sumsq(const adt_segment *segs, int nseg, double *seg_sumsq,
              double *partials, void *stream);

/*
 * Fused momentum-SGD step + pack + norm. Per weight, in
 * float32 with the reference's rounding at every operation (net.py:236-246):
 *   g' = g + weight_decay*W (only if weight_decay != 0); v = v*momentum + g';
 *   W = W - lr*v
 * then W's top round_to bytes go to the packed buffer and, with partials /
 * seg_sumsq, W's float64 sums of squares are fused in (as adt_pack). One pass
 * reads W, v, g (12 B/weight) and writes W, v, packed (8 + r B/weight).
 */
int adt_sgd_pack(const adt_sgd_segment *segs, int nseg, float lr, float momentum, float weight_decay,
                 uint8_t *packed, double *seg_sumsq, double *partials, void *stream);

/*
 * Gradient return path fused with the update and the pack (SURVEY.md §8f
 * item 4). Replaces net.gather_and_update's weight half (net.py:203-246) fed
 * by transfer.TransferBoundary.return_gradients (transfer.py:247-251):
 *   g  = pairwise_sum_c( g_c * f32(sample_counts[c]) ) / f32(sum of sample_counts)
 *        (pairwise_sum's association tree, net.py:186-200; float32, rounded
 *        after every operation)
 * then the momentum step of adt_sgd_pack, the pack of W' and (optionally) its
 * fused norm.  grads[c] (c < ncontrib <= ADT_MAX_SOURCES) are the workers'
 * gradient buffers: local device memory, or the peer ranks' gradient buckets
 * mapped with adt_ipc_open — then the reduce-scatter onto this rank's master
 * shard IS this kernel's load stage (the gradients cross NVLink once, are
 * combined in registers, and never land in HBM as a reduced copy).
 */
int adt_reduce_sgd_pack(const adt_grad_segment *segs, int nseg, const float *const *grads,
                        const int64_t *sample_counts, int ncontrib, float lr, float momentum,
                        float weight_decay, uint8_t *packed, double *seg_sumsq, double *partials,
                        const uint32_t *abort, void *stream);

/*
 * Device-resident AWP step (single-device WeightSync(awp_on_device=True)).
 * The reference decides widths on the host between two packs
 * (precision.py:125-141, training.py:246-254, then :209-213); here the
 * decision runs on the GPU so a whole step replays as one CUDA graph with no
 * device->host read. Layers use capacity offsets (room for 4 bytes/weight,
 * segs[l].round_to must be 4); the width in force for layer l is A[l]
 * (device memory). Per step:
 *   adt_pack_dyn(A) -> [adt_norm_finalize -> adt_awp_observe(-> B)] || adt_unpack_dyn(A)
 *   -> adt_awp_fixup(A, B) -> copy B to A
 * adt_awp_observe advances each group's state, writes one trace row per layer
 * (TRACE_HEADER, precision.py:18) into a ring of ring_steps steps, stores
 * the new widths in widths_out (B) and lists the layers whose width rose; the
 * fixup re-packs (from the masters) and re-unpacks only those (with none, its
 * CTAs exit after one load).
 */
typedef struct adt_awp_config {
    double threshold;        /* T (precision.py:46-54) */
    int32_t interval;        /* INTERVAL */
    int32_t step_bits;       /* N */
    int32_t max_bits;
    int32_t consecutive;     /* 0 = cumulative counter (the default) */
} adt_awp_config;

typedef struct adt_awp_group {   /* LayerPrecisionState, precision.py:67-74 */
    double prev_norm;
    double last_delta;
    int32_t bits;
    int32_t counter;
    int32_t has_prev;            /* prev_norm is not None */
    int32_t has_delta;           /* last_delta is not None */
} adt_awp_group;

typedef struct adt_awp_row {     /* (batch, layer, norm, delta, counter, bits) */
    double norm;
    double delta;                /* valid when has_delta */
    int32_t batch;
    int32_t layer;
    int32_t counter;
    int32_t bits;
    int32_t has_delta;
    int32_t pad;
} adt_awp_row;

typedef struct adt_awp_device {  /* all pointers: device memory */
    adt_awp_group *groups;       /* [ngroups] */
    const int32_t *members;      /* [nlayers] layer ids grouped by group, in layer order within a group */
    const int32_t *member_start; /* [ngroups + 1] */
    const uint8_t *widths_in;    /* [nlayers] bytes per weight the step's pack used (A) */
    uint8_t *widths_out;         /* [nlayers] bytes per weight after this observation (B, 1..4) */
    int32_t *escalated;          /* [nlayers + 1]: count, then the layers with B != A (any order) */
    adt_awp_row *ring;           /* [ring_steps * nlayers] trace rows, step slot = counter[0] % ring_steps */
    int64_t *counter;            /* [2]: observations so far, batch label of the next observation */
    int32_t nlayers;
    int32_t ngroups;
    int32_t ring_steps;
    int32_t reserved;            /* 0 */
} adt_awp_device;

/* adt_pack (norm partials only, finalize separately) with the widths read from device memory. */
int adt_pack_dyn(const adt_segment *segs, int nseg, uint8_t *packed, double *partials, const uint8_t *widths,
                 void *stream);
/* adt_unpack with the widths read from device memory. */
int adt_unpack_dyn(const adt_segment *segs, int nseg, const uint8_t *packed, const uint8_t *widths, void *stream);
/* adt_sgd_pack / adt_reduce_sgd_pack (norm partials only) with the widths read from device memory. */
int adt_sgd_pack_dyn(const adt_sgd_segment *segs, int nseg, float lr, float momentum, float weight_decay,
                     uint8_t *packed, double *partials, const uint8_t *widths, void *stream);
int adt_reduce_sgd_pack_dyn(const adt_grad_segment *segs, int nseg, const float *const *grads,
                            const int64_t *sample_counts, int ncontrib, float lr, float momentum,
                            float weight_decay, uint8_t *packed, double *partials, const uint8_t *widths,
                            const uint32_t *abort, void *stream);
/* One AWP observation of every layer from the finalized sums of squares. */
int adt_awp_observe(const double *seg_sumsq, const adt_awp_device *dev, const adt_awp_config *cfg,
                    const uint32_t *abort, void *stream);
/* Re-pack + re-unpack, at widths_new, of the layers listed in `escalated` (as written by
 * adt_awp_observe); masters[l] and replicas[l] share count / offset (capacity layout,
 * round_to 4). */
int adt_awp_fixup(const adt_segment *masters, const adt_segment *replicas, int nseg, uint8_t *packed,
                  const int32_t *escalated, const uint8_t *widths_new, void *stream);

/* Multi-rank device AWP (ShardedWeightSync(transport="p2p", awp_on_device=True)): segments are
 * layer pieces, seg_layer[i] the global layer of piece i (host array).
 *   adt_unpack_multi_dyn: adt_unpack_multi with per-piece widths from device memory;
 *   adt_awp_combine:      per-layer sums of squares from the gathered per-piece sums tails[k]
 *                         (piece_layer[k], device, -1 = empty slot), added in k order
 *                         (rank-major, as ShardPlan.combine_sumsq) — identical on every rank;
 *   adt_awp_fixup_pieces: adt_awp_fixup for this rank's pieces (re-pack into its send buffer,
 *                         write its replica pieces);
 *   adt_awp_fixup_gather: re-unpack the escalated pieces of every rank from their (re-packed)
 *                         send buffers, at widths_new (per piece). */
int adt_unpack_multi_dyn(const adt_segment *segs, int nseg, const uint8_t *const *sources, int nsrc,
                         const uint8_t *widths, const uint32_t *abort, void *stream);
int adt_awp_combine(const double *tails, int npieces_total, const int32_t *piece_layer, int nlayers,
                    double *seg_sumsq, const uint32_t *abort, void *stream);
int adt_awp_fixup_pieces(const adt_segment *masters, const adt_segment *replicas, int nseg, const int32_t *seg_layer,
                         uint8_t *packed, const int32_t *escalated, const uint8_t *widths_new, const uint32_t *abort,
                         void *stream);
int adt_awp_fixup_gather(const adt_segment *replicas, int nseg, const int32_t *seg_layer,
                         const uint8_t *const *sources, int nsrc, const int32_t *escalated,
                         const uint8_t *widths_new, const uint32_t *abort, void *stream);

/*
 * Host (CPU) pack: the paper's Bitpack stage for CPU-resident master weights
 * (PAPER.md:219-229, 259-268, 351-452). Same bytes as adt_pack / codec.pack
 * (codec.py:116-180) and, with seg_sumsq != NULL, the float64 sum of squares
 * of every layer (precision.py:25-28) fused into the same read. segs[l].weights
 * are HOST pointers (4-B aligned), `packed` is host memory (pinned for DMA).
 * Runs on `threads` host threads (<= 0: all of the process's CPU affinity) —
 * a persistent worker pool owned by the library (created on first use;
 * concurrent calls queue). Work is cut into fixed 64K-weight units, so bytes
 * and sums never depend on the thread count. AVX-512 VBMI when the CPU has
 * it (adt_host_simd() == 512), else a scalar loop. Synchronous.
 */
int adt_pack_host(const adt_segment *segs, int nseg, uint8_t *packed, double *seg_sumsq, int threads);

/*
 * The CPU-master transfer, pipelined: adt_pack_host of host_segs into the
 * pinned staging buffer host_packed; while the host threads pack, the calling
 * thread queues cudaMemcpyAsync (on `stream`) of every finished run of the
 * packed stream (>= min_copy_bytes; 0 = automatic: 1 MiB, or a quarter of a
 * stream under 4 MiB but >= 64 KiB) into dev_packed, so the PCIe
 * DMA overlaps the packing; then adt_unpack of dev_segs (device replicas, the
 * same counts / offsets / round_to, payloads in increasing offset order) from
 * dev_packed — or no unpack when dev_segs is NULL (the caller queues it). Only Σ n·r (+ pad) bytes cross the link instead of 4n.
 * Returns once the host work is done and the copies + unpack are queued: the
 * caller must not rewrite host_packed before `stream` has passed this point.
 * seg_sumsq (host memory) receives the per-layer sums of squares.
 */
int adt_host_to_device(const adt_segment *host_segs, const adt_segment *dev_segs, int nseg, uint8_t *host_packed,
                       uint8_t *dev_packed, uint64_t packed_bytes, double *seg_sumsq, int threads,
                       uint64_t min_copy_bytes, void *stream);

/*
 * adt_host_to_device with options. flags:
 *   ADT_H2D_DIRECT_FULL — layers at round_to 4 whose host words are page-locked
 *     (both ends of the range registered with CUDA) are not packed on the host:
 *     the DMA copies their FP32 words straight into dev_segs[l].weights (the
 *     replica equals the master at full width, so the result is identical;
 *     4n bytes cross the link either way) before the packed stream, and their
 *     unpack is skipped. Their seg_sumsq entries still come from a host pass
 *     (read only; bit-identical to the packed path's sums). Host DRAM then
 *     carries their 4n bytes once instead of three times. Needs dev_segs.
 *   ADT_H2D_SKIP_DIRECT_NORMS — with DIRECT_FULL: no host norm pass over the
 *     direct layers (their seg_sumsq entries are set to NaN); the caller takes
 *     them from the replicas on the device (adt_sumsq: the replica IS the
 *     master at full width). Measured on the B200 host: a host read of the
 *     direct layers running beside their DMA slows the DMA by up to 40 %
 *     (profiles/r02_host_direct.md).
 *   ADT_H2D_ZERO_COPY — no staging copies: host_packed must be page-locked
 *     (device-mapped), and the unpack reads the packed stream from it across
 *     the link once the host has packed it (dev_packed is not written). For
 *     small streams, where one copy's fixed cost exceeds its transfer time
 *     (profiles/r02_small_host.md). Needs dev_segs.
 * direct_out (nseg bytes, may be NULL) receives 1 for every layer sent that way.
 * Everything else as adt_host_to_device (which is this call with flags 0).
 */
#define ADT_H2D_DIRECT_FULL 1u
#define ADT_H2D_SKIP_DIRECT_NORMS 2u
#define ADT_H2D_ZERO_COPY 4u
int adt_host_to_device_ex(const adt_segment *host_segs, const adt_segment *dev_segs, int nseg, uint8_t *host_packed,
                          uint8_t *dev_packed, uint64_t packed_bytes, double *seg_sumsq, int threads,
                          uint64_t min_copy_bytes, uint32_t flags, uint8_t *direct_out, void *stream);

/*
 * adt_host_to_device through a small pinned RING instead of a staging buffer
 * as large as the stream: the stream is cut into chunks (runs of 64K-weight
 * units) of at most slot_bytes (>= 256 KiB + 64); chunk c is packed into slot
 * c % (ring_bytes / slot_bytes) once the copy of the slot's previous chunk has
 * completed, and the calling thread queues each chunk's copy (in order) as
 * soon as it is packed. The ring stays cache-resident, so the copies read the
 * packed bytes from the host's last-level cache rather than DRAM, and only the
 * masters stream through host memory. Same bytes, sums and unpack as
 * adt_host_to_device; needs more slots than host threads.
 */
int adt_host_to_device_ring(const adt_segment *host_segs, const adt_segment *dev_segs, int nseg, uint8_t *ring,
                            uint64_t ring_bytes, uint64_t slot_bytes, uint8_t *dev_packed, uint64_t packed_bytes,
                            double *seg_sumsq, int threads, void *stream);

/* Host threads adt_pack_host uses at most (the process's CPU affinity). */
int adt_host_threads(int *n);
/* 512 when the host packer runs its AVX-512 VBMI path, 0 for the scalar path. */
int adt_host_simd(void);

/*
 * Float64-input norm: *out = sum of x[i]^2 over n float64 words (device
 * memory, 8-B aligned) — precision.l2_norm (precision.py:25-28) of an array
 * that is not float32 (the reference converts any array-like to float64).
 * Fixed grid and reduction order: bit-identical run to run. `partials` holds
 * adt_sumsq_f64_partials(n) doubles of scratch.
 */
int adt_sumsq_f64_partials(uint64_t n, uint64_t *npartials);
int adt_sumsq_f64(const double *x, uint64_t n, double *partials, double *out, void *stream);

/*
 * One-launch step for small sets (latency-bound: LeNet is 106 tiles): pack
 * masters -> packed with the fused norm, grid barrier, unpack packed ->
 * replicas (each CTA unpacks a tile another CTA packed), per-layer sums of
 * squares -> seg_sumsq (same fixed order as adt_norm_finalize). Same results as
 * adt_pack(+finalize) followed by adt_unpack. Requires nseg <= 16 and at most
 * adt_roundtrip_max_tiles() tiles (one CTA per SM, launched cooperatively, so
 * the grid barrier never waits on an unscheduled CTA); ADT_ERR_ARG otherwise.
 * barrier: 2 uint32 of device memory, zero-initialised once, owned by the
 * caller and not shared by concurrent launches. partials: adt_partials_count.
 */
int adt_roundtrip(const adt_segment *masters, const adt_segment *replicas, int nseg, uint8_t *packed,
                  double *seg_sumsq, double *partials, uint32_t *barrier, void *stream);
int adt_roundtrip_max_tiles(int *tiles);

/* Number of SMs of the current device (cached). */
int adt_device_sm_count(int *sm_count);

#ifdef __cplusplus
}
#endif

#endif /* ADT_H */
