// adt_f64.cuh — float64-input sum of squares (precision.l2_norm of any array).
// Included by adt_kernels.cu inside its anonymous namespace.
//
// The reference's l2_norm (precision.py:25-28) converts ANY array-like to
// float64 and takes sqrt(dot(x, x)). Float32 inputs go through the fused pack /
// norm-only pass (widening is exact); everything else arrives here as float64
// words: each CTA of a fixed grid sums a grid-stride slice with FMA (x*x + acc,
// as a vectorised ddot does), lanes and warps reduce in a fixed tree, one
// partial per CTA; one CTA then adds the partials in index order. The grid
// depends only on n, so the result is bit-identical run to run.
constexpr int kF64Threads = 256;
constexpr int kF64MaxCtas = 1184;            // 8 x 148 SMs

__host__ __device__ inline int f64_ctas(uint64_t n) {
    const uint64_t per = static_cast<uint64_t>(kF64Threads) * 16;
    const uint64_t c = (n + per - 1) / per;
    return static_cast<int>(c < 1 ? 1 : (c > kF64MaxCtas ? kF64MaxCtas : c));
}

__global__ void __launch_bounds__(kF64Threads)
adt_sumsq_f64_kernel(const double *__restrict__ x, uint64_t n, double *__restrict__ partials) {
    __shared__ double red[kF64Threads / 32];
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * kF64Threads;
    double a0 = 0.0, a1 = 0.0;
    uint64_t i = static_cast<uint64_t>(blockIdx.x) * kF64Threads + threadIdx.x;
    for (; i + stride < n; i += 2 * stride) {
        const double u = __ldcs(x + i), v = __ldcs(x + i + stride);
        a0 = fma(u, u, a0);
        a1 = fma(v, v, a1);
    }
    if (i < n) {
        const double u = __ldcs(x + i);
        a0 = fma(u, u, a0);
    }
    double a = a0 + a1;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) a += __shfl_down_sync(0xFFFFFFFFu, a, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = a;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
#pragma unroll
        for (int w = 0; w < kF64Threads / 32; ++w) t += red[w];
        partials[blockIdx.x] = t;
    }
}

__global__ void __launch_bounds__(32) adt_sumsq_f64_finalize(const double *__restrict__ partials, int np,
                                                            double *__restrict__ out) {
    double a = 0.0;
    for (int k = threadIdx.x; k < np; k += 32) a += partials[k];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) a += __shfl_down_sync(0xFFFFFFFFu, a, o);
    if (threadIdx.x == 0) *out = a;
}
