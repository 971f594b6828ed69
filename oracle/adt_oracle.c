/*
 * CPU ORACLE — TEST INFRASTRUCTURE ONLY (never linked into the product).
 *
 * Plain-C restatement of the reference ADT codec (weightpack, pure NumPy):
 *   oracle_pack    /root/reference/pkg/src/weightpack/codec.py:116-130 (scalar pack:
 *                  per weight, the top r bytes of the big-endian word)
 *   oracle_unpack  codec.py:183-197 (kept bytes -> word MSBs, low bytes zero)
 *   oracle_sumsq   precision.py:25-28 (float64 sum of squares; sequential order —
 *                  the reference's order is OpenBLAS ddot's and is not pinned)
 * Used by tests/ to check the CUDA path at sizes where the NumPy oracle is slow;
 * pinned against the reference-generated fixtures in tests/golden/ by
 * tests/test_oracle.py.
 */
#include <stddef.h>
#include <stdint.h>

int oracle_pack(const uint32_t *words, size_t n, int r, uint8_t *out) {
    if (r < 1 || r > 4) return -1;
    for (size_t i = 0; i < n; ++i) {
        const uint32_t w = words[i];
        for (int k = 0; k < r; ++k) out[i * r + k] = (uint8_t)(w >> (24 - 8 * k));
    }
    return 0;
}

int oracle_unpack(const uint8_t *in, size_t n, int r, uint32_t *out) {
    if (r < 1 || r > 4) return -1;
    for (size_t i = 0; i < n; ++i) {
        uint32_t w = 0;
        for (int k = 0; k < r; ++k) w |= (uint32_t)in[i * r + k] << (24 - 8 * k);
        out[i] = w;
    }
    return 0;
}

double oracle_sumsq(const float *x, size_t n) {
    double s = 0.0;
    for (size_t i = 0; i < n; ++i) s += (double)x[i] * (double)x[i];
    return s;
}
