// triinv.cuh -- recursive block inverse of a small triangle held in shared memory.
//
// X = T^-1 for T lower unit (UPPER = false) or upper non-unit (UPPER = true), size R (a power
// of two, >= 16) with the live part t <= R; rows/columns >= t are treated as identity.
// 8 x 8 leaves by substitution, then for block sizes 16 .. R every diagonal block
// [X11 0; X21 X22] gets X21 = -X22 (L21 X11)  (upper: X12 = -X11 (U12 X22)): log-depth,
// each level two small products over shared memory.  Dot products are exact in u64
// (<= R/2 terms of < 2^52), one Barrett fold per entry.  All threads of the CTA call it.
#pragma once

#include "common.cuh"

namespace ffg {

template <bool UPPER, int R>
__device__ void tri_inverse_smem(const uint32_t* S, int ss, uint32_t* X, int xs, uint32_t* W, uint32_t* dinv, uint32_t t,
                                 uint32_t p, uint64_t mu) {
    constexpr int LEAF = 8;
    const uint32_t tid = threadIdx.x, nth = blockDim.x;
    for (uint32_t idx = tid; idx < (uint32_t)R * R; idx += nth) X[(idx / R) * xs + idx % R] = 0u;
    for (uint32_t i = tid; i < (uint32_t)R; i += nth)
        dinv[i] = (!UPPER || i >= t) ? 1u : inv_mod32(S[i * ss + i], p);
    __syncthreads();
    if (tid < (uint32_t)R) {  // leaves: thread per (leaf block, column)
        const uint32_t base = (tid / LEAF) * LEAF, j = tid % LEAF;
        uint32_t x[LEAF];
#pragma unroll
        for (int i = 0; i < LEAF; ++i) x[i] = 0;
        x[j] = dinv[base + j];
        if (!UPPER) {
#pragma unroll
            for (int i = 0; i < LEAF; ++i) {
                if (i <= (int)j) continue;
                uint64_t s = 0;
#pragma unroll
                for (int k = 0; k < LEAF; ++k)
                    if (k >= (int)j && k < i && base + i < t && base + k < t) s += (uint64_t)S[(base + i) * ss + base + k] * x[k];
                const uint32_t v = mod_u64(s, p, mu);
                x[i] = v ? p - v : 0u;
            }
        } else {
#pragma unroll
            for (int i = LEAF - 1; i >= 0; --i) {
                if (i >= (int)j) continue;
                uint64_t s = 0;
#pragma unroll
                for (int k = 0; k < LEAF; ++k)
                    if (k > i && k <= (int)j && base + i < t && base + k < t) s += (uint64_t)S[(base + i) * ss + base + k] * x[k];
                uint32_t v = mod_u64(s, p, mu);
                v = v ? p - v : 0u;
                x[i] = mul_mod(v, dinv[base + i], p, mu);
            }
        }
#pragma unroll
        for (int i = 0; i < LEAF; ++i) X[(base + i) * xs + base + j] = x[i];
    }
    __syncthreads();
    for (uint32_t b = 2 * LEAF; b <= (uint32_t)R; b *= 2) {
        const uint32_t h = b / 2, nblk = R / b, per = h * h;
        for (uint32_t idx = tid; idx < nblk * per; idx += nth) {
            const uint32_t blk = idx / per, e = idx % per, i = e / h, c = e % h, ob = blk * b;
            uint64_t s = 0;
            if (!UPPER) {  // W = L21 X11 (X11 lower: k >= c)
                const uint32_t row = ob + h + i;
                if (row < t)
                    for (uint32_t k = c; k < h; ++k)
                        if (ob + k < t) s += (uint64_t)S[row * ss + ob + k] * X[(ob + k) * xs + ob + c];
            } else {  // W = U12 X22 (X22 upper: k <= c)
                const uint32_t row = ob + i;
                if (row < t)
                    for (uint32_t k = 0; k <= c; ++k)
                        if (ob + h + k < t) s += (uint64_t)S[row * ss + ob + h + k] * X[(ob + h + k) * xs + ob + h + c];
            }
            W[blk * per + i * h + c] = mod_u64(s, p, mu);
        }
        __syncthreads();
        for (uint32_t idx = tid; idx < nblk * per; idx += nth) {
            const uint32_t blk = idx / per, e = idx % per, i = e / h, c = e % h, ob = blk * b;
            const uint32_t* w = W + blk * per;
            uint64_t s = 0;
            if (!UPPER) {  // X21 = -X22 W (X22 lower: k <= i)
                for (uint32_t k = 0; k <= i; ++k) s += (uint64_t)X[(ob + h + i) * xs + ob + h + k] * w[k * h + c];
                const uint32_t v = mod_u64(s, p, mu);
                X[(ob + h + i) * xs + ob + c] = v ? p - v : 0u;
            } else {  // X12 = -X11 W (X11 upper: k >= i)
                for (uint32_t k = i; k < h; ++k) s += (uint64_t)X[(ob + i) * xs + ob + k] * w[k * h + c];
                const uint32_t v = mod_u64(s, p, mu);
                X[(ob + i) * xs + ob + h + c] = v ? p - v : 0u;
            }
        }
        __syncthreads();
    }
}

}  // namespace ffg
