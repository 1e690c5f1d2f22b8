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

// One doubling level (block size BS = 2h) of tri_inverse_smem, sizes compile-time so the
// index arithmetic is shifts.  A thread owns 4 consecutive rows x 1 column of an h x h
// product: one load of the shared operand column feeds four exact u64 accumulators.
// barrier over the participating threads: the whole CTA (id 0) or a named subset
__device__ __forceinline__ void tri_bar(uint32_t id, uint32_t nth) {
    if (id == 0)
        __syncthreads();
    else
        asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nth) : "memory");
}

template <bool UPPER, int R, int BS>
__device__ __forceinline__ void tri_inverse_levels(const uint32_t* S, int ss, uint32_t* X, int xs, uint32_t* W,
                                                   uint32_t t, uint32_t p, uint64_t mu, uint32_t tid, uint32_t nth,
                                                   uint32_t bar) {
    if constexpr (BS <= R) {
        constexpr uint32_t h = BS / 2, nblk = R / BS, per_blk = (h / 4) * h;
        for (uint32_t tile = tid; tile < nblk * per_blk; tile += nth) {
            const uint32_t blk = tile / per_blk, e = tile % per_blk, i0 = (e / h) * 4, c = e % h, ob = blk * BS;
            uint64_t s[4] = {0, 0, 0, 0};
            if (!UPPER) {  // W = L21 X11 (X11 lower: k >= c); rows/cols >= t contribute nothing
                const uint32_t row0 = ob + h + i0;
                const uint32_t kend = t > ob ? min(h, t - ob) : 0u;
#pragma unroll 4
                for (uint32_t k = c; k < kend; ++k) {
                    const uint64_t xk = X[(ob + k) * xs + ob + c];
#pragma unroll
                    for (int a = 0; a < 4; ++a) s[a] += (uint64_t)S[(row0 + a) * ss + ob + k] * xk;
                }
#pragma unroll
                for (int a = 0; a < 4; ++a) W[blk * h * h + (i0 + a) * h + c] = row0 + a < t ? mod_u64(s[a], p, mu) : 0u;
            } else {  // W = U12 X22 (X22 upper: k <= c)
                const uint32_t row0 = ob + i0;
                const uint32_t kend = t > ob + h ? min(c + 1, t - ob - h) : 0u;
#pragma unroll 4
                for (uint32_t k = 0; k < kend; ++k) {
                    const uint64_t xk = X[(ob + h + k) * xs + ob + h + c];
#pragma unroll
                    for (int a = 0; a < 4; ++a) s[a] += (uint64_t)S[(row0 + a) * ss + ob + h + k] * xk;
                }
#pragma unroll
                for (int a = 0; a < 4; ++a) W[blk * h * h + (i0 + a) * h + c] = row0 + a < t ? mod_u64(s[a], p, mu) : 0u;
            }
        }
        tri_bar(bar, nth);
        for (uint32_t tile = tid; tile < nblk * per_blk; tile += nth) {
            const uint32_t blk = tile / per_blk, e = tile % per_blk, i0 = (e / h) * 4, c = e % h, ob = blk * BS;
            const uint32_t* w = W + blk * h * h;
            uint64_t s[4] = {0, 0, 0, 0};
            if (!UPPER) {  // X21 = -X22 W (X22 lower: k <= i; the zeros above its diagonal pad)
#pragma unroll 4
                for (uint32_t k = 0; k < i0 + 4; ++k) {
                    const uint64_t wk = w[k * h + c];
#pragma unroll
                    for (int a = 0; a < 4; ++a) s[a] += (uint64_t)X[(ob + h + i0 + a) * xs + ob + h + k] * wk;
                }
#pragma unroll
                for (int a = 0; a < 4; ++a) {
                    const uint32_t v = mod_u64(s[a], p, mu);
                    X[(ob + h + i0 + a) * xs + ob + c] = v ? p - v : 0u;
                }
            } else {  // X12 = -X11 W (X11 upper: k >= i)
#pragma unroll 4
                for (uint32_t k = i0; k < h; ++k) {
                    const uint64_t wk = w[k * h + c];
#pragma unroll
                    for (int a = 0; a < 4; ++a) s[a] += (uint64_t)X[(ob + i0 + a) * xs + ob + k] * wk;
                }
#pragma unroll
                for (int a = 0; a < 4; ++a) {
                    const uint32_t v = mod_u64(s[a], p, mu);
                    X[(ob + i0 + a) * xs + ob + h + c] = v ? p - v : 0u;
                }
            }
        }
        tri_bar(bar, nth);
        tri_inverse_levels<UPPER, R, BS * 2>(S, ss, X, xs, W, t, p, mu, tid, nth, bar);
    }
}

// All participating threads call it: the whole CTA (tri_inverse_smem) or a subset of nth
// threads with local index tid synchronising on named barrier `bar` (tri_inverse_part), so two
// inverses can run side by side in one CTA.
template <bool UPPER, int R>
__device__ void tri_inverse_part(const uint32_t* S, int ss, uint32_t* X, int xs, uint32_t* W, uint32_t* dinv,
                                 uint32_t t, uint32_t p, uint64_t mu, uint32_t tid, uint32_t nth, uint32_t bar) {
    constexpr int LEAF = 8;
    for (uint32_t idx = tid; idx < (uint32_t)R * R; idx += nth) X[(idx / R) * xs + idx % R] = 0u;
    if (!UPPER) {
        for (uint32_t i = tid; i < (uint32_t)R; i += nth) dinv[i] = 1u;
    } else if (tid < 32) {
        // batch inversion of the diagonal in one warp, 64 entries (two per lane) per round:
        // prefix products D_e = prod_{j<e} d_j, one inverse of the total, 1/d_e = D_e / D_{e+1} --
        // one extended Euclid per 64 entries instead of 64 divergent ones
        const uint32_t FULL = 0xffffffffu, lane = tid;
        for (uint32_t o = 0; o < (uint32_t)R; o += 64) {
            const uint32_t e0 = o + 2 * lane, e1 = e0 + 1;
            const uint32_t v0 = (e0 < t && e0 < (uint32_t)R) ? S[e0 * ss + e0] : 1u % p;
            const uint32_t v1 = (e1 < t && e1 < (uint32_t)R) ? S[e1 * ss + e1] : 1u % p;
            uint32_t inc = mul_mod(v0, v1, p, mu);
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                const uint32_t u = __shfl_up_sync(FULL, inc, off);
                if (lane >= (uint32_t)off) inc = mul_mod(inc, u, p, mu);
            }
            uint32_t D0 = __shfl_up_sync(FULL, inc, 1);
            if (lane == 0) D0 = 1u % p;
            const uint32_t D1 = mul_mod(D0, v0, p, mu);
            const uint32_t total = __shfl_sync(FULL, inc, 31);
            const uint32_t tinv = __shfl_sync(FULL, lane == 0 ? inv_mod_bin(total, p) : 0u, 0);
            uint32_t suf = mul_mod(v0, v1, p, mu);
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                const uint32_t u = __shfl_down_sync(FULL, suf, off);
                if (lane + off < 32) suf = mul_mod(suf, u, p, mu);
            }
            const uint32_t sufx = __shfl_down_sync(FULL, suf, 1);
            const uint32_t iD2 = mul_mod(tinv, lane == 31 ? 1u % p : sufx, p, mu);  // 1 / D_{e0 + 2}
            const uint32_t iD1 = mul_mod(iD2, v1, p, mu);                           // 1 / D_{e0 + 1}
            // a zero diagonal entry (singular input; uniform) keeps the per-entry inverses (0 for it)
            const bool sing = total == 0u;
            if (e0 < (uint32_t)R) dinv[e0] = e0 >= t ? 1u : (sing ? inv_mod_bin(v0, p) : mul_mod(D0, iD1, p, mu));
            if (e1 < (uint32_t)R) dinv[e1] = e1 >= t ? 1u : (sing ? inv_mod_bin(v1, p) : mul_mod(D1, iD2, p, mu));
        }
    }
    tri_bar(bar, nth);
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
    tri_bar(bar, nth);
    tri_inverse_levels<UPPER, R, 2 * LEAF>(S, ss, X, xs, W, t, p, mu, tid, nth, bar);
}

template <bool UPPER, int R>
__device__ void tri_inverse_smem(const uint32_t* S, int ss, uint32_t* X, int xs, uint32_t* W, uint32_t* dinv, uint32_t t,
                                 uint32_t p, uint64_t mu) {
    tri_inverse_part<UPPER, R>(S, ss, X, xs, W, dinv, t, p, mu, threadIdx.x, blockDim.x, 0);
}

}  // namespace ffg
