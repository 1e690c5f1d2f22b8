// trsm.cu -- modular triangular solves, recursive onto the tcgen05 GEMM.
//
// Replaces ftrsm / pftrsm / trsm_left / trsm_right (blas.hpp:285-419).  The
// solution of a triangular system mod p is unique, so any exact evaluation
// order gives the reference's bits.  Structure:
//   1. one launch inverts every TB x TB diagonal block of the triangle
//      (tri_inv_kernel, one CTA per block, exact column substitution in SMEM);
//   2. a recursion split at multiples of TB turns the off-diagonal work into
//      Schur GEMMs  B2 -= T21 X1  (fgemm, alpha = p-1, beta = 1);
//   3. each leaf is the GEMM  X = inv(T_bb) B_b  (alpha = 1, beta = 0) written
//      in place -- safe because the GEMM reads limb copies made before it runs.
// Only the selected triangle (plus the diagonal when nonunit) is read, so T can
// be the packed L\U square that tile_rec passes (rankrev.hpp:112,114).
#include <mutex>

#include "pluq.cuh"
#include "ptx.cuh"
#include "triinv.cuh"

namespace ffg {

constexpr int TB = 128;  // diagonal block (= GEMM K-block, so leaf GEMMs have no K padding)

// Inverse of diagonal block b of T (t x t) into Tinv + b*TB*TB (TB x TB, zero padded).
// One warp per column j of the inverse (32 columns per CTA, TB/32 CTAs per block), solving
// T x = e_j by substitution in 32-row chunks with lane = row within the chunk:
//   1. each lane accumulates its row's dot product with the x entries of earlier chunks
//      (independent per lane: no reduction, x broadcast by shuffles);
//   2. the 32 x 32 diagonal sub-block is solved with one shuffle + one MAC per step.
// Sums stay exact in u64 (< 128 products of < 2^52); one Barrett fold per entry.
constexpr int TRI_COLS = 32;
constexpr int TSTR = TB + 1;  // padded row stride: lanes read different rows of one column
template <bool UPPER, bool UNIT>
__global__ void __launch_bounds__(TRI_COLS * 32) tri_inv_kernel(const uint32_t* __restrict__ T, uint64_t ldt,
                                                               uint32_t t, uint32_t* __restrict__ Tinv, uint32_t p,
                                                               uint64_t mu) {
    extern __shared__ uint32_t sm[];
    uint32_t* S = sm;                 // TB x TSTR block of T
    uint32_t* dinv = sm + TB * TSTR;  // TB inverses of the diagonal (nonunit)
    uint32_t* dinvp = dinv + TB;      // their Shoup factors
    const uint32_t b = blockIdx.x / (TB / TRI_COLS), cblk = blockIdx.x % (TB / TRI_COLS);
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t o = b * TB;
    const uint32_t tb = min((uint32_t)TB, t - o);
    for (uint32_t r = warp; r < (uint32_t)TB; r += TRI_COLS)
        for (uint32_t c = lane; c < (uint32_t)TB; c += 32)
            S[r * TSTR + c] = (r < tb && c < tb) ? T[(uint64_t)(o + r) * ldt + o + c] : 0u;
    __syncthreads();
    if (!UNIT)
        for (uint32_t i = threadIdx.x; i < tb; i += blockDim.x) {
            dinv[i] = inv_mod32(S[i * TSTR + i], p);
            dinvp[i] = shoup_pre(dinv[i], p, mu);
        }
    __syncthreads();
    const uint32_t j = cblk * TRI_COLS + warp;  // column of the inverse owned by this warp
    uint32_t x[TB / 32];                         // x[q] = X[q*32 + lane][j]
#pragma unroll
    for (int q = 0; q < TB / 32; ++q) x[q] = 0;
    if (j < tb) {
        const uint32_t xj = UNIT ? 1u : dinv[j];
        const int cj = (int)(j >> 5);
#pragma unroll
        for (int cc = 0; cc < TB / 32; ++cc) {
            const int c = UPPER ? (TB / 32 - 1 - cc) : cc;
            if (UPPER ? (c > cj) : (c < cj)) continue;  // chunk entirely zero for this column
            const uint32_t i = (uint32_t)c * 32 + lane;  // this lane's row
            uint64_t s = 0;
            // 1. contributions of the already-solved chunks
#pragma unroll
            for (int q = 0; q < TB / 32; ++q) {
                if (UPPER ? (q <= c || q > cj) : (q >= c || q < cj)) continue;
                for (int l2 = 0; l2 < 32; ++l2) {
                    const uint32_t xk = __shfl_sync(0xffffffffu, x[q], l2);
                    s += (uint64_t)S[i * TSTR + q * 32 + l2] * xk;
                }
            }
            // 2. the diagonal 32 x 32 sub-block, one row per step
            uint32_t mine = 0;
            for (int s2 = 0; s2 < 32; ++s2) {
                const int kk = UPPER ? 31 - s2 : s2;
                const uint32_t k = (uint32_t)c * 32 + kk;
                uint32_t v = 0;
                if (lane == (uint32_t)kk) {
                    if (k == j) {
                        v = xj;
                    } else if (UPPER ? (k < j) : (k > j)) {
                        v = mod_u64(s, p, mu);
                        v = v ? p - v : 0u;
                        if (!UNIT && k < tb) v = shoup_mul(v, dinv[k], dinvp[k], p);
                        if (k >= tb) v = 0;
                    }
                    mine = v;
                }
                const uint32_t xk = __shfl_sync(0xffffffffu, v, kk);
                if (UPPER ? (lane < (uint32_t)kk) : (lane > (uint32_t)kk)) s += (uint64_t)S[i * TSTR + k] * xk;
            }
            x[c] = mine;
        }
    }
    uint32_t* out = Tinv + (uint64_t)b * TB * TB;
    if (j < (uint32_t)TB) {
#pragma unroll
        for (int q = 0; q < TB / 32; ++q) out[(uint64_t)(q * 32 + lane) * TB + j] = x[q];
    }
}

// Recursive block inverse of diagonal block b (log depth instead of a TB-step chain):
// 8 x 8 leaves by substitution, then for block sizes 16, 32, 64, 128 every diagonal
// block [X11 0; X21 X22] (lower) gets X21 = -X22 (L21 X11); upper: X12 = -X11 (U12 X22).
// Each level is two small products over shared memory, all blocks of the level at once;
// dot products are exact in u64 (<= 64 terms < 2^52), one Barrett fold per entry.
constexpr int RI_THREADS = 512;
constexpr int LEAF = 8;
template <bool UPPER, bool UNIT>
__global__ void __launch_bounds__(RI_THREADS) tri_inv_rec_kernel(const uint32_t* __restrict__ T, uint64_t ldt,
                                                                uint32_t t, uint32_t* __restrict__ Tinv, uint32_t p,
                                                                uint64_t mu) {
    extern __shared__ uint32_t sm[];
    uint32_t* S = sm;                    // TB x TSTR: the triangle
    uint32_t* X = S + TB * TSTR;         // TB x TSTR: its inverse
    uint32_t* W = X + TB * TSTR;         // (TB/2) x (TB/2 + 1) temporaries
    ptx::pdl_enter();
    uint32_t* dinv = W + (TB / 2) * (TB / 2 + 1);
    const uint32_t tid = threadIdx.x, o = blockIdx.x * TB;
    const uint32_t tb = min((uint32_t)TB, t - o);
    for (uint32_t idx = tid; idx < (uint32_t)TB * TB; idx += RI_THREADS) {
        const uint32_t r = idx / TB, c = idx % TB;
        S[r * TSTR + c] = (r < tb && c < tb) ? T[(uint64_t)(o + r) * ldt + o + c] : 0u;
        X[r * TSTR + c] = 0u;
    }
    __syncthreads();
    if constexpr ((!UPPER && UNIT) || (UPPER && !UNIT)) {
        // tile_rec's two triangles: the compile-time-level inverse with register tiles (triinv.cuh)
        tri_inverse_smem<UPPER, TB>(S, TSTR, X, TSTR, W, dinv, tb, p, mu);
        uint32_t* out = Tinv + (uint64_t)blockIdx.x * TB * TB;
        for (uint32_t idx = tid; idx < (uint32_t)TB * TB; idx += RI_THREADS) {
            const uint32_t r = idx / TB, c = idx % TB;
            out[idx] = (r < tb && c < tb) ? X[r * TSTR + c] : 0u;
        }
        return;
    }
    for (uint32_t i = tid; i < (uint32_t)TB; i += RI_THREADS)
        dinv[i] = UNIT ? 1u : (i < tb ? inv_mod32(S[i * TSTR + i], p) : 1u);
    __syncthreads();
    // leaves: thread per (leaf block, column)
    if (tid < (uint32_t)TB) {
        const uint32_t lb = tid / LEAF, j = tid % LEAF, base = lb * LEAF;
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
                    if (k >= (int)j && k < i) s += (uint64_t)S[(base + i) * TSTR + base + k] * x[k];
                uint32_t v = mod_u64(s, p, mu);
                v = v ? p - v : 0u;
                x[i] = UNIT ? v : mul_mod(v, dinv[base + i], p, mu);
            }
        } else {
#pragma unroll
            for (int i = LEAF - 1; i >= 0; --i) {
                if (i >= (int)j) continue;
                uint64_t s = 0;
#pragma unroll
                for (int k = 0; k < LEAF; ++k)
                    if (k > i && k <= (int)j) s += (uint64_t)S[(base + i) * TSTR + base + k] * x[k];
                uint32_t v = mod_u64(s, p, mu);
                v = v ? p - v : 0u;
                x[i] = UNIT ? v : mul_mod(v, dinv[base + i], p, mu);
            }
        }
#pragma unroll
        for (int i = 0; i < LEAF; ++i) X[(base + i) * TSTR + base + j] = x[i];
    }
    __syncthreads();
    for (uint32_t b = 2 * LEAF; b <= (uint32_t)TB; b *= 2) {
        const uint32_t h = b / 2, nblk = TB / b, per = h * h;
        // W_blk = L21 X11 (lower) or U12 X22 (upper), stored per block at W + blk*per (fits: nblk*per = TB*h/2)
        for (uint32_t idx = tid; idx < nblk * per; idx += RI_THREADS) {
            const uint32_t blk = idx / per, e = idx % per, i = e / h, c = e % h, ob = blk * b;
            uint64_t s = 0;
            if (!UPPER) {  // L21[i][k] * X11[k][c], X11 lower -> k >= c
                const uint32_t* lrow = S + (ob + h + i) * TSTR + ob;
                for (uint32_t k = c; k < h; ++k) s += (uint64_t)lrow[k] * X[(ob + k) * TSTR + ob + c];
            } else {  // U12[i][k] * X22[k][c], X22 upper -> k <= c
                const uint32_t* urow = S + (ob + i) * TSTR + ob + h;
                for (uint32_t k = 0; k <= c; ++k) s += (uint64_t)urow[k] * X[(ob + h + k) * TSTR + ob + h + c];
            }
            W[blk * per + i * h + c] = mod_u64(s, p, mu);
        }
        __syncthreads();
        for (uint32_t idx = tid; idx < nblk * per; idx += RI_THREADS) {
            const uint32_t blk = idx / per, e = idx % per, i = e / h, c = e % h, ob = blk * b;
            const uint32_t* w = W + blk * per;
            uint64_t s = 0;
            if (!UPPER) {  // X21[i][c] = -sum_{k<=i} X22[i][k] W[k][c]
                const uint32_t* xrow = X + (ob + h + i) * TSTR + ob + h;
                for (uint32_t k = 0; k <= i; ++k) s += (uint64_t)xrow[k] * w[k * h + c];
                const uint32_t v = mod_u64(s, p, mu);
                X[(ob + h + i) * TSTR + ob + c] = v ? p - v : 0u;
            } else {  // X12[i][c] = -sum_{k>=i} X11[i][k] W[k][c]
                const uint32_t* xrow = X + (ob + i) * TSTR + ob;
                for (uint32_t k = i; k < h; ++k) s += (uint64_t)xrow[k] * w[k * h + c];
                const uint32_t v = mod_u64(s, p, mu);
                X[(ob + i) * TSTR + ob + h + c] = v ? p - v : 0u;
            }
        }
        __syncthreads();
    }
    uint32_t* out = Tinv + (uint64_t)blockIdx.x * TB * TB;
    for (uint32_t idx = tid; idx < (uint32_t)TB * TB; idx += RI_THREADS) {
        const uint32_t r = idx / TB, c = idx % TB;
        out[idx] = (r < tb && c < tb) ? X[r * TSTR + c] : 0u;
    }
}

// Direct small triangular solve (t <= TB): one launch, no inverse matrix, no limb staging.
// Every case is rewritten as a forward substitution over "vectors" (columns of B for a
// left solve, rows of B for a right solve) with coefficients C[i][k], k < i:
//   left  lower: C = T,        forward      right upper: C = T^T,  forward
//   left  upper: C = T,        reversed     right lower: C = T^T,  reversed
// x_i = (b_i - sum_{k<i} C[i][k] x_k) * d_i,  d_i = 1 (unit) or T[i][i]^-1 (nonunit).
// A CTA owns 64 vectors; rows go in chunks of 16: (1) all 256 threads form the chunk's
// dot products with the solved rows (u64, exact), (2) 64 threads finish the 16 x 16
// diagonal block with register-resident x.  Exact residues throughout.
constexpr int SV = 64;   // vectors per CTA
constexpr int SCH = 16;  // rows per chunk
template <int SIDE, bool REV, bool UNIT>
__global__ void __launch_bounds__(256) trsm_small_kernel(const uint32_t* __restrict__ T, uint64_t ldt, uint32_t t,
                                                         uint32_t* __restrict__ B, uint64_t ldb, uint32_t nvec,
                                                         uint32_t p, uint64_t mu) {
    extern __shared__ __align__(16) uint32_t sm[];
    uint32_t* C = sm;                       // TB x TSTR
    uint32_t* X = C + TB * TSTR;            // TB x (SV + 1)
    uint32_t* Acc = X + TB * (SV + 1);      // SCH x SV
    uint32_t* dg = Acc + SCH * SV;          // TB
    uint32_t* dgp = dg + TB;                // TB
    const uint32_t tid = threadIdx.x, v0 = blockIdx.x * SV;
    const uint32_t nv = min((uint32_t)SV, nvec - v0);
    // coefficients in forward order
    for (uint32_t idx = tid; idx < t * t; idx += 256) {
        const uint32_t i = idx / t, k = idx % t;
        if (k > i || (UNIT && k == i)) continue;
        const uint32_t oi = REV ? t - 1 - i : i, ok = REV ? t - 1 - k : k;
        C[i * TSTR + k] = SIDE == 0 ? T[(uint64_t)oi * ldt + ok] : T[(uint64_t)ok * ldt + oi];
    }
    // vectors: X[i][v] = b_{oi} of vector v
    if (SIDE == 0) {
        for (uint32_t idx = tid; idx < t * SV; idx += 256) {
            const uint32_t i = idx / SV, v = idx % SV;
            const uint32_t oi = REV ? t - 1 - i : i;
            X[i * (SV + 1) + v] = v < nv ? B[(uint64_t)oi * ldb + v0 + v] : 0u;
        }
    } else {
        for (uint32_t idx = tid; idx < t * SV; idx += 256) {
            const uint32_t v = idx / t, i = idx % t;
            const uint32_t oi = REV ? t - 1 - i : i;
            X[i * (SV + 1) + v] = v < nv ? B[(uint64_t)(v0 + v) * ldb + oi] : 0u;
        }
    }
    __syncthreads();
    if (!UNIT)
        for (uint32_t i = tid; i < t; i += 256) {
            dg[i] = inv_mod32(C[i * TSTR + i], p);
            dgp[i] = shoup_pre(dg[i], p, mu);
        }
    const uint32_t v = tid % SV, rl = tid / SV;  // step-1 mapping: 4 row lanes x 64 vectors
    for (uint32_t i0 = 0; i0 < t; i0 += SCH) {
        // (1) dot products of the chunk rows with the already-solved rows k < i0
        if (i0 > 0) {
            for (uint32_t q = 0; q < SCH / 4; ++q) {
                const uint32_t i = i0 + rl + 4 * q;
                if (i >= t) continue;
                uint64_t s = 0;
                const uint32_t* crow = C + i * TSTR;
                for (uint32_t k = 0; k < i0; ++k) s += (uint64_t)crow[k] * X[k * (SV + 1) + v];
                Acc[(rl + 4 * q) * SV + v] = mod_u64(s, p, mu);
            }
        } else {
            for (uint32_t q = 0; q < SCH / 4; ++q) Acc[(rl + 4 * q) * SV + v] = 0u;
        }
        __syncthreads();
        // (2) the diagonal SCH x SCH block, one vector per thread
        if (tid < SV) {
            uint32_t xr[SCH];
#pragma unroll
            for (int ii = 0; ii < SCH; ++ii) {
                const uint32_t i = i0 + ii;
                uint32_t val = 0;
                if (i < t) {
                    uint64_t s = Acc[ii * SV + v];
                    const uint32_t* crow = C + i * TSTR + i0;
#pragma unroll
                    for (int k = 0; k < ii; ++k) s += (uint64_t)crow[k] * xr[k];
                    const uint32_t sm_ = mod_u64(s, p, mu);
                    const uint32_t b = X[i * (SV + 1) + v];
                    val = b >= sm_ ? b - sm_ : b + p - sm_;
                    if (!UNIT) val = shoup_mul(val, dg[i], dgp[i], p);
                    X[i * (SV + 1) + v] = val;
                }
                xr[ii] = val;
            }
        }
        __syncthreads();
    }
    if (SIDE == 0) {
        for (uint32_t idx = tid; idx < t * SV; idx += 256) {
            const uint32_t i = idx / SV, vv = idx % SV;
            if (vv >= nv) continue;
            const uint32_t oi = REV ? t - 1 - i : i;
            B[(uint64_t)oi * ldb + v0 + vv] = X[i * (SV + 1) + vv];
        }
    } else {
        for (uint32_t idx = tid; idx < t * SV; idx += 256) {
            const uint32_t vv = idx / t, i = idx % t;
            if (vv >= nv) continue;
            const uint32_t oi = REV ? t - 1 - i : i;
            B[(uint64_t)(v0 + vv) * ldb + oi] = X[i * (SV + 1) + vv];
        }
    }
}

// Leaf of a panel solve: X = inv(L) B (left) or X = B inv(U) (right), in place, with the
// inverse cached by the base case (d <= 64).  A CTA owns 64 vectors (columns of B for left,
// rows for right) and stages them in shared memory before writing, so in place is safe.
// 256 threads x (4 x 4) register tiles fed by two 16-byte shared loads per k (coefficients
// stored transposed), exact u64 dot products (<= 64 terms), results staged back through shared
// memory so both sides store whole rows.
constexpr int LA = 64;
constexpr int LAS = LA + 4;  // 16-byte aligned rows
// qp (right side only, may be null): the vectors' elements are read through this local column
// permutation first (the base case's column pivots applied to its bottom panel, in place)
template <int SIDE>
__global__ void __launch_bounds__(256) leaf_apply_kernel(const uint32_t* __restrict__ inv, uint32_t d,
                                                         uint32_t* __restrict__ B, uint64_t ldb, uint32_t nvec,
                                                         uint32_t p, uint64_t mu, const uint32_t* __restrict__ qp) {
    __shared__ __align__(16) uint32_t Ct[LA][LAS];  // Ct[k][i] = coefficient of x_k in output i
    __shared__ __align__(16) uint32_t Bs[LA][LAS];  // Bs[k][v] = element k of vector v (later outputs)
    const uint32_t tid = threadIdx.x;
    constexpr int PER = LA * LA / 256;
    uint32_t rb[PER];
    // the strip's loads, all in flight at once (a rolled loop serialises their latencies)
    auto load = [&](uint32_t v0) {
        const uint32_t nv = min((uint32_t)LA, nvec - v0);
#pragma unroll
        for (int r = 0; r < PER; ++r) {
            const uint32_t idx = tid + 256 * r, hi = idx / LA, lo = idx % LA;
            if (SIDE == 0)  // hi = k, lo = v
                rb[r] = (hi < d && lo < nv) ? B[(uint64_t)hi * ldb + v0 + lo] : 0u;
            else  // hi = v, lo = k
                rb[r] = (lo < d && hi < nv) ? B[(uint64_t)(v0 + hi) * ldb + (qp ? qp[lo] : lo)] : 0u;
        }
    };
    ptx::pdl_enter();
    {
        uint32_t rc[PER];
#pragma unroll
        for (int r = 0; r < PER; ++r) {
            const uint32_t idx = tid + 256 * r, hi = idx / LA, lo = idx % LA;
            rc[r] = (lo < d && hi < d) ? inv[hi * d + lo] : 0u;  // coalesced rows of the inverse
        }
        if (blockIdx.x * LA < nvec) load(blockIdx.x * LA);
#pragma unroll
        for (int r = 0; r < PER; ++r) {
            const uint32_t idx = tid + 256 * r;
            if (SIDE == 0)  // Ct[k][i] = inv(L)[i][k]: transposed on the shared-memory store (a
                Ct[idx % LA][idx / LA] = rc[r];  // strided global read cost 32 lines per warp load)
            else
                Ct[idx / LA][idx % LA] = rc[r];
        }
    }
    // strips blockIdx.x, blockIdx.x + gridDim.x, ...: the next strip's loads fly during this one's math
    for (uint32_t v0 = blockIdx.x * LA; v0 < nvec; v0 += gridDim.x * LA) {
        const uint32_t nv = min((uint32_t)LA, nvec - v0);
        __syncthreads();  // the previous strip's outputs are written out
#pragma unroll
        for (int r = 0; r < PER; ++r) {
            const uint32_t idx = tid + 256 * r, hi = idx / LA, lo = idx % LA;
            if (SIDE == 0)
                Bs[hi][lo] = rb[r];
            else
                Bs[lo][hi] = rb[r];
        }
        __syncthreads();
        if (v0 + gridDim.x * LA < nvec) load(v0 + gridDim.x * LA);
        const uint32_t ti = tid / 16, tv = tid % 16;
        uint64_t acc[4][4] = {};
        // both inverses are triangular in the output index: output i only takes k <= i
        const uint32_t kend = min(d, ti * 4 + 4);
        for (uint32_t k = 0; k < kend; ++k) {
            const uint4 c = *reinterpret_cast<const uint4*>(&Ct[k][ti * 4]);
            const uint4 x = *reinterpret_cast<const uint4*>(&Bs[k][tv * 4]);
            const uint32_t cc[4] = {c.x, c.y, c.z, c.w}, xx[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int q = 0; q < 4; ++q) acc[a][q] += (uint64_t)cc[a] * xx[q];
        }
        __syncthreads();  // every thread is done reading Bs: reuse it for the outputs Os[i][v]
#pragma unroll
        for (int a = 0; a < 4; ++a) {
            uint4 o;
            o.x = mod_u64(acc[a][0], p, mu);
            o.y = mod_u64(acc[a][1], p, mu);
            o.z = mod_u64(acc[a][2], p, mu);
            o.w = mod_u64(acc[a][3], p, mu);
            *reinterpret_cast<uint4*>(&Bs[ti * 4 + a][tv * 4]) = o;
        }
        __syncthreads();
        if (SIDE == 0) {
            for (uint32_t idx = tid; idx < LA * LA; idx += 256) {
                const uint32_t i = idx / LA, v = idx % LA;
                if (i < d && v < nv) B[(uint64_t)i * ldb + v0 + v] = Bs[i][v];
            }
        } else {
            for (uint32_t idx = tid; idx < LA * LA; idx += 256) {
                const uint32_t v = idx / LA, i = idx % LA;
                if (i < d && v < nv) B[(uint64_t)(v0 + v) * ldb + i] = Bs[i][v];
            }
        }
    }
}

// Fused small TRSM (t <= R <= 128): every CTA inverts the triangle in shared memory
// (tri_inverse_smem, log depth) and applies it to its own 64 vectors in place --
// one launch instead of inverse + limb split + tensor GEMM.  The inverse is recomputed per
// CTA, which is cheap next to the launch chain it replaces for the small TRSMs of the
// bottom recursion levels.
template <int SIDE, bool UPPER, bool UNIT, int R>
__global__ void __launch_bounds__(512) trsm_fused_kernel(const uint32_t* __restrict__ T, uint64_t ldt, uint32_t t,
                                                         uint32_t* __restrict__ B, uint64_t ldb, uint32_t nvec,
                                                         uint32_t p, uint64_t mu) {
    extern __shared__ __align__(16) uint32_t sm[];
    constexpr int RS = R + 1;
    uint32_t* Ts = sm;              // R x RS triangle, later the vector strip (R x 65)
    uint32_t* Xs = Ts + R * RS;     // R x RS inverse
    uint32_t* Ws = Xs + R * RS;     // (R/2)^2
    uint32_t* dv = Ws + (R / 2) * (R / 2);
    const uint32_t tid = threadIdx.x, v0 = blockIdx.x * LA;
    const uint32_t nv = min((uint32_t)LA, nvec - v0);
    ptx::pdl_enter();
    for (uint32_t idx = tid; idx < t * t; idx += 512) {
        const uint32_t i = idx / t, k = idx % t;
        Ts[i * RS + k] = T[(uint64_t)i * ldt + k];
    }
    __syncthreads();
    if (UNIT) {
        tri_inverse_smem<false, R>(Ts, RS, Xs, RS, Ws, dv, t, p, mu);  // unit lower
    } else {
        tri_inverse_smem<true, R>(Ts, RS, Xs, RS, Ws, dv, t, p, mu);   // upper (tile_rec's pair)
    }
    // vectors into the triangle's frame: Bs[k][v]
    uint32_t* Bs = Ts;
    if (SIDE == 0) {
        for (uint32_t idx = tid; idx < t * LA; idx += 512) {
            const uint32_t k = idx / LA, v = idx % LA;
            Bs[k * (LA + 1) + v] = v < nv ? B[(uint64_t)k * ldb + v0 + v] : 0u;
        }
    } else {
        for (uint32_t idx = tid; idx < t * LA; idx += 512) {
            const uint32_t v = idx / t, k = idx % t;
            Bs[k * (LA + 1) + v] = v < nv ? B[(uint64_t)(v0 + v) * ldb + k] : 0u;
        }
    }
    __syncthreads();
    // out(i, v) = sum_k C[i][k] Bs[k][v], C = X (left) or X^T (right); 512 threads = 32 row
    // groups x 16 vector groups, each R/32 rows x 4 vectors
    constexpr int RPT = R / 32;
    const uint32_t tr = tid / 16, tv = tid % 16;
    uint64_t acc[RPT][4];
#pragma unroll
    for (int a = 0; a < RPT; ++a)
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[a][q] = 0;
    for (uint32_t k = 0; k < t; ++k) {
        uint32_t x[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) x[q] = Bs[k * (LA + 1) + tv * 4 + q];
#pragma unroll
        for (int a = 0; a < RPT; ++a) {
            const uint32_t i = tr * RPT + a;
            const uint32_t c = SIDE == 0 ? Xs[i * RS + k] : Xs[k * RS + i];
#pragma unroll
            for (int q = 0; q < 4; ++q) acc[a][q] += (uint64_t)c * x[q];
        }
    }
#pragma unroll
    for (int a = 0; a < RPT; ++a) {
        const uint32_t i = tr * RPT + a;
        if (i >= t) continue;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const uint32_t v = tv * 4 + q;
            if (v >= nv) continue;
            const uint32_t val = mod_u64(acc[a][q], p, mu);
            if (SIDE == 0)
                B[(uint64_t)i * ldb + v0 + v] = val;
            else
                B[(uint64_t)(v0 + v) * ldb + i] = val;
        }
    }
}

template <int R>
void trsm_fused_launch(const Blas& b, int side, int upper, int unit, DView T, DView B) {
    const size_t nvec = side == 0 ? B.cols : B.rows;
    const size_t smem = (2 * R * (R + 1) + (R / 2) * (R / 2) + R + 4) * sizeof(uint32_t);
    using K = void (*)(const uint32_t*, uint64_t, uint32_t, uint32_t*, uint64_t, uint32_t, uint32_t, uint64_t);
    // tile_rec pairs: (left, lower, unit) and (right, upper, nonunit); others use the generic path
    K k = side == 0 ? trsm_fused_kernel<0, false, true, R> : trsm_fused_kernel<1, true, false, R>;
    static PerDeviceOnce once;
    once([&] {
        FFG_CUDA(cudaFuncSetAttribute(trsm_fused_kernel<0, false, true, R>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        FFG_CUDA(cudaFuncSetAttribute(trsm_fused_kernel<1, true, false, R>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    });
    b.ws.prof.begin(b.st);
    launch_k(k, dim3((unsigned)ceil_div(nvec, LA)), dim3(512), smem, b.st, T.d, T.ld, (uint32_t)T.rows, B.d, B.ld,
             (uint32_t)nvec, b.F.p, b.F.mu);
    FFG_CUDA(cudaGetLastError());
    b.ws.prof.end(b.st, PROF_TRINV, 8.0 * (double)T.rows * nvec);
    b.count();
}

// Both factor inverses of a packed t x t block (t <= 64, full rank): inv(L) (unit lower) by
// threads 0..255 and inv(U) (upper, non-unit) by threads 256..511 side by side, each half
// synchronising on its own named barrier.  inv[0, t*t) = inv(L), inv[t*t, 2t*t) = inv(U), ld t.
// The panel schedule computes them once per base case; every strip of its right / bottom panel
// then only applies them (leaf_apply_kernel) instead of re-inverting per CTA.
constexpr int PI_RS = 65;
__global__ void __launch_bounds__(512) panel_inv_kernel(const uint32_t* __restrict__ T, uint64_t ldt, uint32_t t,
                                                        uint32_t* __restrict__ inv, uint32_t p, uint64_t mu) {
    extern __shared__ __align__(16) uint32_t sm[];
    uint32_t* Ts = sm;  // 64 x 65
    const uint32_t tid = threadIdx.x, half = tid >> 8, lt = tid & 255;
    uint32_t* X = Ts + 64 * PI_RS + half * (64 * PI_RS + 32 * 32 + 64);
    uint32_t* W = X + 64 * PI_RS;
    uint32_t* dv = W + 32 * 32;
    ptx::pdl_enter();
    {
        uint32_t r[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const uint32_t idx = tid + 512 * q, i = idx / 64, k = idx % 64;
            r[q] = (i < t && k < t) ? T[(uint64_t)i * ldt + k] : 0u;
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const uint32_t idx = tid + 512 * q;
            Ts[(idx / 64) * PI_RS + idx % 64] = r[q];
        }
    }
    __syncthreads();
    if (gridDim.x == 2) {  // one triangle per CTA, all 512 threads on it
        uint32_t* Xc = Ts + 64 * PI_RS;
        uint32_t* Wc = Xc + 64 * PI_RS;
        uint32_t* dvc = Wc + 32 * 32;
        if (blockIdx.x == 0)
            tri_inverse_smem<false, 64>(Ts, PI_RS, Xc, PI_RS, Wc, dvc, t, p, mu);
        else
            tri_inverse_smem<true, 64>(Ts, PI_RS, Xc, PI_RS, Wc, dvc, t, p, mu);
        __syncthreads();
        uint32_t* out = inv + (size_t)blockIdx.x * t * t;
        for (uint32_t idx = tid; idx < t * t; idx += 512) out[idx] = Xc[(idx / t) * PI_RS + idx % t];
        return;
    }
    if (half == 0)
        tri_inverse_part<false, 64>(Ts, PI_RS, X, PI_RS, W, dv, t, p, mu, lt, 256, 1);
    else
        tri_inverse_part<true, 64>(Ts, PI_RS, X, PI_RS, W, dv, t, p, mu, lt, 256, 2);
    uint32_t* out = inv + (size_t)half * t * t;
    for (uint32_t idx = lt; idx < t * t; idx += 256) out[idx] = X[(idx / t) * PI_RS + idx % t];
}

void panel_inverses_dev(const Blas& b, DView T, uint32_t* inv) {
    const uint32_t t = (uint32_t)T.rows;
    if (t == 0 || t > 64 || T.cols != T.rows) throw Error(FFG_ERR_INTERNAL, "panel_inverses: block must be square <= 64");
    const size_t smem = (64 * PI_RS + 2 * (64 * PI_RS + 32 * 32 + 64)) * 4;
    static PerDeviceOnce once;
    once([smem] {
        FFG_CUDA(cudaFuncSetAttribute(panel_inv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    });
    b.ws.prof.begin(b.st);
    static const bool one = knob_on("FFG_INV_ONE_CTA");
    launch_k(panel_inv_kernel, dim3(one ? 1 : 2), dim3(512), smem, b.st, T.d, T.ld, t, inv, b.F.p, b.F.mu);
    FFG_CUDA(cudaGetLastError());
    b.ws.prof.end(b.st, PROF_TRINV, 8.0 * t * t);
    b.count();
}

// CTAs of a panel apply: one per strip up to FFG_APPLY_CTAS (default: no cap); fewer CTAs loop
// over strips and leave SMs to concurrent work
static unsigned apply_grid(size_t nvec) {
    const char* e = knob_str("FFG_APPLY_CTAS");
    const size_t cap = e ? (size_t)std::max(1, atoi(e)) : (size_t)1 << 30;
    return (unsigned)std::min(ceil_div(nvec, (size_t)LA), cap);
}

// side 0: B <- inv(L) B; side 1: B <- B inv(U), with the inverses of panel_inverses_dev
void panel_apply_dev(const Blas& b, int side, const uint32_t* inv, size_t t, DView B, const uint32_t* qperm) {
    if (B.empty()) return;
    const size_t nvec = side == 0 ? B.cols : B.rows;
    b.ws.prof.begin(b.st);
    if (side == 0)
        launch_k(leaf_apply_kernel<0>, dim3(apply_grid(nvec)), dim3(256), 0, b.st, inv, (uint32_t)t, B.d, B.ld,
                 (uint32_t)nvec, b.F.p, b.F.mu, (const uint32_t*)nullptr);
    else
        launch_k(leaf_apply_kernel<1>, dim3(apply_grid(nvec)), dim3(256), 0, b.st, inv + t * t, (uint32_t)t, B.d,
                 B.ld, (uint32_t)nvec, b.F.p, b.F.mu, qperm);
    FFG_CUDA(cudaGetLastError());
    b.ws.prof.end(b.st, PROF_TRINV, 8.0 * (double)t * nvec);
    b.count();
}

// The next block's columns and rows of a leaf's panels (X = inv(L) X, t x w and Y = Y[:, q] inv(U),
// h x t; w, h <= 64) in one launch, 16 vectors per CTA: the right side's strips first, then the
// bottom side's.  A thread owns one output row x 4 vectors; both inverses are triangular in the
// output index (k <= i).  Small CTAs: this sits on the critical path between two base cases.
constexpr int MV = 16;
__global__ void __launch_bounds__(256) panel_mini_kernel(const uint32_t* __restrict__ inv, uint32_t d,
                                                         uint32_t* __restrict__ X, uint64_t ldx, uint32_t w,
                                                         uint32_t* __restrict__ Y, uint64_t ldy, uint32_t h,
                                                         const uint32_t* __restrict__ qp, uint32_t p, uint64_t mu) {
    __shared__ __align__(16) uint32_t Ct[64][68];  // Ct[k][i] = coefficient of x_k in output i
    __shared__ __align__(16) uint32_t Bs[64][MV + 4];  // Bs[k][v]
    const uint32_t tid = threadIdx.x, nr = (w + MV - 1) / MV;
    const bool right = blockIdx.x < nr;
    const uint32_t v0 = (right ? blockIdx.x : blockIdx.x - nr) * MV, nvec = right ? w : h;
    const uint32_t nv = min((uint32_t)MV, nvec - v0);
    const uint32_t* invp = right ? inv : inv + d * d;
    ptx::pdl_enter();
    uint32_t rc[16], rb[4];
#pragma unroll
    for (int r = 0; r < 16; ++r) {
        const uint32_t idx = tid + 256 * r, k = idx / 64, i = idx % 64;
        rc[r] = (i < d && k < d) ? invp[k * d + i] : 0u;  // row k of the inverse, coalesced
    }
#pragma unroll
    for (int r = 0; r < 4; ++r) {
        // right: 16 consecutive columns of row k; bottom: 64 consecutive columns of row v
        const uint32_t idx = tid + 256 * r, k = right ? idx / MV : idx % 64, v = right ? idx % MV : idx / 64;
        rb[r] = 0u;
        if (k < d && v < nv)
            rb[r] = right ? X[(uint64_t)k * ldx + v0 + v] : Y[(uint64_t)(v0 + v) * ldy + (qp ? qp[k] : k)];
    }
#pragma unroll
    for (int r = 0; r < 16; ++r) {
        const uint32_t idx = tid + 256 * r;
        if (right)  // Ct[k][i] = inv(L)[i][k]: transposed on the shared-memory store
            Ct[idx % 64][idx / 64] = rc[r];
        else
            Ct[idx / 64][idx % 64] = rc[r];
    }
#pragma unroll
    for (int r = 0; r < 4; ++r) {
        const uint32_t idx = tid + 256 * r;
        if (right)
            Bs[idx / MV][idx % MV] = rb[r];
        else
            Bs[idx % 64][idx / 64] = rb[r];
    }
    __syncthreads();
    const uint32_t i = tid >> 2, vg = (tid & 3) * 4;
    uint64_t acc[4] = {0, 0, 0, 0};
    const uint32_t kend = min(d, i + 1);
#pragma unroll 4
    for (uint32_t k = 0; k < kend; ++k) {
        const uint64_t c = Ct[k][i];
        const uint4 x = *reinterpret_cast<const uint4*>(&Bs[k][vg]);
        acc[0] += c * x.x;
        acc[1] += c * x.y;
        acc[2] += c * x.z;
        acc[3] += c * x.w;
    }
    if (i < d) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const uint32_t v = vg + q;
            if (v >= nv) continue;
            const uint32_t val = mod_u64(acc[q], p, mu);
            if (right)
                X[(uint64_t)i * ldx + v0 + v] = val;
            else
                Y[(uint64_t)(v0 + v) * ldy + i] = val;
        }
    }
}

void panel_mini_dev(const Blas& b, const uint32_t* inv, size_t t, DView X, DView Y, const uint32_t* qperm) {
    const size_t w = X.empty() ? 0 : X.cols, h = Y.empty() ? 0 : Y.rows;
    if (!w && !h) return;
    if (t > 64 || w > 64 || h > 64) throw Error(FFG_ERR_INTERNAL, "panel_mini: blocks wider than 64");
    const unsigned grid = (unsigned)(ceil_div(w, (size_t)MV) + ceil_div(h, (size_t)MV));
    b.ws.prof.begin(b.st);
    launch_k(panel_mini_kernel, dim3(grid), dim3(256), 0, b.st, inv, (uint32_t)t, X.d, X.ld, (uint32_t)w, Y.d, Y.ld,
             (uint32_t)h, qperm, b.F.p, b.F.mu);
    FFG_CUDA(cudaGetLastError());
    b.ws.prof.end(b.st, PROF_TRINV, 8.0 * (double)t * (w + h));
    b.count();
}

// C -= Y X (C h x w with h <= 64, any w; Y h x t, X t x w, any t: 64-deep chunks through shared
// memory, one exact u64 sum per entry -- t <= 2^13 keeps it below 2^64 for p < 2^26), 16 columns
// of C per CTA: R's update inside a two-leaf node and the corner of larger nodes, in small CTAs.
__global__ void __launch_bounds__(256) panel_update_kernel(const uint32_t* __restrict__ Y, uint64_t ldy,
                                                           const uint32_t* __restrict__ X, uint64_t ldx,
                                                           uint32_t* __restrict__ C, uint64_t ldc, uint32_t h,
                                                           uint32_t t, uint32_t w, uint32_t p, uint64_t mu) {
    __shared__ __align__(16) uint32_t Ys[64][65];  // Ys[i][k] of the current chunk
    __shared__ __align__(16) uint32_t Xs[64][MV];  // Xs[k][v]
    const uint32_t tid = threadIdx.x, v0 = blockIdx.x * MV, nv = min((uint32_t)MV, w - v0);
    const uint32_t i = tid >> 2, vg = (tid & 3) * 4;
    ptx::pdl_enter();
    uint64_t acc[4] = {0, 0, 0, 0};
    for (uint32_t kc = 0; kc < t; kc += 64) {
        const uint32_t kn = min(64u, t - kc);
        uint32_t ry[16], rx[4];
#pragma unroll
        for (int r = 0; r < 16; ++r) {
            const uint32_t idx = tid + 256 * r, ii = idx / 64, k = idx % 64;
            ry[r] = (ii < h && k < kn) ? Y[(uint64_t)ii * ldy + kc + k] : 0u;
        }
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const uint32_t idx = tid + 256 * r, k = idx / MV, v = idx % MV;
            rx[r] = (k < kn && v < nv) ? X[(uint64_t)(kc + k) * ldx + v0 + v] : 0u;
        }
        if (kc) __syncthreads();  // the previous chunk is consumed
#pragma unroll
        for (int r = 0; r < 16; ++r) {
            const uint32_t idx = tid + 256 * r;
            Ys[idx / 64][idx % 64] = ry[r];
        }
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const uint32_t idx = tid + 256 * r;
            Xs[idx / MV][idx % MV] = rx[r];
        }
        __syncthreads();
#pragma unroll 4
        for (uint32_t k = 0; k < kn; ++k) {
            const uint64_t y = Ys[i][k];
            const uint4 x = *reinterpret_cast<const uint4*>(&Xs[k][vg]);
            acc[0] += y * x.x;
            acc[1] += y * x.y;
            acc[2] += y * x.z;
            acc[3] += y * x.w;
        }
    }
    if (i >= h) return;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const uint32_t v = vg + q;
        if (v >= nv) continue;
        uint32_t* c = C + (uint64_t)i * ldc + v0 + v;
        const uint32_t yx = mod_u64(acc[q], p, mu), cv = *c;
        *c = cv >= yx ? cv - yx : cv + p - yx;
    }
}

void panel_update_dev(const Blas& b, DView Y, DView X, DView C) {
    if (C.empty() || Y.cols == 0) return;
    if (C.rows > 64 || Y.cols > 8192 || Y.rows != C.rows || X.cols != C.cols || X.rows != Y.cols)
        throw Error(FFG_ERR_INTERNAL, "panel_update: bad shapes");
    b.ws.prof.begin(b.st);
    launch_k(panel_update_kernel, dim3((unsigned)ceil_div(C.cols, (size_t)MV)), dim3(256), 0, b.st, Y.d, Y.ld, X.d,
             X.ld, C.d, C.ld, (uint32_t)C.rows, (uint32_t)Y.cols, (uint32_t)C.cols, b.F.p, b.F.mu);
    FFG_CUDA(cudaGetLastError());
    b.ws.prof.end(b.st, PROF_TRINV, 8.0 * C.rows * C.cols * (double)Y.cols);
    b.count();
}

// true when the fused kernel handled the solve
bool trsm_fused(const Blas& b, int side, int upper, int unit, DView T, DView B) {
    static const bool off = knob_on("FFG_NO_FUSED_TRSM");
    if (off) return false;
    const bool pair = (side == 0 && !upper && unit) || (side == 1 && upper && !unit);
    if (!pair || T.rows > 128 || T.rows == 0) return false;
    if (T.rows <= 64)
        trsm_fused_launch<64>(b, side, upper, unit, T, B);
    else
        trsm_fused_launch<128>(b, side, upper, unit, T, B);
    return true;
}

// smallest i with T[i][i] == 0 (blas.hpp:291-297 / 347-353)
__global__ void first_zero_diag_kernel(const uint32_t* T, uint64_t ldt, uint32_t t, uint32_t* out) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < t && T[(uint64_t)i * ldt + i] == 0) atomicMin(out, i);
}

namespace {

struct TrsmCtx {
    const Blas& b;
    int side, upper, unit;
    DView T;
    const uint32_t* Tinv;  // one TB x TB inverse per diagonal block (nullptr: direct leaves)
};

void trsm_small(const Blas& b, int side, int upper, int unit, DView T, DView B) {
    const size_t t = T.rows;
    const size_t nvec = side == 0 ? B.cols : B.rows;
    const size_t smem = (TB * TSTR + TB * (SV + 1) + SCH * SV + 2 * TB) * sizeof(uint32_t);
    using K = void (*)(const uint32_t*, uint64_t, uint32_t, uint32_t*, uint64_t, uint32_t, uint32_t, uint64_t);
    static K kerns[8] = {trsm_small_kernel<0, false, false>, trsm_small_kernel<0, false, true>,
                         trsm_small_kernel<0, true, false>,  trsm_small_kernel<0, true, true>,
                         trsm_small_kernel<1, false, false>, trsm_small_kernel<1, false, true>,
                         trsm_small_kernel<1, true, false>,  trsm_small_kernel<1, true, true>};
    static PerDeviceOnce once;
    once([&] {
        for (auto k : kerns) FFG_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    });
    // forward order: left lower / right upper; reversed: left upper / right lower
    const bool rev = side == 0 ? upper != 0 : upper == 0;
    K k = kerns[side * 4 + (rev ? 2 : 0) + (unit ? 1 : 0)];
    b.ws.prof.begin(b.st);
    k<<<(unsigned)ceil_div(nvec, SV), 256, smem, b.st>>>(T.d, T.ld, (uint32_t)t, B.d, B.ld, (uint32_t)nvec, b.F.p,
                                                         b.F.mu);
    FFG_CUDA(cudaGetLastError());
    b.ws.prof.end(b.st, PROF_TRINV, 4.0 * (double)t * (t + 2.0 * nvec));
    b.count();
}

// solve on the diagonal range [o, o + t) of T (o a multiple of TB) against B
void trsm_rec(const TrsmCtx& c, size_t o, size_t t, DView B) {
    const uint32_t pm1 = c.b.F.p - 1;
    if (t <= (size_t)TB) {
        if (!c.Tinv) {
            trsm_small(c.b, c.side, c.upper, c.unit, c.T.sub(o, o, t, t), B);
            return;
        }
        DView inv{const_cast<uint32_t*>(c.Tinv) + (o / TB) * TB * TB, t, t, (size_t)TB};
        if (c.side == 0) {
            c.b.gemm(1, inv, B, 0, B);  // t <= 128 rows: in place on B is safe in the direct GEMM
        } else {
            // X = B inv in place would alias the A operand across column tiles (split path);
            // out of place through a pooled temporary keeps it on the one-launch direct GEMM
            uint32_t* tmp = nullptr;
            FFG_CUDA(cudaMallocAsync(&tmp, B.rows * B.cols * 4, c.b.st));
            DView X{tmp, B.rows, B.cols, B.cols};
            c.b.gemm(1, B, inv, 0, X);
            copy_block_dev(c.b, X, B);
            FFG_CUDA(cudaFreeAsync(tmp, c.b.st));
        }
        return;
    }
    const size_t nb = ceil_div(t, TB);
    const size_t t1 = ((nb + 1) / 2) * TB, t2 = t - t1;
    DView T11 = c.T.sub(o, o, t1, t1), T22 = c.T.sub(o + t1, o + t1, t2, t2);
    (void)T11;
    (void)T22;
    if (c.side == 0) {
        DView B1 = B.sub(0, 0, t1, B.cols), B2 = B.sub(t1, 0, t2, B.cols);
        if (!c.upper) {  // L X = B
            trsm_rec(c, o, t1, B1);
            c.b.gemm(pm1, c.T.sub(o + t1, o, t2, t1), B1, 1, B2);
            trsm_rec(c, o + t1, t2, B2);
        } else {  // U X = B
            trsm_rec(c, o + t1, t2, B2);
            c.b.gemm(pm1, c.T.sub(o, o + t1, t1, t2), B2, 1, B1);
            trsm_rec(c, o, t1, B1);
        }
    } else {
        DView B1 = B.sub(0, 0, B.rows, t1), B2 = B.sub(0, t1, B.rows, t2);
        if (c.upper) {  // X U = B
            trsm_rec(c, o, t1, B1);
            c.b.gemm(pm1, B1, c.T.sub(o, o + t1, t1, t2), 1, B2);
            trsm_rec(c, o + t1, t2, B2);
        } else {  // X L = B
            trsm_rec(c, o + t1, t2, B2);
            c.b.gemm(pm1, B2, c.T.sub(o + t1, o, t2, t1), 1, B1);
            trsm_rec(c, o, t1, B1);
        }
    }
}

}  // namespace

void ftrsm_dev(const Blas& b, int side, int uplo, int diag, DView A, DView B, bool check_diag) {
    const size_t need = side == 0 ? B.rows : B.cols;
    if (A.rows != A.cols) throw Error(FFG_ERR_DIM_MISMATCH, "trsm: triangle must be square");
    if (A.rows != need) throw Error(FFG_ERR_DIM_MISMATCH, "trsm: triangle does not match B");
    if (A.rows == 0 || B.rows == 0 || B.cols == 0) return;  // blas.hpp:393
    const size_t t = A.rows;
    const uint32_t p = b.F.p;
    if (check_diag && diag == 1) {
        uint32_t* d = nullptr;
        FFG_CUDA(cudaMallocAsync(&d, sizeof(uint32_t), b.st));
        FFG_CUDA(cudaMemsetAsync(d, 0xFF, sizeof(uint32_t), b.st));
        first_zero_diag_kernel<<<(unsigned)ceil_div(t, 256), 256, 0, b.st>>>(A.d, A.ld, (uint32_t)t, d);
        b.count();
        uint32_t h = 0;
        FFG_CUDA(cudaMemcpyAsync(&h, d, sizeof(uint32_t), cudaMemcpyDeviceToHost, b.st));
        FFG_CUDA(cudaFreeAsync(d, b.st));
        FFG_CUDA(cudaStreamSynchronize(b.st));
        if (h != 0xFFFFFFFFu)
            throw Error(FFG_ERR_SINGULAR_DIAGONAL, "zero diagonal entry " + std::to_string(h) + " in triangular solve",
                        h);
    }
    const int upper = uplo == 1, unit = diag == 0;
    if (trsm_fused(b, side, upper, unit, A, B)) return;
    static const bool inverse_leaves = !(knob_on("FFG_TRSM_DIRECT"));
    if (!inverse_leaves) {  // default: direct CUDA-core leaves, tensor-core Schur updates between them
        TrsmCtx c{b, side, upper, unit, A, nullptr};
        trsm_rec(c, 0, t, B);
        return;
    }
    const size_t nblk = ceil_div(t, TB);
    uint32_t* Tinv = nullptr;
    FFG_CUDA(cudaMallocAsync(&Tinv, nblk * TB * TB * sizeof(uint32_t), b.st));
    static const bool column_inverse = knob_on("FFG_TRI_COLUMN");
    b.ws.prof.begin(b.st);
    if (column_inverse) {  // per-column substitution (kept for A/B comparison)
        const size_t smem = (TB * TSTR + 2 * TB) * sizeof(uint32_t);
        static PerDeviceOnce once;
        once([&] {
            FFG_CUDA(cudaFuncSetAttribute(tri_inv_kernel<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            FFG_CUDA(cudaFuncSetAttribute(tri_inv_kernel<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            FFG_CUDA(cudaFuncSetAttribute(tri_inv_kernel<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            FFG_CUDA(cudaFuncSetAttribute(tri_inv_kernel<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        });
        auto kern = upper ? (unit ? tri_inv_kernel<true, true> : tri_inv_kernel<true, false>)
                          : (unit ? tri_inv_kernel<false, true> : tri_inv_kernel<false, false>);
        kern<<<(unsigned)(nblk * (TB / TRI_COLS)), TRI_COLS * 32, smem, b.st>>>(A.d, A.ld, (uint32_t)t, Tinv, p, b.F.mu);
    } else {
        const size_t smem = (2 * TB * TSTR + (TB / 2) * (TB / 2 + 1) + TB) * sizeof(uint32_t);
        static PerDeviceOnce once2;
        once2([&] {
            FFG_CUDA(cudaFuncSetAttribute(tri_inv_rec_kernel<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            FFG_CUDA(cudaFuncSetAttribute(tri_inv_rec_kernel<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            FFG_CUDA(cudaFuncSetAttribute(tri_inv_rec_kernel<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            FFG_CUDA(cudaFuncSetAttribute(tri_inv_rec_kernel<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        });
        auto kern = upper ? (unit ? tri_inv_rec_kernel<true, true> : tri_inv_rec_kernel<true, false>)
                          : (unit ? tri_inv_rec_kernel<false, true> : tri_inv_rec_kernel<false, false>);
        launch_k(kern, dim3((unsigned)nblk), dim3(RI_THREADS), smem, b.st, A.d, A.ld, (uint32_t)t, Tinv, p, b.F.mu);
    }
    FFG_CUDA(cudaGetLastError());
    b.ws.prof.end(b.st, PROF_TRINV, 8.0 * nblk * TB * TB);
    b.count();
    TrsmCtx c{b, side, upper, unit, A, Tinv};
    trsm_rec(c, 0, t, B);
    FFG_CUDA(cudaFreeAsync(Tinv, b.st));
}

}  // namespace ffg
