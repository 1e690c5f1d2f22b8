// base.cu -- the rank-profile revealing base case (rr_base, rankrev.hpp:29-78) as one CTA.
//
// The reference eliminates Crout-lazily and physically rotates rows and
// columns after each pivot.  Its output is fully determined by the pivot
// sequence: pivot k is the first remaining row (original order) whose Schur
// row is nonzero, at the first nonzero non-pivot column (original order) --
// rotations keep non-pivot rows/columns in original relative order
// (perm.hpp:11-13).  Given the pivot sequence, P A Q = L U has unique packed
// factors, so this kernel eliminates eagerly on the block held in shared
// memory with rows and columns left in place, and applies the permutations
// once when writing the block back:
//     P = [pivot rows in discovery order, non-pivot rows ascending]
//     Q = [pivot cols in discovery order, non-pivot cols ascending]
//
// Phase 1 (pivot discovery) is fraction-free: at pivot k every later row becomes
//     S_i <- piv_k * S_i - S_i[q_k] * S_{p_k}        (mod p),
// the true Schur row times the common nonzero factor piv_0 ... piv_k.  Nonzero
// scaling keeps the zero pattern, so the search sees exactly what rr_base sees,
// and no modular inverse sits on the serial path.  Eliminating column q_k zeroes
// it in every later row, so the update runs over whole rows without pivot-column
// masks (the L numerator S_i[q_k] is saved to Lb first) and the row search is a
// plain first-nonzero scan.  Phase 2 recovers the exact factors in parallel:
//     L[i][k] = Lb[i][k] / piv_k,    U[k][:] = S_{p_k}[:] / (piv_0 ... piv_{k-1}).
// Exhausted rows (rankrev.hpp:54-57) keep their zero Schur rows and zero L
// entries for later pivots, as in the reference.
#include <cstdio>
#include <mutex>
#include <vector>

#include "pluq.cuh"
#include "ptx.cuh"
#include "triinv.cuh"

namespace ffg {

constexpr int BASE_THREADS = 256;
constexpr size_t BASE_SMEM_LIMIT = 200 * 1024;
constexpr uint32_t NONE = 0xFFFFFFFFu;
constexpr uint32_t INV_MAX = 64;  // largest base-case rank whose factor inverses are cached

__device__ __forceinline__ uint32_t sub_mod(uint32_t a, uint32_t b, uint32_t p) { return a >= b ? a - b : a + p - b; }

// diagnostics (FFG_BASE_DBG): per launch {clock64, globaltimer} at entry, end of pivoting, exit
__device__ unsigned long long* g_base_dbg = nullptr;
__device__ unsigned int g_base_dbg_n = 0;
__device__ int g_base_skip = 0;  // experiment: skip the update arithmetic (timing only)
__device__ __forceinline__ void base_stamp(unsigned long long* slot) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    slot[0] = clock64();
    slot[1] = t;
}

struct BaseLayout {
    uint32_t m, n, ns, rmax;  // ns = padded row stride of S (multiple of 8)
};

constexpr int BASE_THREADS_REG = 512;
template <bool IN_SMEM, bool REG>
__global__ void __launch_bounds__(REG ? BASE_THREADS_REG : BASE_THREADS, 1)
    rr_base_kernel(uint32_t* __restrict__ A, uint64_t lda, BaseLayout lay, uint32_t* __restrict__ scratch,
                   uint32_t* __restrict__ Pd, uint32_t* __restrict__ Qd, BaseInfo* __restrict__ info, uint32_t p,
                   uint64_t mu, uint32_t* __restrict__ inv_out, uint32_t seq) {
    extern __shared__ __align__(16) uint32_t sm[];
    const uint32_t m = lay.m, n = lay.n, ns = lay.ns, rmax = lay.rmax;
    unsigned long long* dbg = nullptr;
    if (g_base_dbg && threadIdx.x == 0) {
        dbg = g_base_dbg + 6 * (atomicAdd(&g_base_dbg_n, 1u) % 4096);
        base_stamp(dbg);
    }
    // shared: prow | pcol | pivv | invp | invD (rmax each) | Psh m | Qsh n | rowrank m | colrank n
    uint32_t* prow = sm;
    uint32_t* pcol = prow + rmax;
    uint32_t* pivv = pcol + rmax;
    uint32_t* invp = pivv + rmax;
    uint32_t* invD = invp + rmax;
    uint32_t* Psh = invD + rmax;
    uint32_t* Qsh = Psh + m;
    uint32_t* rowrank = Qsh + n;
    uint32_t* colrank = rowrank + m;
    uint32_t* tail = colrank + n;
    tail += (4 - (reinterpret_cast<uintptr_t>(tail) / 4) % 4) % 4;  // 16-byte align
    uint32_t* S = IN_SMEM ? tail : scratch;             // m x ns
    uint32_t* Lb = IN_SMEM ? tail + (size_t)m * ns : scratch + (size_t)m * ns;  // m x rmax numerators

    constexpr uint32_t NTH = REG ? BASE_THREADS_REG : BASE_THREADS;
    const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, nwarps = NTH / 32;
    uint32_t r = 0;
    if constexpr (REG) {
        // ---- phase 1, register-resident (m, n <= 64).  Row i lives in the registers of the 8
        // lanes 8i..8i+7 (8 columns each; 16 warps x 4 rows) and, for indexed reads, in S.
        // Values are kept lazily reduced in [0, 4p): an update is two Shoup products without
        // their final corrections plus one add (7 instructions per element); zero tests and
        // the pivot row use fully reduced values.  Per pivot one barrier: the warp holding the
        // first row after the pivot finds the next pivot (first nonzero row, first nonzero
        // column: rr_base's row-major search, rankrev.hpp:40-57) and publishes it; only when
        // that warp's rows are all zero (rank deficiency) does every warp search (slow path).
        constexpr uint32_t FULL = 0xffffffffu;
        constexpr uint32_t LEAD_NONE = NONE - 1;  // the lead warp found no nonzero row
        uint32_t* hdr = Lb + (size_t)m * rmax;    // [2] x {row, col, value, shoup(value)}
        hdr += (4 - (reinterpret_cast<uintptr_t>(hdr) / 4) % 4) % 4;
        uint32_t* cand = hdr + 8;                 // [2][64] pivot row (reduced)
        uint32_t* srow = cand + 128;              // [16] slow path: candidate row per warp
        uint32_t* sval = srow + 16;               // [16][64] slow path: candidate values
        uint32_t* shdr = sval + 16 * 64;          // [16] x {col, value, shoup(value), -}
        const uint32_t i = tid >> 3, c0 = (tid & 7) * 8;
        const uint32_t p2 = 2 * p;
        auto red = [&](uint32_t x) {  // [0, 4p) -> [0, p)
            x = min(x, x - p2);
            return min(x, x - p);
        };
        uint32_t v[8];
        {
            const uint32_t* src = A + (uint64_t)(i < m ? i : 0) * lda;
#pragma unroll
            for (int u = 0; u < 8; ++u) v[u] = (i < m && c0 + u < n) ? src[c0 + u] : 0u;
        }
        auto store_row = [&]() {
            if (i < m && c0 < ns) {
                uint4* d = reinterpret_cast<uint4*>(S + (size_t)i * ns + c0);
                d[0] = make_uint4(v[0], v[1], v[2], v[3]);
                d[1] = make_uint4(v[4], v[5], v[6], v[7]);
            }
        };
        store_row();  // numerators are read back from S by column index
        for (uint32_t idx = tid; idx < m * rmax; idx += NTH) Lb[idx] = 0u;
        // first nonzero row >= first of this warp: reduced-OR per row, ballot over the warp
        auto warp_first = [&](uint32_t first) -> uint32_t {
            uint32_t o = 0;
#pragma unroll
            for (int u = 0; u < 8; ++u) o |= red(v[u]);
            o |= __shfl_xor_sync(FULL, o, 1);
            o |= __shfl_xor_sync(FULL, o, 2);
            o |= __shfl_xor_sync(FULL, o, 4);
            const uint32_t bal = __ballot_sync(FULL, i < m && i >= first && o != 0);
            return bal ? (warp * 4 + ((__ffs(bal) - 1) >> 3)) : NONE;
        };
        // the row c of this warp becomes a candidate: its reduced values to dst[64], then the
        // first nonzero column by two ballots over the stored row
        auto emit = [&](uint32_t c, uint32_t* dst, uint32_t* out_col, uint32_t* out_val, uint32_t* out_pre) {
            if (i == c) {
#pragma unroll
                for (int u = 0; u < 8; ++u) v[u] = red(v[u]);
                uint4* d = reinterpret_cast<uint4*>(dst + c0);
                d[0] = make_uint4(v[0], v[1], v[2], v[3]);
                d[1] = make_uint4(v[4], v[5], v[6], v[7]);
            }
            __syncwarp();
            const uint32_t x0 = dst[lane], x1 = dst[lane + 32];
            const uint32_t b0 = __ballot_sync(FULL, x0 != 0), b1 = __ballot_sync(FULL, x1 != 0);
            const uint32_t pj = b0 ? __ffs(b0) - 1 : 31 + __ffs(b1);
            if (lane == 0) {
                const uint32_t pv = dst[pj];
                *out_col = pj;
                *out_val = pv;
                *out_pre = shoup_pre(pv, p, mu);
            }
        };
        auto lead_publish = [&](uint32_t buf, uint32_t first) {  // rows >= first are eligible
            if (first >= m) {
                if (tid == 0) hdr[buf * 4] = NONE;
                return;
            }
            if (warp != first / 4) return;
            const uint32_t c = warp_first(first);
            if (c == NONE) {
                if (lane == 0) hdr[buf * 4] = LEAD_NONE;
                return;
            }
            emit(c, cand + buf * 64, hdr + buf * 4 + 1, hdr + buf * 4 + 2, hdr + buf * 4 + 3);
            if (lane == 0) hdr[buf * 4] = c;
        };
        lead_publish(0, 0);
        __syncthreads();
        uint32_t buf = 0, first = 0;
        const uint32_t warp_last_row = warp * 4 + 3;
        while (r < n) {
            const uint4 hh = reinterpret_cast<const uint4*>(hdr)[buf];
            uint32_t pi = hh.x, pj = hh.y, pv = hh.z, pvp = hh.w;
            const uint32_t* prw = cand + buf * 64;
            if (pi == LEAD_NONE) {  // slow path (uniform): every warp offers its first nonzero row
                const uint32_t c = warp_first(first);
                if (lane == 0) srow[warp] = c;
                if (c != NONE) emit(c, sval + warp * 64, shdr + warp * 4, shdr + warp * 4 + 1, shdr + warp * 4 + 2);
                __syncthreads();
                uint32_t ws = NONE;
                for (uint32_t w = 0; w < nwarps && ws == NONE; ++w)
                    if (srow[w] != NONE) ws = w;
                if (ws == NONE) break;  // uniform: no nonzero row left
                pi = srow[ws];
                pj = shdr[ws * 4];
                pv = shdr[ws * 4 + 1];
                pvp = shdr[ws * 4 + 2];
                prw = sval + ws * 64;
            } else if (pi == NONE) {
                break;  // uniform
            }
            if (tid == 0) {
                prow[r] = pi;
                pcol[r] = pj;
                pivv[r] = pv;
            }
            if (!g_base_skip && warp_last_row > pi && i > pi && i < m) {  // warps past their last row only keep step
                const uint32_t numer = red(S[(size_t)i * ns + pj]);
                if ((tid & 7) == 0) Lb[(size_t)i * rmax + r] = numer;
                const uint32_t nump = shoup_pre(numer, p, mu);
                const uint4 b0 = reinterpret_cast<const uint4*>(prw + c0)[0];
                const uint4 b1 = reinterpret_cast<const uint4*>(prw + c0)[1];
                const uint32_t b[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const uint32_t a = v[u] * pv - __umulhi(v[u], pvp) * p;   // [0, 2p)
                    const uint32_t s = b[u] * numer - __umulhi(b[u], nump) * p;  // [0, 2p)
                    v[u] = a + p2 - s;                                          // (0, 4p)
                }
                store_row();
            }
            ++r;
            buf ^= 1;
            first = pi + 1;
            lead_publish(buf, first);
            __syncthreads();
        }
        // reduced final rows for phase 2
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = red(v[u]);
        store_row();
        __syncthreads();
    } else {
        for (uint32_t t = warp; t < m; t += nwarps) {
            for (uint32_t u = lane; u < ns; u += 32) S[(size_t)t * ns + u] = u < n ? A[(uint64_t)t * lda + u] : 0u;
            for (uint32_t u = lane; u < rmax; u += 32) Lb[(size_t)t * rmax + u] = 0u;
        }
        __syncthreads();

        const uint32_t ngroups = ns / 8;
        uint32_t lg = 0;  // row segment = 2^lg lanes >= ngroups
        while ((1u << lg) < ngroups) ++lg;
        const uint32_t seg = 1u << lg;
        uint32_t cur = 0;
        while (cur < m && r < n) {
            // row-major pivot search (rankrev.hpp:40-57), done redundantly by every warp so no
            // barrier separates it from the update; pivot columns are already 0 in rows >= cur,
            // and rows in [cur, pi] are never written during this step
            uint32_t pi = m, pj = n;
            for (uint32_t i = cur; i < m && pi == m; ++i) {
                const uint32_t* row = S + (size_t)i * ns;
                for (uint32_t jc = 0; jc < n; jc += 32) {
                    const uint32_t j = jc + lane;
                    const uint32_t bal = __ballot_sync(0xffffffffu, j < n && row[j] != 0);
                    if (bal) {
                        pi = i;
                        pj = jc + __ffs(bal) - 1;
                        break;
                    }
                }
            }
            if (pi >= m) break;  // uniform: every warp found the same (pi, pj)
            const uint32_t* prw = S + (size_t)pi * ns;
            const uint32_t pv = prw[pj];
            const uint32_t pvp = shoup_pre(pv, p, mu);
            if (tid == 0) {
                prow[r] = pi;
                pcol[r] = pj;
                pivv[r] = pv;
            }
            const uint32_t rows_below = m - pi - 1;
            if (seg <= 32) {
                // a row's column groups sit in one warp segment of `seg` lanes: the lane holding
                // column pj broadcasts the numerator by shuffle before anyone overwrites it
                const uint32_t lseg = lane & (seg - 1), sbase = lane - lseg, owner = sbase + (pj >> 3);
                const uint32_t q = pj & 7;
                for (uint32_t r0 = warp << (5 - lg); r0 < rows_below; r0 += nwarps << (5 - lg)) {
                    const uint32_t i = pi + 1 + r0 + (lane >> lg);
                    const bool live = i < m && lseg < ngroups;
                    const uint32_t g = live ? lseg : 0u;
                    uint32_t* row = S + (size_t)(live ? i : pi) * ns + g * 8;
                    const uint4 a0 = reinterpret_cast<const uint4*>(row)[0], a1 = reinterpret_cast<const uint4*>(row)[1];
                    const uint4 b0 = reinterpret_cast<const uint4*>(prw + g * 8)[0];
                    const uint4 b1 = reinterpret_cast<const uint4*>(prw + g * 8)[1];
                    const uint32_t lo = (q & 2) ? ((q & 1) ? a0.w : a0.z) : ((q & 1) ? a0.y : a0.x);
                    const uint32_t hi = (q & 2) ? ((q & 1) ? a1.w : a1.z) : ((q & 1) ? a1.y : a1.x);
                    const uint32_t numer = __shfl_sync(0xffffffffu, (q & 4) ? hi : lo, owner);
                    if (!live) continue;
                    const uint32_t nump = shoup_pre(numer, p, mu);
                    uint4 o0, o1;
                    o0.x = sub_mod(shoup_mul(a0.x, pv, pvp, p), shoup_mul(b0.x, numer, nump, p), p);
                    o0.y = sub_mod(shoup_mul(a0.y, pv, pvp, p), shoup_mul(b0.y, numer, nump, p), p);
                    o0.z = sub_mod(shoup_mul(a0.z, pv, pvp, p), shoup_mul(b0.z, numer, nump, p), p);
                    o0.w = sub_mod(shoup_mul(a0.w, pv, pvp, p), shoup_mul(b0.w, numer, nump, p), p);
                    o1.x = sub_mod(shoup_mul(a1.x, pv, pvp, p), shoup_mul(b1.x, numer, nump, p), p);
                    o1.y = sub_mod(shoup_mul(a1.y, pv, pvp, p), shoup_mul(b1.y, numer, nump, p), p);
                    o1.z = sub_mod(shoup_mul(a1.z, pv, pvp, p), shoup_mul(b1.z, numer, nump, p), p);
                    o1.w = sub_mod(shoup_mul(a1.w, pv, pvp, p), shoup_mul(b1.w, numer, nump, p), p);
                    if (lseg == (pj >> 3)) Lb[(size_t)i * rmax + r] = numer;
                    reinterpret_cast<uint4*>(row)[0] = o0;
                    reinterpret_cast<uint4*>(row)[1] = o1;
                }
            } else {
                // wide rows: save the L numerators of column pj before the update zeroes it
                __syncthreads();  // every warp has finished reading the pivot row / numerators
                for (uint32_t i = pi + 1 + tid; i < m; i += NTH)
                    Lb[(size_t)i * rmax + r] = S[(size_t)i * ns + pj];
                __syncthreads();
                for (uint32_t idx = tid; idx < rows_below * ngroups; idx += NTH) {
                    const uint32_t i = pi + 1 + idx / ngroups, g = idx % ngroups;
                    uint32_t* row = S + (size_t)i * ns + g * 8;
                    const uint32_t numer = Lb[(size_t)i * rmax + r];
                    const uint32_t nump = shoup_pre(numer, p, mu);
                    const uint4 a0 = reinterpret_cast<const uint4*>(row)[0], a1 = reinterpret_cast<const uint4*>(row)[1];
                    const uint4 b0 = reinterpret_cast<const uint4*>(prw + g * 8)[0];
                    const uint4 b1 = reinterpret_cast<const uint4*>(prw + g * 8)[1];
                    uint4 o0, o1;
                    o0.x = sub_mod(shoup_mul(a0.x, pv, pvp, p), shoup_mul(b0.x, numer, nump, p), p);
                    o0.y = sub_mod(shoup_mul(a0.y, pv, pvp, p), shoup_mul(b0.y, numer, nump, p), p);
                    o0.z = sub_mod(shoup_mul(a0.z, pv, pvp, p), shoup_mul(b0.z, numer, nump, p), p);
                    o0.w = sub_mod(shoup_mul(a0.w, pv, pvp, p), shoup_mul(b0.w, numer, nump, p), p);
                    o1.x = sub_mod(shoup_mul(a1.x, pv, pvp, p), shoup_mul(b1.x, numer, nump, p), p);
                    o1.y = sub_mod(shoup_mul(a1.y, pv, pvp, p), shoup_mul(b1.y, numer, nump, p), p);
                    o1.z = sub_mod(shoup_mul(a1.z, pv, pvp, p), shoup_mul(b1.z, numer, nump, p), p);
                    o1.w = sub_mod(shoup_mul(a1.w, pv, pvp, p), shoup_mul(b1.w, numer, nump, p), p);
                    reinterpret_cast<uint4*>(row)[0] = o0;
                    reinterpret_cast<uint4*>(row)[1] = o1;
                }
            }
            ++r;
            cur = pi + 1;
            __syncthreads();
        }
    }

    if (dbg) base_stamp(dbg + 2);
    // ---- phase 2: exact values (pivot inverses in parallel, prefix products, scaling)
    for (uint32_t k = tid; k < r; k += NTH) invp[k] = inv_mod_bin(pivv[k], p);
    for (uint32_t i = tid; i < m; i += NTH) rowrank[i] = NONE;
    for (uint32_t j = tid; j < n; j += NTH) colrank[j] = NONE;
    __syncthreads();
    for (uint32_t k = tid; k < r; k += NTH) {
        rowrank[prow[k]] = k;
        colrank[pcol[k]] = k;
    }
    __syncthreads();
    if (warp == 0) {  // invD[k] = 1 / (piv_0 ... piv_{k-1}): exclusive prefix product, 32 per round
        uint32_t carry = 1 % p;
        for (uint32_t c = 0; c < r; c += 32) {
            const uint32_t k = c + lane;
            uint32_t v = k < r ? invp[k] : 1u % p;
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {  // inclusive scan (Hillis-Steele)
                const uint32_t o = __shfl_up_sync(0xffffffffu, v, off);
                if (lane >= (uint32_t)off) v = mul_mod(v, o, p, mu);
            }
            uint32_t ex = __shfl_up_sync(0xffffffffu, v, 1);
            if (lane == 0) ex = 1u % p;
            if (k < r) invD[k] = mul_mod(carry, ex, p, mu);
            carry = mul_mod(carry, __shfl_sync(0xffffffffu, v, 31), p, mu);
        }
    }
    __syncthreads();

    // ---- permutations: pivots in discovery order, then the rest ascending (warp 0: P, warp 1: Q),
    // built in shared memory with ballot compaction, moved ranges by warp min/max reductions
    if (warp < 2) {
        const uint32_t dim = warp == 0 ? m : n;
        const uint32_t* rank_of = warp == 0 ? rowrank : colrank;
        const uint32_t* order = warp == 0 ? prow : pcol;
        uint32_t* out = warp == 0 ? Psh : Qsh;
        uint32_t base = 0;
        for (uint32_t c = 0; c < dim; c += 32) {
            const uint32_t i = c + lane;
            const bool np = i < dim && rank_of[i] == NONE;
            const uint32_t bal = __ballot_sync(0xffffffffu, np);
            if (np) out[r + base + __popc(bal & ((1u << lane) - 1u))] = i;
            base += __popc(bal);
        }
        for (uint32_t k = lane; k < r; k += 32) out[k] = order[k];
        __syncwarp();
        uint32_t lo = NONE, hi = 0;
        for (uint32_t i = lane; i < dim; i += 32)
            if (out[i] != i) {
                lo = min(lo, i);
                hi = max(hi, i + 1);
            }
        lo = __reduce_min_sync(0xffffffffu, lo);
        hi = __reduce_max_sync(0xffffffffu, hi);
        if (lane == 0) {
            if (warp == 0) {
                info->rank = r;
                info->plo = lo < hi ? lo : 0;
                info->phi = lo < hi ? hi : 0;
            } else {
                info->qlo = lo < hi ? lo : 0;
                info->qhi = lo < hi ? hi : 0;
            }
        }
    }
    __syncthreads();
    if (dbg) base_stamp(dbg + 4);
    for (uint32_t i = tid; i < m; i += NTH) Pd[i] = Psh[i];
    for (uint32_t j = tid; j < n; j += NTH) Qd[j] = Qsh[j];
    // packed output: out[t][u] for original row i = P[t], column j = Q[u]
    for (uint32_t t = warp; t < m; t += nwarps) {
        const uint32_t i = Psh[t];
        const uint32_t k = rowrank[i];
        const uint32_t du = k < r ? invD[k] : 0u, dup = k < r ? shoup_pre(du, p, mu) : 0u;
        const uint32_t* srow = S + (size_t)i * ns;
        const uint32_t* lrow = Lb + (size_t)i * rmax;
        uint32_t* dst = A + (uint64_t)t * lda;
        for (uint32_t u = lane; u < n; u += 32) {
            const uint32_t j = Qsh[u];
            const uint32_t tc = colrank[j];
            uint32_t v;
            if (tc < r && tc < k)  // L entry for pivot tc (k == NONE for non-pivot rows)
                v = mul_mod(lrow[tc], invp[tc], p, mu);
            else if (k < r)  // U row k
                v = shoup_mul(srow[j], du, dup, p);
            else  // non-pivot row, non-pivot column: the zero Schur complement
                v = srow[j];
            dst[u] = v;
        }
    }
    // inverses of the leading r x r factors (L unit lower, U upper) for the TRSMs that will use
    // this block as their triangle: a base case is a leaf of every such TRSM
    if (IN_SMEM && inv_out != nullptr && (r == 0 || r > INV_MAX)) {
        if (tid == 0) info->cached = 0;
    } else if (IN_SMEM && inv_out != nullptr) {
        __syncthreads();  // the packed block in A (global) is complete and visible to the CTA
        uint32_t* Ts = S + (size_t)m * ns + (size_t)m * rmax;  // scratch after S and Lb
        Ts += (4 - (reinterpret_cast<uintptr_t>(Ts) / 4) % 4) % 4;
        uint32_t* Xs = Ts + INV_MAX * (INV_MAX + 1);
        uint32_t* Ws = Xs + INV_MAX * (INV_MAX + 1);
        uint32_t* dv = Ws + (INV_MAX / 2) * (INV_MAX / 2);
        for (uint32_t idx = tid; idx < r * r; idx += NTH) {
            const uint32_t i = idx / r, j = idx % r;
            Ts[i * (INV_MAX + 1) + j] = A[(uint64_t)i * lda + j];
        }
        __syncthreads();
        for (int which = 0; which < 2; ++which) {
            if (r <= 16) {
                if (which == 0) tri_inverse_smem<false, 16>(Ts, INV_MAX + 1, Xs, INV_MAX + 1, Ws, dv, r, p, mu);
                else tri_inverse_smem<true, 16>(Ts, INV_MAX + 1, Xs, INV_MAX + 1, Ws, dv, r, p, mu);
            } else if (r <= 32) {
                if (which == 0) tri_inverse_smem<false, 32>(Ts, INV_MAX + 1, Xs, INV_MAX + 1, Ws, dv, r, p, mu);
                else tri_inverse_smem<true, 32>(Ts, INV_MAX + 1, Xs, INV_MAX + 1, Ws, dv, r, p, mu);
            } else {
                if (which == 0) tri_inverse_smem<false, 64>(Ts, INV_MAX + 1, Xs, INV_MAX + 1, Ws, dv, r, p, mu);
                else tri_inverse_smem<true, 64>(Ts, INV_MAX + 1, Xs, INV_MAX + 1, Ws, dv, r, p, mu);
            }
            uint32_t* out = inv_out + (size_t)which * r * r;
            for (uint32_t idx = tid; idx < r * r; idx += NTH) out[idx] = Xs[(idx / r) * (INV_MAX + 1) + idx % r];
            __syncthreads();
        }
        if (tid == 0) info->cached = 1;
    }
    // completion mailbox: every info field above is written before the sequence number the host
    // spins on (barrier + system fence by the publishing thread, which is cumulative)
    __syncthreads();
    if (tid == 0) {
        __threadfence_system();
        *reinterpret_cast<volatile uint32_t*>(&info->seq) = seq;
    }
}

// ---------------------------------------------------------------------------------------------
// Blocked base case for m, n <= 64: rr_base evaluated as the reference's slab algorithm
// (pluq_slab_iterative, rankrev.hpp:244-282, which equals rr_base for every slab height --
// tests/test_oracle_pins.py::test_rr_base_equals_slab_iterative), rows and columns left in
// place, 16-row slabs, one warp per slab row (2 columns per lane):
//   (A) the slab rows' exact Schur complements w.r.t. the R earlier pivots: each warp sweeps
//       k = 0..R-1 right-looking with the EXACT earlier U rows (l_ik = S_i[q_k] / U_k[q_k],
//       S_i -= l_ik U_k), using per-column Shoup factors of U and Shoup-ready pivot inverses --
//       one shuffle and a few multiplies per pivot, no barrier;
//   (B) rr_base's greedy search on the slab (rankrev.hpp:40-57): fraction-free, lazily reduced
//       values in registers, one barrier per pivot, every eligible warp publishing its row into
//       a double-buffered slot and the lowest row winning through a shared atomicMin;
//   (C) the slab's pivots normalised with ONE modular inverse (prefix products): exact U rows
//       (+ their Shoup factors for later slabs), exact pivot inverses, exact in-slab L.
constexpr int SLAB = 16;
constexpr int SL_THREADS = 512;
constexpr int SS = 68;  // row stride of the block (16-byte rows, banks shifted per row)
constexpr int LS = 65;  // row stride of L

__device__ __forceinline__ uint32_t red4p(uint32_t x, uint32_t p) {  // [0, 4p) -> [0, p)
    x = min(x, x - 2 * p);
    return min(x, x - p);
}

__global__ void __launch_bounds__(SL_THREADS, 1)
    rr_base_slab_kernel(uint32_t* __restrict__ A, uint64_t lda, uint32_t m, uint32_t n, uint32_t* __restrict__ Pd,
                        uint32_t* __restrict__ Qd, BaseInfo* __restrict__ info, uint32_t p, uint64_t mu,
                        uint32_t seq) {
    extern __shared__ __align__(16) uint32_t sm[];
    uint32_t* S = sm;                    // 64 x SS: the block; exact U rows after normalisation
    uint32_t* Uf = S + 64 * SS;          // 64 x SS: Shoup factors of the exact U rows (by pivot index)
    uint32_t* Lx = Uf + 64 * SS;         // 64 x LS: exact L (row i, pivot k)
    uint32_t* slot = Lx + 64 * LS;       // [2][16] x 132: candidate rows: 64 values, 64 Shoup
                                         // factors, {row, col, val, shoup(val)}
    uint32_t* prow = slot + 2 * 16 * 132;  // 64
    uint32_t* pcol = prow + 64;          // 64
    uint32_t* ipv = pcol + 64;           // 64 inverses of the exact pivot values
    uint32_t* ipf = ipv + 64;            // 64 their Shoup factors
    uint32_t* sl = ipf + 64;             // per slab: piv_ff[16], D[16], invD[16], invp[16]
    uint32_t* Psh = sl + 64;             // 64
    uint32_t* Qsh = Psh + 64;            // 64
    uint32_t* rowrank = Qsh + 64;        // 64
    uint32_t* colrank = rowrank + 64;    // 64
    uint32_t* misc = colrank + 64;       // [0] slab rank, [2..4] winning row, rotating per step
    const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    constexpr uint32_t FULL = 0xffffffffu;
    unsigned long long ph[8] = {0, 0, 0, 0, 0, 0, 0, 0}, tq = clock64();
    auto stamp = [&](int k) {
        const unsigned long long t2 = clock64();
        ph[k] += t2 - tq;
        tq = t2;
    };
    ptx::pdl_enter();

    for (uint32_t idx = tid; idx < 64 * 64; idx += SL_THREADS) {
        const uint32_t i = idx >> 6, j = idx & 63;
        S[i * SS + j] = (i < m && j < n) ? A[(uint64_t)i * lda + j] : 0u;
        Lx[i * LS + j] = 0u;
    }
    __syncthreads();
    stamp(0);

    uint32_t R = 0;
    for (uint32_t i0 = 0; i0 < m; i0 += SLAB) {
        const uint32_t rows = min((uint32_t)SLAB, m - i0);
        const uint32_t i = i0 + warp;
        const bool live = warp < rows;
        uint32_t x0 = live ? S[i * SS + lane] : 0u, x1 = live ? S[i * SS + lane + 32] : 0u;
        // (A) exact Schur rows against the earlier pivots (x stays in [0, p) after each step)
        if (live) {
#pragma unroll 2
            for (uint32_t k = 0; k < R; ++k) {
                const uint32_t q = pcol[k];
                const uint32_t* u = S + prow[k] * SS;
                const uint32_t* uf = Uf + k * SS;
                const uint32_t u0 = u[lane], u1 = u[lane + 32], f0 = uf[lane], f1 = uf[lane + 32];
                const uint32_t v = __shfl_sync(FULL, q < 32 ? x0 : x1, q & 31);
                const uint32_t l = shoup_mul(v, ipv[k], ipf[k], p);  // exact multiplier
                if (lane == 0) Lx[i * LS + k] = l;
                x0 = red4p(x0 + 2 * p - (l * u0 - __umulhi(l, f0) * p), p);
                x1 = red4p(x1 + 2 * p - (l * u1 - __umulhi(l, f1) * p), p);
            }
        }
        stamp(1);
        // (B) sequential pivoting inside the slab: warp w <-> row i0 + w
        // Normally only the warp of the next row publishes (the lead): on full-rank input the next
        // row always is the pivot.  If that row is zero the lead posts SLOW and every warp offers its
        // row in an extra round (rank deficiency only).
        constexpr uint32_t SLOW = NONE - 1;
        uint32_t first = i0;  // rows < first are done
        uint32_t t = 0;
        bool is_pivot = false;
        if (tid == 0) misc[2] = misc[3] = misc[4] = NONE;
        __syncthreads();
        // one barrier per pivot: slots are double-buffered and the winner cell rotates over three,
        // so a cell is reset only after every thread has passed the barrier following its last read
        uint32_t rot = 0;
        auto offer = [&](uint32_t* my, uint32_t* cell) -> bool {  // whole warp; true if nonzero
            x0 = red4p(x0, p);
            x1 = red4p(x1, p);
            const uint32_t b0 = __ballot_sync(FULL, x0 != 0u), b1 = __ballot_sync(FULL, x1 != 0u);
            if (!(b0 | b1)) return false;
            my[lane] = x0;
            my[lane + 32] = x1;
            my[64 + lane] = shoup_pre(x0, p, mu);
            my[96 + lane] = shoup_pre(x1, p, mu);
            const uint32_t pj = b0 ? __ffs(b0) - 1 : 31 + __ffs(b1);
            const uint32_t pv = __shfl_sync(FULL, pj < 32 ? x0 : x1, pj & 31);
            if (lane == 0) {
                my[128] = i;
                my[129] = pj;
                my[130] = pv;
                my[131] = shoup_pre(pv, p, mu);
                atomicMin(cell, i);
            }
            return true;
        };
        while (R + t < n) {
            const uint32_t par = t & 1;
            uint32_t* my = slot + (par * 16 + warp) * 132;
            uint32_t* cell = misc + 2 + rot;
            if (live && i == first && !offer(my, cell) && lane == 0) atomicMin(cell, SLOW);
            if (tid == 0) misc[2 + (rot == 2 ? 0 : rot + 1)] = NONE;  // the next step's cell
            __syncthreads();
            uint32_t pi = *cell;
            rot = rot == 2 ? 0 : rot + 1;
            if (pi == SLOW) {  // uniform: the next row is zero -- every later row offers itself
                if (tid == 0) misc[5] = NONE;
                __syncthreads();
                if (live && i > first && !is_pivot) offer(my, misc + 5);
                __syncthreads();
                pi = misc[5];
            }
            if (pi == NONE) break;  // uniform: the slab has no nonzero row left
            const uint32_t* pr = slot + (par * 16 + (pi - i0)) * 132;
            const uint32_t pj = pr[129], pv = pr[130], pvp = pr[131];
            const uint32_t k = R + t;
            if (tid == 0) {
                prow[k] = pi;
                pcol[k] = pj;
                sl[t] = pv;  // fraction-free pivot value
            }
            if (live && i > pi) {
                const uint32_t numer = red4p(__shfl_sync(FULL, pj < 32 ? x0 : x1, pj & 31), p);
                if (lane == 0) Lx[i * LS + k] = numer;  // fraction-free numerator, scaled below
                const uint32_t b0 = pr[lane], b1 = pr[lane + 32], f0 = pr[64 + lane], f1 = pr[96 + lane];
                x0 = (x0 * pv - __umulhi(x0, pvp) * p) + 2 * p - (numer * b0 - __umulhi(numer, f0) * p);
                x1 = (x1 * pv - __umulhi(x1, pvp) * p) + 2 * p - (numer * b1 - __umulhi(numer, f1) * p);
            }
            if (i == pi) is_pivot = true;  // its registers hold the published (reduced) row
            first = pi + 1;                // rows between the previous pivot and pi were zero
            ++t;
        }
        __syncthreads();
        if (live) {  // pivot rows: scaled U; other rows: zero Schur complement
            S[i * SS + lane] = red4p(x0, p);
            S[i * SS + lane + 32] = red4p(x1, p);
        }
        if (tid == 0) misc[0] = t;
        __syncthreads();
        stamp(2);
        const uint32_t rs = misc[0];
        if (rs == 0) continue;
        // (C) D_t = prod_{j<t} piv_j; one inverse of the total, suffix products for the rest
        if (warp == 0) {
            const uint32_t v = lane < rs ? sl[lane] : 1u;
            uint32_t inc = v;
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                const uint32_t o = __shfl_up_sync(FULL, inc, off);
                if (lane >= (uint32_t)off) inc = mul_mod(inc, o, p, mu);
            }
            uint32_t exc = __shfl_up_sync(FULL, inc, 1);
            if (lane == 0) exc = 1u % p;
            const uint32_t total = __shfl_sync(FULL, inc, rs - 1);
            const uint32_t tinv = __shfl_sync(FULL, lane == 0 ? inv_mod_bin(total, p) : 0u, 0);
            uint32_t suf = lane + 1 < rs ? sl[lane + 1] : 1u;  // prod_{j>t} piv_j by a suffix scan
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                const uint32_t o = __shfl_down_sync(FULL, suf, off);
                if (lane + off < 32) suf = mul_mod(suf, o, p, mu);
            }
            const uint32_t inv_incl = mul_mod(tinv, suf, p, mu);  // 1 / prod_{j<=t}
            const uint32_t inv_exc = __shfl_up_sync(FULL, inv_incl, 1);
            if (lane < rs) {
                const uint32_t invD = lane == 0 ? 1u % p : inv_exc;
                const uint32_t invp = mul_mod(exc, inv_incl, p, mu);  // 1 / piv_t
                sl[32 + lane] = invD;
                sl[48 + lane] = invp;
                // exact pivot value piv_t / D_t; its inverse D_t / piv_t
                const uint32_t ip = mul_mod(exc, invp, p, mu);
                ipv[R + lane] = ip;
                ipf[R + lane] = shoup_pre(ip, p, mu);
            }
        }
        __syncthreads();
        // exact U rows (and their Shoup factors) and the slab's exact L entries
        for (uint32_t idx = tid; idx < rs * 64; idx += SL_THREADS) {
            const uint32_t tt = idx >> 6, j = idx & 63;
            uint32_t* u = S + prow[R + tt] * SS;
            const uint32_t e = mul_mod(u[j], sl[32 + tt], p, mu);
            u[j] = e;
            Uf[(R + tt) * SS + j] = shoup_pre(e, p, mu);
        }
        for (uint32_t idx = tid; idx < rows * rs; idx += SL_THREADS) {
            const uint32_t ii = i0 + idx / rs, tt = idx % rs;
            if (ii > prow[R + tt]) Lx[ii * LS + R + tt] = mul_mod(Lx[ii * LS + R + tt], sl[48 + tt], p, mu);
        }
        __syncthreads();
        stamp(3);
        R += rs;
    }
    const uint32_t r = R;

    // ---- permutations and packed output (exact L and U already in place)
    for (uint32_t ii = tid; ii < 64; ii += SL_THREADS) {
        rowrank[ii] = NONE;
        colrank[ii] = NONE;
    }
    __syncthreads();
    for (uint32_t k = tid; k < r; k += SL_THREADS) {
        rowrank[prow[k]] = k;
        colrank[pcol[k]] = k;
    }
    __syncthreads();
    if (warp < 2) {
        const uint32_t dim = warp == 0 ? m : n;
        const uint32_t* rank_of = warp == 0 ? rowrank : colrank;
        const uint32_t* order = warp == 0 ? prow : pcol;
        uint32_t* out = warp == 0 ? Psh : Qsh;
        uint32_t base = 0;
        for (uint32_t c = 0; c < dim; c += 32) {
            const uint32_t ii = c + lane;
            const bool np = ii < dim && rank_of[ii] == NONE;
            const uint32_t bal = __ballot_sync(FULL, np);
            if (np) out[r + base + __popc(bal & ((1u << lane) - 1u))] = ii;
            base += __popc(bal);
        }
        for (uint32_t k = lane; k < r; k += 32) out[k] = order[k];
        __syncwarp();
        uint32_t lo = NONE, hi = 0;
        for (uint32_t ii = lane; ii < dim; ii += 32)
            if (out[ii] != ii) {
                lo = min(lo, ii);
                hi = max(hi, ii + 1);
            }
        lo = __reduce_min_sync(FULL, lo);
        hi = __reduce_max_sync(FULL, hi);
        if (lane == 0) misc[5 + warp] = lo < hi ? 1u : 0u;  // this permutation moves something
        if (lane == 0) {
            if (warp == 0) {
                info->rank = r;
                info->plo = lo < hi ? lo : 0;
                info->phi = lo < hi ? hi : 0;
            } else {
                info->qlo = lo < hi ? lo : 0;
                info->qhi = lo < hi ? hi : 0;
            }
        }
    }
    __syncthreads();
    for (uint32_t ii = tid; ii < m; ii += SL_THREADS) Pd[ii] = Psh[ii];
    for (uint32_t j = tid; j < n; j += SL_THREADS) Qd[j] = Qsh[j];
    for (uint32_t idx = tid; idx < m * n; idx += SL_THREADS) {
        const uint32_t tt = idx / n, u = idx % n;
        const uint32_t ii = Psh[tt], j = Qsh[u];
        const uint32_t k = rowrank[ii], tc = colrank[j];
        uint32_t v;
        if (tc < r && tc < k)  // L entry (k == NONE for non-pivot rows)
            v = Lx[ii * LS + tc];
        else  // U row k, or the zero Schur complement of a non-pivot row
            v = S[ii * SS + j];
        A[(uint64_t)tt * lda + u] = v;
    }
    __syncthreads();
    stamp(7);
    if (tid == 0 && g_base_dbg) {
        unsigned long long* d = g_base_dbg + 6 * 4096 + 8 * (atomicAdd(&g_base_dbg_n, 1u) % 64);
        for (int q = 0; q < 8; ++q) d[q] = ph[q];
    }
    if (tid == 0) {
        info->cached = 0;
        // speculative launch (top bit of seq): the host assumed full rank and identity P, Q
        if ((seq & SPEC_BIT) && (r != min(m, n) || misc[5] || misc[6])) {
            volatile uint32_t* sf = &info->spec_fail;
            if (!*sf) *reinterpret_cast<volatile uint32_t*>(&info->fail_seq) = seq;  // the first failure
            *sf = 1u;
        }
        __threadfence_system();
        *reinterpret_cast<volatile uint32_t*>(&info->seq) = seq;
    }
}

// ---------------------------------------------------------------------------------------------
// Speculative base case (m, n <= 64): the caller assumed full rank with identity permutations,
// i.e. that the pivot of step k is (k, k).  Then rr_base is plain LU without pivoting -- the
// pivot search picks row k (the first remaining row; it is nonzero at column k) and column k (its
// first nonzero entry, every earlier column having been eliminated) -- so the kernel runs that LU
// with no search and checks the guess: a zero diagonal pivot raises spec_fail and the caller
// reruns exactly (the outputs of a failed launch are never used).
//
// Fraction-free over the whole block: row_i <- pv_k * row_i - row_i[k] * row_k keeps row_i =
// D_k * (exact Schur row) with D_k = prod_{j<k} pv_j, so no inverse is needed while eliminating;
// at the end one modular inverse (prefix / suffix products) gives U_k = row_k / D_k and
// L_ik = numer_ik / pv_k (numer_ik = row_i[k] at step k, frozen in place in the register of
// column k).  Rows stay in registers (warp w owns rows w, w+16, w+32, w+48; lane l columns l and
// l+32); the owner of row k+1 publishes it (reduced, with Shoup factors) right after its step-k
// update into a double-buffered slot -- one barrier per pivot, no slab phases.
#ifndef FFG_SP_WARPS
#define FFG_SP_WARPS 16
#endif
constexpr int SP_WARPS = FFG_SP_WARPS;
constexpr int SP_THREADS = SP_WARPS * 32;
constexpr int SP_RPW = 64 / SP_WARPS;  // rows per warp

// allow_q (panel schedule, square blocks): the guess is only "full rank"; a zero diagonal Schur
// entry is handled like rr_base does -- the pivot of row k is its first nonzero column among the
// columns not yet chosen (rr_base's rotations keep the remaining columns in original order), so
// the kernel tracks physical pivot columns c_k and writes the block in logical (rotated) order,
// with Q[t] = c_t.  Full rank implies P = identity.  Without allow_q any c_k != k fails the guess.
// FULLB: a 64 x 64 block (every base case of a square matrix whose order is a multiple of 64):
// the bounds checks fold away.
template <bool FULLB>
__global__ void __launch_bounds__(SP_THREADS, 1)
    rr_base_spec_kernel(uint32_t* __restrict__ A, uint64_t lda, uint32_t m_, uint32_t n_, uint32_t* __restrict__ Pd,
                        uint32_t* __restrict__ Qd, BaseInfo* __restrict__ info, uint32_t p, uint64_t mu,
                        uint32_t seq, uint32_t allow_q) {
    __shared__ __align__(16) uint32_t buf[2][128];  // published pivot row: 64 values, 64 Shoup factors
    __shared__ uint32_t pvs[64];                     // fraction-free pivots
    __shared__ uint32_t pcol[64];                    // physical column of pivot k
    __shared__ uint32_t invd[64], invdf[64];         // 1 / D_k and its Shoup factor
    __shared__ uint32_t invp[64], invpf[64];         // 1 / pv_k and its Shoup factor
    __shared__ uint32_t fail;
    const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    constexpr uint32_t FULL = 0xffffffffu;
    const uint32_t m = FULLB ? 64u : m_, n = FULLB ? 64u : n_;
    const uint32_t r = min(m, n);
    ptx::pdl_enter();

    uint32_t x[SP_RPW][2];
#pragma unroll
    for (int j = 0; j < SP_RPW; ++j) {
        const uint32_t i = warp + SP_WARPS * j;
        const uint32_t* row = A + (uint64_t)i * lda;
        x[j][0] = (i < m && lane < n) ? row[lane] : 0u;
        x[j][1] = (i < m && lane + 32 < n) ? row[lane + 32] : 0u;
    }
    // publish row k (reduced, with Shoup factors)
    auto publish = [&](uint32_t& a0, uint32_t& a1, uint32_t* dst) {
        a0 = red4p(a0, p);
        a1 = red4p(a1, p);
        dst[lane] = a0;
        dst[lane + 32] = a1;
        dst[64 + lane] = shoup_pre(a0, p, mu);
        dst[96 + lane] = shoup_pre(a1, p, mu);
    };
    if (tid == 0) fail = 0u;
    if (warp == 0 && r > 0) publish(x[0][0], x[0][1], buf[0]);
    __syncthreads();

    // Every thread finds the pivot column itself from the published row: while every pivot so far
    // sat on the diagonal (`diag`, uniform) and the diagonal entry is nonzero it is column k at no
    // extra cost; otherwise a ballot over the row picks its first nonzero column outside `used`.
    uint64_t used = 0;  // maintained once the first pivot left the diagonal
    bool diag = true;
    for (uint32_t k = 0; k < r; ++k) {
        const uint32_t* pr = buf[k & 1];
        const uint32_t b0 = pr[lane], b1 = pr[lane + 32], f0 = pr[64 + lane], f1 = pr[96 + lane];
        uint32_t c = k, pv = pr[k], pvp = pr[64 + k];
        if (!diag || pv == 0u) {  // uniform
            if (diag) used = k ? (~0ull >> (64 - k)) : 0ull;  // columns < k
            const uint32_t m0 = __ballot_sync(FULL, b0 != 0u && lane < n && !((used >> lane) & 1u));
            const uint32_t m1 = __ballot_sync(FULL, b1 != 0u && lane + 32 < n && !((used >> (lane + 32)) & 1u));
            c = m0 ? (uint32_t)__ffs(m0) - 1 : (m1 ? 31u + (uint32_t)__ffs(m1) : 64u);
            if (c == 64u || (!allow_q && c != k)) {
                if (tid == 0) fail = 1u;
                c = k;  // keep going on a harmless column; the outputs are discarded
            }
            pv = pr[c];
            pvp = pr[64 + c];
            diag = diag && c == k;
        }
        if (tid == 0) {
            pvs[k] = pv;
            pcol[k] = c;
        }
        const uint32_t nxt = k + 1;
        if (diag && k >= 32) {  // uniform: pivot (k, k) in the second column half; the first half is final
#pragma unroll
            for (int j = 0; j < SP_RPW; ++j) {
                const uint32_t i = warp + SP_WARPS * j;
                if (i > k && i < m) {  // warp-uniform
                    const uint32_t numer = red4p(__shfl_sync(FULL, x[j][1], k & 31), p);
                    const uint32_t u1 = (x[j][1] * pv - __umulhi(x[j][1], pvp) * p) + 2 * p -
                                        (numer * b1 - __umulhi(numer, f1) * p);
                    x[j][1] = lane + 32 > k ? u1 : (lane + 32 == k ? numer : x[j][1]);
                    if (i == nxt && nxt < r) publish(x[j][0], x[j][1], buf[nxt & 1]);
                }
            }
        } else if (diag) {  // uniform: the pivot is (k, k)
#pragma unroll
            for (int j = 0; j < SP_RPW; ++j) {
                const uint32_t i = warp + SP_WARPS * j;
                if (i > k && i < m) {  // warp-uniform
                    const uint32_t numer = red4p(__shfl_sync(FULL, k < 32 ? x[j][0] : x[j][1], k & 31), p);
                    const uint32_t u0 = (x[j][0] * pv - __umulhi(x[j][0], pvp) * p) + 2 * p -
                                        (numer * b0 - __umulhi(numer, f0) * p);
                    const uint32_t u1 = (x[j][1] * pv - __umulhi(x[j][1], pvp) * p) + 2 * p -
                                        (numer * b1 - __umulhi(numer, f1) * p);
                    // columns > k take the update; column k keeps the L numerator; earlier ones stay
                    x[j][0] = lane > k ? u0 : (lane == k ? numer : x[j][0]);
                    x[j][1] = lane + 32 > k ? u1 : (lane + 32 == k ? numer : x[j][1]);
                    if (i == nxt && nxt < r) publish(x[j][0], x[j][1], buf[nxt & 1]);
                }
            }
        } else {  // pivot (k, c): the columns outside `used` and c take the update
            used |= 1ull << c;
            const bool up0 = !((used >> lane) & 1u), up1 = !((used >> (lane + 32)) & 1u);
#pragma unroll
            for (int j = 0; j < SP_RPW; ++j) {
                const uint32_t i = warp + SP_WARPS * j;
                if (i > k && i < m) {  // warp-uniform
                    const uint32_t numer = red4p(__shfl_sync(FULL, c < 32 ? x[j][0] : x[j][1], c & 31), p);
                    const uint32_t u0 = (x[j][0] * pv - __umulhi(x[j][0], pvp) * p) + 2 * p -
                                        (numer * b0 - __umulhi(numer, f0) * p);
                    const uint32_t u1 = (x[j][1] * pv - __umulhi(x[j][1], pvp) * p) + 2 * p -
                                        (numer * b1 - __umulhi(numer, f1) * p);
                    x[j][0] = up0 ? u0 : (lane == c ? numer : x[j][0]);
                    x[j][1] = up1 ? u1 : (lane + 32 == c ? numer : x[j][1]);
                    if (i == nxt && nxt < r) publish(x[j][0], x[j][1], buf[nxt & 1]);
                }
            }
        }
        __syncthreads();
    }

    // ---- one inverse: D_k = prod_{j<k} pv_j, 1/D_k and 1/pv_k = D_k / D_{k+1}
    if (warp == 0 && r > 0 && !fail) {
        const uint32_t e0 = 2 * lane, e1 = 2 * lane + 1;
        const uint32_t v0 = e0 < r ? pvs[e0] : 1u, v1 = e1 < r ? pvs[e1] : 1u;
        uint32_t inc = mul_mod(v0, v1, p, mu);  // inclusive scan of pair products
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const uint32_t o = __shfl_up_sync(FULL, inc, off);
            if (lane >= (uint32_t)off) inc = mul_mod(inc, o, p, mu);
        }
        uint32_t exc = __shfl_up_sync(FULL, inc, 1);
        if (lane == 0) exc = 1u % p;
        const uint32_t D0 = exc, D1 = mul_mod(exc, v0, p, mu);  // D_{e0}, D_{e1}
        const uint32_t total = __shfl_sync(FULL, inc, 31);
        const uint32_t tinv = __shfl_sync(FULL, lane == 0 ? inv_mod_bin(total, p) : 0u, 0);
        uint32_t suf = mul_mod(v0, v1, p, mu);  // inclusive suffix scan of pair products
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const uint32_t o = __shfl_down_sync(FULL, suf, off);
            if (lane + off < 32) suf = mul_mod(suf, o, p, mu);
        }
        // 1/D_e = tinv * prod_{j >= e} pv_j
        const uint32_t iD0 = mul_mod(tinv, suf, p, mu);
        const uint32_t sufx = __shfl_down_sync(FULL, suf, 1);
        const uint32_t iD2 = mul_mod(tinv, lane == 31 ? 1u % p : sufx, p, mu);  // 1/D_{e0+2}
        const uint32_t iD1 = mul_mod(iD2, v1, p, mu);
        if (e0 < r) {
            invd[e0] = iD0;
            invdf[e0] = shoup_pre(iD0, p, mu);
            const uint32_t ip = mul_mod(D0, iD1, p, mu);  // D_e0 / D_{e0+1}
            invp[e0] = ip;
            invpf[e0] = shoup_pre(ip, p, mu);
        }
        if (e1 < r) {
            invd[e1] = iD1;
            invdf[e1] = shoup_pre(iD1, p, mu);
            const uint32_t ip = mul_mod(D1, iD2, p, mu);
            invp[e1] = ip;
            invpf[e1] = shoup_pre(ip, p, mu);
        }
    }
    __syncthreads();
    if (!fail) {
        // logical column t of the output holds physical column pcol[t] (t < r); beyond r (wide
        // blocks, identity guess only) the columns stay in place
        const uint32_t s0 = (!diag && lane < r) ? pcol[lane] : lane;
        const uint32_t s1 = (!diag && lane + 32 < r) ? pcol[lane + 32] : lane + 32;
#pragma unroll
        for (int j = 0; j < SP_RPW; ++j) {
            const uint32_t i = warp + SP_WARPS * j;
            if (i >= m) continue;  // warp-uniform
            uint32_t g[2] = {x[j][0], x[j][1]};
            if (!diag) {  // uniform: gather the logical columns
                const uint32_t g00 = __shfl_sync(FULL, x[j][0], s0 & 31), g01 = __shfl_sync(FULL, x[j][1], s0 & 31);
                const uint32_t g10 = __shfl_sync(FULL, x[j][0], s1 & 31), g11 = __shfl_sync(FULL, x[j][1], s1 & 31);
                g[0] = s0 < 32 ? g00 : g01;
                g[1] = s1 < 32 ? g10 : g11;
            }
            uint32_t* row = A + (uint64_t)i * lda;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const uint32_t c = lane + 32 * h;
                if (c >= n) continue;
                uint32_t v;
                if (c < i)  // L entry (c < r: every column is a pivot column when i >= r)
                    v = shoup_mul(g[h], invp[c], invpf[c], p);
                else  // U entry of pivot row i < r
                    v = shoup_mul(g[h], invd[i], invdf[i], p);
                row[c] = v;
            }
        }
    }
    for (uint32_t ii = tid; ii < m; ii += SP_THREADS) Pd[ii] = ii;
    for (uint32_t jj = tid; jj < n; jj += SP_THREADS) Qd[jj] = jj < r ? pcol[jj] : jj;
    __syncthreads();
    if (tid == 0) {
        info->rank = r;
        info->plo = info->phi = info->qlo = info->qhi = 0;
        info->cached = 0;
        if ((seq & SPEC_BIT) && fail) {
            volatile uint32_t* sf = &info->spec_fail;
            if (!*sf) *reinterpret_cast<volatile uint32_t*>(&info->fail_seq) = seq;  // the first failure
            *sf = 1u;
        }
        __threadfence_system();
        *reinterpret_cast<volatile uint32_t*>(&info->seq) = seq;
    }
}

void base_dbg_init() {
    static bool done = false;
    if (done || !knob_set("FFG_BASE_DBG")) return;
    done = true;
    unsigned long long* buf = nullptr;
    FFG_CUDA(cudaMalloc(&buf, (4096 * 6 + 8 * 64) * 8));
    FFG_CUDA(cudaMemcpyToSymbol(g_base_dbg, &buf, sizeof(buf)));
    if (knob_str("FFG_BASE_SKIP")) {
        int one = 1;
        FFG_CUDA(cudaMemcpyToSymbol(g_base_skip, &one, sizeof(one)));
    }
}

void base_dbg_dump() {
    if (!knob_set("FFG_BASE_DBG")) return;
    unsigned long long* buf = nullptr;
    unsigned int n = 0;
    FFG_CUDA(cudaDeviceSynchronize());
    FFG_CUDA(cudaMemcpyFromSymbol(&buf, g_base_dbg, sizeof(buf)));
    FFG_CUDA(cudaMemcpyFromSymbol(&n, g_base_dbg_n, sizeof(n)));
    if (!buf || n == 0) return;
    {
        std::vector<unsigned long long> ph(8 * 64);
        FFG_CUDA(cudaMemcpy(ph.data(), buf + 6 * 4096, ph.size() * 8, cudaMemcpyDeviceToHost));
        double acc[8] = {0};
        const unsigned cnt = std::min(n, 64u);
        for (unsigned i = 0; i < cnt; ++i)
            for (int q = 0; q < 8; ++q) acc[q] += ph[8 * i + q];
        fprintf(stderr, "SLAB_DBG cycles/launch: load %.0f schur %.0f pivot %.0f norm %.0f - %.0f - %.0f out %.0f (%.0f)\n",
                acc[0] / cnt, acc[1] / cnt, acc[2] / cnt, acc[3] / cnt, acc[4] / cnt, acc[5] / cnt, acc[6] / cnt,
                acc[7] / cnt);
    }
    n = std::min(n, 4096u);
    std::vector<unsigned long long> h(6 * (size_t)n);
    FFG_CUDA(cudaMemcpy(h.data(), buf, h.size() * 8, cudaMemcpyDeviceToHost));
    double piv_us = 0, tot_us = 0, mhz = 0;
    for (unsigned i = 0; i < n; ++i) {
        const unsigned long long* d = &h[6 * i];
        piv_us += (d[3] - d[1]) / 1e3;
        tot_us += (d[5] - d[1]) / 1e3;
        mhz += (double)(d[4] - d[0]) / ((d[5] - d[1]) / 1e3);
    }
    fprintf(stderr, "BASE_DBG %u launches: pivoting %.2f us, to output %.2f us avg, SM clock %.0f MHz avg\n", n,
            piv_us / n, tot_us / n, mhz / n);
    unsigned int zero = 0;
    FFG_CUDA(cudaMemcpyToSymbol(g_base_dbg_n, &zero, sizeof(zero)));
}

bool rr_base_launch(const Blas& b, DView a, uint32_t* Pd, uint32_t* Qd, void* info_dev, uint32_t* inv_out,
                    uint32_t seq, bool allow_q) {
    base_dbg_init();
    BaseLayout lay;
    lay.m = (uint32_t)a.rows;
    lay.n = (uint32_t)a.cols;
    lay.ns = (uint32_t)round_up(a.cols, 8);
    lay.rmax = (uint32_t)std::min(a.rows, a.cols);
    const size_t fixed = ((size_t)5 * lay.rmax + 2 * ((size_t)lay.m + lay.n) + 4) * 4;
    const size_t blk = ((size_t)lay.m * lay.ns + (size_t)lay.m * lay.rmax) * 4;
    BaseInfo* info = static_cast<BaseInfo*>(info_dev);
    // panel schedule: square speculative block with an inverse slot -> the fused base + inverses
    // kernel (baseinv.cu), which also writes inv(L) and inv(U) into inv_out
    static const bool no_fused_inv = (knob_int("FFG_BASE_INV", 1) == 0);
    if ((seq & SPEC_BIT) && inv_out && !no_fused_inv && lay.m == lay.n && lay.m <= 64 && lay.m > 0) {
        rr_base_inv_launch(b, a, Pd, Qd, info, inv_out, seq, allow_q);
        return true;
    }
    // room for the factor inverses (two INV_MAX frames + workspace), only for ranks <= INV_MAX
    const size_t inv_bytes = (2 * INV_MAX * (INV_MAX + 1) + (INV_MAX / 2) * (INV_MAX / 2) + INV_MAX + 8) * 4;
    if (inv_out && (fixed + blk + inv_bytes > BASE_SMEM_LIMIT)) inv_out = nullptr;
    b.ws.prof.begin(b.st);
    // kernel choice (read per launch so tests can exercise every path): FFG_BASE_SMEM=1 forces the
    // shared-memory right-looking kernel, FFG_BASE_NO_SLAB=1 the register right-looking one
    const char* e_smem = knob_str("FFG_BASE_SMEM");
    const char* e_slab = knob_str("FFG_BASE_NO_SLAB");
    const bool spec = (seq & SPEC_BIT) != 0;  // speculative launches need the slab kernel's check
    const bool no_reg = !spec && e_smem && atoi(e_smem) != 0;
    const bool no_slab = !spec && e_slab && atoi(e_slab) != 0;
    const char* e_spec = knob_str("FFG_SPEC_SLAB");  // diagnostics: speculative launches on the slab kernel
    if (spec && lay.m <= 64 && lay.n <= 64 && !(e_spec && atoi(e_spec) != 0)) {
        if (lay.m == 64 && lay.n == 64)
            launch_k(rr_base_spec_kernel<true>, dim3(1), dim3(SP_THREADS), 0, b.st, a.d, a.ld, lay.m, lay.n, Pd, Qd,
                     info, b.F.p, b.F.mu, seq, (uint32_t)allow_q);
        else
            launch_k(rr_base_spec_kernel<false>, dim3(1), dim3(SP_THREADS), 0, b.st, a.d, a.ld, lay.m, lay.n, Pd, Qd,
                     info, b.F.p, b.F.mu, seq, (uint32_t)(allow_q && lay.m == lay.n));
        FFG_CUDA(cudaGetLastError());
        b.ws.prof.end(b.st, PROF_BASE, 2.0 * lay.m * lay.n * 4, 2.0 * lay.rmax * (double)lay.m * lay.n);
        b.count();
        return false;
    }
    if (!no_reg && !no_slab && lay.m <= 64 && lay.n <= 64) {
        const size_t smem = (2 * 64 * SS + 64 * LS + 2 * 16 * 132 + 64 * 11 + 8) * 4;
        static PerDeviceOnce once;
        once([smem] {
            FFG_CUDA(cudaFuncSetAttribute(rr_base_slab_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        });
        launch_k(rr_base_slab_kernel, dim3(1), dim3(SL_THREADS), smem, b.st, a.d, a.ld, lay.m, lay.n, Pd, Qd, info,
                 b.F.p, b.F.mu, seq);
        FFG_CUDA(cudaGetLastError());
        b.ws.prof.end(b.st, PROF_BASE, 2.0 * lay.m * lay.n * 4, 2.0 * lay.rmax * (double)lay.m * lay.n);
        b.count();
        return false;
    }
    const bool reg = !no_reg && lay.m <= 64 && lay.n <= 64;
    const size_t slots = (8 + 128 + 16 + 16 * 64 + 64 + 4) * 4;  // candidate slots of the register path
    if (reg && fixed + blk + slots <= BASE_SMEM_LIMIT) {
        inv_out = nullptr;  // the register path does not cache factor inverses
        static PerDeviceOnce once;
        once([] {
            FFG_CUDA(cudaFuncSetAttribute(rr_base_kernel<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)BASE_SMEM_LIMIT));
        });
        rr_base_kernel<true, true><<<1, BASE_THREADS_REG, fixed + blk + slots, b.st>>>(a.d, a.ld, lay, nullptr, Pd, Qd,
                                                                                   info, b.F.p, b.F.mu, nullptr, seq);
    } else if (fixed + blk <= BASE_SMEM_LIMIT) {
        static PerDeviceOnce once;
        once([] {
            FFG_CUDA(cudaFuncSetAttribute(rr_base_kernel<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)BASE_SMEM_LIMIT));
        });
        rr_base_kernel<true, false><<<1, BASE_THREADS, fixed + blk + (inv_out ? inv_bytes : 0), b.st>>>(
            a.d, a.ld, lay, nullptr, Pd, Qd, info, b.F.p, b.F.mu, inv_out, seq);
    } else {
        inv_out = nullptr;
        if (fixed > BASE_SMEM_LIMIT) throw Error(FFG_ERR_INVALID_BLOCK, "base case block too large");
        static PerDeviceOnce once;
        once([] {
            FFG_CUDA(cudaFuncSetAttribute(rr_base_kernel<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)BASE_SMEM_LIMIT));
        });
        uint32_t* scratch = nullptr;
        FFG_CUDA(cudaMallocAsync(&scratch, blk, b.st));
        rr_base_kernel<false, false><<<1, BASE_THREADS, fixed, b.st>>>(a.d, a.ld, lay, scratch, Pd, Qd, info, b.F.p,
                                                                       b.F.mu, nullptr, seq);
        FFG_CUDA(cudaFreeAsync(scratch, b.st));
    }
    FFG_CUDA(cudaGetLastError());
    b.ws.prof.end(b.st, PROF_BASE, 2.0 * lay.m * lay.n * 4, 2.0 * lay.rmax * (double)lay.m * lay.n);
    b.count();
    return inv_out != nullptr;
}

}  // namespace ffg
