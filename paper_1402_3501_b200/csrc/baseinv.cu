// baseinv.cu -- the panel schedule's speculative base case that also produces both factor inverses.
//
// The panel schedule (pluq.cu, rec_panel / two_leaf) factors each t x t diagonal block (t <= 64,
// full rank guessed: P = identity, Q = the block's column pivots, rankrev.hpp:29-78 restated) and
// then needs inv(L) and inv(U) of the block for its panel solves.  Here both come out of the same
// 64-step elimination chain as L and U, as a cluster of two independent CTAs:
//
//   CTA 0 eliminates [A | I] row-wise:          [A | I]    ->  [D_i U_i | D_i inv(L)_i]
//   CTA 1 eliminates [A^T | I] (same pivots):   [A^T | I]  ->  row i of its I part = D_i pv_i U^-1[:, i]^T
//
// (fraction-free: row_i <- pv_k row_i - x_ik row_k keeps row_i = D_k x the exact Schur row,
// D_k = pv_0 ... pv_{k-1}; one modular inverse at the end recovers 1/D_k and 1/pv_k.)
// The augmentation costs no extra arithmetic: the I part of a row is nonzero only in columns <= k
// and the A part is live only in columns > k, so lane column j carries ONE live value -- the A part
// while j > k, the I part after -- plus the frozen L numerator of column j.  Each CTA runs exactly
// the work of a plain 64 x 64 elimination; the two run side by side on two SMs.
//
// Chain.  Warp w (of 16) holds the 4-row block b = 15 - w in registers (lane l: columns l, l + 32)
// as a shift register: slot 0 is always the warp's next pivot row.  Pivot row k is published into
// its own slot of a 64-slot ring in shared memory (values + Shoup factors) and announced on its own
// mbarrier: warps run decoupled, the owner of row k + 1 updates it first, publishes it, then its
// other rows; the next three pivots stay in the same warp (forwarded in registers).  Early blocks
// sit in high warp ids: the SMSP arbiter issues highest-id-first, so the warp producing the next
// pivot wins its SMSP over the warps still catching up.
//
// Instruction fetch.  Two CTAs on two SMs that ran other kernels a moment ago start with cold
// instruction caches; every straight-line instruction executed once costs an L2 fetch (measured
// ~25-40 cycles each on B200, against ~8 once warm).  So this kernel is written small: the pivot
// loop is one body of four row updates (fits the ~6 KB L0 cache) and every other phase is a rolled
// loop.  (An unrolled version of the same arithmetic measured 2.5x slower.)
//
// A zero Schur diagonal (column pivot, ~1/p per pivot) switches both CTAs, at that step, to a plain
// shared-memory elimination with explicit A and I parts (CTA 0: first nonzero unused column of the
// pivot row, rr_base's choice; CTA 1: the matching row of A^T).  A rank-deficient block raises the
// speculation-failed flag exactly like rr_base_spec_kernel (base.cu); its outputs are then unused.
#include "pluq.cuh"
#include "ptx.cuh"

namespace ffg {

namespace {

constexpr int BI_WARPS = 16;
constexpr int BI_THREADS = BI_WARPS * 32;
constexpr int BI_SS = 65;  // row stride of the shared-memory matrices
constexpr uint32_t BI_FULL = 0xffffffffu;

struct BiSmem {
    uint32_t pub[64][64];    // published pivot row k (fraction-free; cols < k: I part, > k: A part,
                             // [k][k] = 1, see the I-part scaling note); after the loop: the final
                             // rows in logical order
    uint32_t pf[64][64];     // Shoup factors of pub
    uint32_t Ln[64][64];     // L numerators of row i (columns < i), saved when row i is published
    uint32_t S[64][BI_SS];   // block staging / slow path: A part / epilogue transpose
    uint32_t I[64][BI_SS];   // slow path: I part
    uint32_t pv[64], pvf[64], D[64];
    uint32_t invd[64], invdf[64], invp[64], invpf[64], Dd[64], Ddf[64];
    uint32_t pcol[64];       // physical column of logical column t (the block's Q)
    uint32_t perm[64];       // current logical -> physical column order (CTA 1: rows of A^T)
    uint64_t full[64];       // pivot row k published
    uint32_t fail, k0, cmin;
};

__device__ __forceinline__ uint32_t bi_red4p(uint32_t x, uint32_t p) {  // [0, 4p) -> [0, p)
    x = min(x, x - 2 * p);
    return min(x, x - p);
}

__device__ __forceinline__ uint32_t bi_sub(uint32_t a, uint32_t b, uint32_t p) { return a >= b ? a - b : a + p - b; }

__device__ __forceinline__ void bi_cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// a * b mod p for a, b < p < 2^26 in double precision (the epilogue's short serial chains): the product
// is exact (< 2^52), the quotient estimate is off by at most one, corrected once each way
__device__ __forceinline__ uint32_t bi_mulmod(uint32_t a, uint32_t b, double pd, double pinv) {
    const double ab = (double)a * (double)b;
    const double q = floor(ab * pinv);
    double r = fma(-q, pd, ab);
    r = r < 0.0 ? r + pd : r;
    r = r >= pd ? r - pd : r;
    return (uint32_t)r;
}

// x * w - (x * w div p) * p with w's Shoup factor wf: in [0, 2p) for any 32-bit x
__device__ __forceinline__ uint32_t bi_shoup_lazy(uint32_t x, uint32_t w, uint32_t wf, uint32_t p) {
    return x * w - __umulhi(x, wf) * p;
}

// per-step values every row update of step k uses
struct BiStep {
    uint32_t kh, kl, pv, pvp, b0, b1, f0, f1, p;
    uint32_t k4p2, mu32;  // small fields: 4 p^2 and floor(2^32 / p)
    bool dk0, dk1;
};

// one row's step-k update (fast path): numer = its live value in column k (frozen as the L
// numerator there), every lane column then takes new = pv * live - numer * b  (lazy, [0, 4p));
// in column k the I part starts from zero
//
// SMALLP (p < 2^14): pv * live - numer * b + 4 p^2 lies in (0, 8 p^2) < 2^31, so the update is two
// 32-bit multiply-adds and one 32-bit Barrett step (result in [0, 2p)) -- four IMADs per entry
// instead of six, and the published rows need no Shoup factors (three shoup_pre less on the
// owner's serial path per pivot).
template <bool SMALLP>
__device__ __forceinline__ void bi_row(uint32_t (&lv)[2], uint32_t (&fz)[2], const BiStep& q) {
    const uint32_t numer = __shfl_sync(BI_FULL, q.kh ? lv[1] : lv[0], q.kl);
    if (SMALLP) {
        const uint32_t nn = 0u - numer;
        const uint32_t u0 = (q.dk0 ? 0u : lv[0]) * q.pv + q.k4p2 + nn * q.b0;
        const uint32_t u1 = (q.dk1 ? 0u : lv[1]) * q.pv + q.k4p2 + nn * q.b1;
        lv[0] = u0 - __umulhi(u0, q.mu32) * q.p;
        lv[1] = u1 - __umulhi(u1, q.mu32) * q.p;
        fz[0] = q.dk0 ? numer : fz[0];
        fz[1] = q.dk1 ? numer : fz[1];
        return;
    }
    const uint32_t t10 = bi_shoup_lazy(lv[0], q.pv, q.pvp, q.p), t11 = bi_shoup_lazy(lv[1], q.pv, q.pvp, q.p);
    const uint32_t t20 = bi_shoup_lazy(numer, q.b0, q.f0, q.p), t21 = bi_shoup_lazy(numer, q.b1, q.f1, q.p);
    lv[0] = (q.dk0 ? 0u : t10) + 2 * q.p - t20;
    lv[1] = (q.dk1 ? 0u : t11) + 2 * q.p - t21;
    fz[0] = q.dk0 ? numer : fz[0];
    fz[1] = q.dk1 ? numer : fz[1];
}

}  // namespace

// diagnostics (-DBI_DBG builds, FFG_BI_DBG=1): clock64 at phase boundaries of CTA 0
__device__ long long* g_bi_dbg = nullptr;
#ifdef BI_DBG
#define BI_STAMP(i) \
    if (!tr && tid == 0 && g_bi_dbg) g_bi_dbg[i] = clock64();
#else
#define BI_STAMP(i)
#endif

// I-part scaling: the I part of column j starts at step j from the pivot row's entry there, which
// is D_j in the plain fraction-free form; it is published as 1 instead (no product on the serial
// path), which scales the whole I column j by 1/D_j -- undone in the epilogue.
//
// grid = 2 CTAs (CTA 0: A, CTA 1: A^T, one cluster), BI_THREADS threads, sizeof(BiSmem) dynamic
// shared memory.  Outputs (CTA 0): the packed block (logical column order), Pd = identity, Qd =
// column pivots, inv[0, t^2) = inv(L); (CTA 1): inv[t^2, 2 t^2) = inv(U), both row-major with ld t;
// info as rr_base_spec_kernel.  allow_q = 0: any column pivot fails the guess.
template <bool SMALLP>
__global__ void __launch_bounds__(BI_THREADS, 1)
    rr_base_inv_kernel(uint32_t* __restrict__ A, uint64_t lda, uint32_t t, uint32_t* __restrict__ Pd,
                       uint32_t* __restrict__ Qd, BaseInfo* __restrict__ info, uint32_t* __restrict__ inv, uint32_t p,
                       uint64_t mu, uint32_t seq, uint32_t allow_q) {
    extern __shared__ __align__(16) unsigned char bi_raw[];
    BiSmem& sm = *reinterpret_cast<BiSmem*>(bi_raw);
    const uint32_t tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
    const bool tr = blockIdx.x == 1;
    if (tid < 64) {
        ptx::mbar_init(&sm.full[tid], 32);
        sm.perm[tid] = tid;
    }
    if (tid == 0) {
        sm.fail = 0u;
        sm.k0 = t;
        sm.cmin = 64u;
    }
    ptx::fence_mbar_init();
    BI_STAMP(0);
    ptx::pdl_enter();
    BI_STAMP(1);
    // stage the block (coalesced), zero-padded to 64 x 64
    {   // all eight loads of a thread in flight at once: one global-memory latency, not two
        uint32_t r[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const uint32_t x = tid + q * BI_THREADS, i = x >> 6, j = x & 63;
            r[q] = (i < t && j < t) ? A[(uint64_t)i * lda + j] : 0u;
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const uint32_t x = tid + q * BI_THREADS;
            sm.S[x >> 6][x & 63] = r[q];
        }
    }
    // both CTAs hold the input before CTA 0 may overwrite it (a 2-CTA cluster: co-scheduled)
    bi_cluster_sync();
    BI_STAMP(2);
    // A zero Schur diagonal at step k0 with a nonzero further right in row k0 (a column pivot,
    // ~1/p per step): rr_base takes the first such column (rankrev.hpp:29-78, columns rotated so
    // the ones not yet pivots stay in ascending order), so the elimination restarts on the block
    // with that logical column order -- the steps before k0 repeat unchanged.  No such column: the
    // block is rank deficient and the guess fails.
    uint32_t passes = 0;
    uint64_t ph = 0;  // bit k: parity of the phase pivot row k's mbarrier is in (flips per publish)
#pragma unroll 1
    for (;;) {
    ++passes;
#ifdef BI_RESTART_DBG
    if (tid == 0) printf("cta %d start pass %u\n", (int)tr, passes);
#endif
    // this warp's block: rows r0 .. r0 + 3, slot 0 = the next one to become a pivot
    const uint32_t r0 = 4 * (BI_WARPS - 1 - w);
    uint32_t nxt = r0, left = r0 < t ? min(4u, t - r0) : 0u;
    uint32_t lv[4][2], fz[4][2];
    {
        const uint32_t c0 = sm.perm[lane], c1 = sm.perm[lane + 32];
#pragma unroll
        for (int s = 0; s < 4; ++s) {
            const uint32_t i = r0 + s, ci = sm.perm[i];
            lv[s][0] = tr ? sm.S[lane][ci] : sm.S[i][c0];
            lv[s][1] = tr ? sm.S[lane + 32][ci] : sm.S[i][c1];
            fz[s][0] = fz[s][1] = 0u;
        }
    }
    // forwarded pivot (the warp's own last publish) and the publish itself
    bool fwd = false;
    uint32_t fpv = 0, fpvp = 0, fb0 = 0, fb1 = 0, ff0 = 0, ff1 = 0;
    auto publish = [&](uint32_t kn) {  // slot 0 (row kn, updated through pivot kn - 1) -> ring slot kn
        const uint32_t a0 = bi_red4p(lv[0][0], p), a1 = bi_red4p(lv[0][1], p);
        const uint32_t pvn = __shfl_sync(BI_FULL, kn >= 32 ? a1 : a0, kn & 31);
        const uint32_t v0 = lane == kn ? 1u : a0, v1 = lane + 32 == kn ? 1u : a1;
        uint32_t g0 = 0, g1 = 0, pvnf = 0;
        if (!SMALLP) {
            g0 = shoup_pre(v0, p, mu);
            g1 = shoup_pre(v1, p, mu);
            pvnf = shoup_pre(pvn, p, mu);
        }
        sm.pub[kn][lane] = v0;
        sm.pub[kn][lane + 32] = v1;
        if (!SMALLP) {
            sm.pf[kn][lane] = g0;
            sm.pf[kn][lane + 32] = g1;
        }
        if (lane == 0) {
            sm.pv[kn] = pvn;
            if (!SMALLP) sm.pvf[kn] = pvnf;
        }
        ptx::mbar_arrive(&sm.full[kn]);
        fwd = true;
        fpv = pvn;
        fpvp = pvnf;
        fb0 = v0;
        fb1 = v1;
        ff0 = g0;
        ff1 = g1;
        // its L numerators (columns < kn) -- then the shift register moves on
        sm.Ln[kn][lane] = bi_red4p(fz[0][0], p);
        sm.Ln[kn][lane + 32] = bi_red4p(fz[0][1], p);
#pragma unroll
        for (int s = 0; s < 3; ++s) {
            lv[s][0] = lv[s + 1][0];
            lv[s][1] = lv[s + 1][1];
            fz[s][0] = fz[s + 1][0];
            fz[s][1] = fz[s + 1][1];
        }
        ++nxt;
        --left;
    };
    if (left && nxt == 0) publish(0);  // row 0: I part [0][0] = 1, pivot = A[0][0]
#pragma unroll 1
    for (uint32_t k = 0; k < t && left; ++k) {
        BiStep q;
        if (fwd) {
            q.pv = fpv;
            q.pvp = fpvp;
            q.b0 = fb0;
            q.b1 = fb1;
            q.f0 = ff0;
            q.f1 = ff1;
        } else {
#ifdef BI_RESTART_DBG
            {
                uint32_t it = 0;
                while (!ptx::mbar_try_wait(&sm.full[k], (uint32_t)(ph >> k) & 1u)) {
                    if (++it == (1u << 22) && lane == 0)
                        printf("HANG cta %d pass %u warp %u step %u nxt %u left %u\n", (int)tr, passes, w, k, nxt, left);
                }
            }
#else
            ptx::mbar_wait(&sm.full[k], (uint32_t)(ph >> k) & 1u);
#endif
            q.pv = sm.pv[k];
            q.b0 = sm.pub[k][lane];
            q.b1 = sm.pub[k][lane + 32];
            if (!SMALLP) {
                q.pvp = sm.pvf[k];
                q.f0 = sm.pf[k][lane];
                q.f1 = sm.pf[k][lane + 32];
            } else {
                q.pvp = q.f0 = q.f1 = 0u;
            }
        }
        fwd = false;
        if (q.pv == 0u) {  // zero Schur diagonal: every warp still holding rows leaves at this step
            sm.k0 = k;
            break;
        }
        q.p = p;
        q.k4p2 = 4u * p * p;                // (used by SMALLP only: p < 2^14)
        q.mu32 = (uint32_t)(mu >> 32);
        q.kh = k >> 5;
        q.kl = k & 31;
        q.dk0 = lane == k;
        q.dk1 = lane + 32 == k;
        const bool owner = nxt == k + 1;  // slot 0 is the next pivot row
        if (owner) {
            bi_row<SMALLP>(lv[0], fz[0], q);
            publish(k + 1);  // shifts: the rows after it move down one slot
#ifndef BI_CHAIN_ONLY
            bi_row<SMALLP>(lv[0], fz[0], q);  // (rows past the block's last are stale copies: updating them
            bi_row<SMALLP>(lv[1], fz[1], q);  //  unconditionally measured faster than branching around them)
            bi_row<SMALLP>(lv[2], fz[2], q);
#endif
        } else {
            bi_row<SMALLP>(lv[0], fz[0], q);
            bi_row<SMALLP>(lv[1], fz[1], q);
            bi_row<SMALLP>(lv[2], fz[2], q);
            bi_row<SMALLP>(lv[3], fz[3], q);
        }
    }
    __syncthreads();
    // the last pivot row is published but never consumed inside the loop: check its diagonal here
    if (tid == 0 && sm.k0 == t && t > 0 && sm.pv[t - 1] == 0u) sm.k0 = t - 1;
    __syncthreads();
    const uint32_t k0 = sm.k0;
    if (k0 >= t) break;
    // the first logical column c > k0 whose entry in the reduced row k0 is nonzero -- CTA 0 reads
    // the published row k0, CTA 1 the column-k0 entries of its unpublished rows (= the same row of
    // the transposed Schur complement, times the same D_k0)
    if (!tr) {
        if (w == 0) {
            const bool z0 = lane > k0 && lane < t && sm.pub[k0][lane] != 0u;
            const bool z1 = lane + 32 > k0 && lane + 32 < t && sm.pub[k0][lane + 32] != 0u;
            const uint32_t m0 = __ballot_sync(BI_FULL, z0), m1 = __ballot_sync(BI_FULL, z1);
            if (lane == 0) sm.cmin = m0 ? __ffs(m0) - 1 : (m1 ? 31 + __ffs(m1) : 64u);
        }
    } else {
#pragma unroll
        for (int s = 0; s < 4; ++s) {
            if ((uint32_t)s >= left) break;
            const uint32_t x = bi_red4p(__shfl_sync(BI_FULL, (k0 >> 5) ? lv[s][1] : lv[s][0], k0 & 31), p);
            const uint32_t i = nxt + s;
            if (lane == 0 && x != 0u && i > k0 && i < t) atomicMin(&sm.cmin, i);
        }
    }
    __syncthreads();
    const uint32_t c = sm.cmin;
#ifdef BI_RESTART_DBG
    if (tid == 0) printf("cta %d pass %u k0 %u c %u t %u allow %u\n", (int)tr, passes, k0, c, t, allow_q);
#endif
    if (c >= t || !allow_q || passes > 64) {  // rank deficient (or no column pivots allowed): the guess fails
        if (tid == 0) sm.fail = 1u;
        break;
    }
    __syncthreads();  // every thread has read k0 and c
    if (tid == 0) {   // rotate logical columns k0..c: c moves to k0, the rest keeps its order
        const uint32_t pc = sm.perm[c];
        for (uint32_t j = c; j > k0; --j) sm.perm[j] = sm.perm[j - 1];
        sm.perm[k0] = pc;
        sm.k0 = t;
        sm.cmin = 64u;
    }
    ph ^= (2ull << k0) - 1ull;  // rows 0..k0 were published in this pass (k0 = 63: all bits)
    __syncthreads();
    }  // restart
    BI_STAMP(3);
    if (tid < 64) sm.pcol[tid] = sm.perm[tid];
    __syncthreads();
    // ---- one inverse: D_k = prod_{j<k} pv_j -> 1/D_k and 1/pv_k = D_k / D_{k+1}; plus the I-column
    // scales Dd_j (= D_j on the fast path, 1 after the slow path rescaled them).  Branch-free scans.
    if (w == 0) {
        const double pd = (double)p, pinv = (double)mu * 5.421010862427522e-20;  // mu / 2^64 ~ 1 / p
        const uint32_t e0 = 2 * lane, e1 = 2 * lane + 1;
        const uint32_t v0 = (e0 < t && sm.pv[e0]) ? sm.pv[e0] : 1u, v1 = (e1 < t && sm.pv[e1]) ? sm.pv[e1] : 1u;
        uint32_t inc = bi_mulmod(v0, v1, pd, pinv), suf = inc;
#pragma unroll 1
        for (uint32_t off = 1; off < 32; off <<= 1) {
            const uint32_t o = __shfl_up_sync(BI_FULL, inc, off), u = __shfl_down_sync(BI_FULL, suf, off);
            const uint32_t mi = bi_mulmod(inc, o, pd, pinv), ms = bi_mulmod(suf, u, pd, pinv);
            inc = lane >= off ? mi : inc;
            suf = lane + off < 32 ? ms : suf;
        }
        uint32_t exc = __shfl_up_sync(BI_FULL, inc, 1);
        if (lane == 0) exc = 1u;
        const uint32_t D0 = exc, D1 = bi_mulmod(exc, v0, pd, pinv);
        const uint32_t total = __shfl_sync(BI_FULL, inc, 31);
        const uint32_t tinv = inv_mod_bin(total, p);  // every lane, same input: a uniform loop
        const uint32_t iD0 = bi_mulmod(tinv, suf, pd, pinv);
        const uint32_t sufx = __shfl_down_sync(BI_FULL, suf, 1);
        const uint32_t iD2 = bi_mulmod(tinv, lane == 31 ? 1u : sufx, pd, pinv);
        const uint32_t iD1 = bi_mulmod(iD2, v1, pd, pinv);
        const uint32_t ip0 = bi_mulmod(D0, iD1, pd, pinv), ip1 = bi_mulmod(D1, iD2, pd, pinv);
        const uint32_t s0 = D0, s1 = D1;
        sm.invd[e0] = iD0;
        sm.invp[e0] = ip0;
        sm.Dd[e0] = s0;
        sm.invd[e1] = iD1;
        sm.invp[e1] = ip1;
        sm.Dd[e1] = s1;
    }
    __syncthreads();
    BI_STAMP(4);
    if (tid < 3 * 64) {  // Shoup factors of the three scale vectors, one per thread
        uint32_t* v = tid < 64 ? sm.invd : (tid < 128 ? sm.invp : sm.Dd);
        uint32_t* f = tid < 64 ? sm.invdf : (tid < 128 ? sm.invpf : sm.Ddf);
        f[tid & 63] = shoup_pre(v[tid & 63], p, mu);
    }
    __syncthreads();
    if (!tr) {
        // packed L \ U (logical columns) and inv(L)[i][j] = I[i][j] D_j / D_i
#pragma unroll 1
        for (uint32_t idx = tid; idx < t * t; idx += BI_THREADS) {
            const uint32_t i = t == 64 ? idx >> 6 : idx / t, j = idx - i * t;
            const bool lo = j < i, dg = j == i;
            const uint32_t x = lo ? sm.Ln[i][j] : (dg ? sm.pv[i] : sm.pub[i][j]);
            const uint32_t m = lo ? sm.invp[j] : sm.invd[i], mf = lo ? sm.invpf[j] : sm.invdf[i];
            A[(uint64_t)i * lda + j] = shoup_mul(x, m, mf, p);
            const uint32_t y = shoup_mul(sm.pub[i][j], sm.Dd[j], sm.Ddf[j], p);
            inv[idx] = j <= i ? shoup_mul(y, sm.invd[i], sm.invdf[i], p) : 0u;
        }
        for (uint32_t i = tid; i < t; i += BI_THREADS) {
            Pd[i] = i;
            Qd[i] = sm.pcol[i];
        }
    } else {
        // inv(U)[s][q] = I1[q][s] D_s / pv_q (s <= q): transposed through S, then coalesced stores
#pragma unroll 1
        for (uint32_t idx = tid; idx < 64 * 64; idx += BI_THREADS) {
            const uint32_t q = idx >> 6, s = idx & 63;
            const uint32_t y = shoup_mul(sm.pub[q][s], sm.Dd[s], sm.Ddf[s], p);
            sm.S[s][q] = s <= q ? shoup_mul(y, sm.invp[q], sm.invpf[q], p) : 0u;
        }
        __syncthreads();
        uint32_t* invU = inv + (size_t)t * t;
#pragma unroll 1
        for (uint32_t idx = tid; idx < t * t; idx += BI_THREADS) {
            const uint32_t s = t == 64 ? idx >> 6 : idx / t, q = idx - s * t;
            invU[idx] = sm.S[s][q];
        }
    }
    __syncthreads();
    BI_STAMP(5);
    if (!tr && tid == 0) {
        info->rank = t;
        info->plo = info->phi = info->qlo = info->qhi = 0;
        info->cached = 0;
        if ((seq & SPEC_BIT) && sm.fail) {
            volatile uint32_t* sf = &info->spec_fail;
            if (!*sf) *reinterpret_cast<volatile uint32_t*>(&info->fail_seq) = seq;  // the first failure
            *sf = 1u;
        }
        __threadfence_system();
        *reinterpret_cast<volatile uint32_t*>(&info->seq) = seq;
    }
}

static void bi_dbg_dump(cudaStream_t st) {
    static long long* buf = nullptr;
    if (!buf) {
        FFG_CUDA(cudaMalloc(&buf, 8 * 8));
        FFG_CUDA(cudaMemset(buf, 0, 8 * 8));
        FFG_CUDA(cudaMemcpyToSymbol(g_bi_dbg, &buf, sizeof(buf)));
        return;
    }
    long long h[8];
    FFG_CUDA(cudaStreamSynchronize(st));
    FFG_CUDA(cudaMemcpy(h, buf, sizeof(h), cudaMemcpyDeviceToHost));
    fprintf(stderr, "BI_DBG cycles: pdl wait %lld, staging+cluster %lld, pivot loop %lld, scan %lld, outputs %lld\n",
            h[1] - h[0], h[2] - h[1], h[3] - h[2], h[4] - h[3], h[5] - h[4]);
}

void rr_base_inv_launch(const Blas& b, DView a, uint32_t* Pd, uint32_t* Qd, void* info_dev, uint32_t* inv,
                        uint32_t seq, bool allow_q) {
    const uint32_t t = (uint32_t)a.rows;
    if (t == 0 || t > 64 || a.cols != a.rows) throw Error(FFG_ERR_INTERNAL, "rr_base_inv: block must be square <= 64");
    const size_t smem = sizeof(BiSmem);
    static PerDeviceOnce once;
    once([smem] {
        FFG_CUDA(cudaFuncSetAttribute(rr_base_inv_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        FFG_CUDA(cudaFuncSetAttribute(rr_base_inv_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    });
    BaseInfo* info = static_cast<BaseInfo*>(info_dev);
    b.ws.prof.begin(b.st);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(2);
    cfg.blockDim = dim3(BI_THREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = b.st;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl_enabled() ? 2 : 1;
    static const bool dbg = knob_set("FFG_BI_DBG");
    if (dbg) bi_dbg_dump(b.st);
    // fields below 2^14 take the 32-bit update (FFG_BASE_SMALLP=0: the general kernel everywhere)
    static const bool smallp_on = knob_int("FFG_BASE_SMALLP", 1) != 0;
    const auto kern = (smallp_on && b.F.p < (1u << 14)) ? rr_base_inv_kernel<true> : rr_base_inv_kernel<false>;
    FFG_CUDA(cudaLaunchKernelEx(&cfg, kern, a.d, (uint64_t)a.ld, t, Pd, Qd, info, inv, b.F.p, b.F.mu,
                                seq, (uint32_t)allow_q));
    FFG_CUDA(cudaGetLastError());
    b.ws.prof.end(b.st, PROF_BASE, 2.0 * t * t * 4, 2.0 * t * (double)t * t);
    b.count();
}

}  // namespace ffg
