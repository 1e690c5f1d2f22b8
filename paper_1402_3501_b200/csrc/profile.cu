// profile.cu -- the profile-first exact path for rank-deficient input.
//
// tile_rec (rankrev.hpp:85-183) on a rank-deficient matrix visits ~(n / threshold)^2 base cases
// whose ranks decide every later shape: on the GPU that is one device -> host round trip and a
// dozen small launches per base case (config 4: 64K base cases, ~600 ms).  The same outputs
// follow from the rank profile matrix R_A alone (rpsim.cu, tests/test_profile.py):
//   phase 1  R_A = the pivots of any rank-profile-revealing elimination.  Here: rr_base's own
//            greedy row-major search (rankrev.hpp:40-57) run blocked -- row slabs of <= 32 rows,
//            each searched by one 16-CTA cluster holding the slab's Schur rows in shared memory
//            (columns split over the CTAs, one cluster barrier per pivot), the slabs' reduced
//            pivot rows V applied to the rows below by the tensor-core GEMM in a row-halving
//            recursion (the bottom half is updated once by the top half's pivots, so the
//            trailing matrix is rewritten log2(m / 32) times, not m / 32 times);
//   phase 2  tile_rec's P and Q from R_A on the host (tile_rec_perms);
//   phase 3  the packed L\U: the unique LU without pivoting of B = A[P][:, Q] on its leading
//            rank x rank block (every leading minor is nonzero -- the full-rank speculative
//            schedule of pluq.cu, whose guess cannot fail here), U2 = L1^-1 B12, L2 = B21 U1^-1
//            (ftrsm), and a zero trailing block (rank-deficient tile_rec stores its exhausted
//            Schur complement, which is zero).
// Every phase is exact integer arithmetic, so the outputs are bit-identical to the reference.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <vector>

#include "profile.cuh"
#include "ptx.cuh"

namespace ffg {

namespace {

constexpr uint32_t RP_THREADS = 512;
constexpr uint32_t RP_KMAX = 32;        // slab rows
constexpr uint32_t RP_SMEM_WORDS = 40960;  // slab values per CTA (160 KB)
constexpr uint32_t NONE = 0xFFFFFFFFu;

#ifdef RP_TIMING
__device__ unsigned long long rp_clk[16];
#define RP_T(k) do { unsigned long long t_ = clock64(); rp_acc[k] += t_ - rp_t0; rp_t0 = t_; } while (0)
#else
#define RP_T(k) do { } while (0)
#endif

struct RpPub {
    uint32_t row, col, pad0, pad1;
    uint32_t vals[RP_KMAX];
};

__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t cluster_size() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// a word of CTA `cta`'s shared memory at the address of `local` in this CTA (DSMEM)
__device__ __forceinline__ uint32_t ld_cluster(const uint32_t* local, uint32_t cta) {
    uint32_t a = ptx::smem_u32(local), ra, v;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"(cta));
    asm volatile("ld.shared::cluster.u32 %0, [%1];" : "=r"(v) : "r"(ra) : "memory");
    return v;
}

// The end phase of a slab search: the slab's pivot rows (shared memory S, kk x w per CTA) brought
// to reduced echelon form V (V[t][c_t'] = delta_tt') by a column-parallel back substitution and
// stored, the pivots and the slab's rank reported (CTA 0).
struct RpEnd {
    uint32_t pubT[RP_KMAX][RP_KMAX];
    uint32_t Tn[RP_KMAX][RP_KMAX + 1];
    uint32_t dinv[RP_KMAX];
};
__device__ __forceinline__ void rp_finish(uint32_t* S, RpEnd& E, const uint32_t* piv_row, const uint32_t* piv_col,
                                          uint32_t rho, uint32_t w, uint32_t wv, uint32_t c0, uint32_t cta,
                                          uint32_t row0, uint32_t* __restrict__ prow_out,
                                          uint32_t* __restrict__ pcol_out, uint32_t* __restrict__ V, uint64_t ldv,
                                          BaseInfo* __restrict__ info, uint32_t seq, uint32_t p, uint64_t mu) {
    const uint32_t tid = threadIdx.x;
    auto& pubT = E.pubT;
    auto& Tn = E.Tn;
    auto& dinv = E.dinv;
    // reduced echelon form of the pivot rows: T[t][t'] = S[row_t][c_t'] (upper triangular in pivot
    // order -- each pivot column is zero in every later pivot row), gathered from the columns' owners
    for (uint32_t idx = tid; idx < rho * rho; idx += RP_THREADS) {
        const uint32_t tc = idx / rho, t = idx % rho;
        if (piv_col[tc] / w == cta) pubT[tc][t] = S[piv_row[t] * w + (piv_col[tc] - c0)];
    }
    cluster_sync_all();
    for (uint32_t idx = tid; idx < rho * rho; idx += RP_THREADS) {
        const uint32_t tc = idx / rho, t = idx % rho;
        const uint32_t v = ld_cluster(&pubT[tc][t], piv_col[tc] / w);
        Tn[t][tc] = v ? p - v : 0u;  // negated: the back substitution subtracts
    }
    __syncthreads();
    if (tid < rho) dinv[tid] = inv_mod32(p - Tn[tid][tid], p);
    __syncthreads();
    for (uint32_t j = tid; j < w; j += RP_THREADS) {
        for (int t = (int)rho - 1; t >= 0; --t) {
            uint64_t acc = S[piv_row[t] * w + j];
            for (uint32_t u = t + 1; u < rho; ++u) acc += (uint64_t)Tn[t][u] * S[piv_row[u] * w + j];
            S[piv_row[t] * w + j] = mul_mod(mod_u64(acc, p, mu), dinv[t], p, mu);
        }
    }
    __syncthreads();
    for (uint32_t t = 0; t < rho; ++t)
        for (uint32_t j = tid; j < wv; j += RP_THREADS) V[(uint64_t)t * ldv + c0 + j] = S[piv_row[t] * w + j];
    if (cta == 0) {
        if (tid < rho) {
            prow_out[tid] = row0 + piv_row[tid];
            pcol_out[tid] = piv_col[tid];
        }
        __syncthreads();
        if (tid == 0) {
            __threadfence_system();
            *reinterpret_cast<volatile uint32_t*>(&info->rank) = rho;
            __threadfence_system();
            *reinterpret_cast<volatile uint32_t*>(&info->seq) = seq;
        }
    }
}

// One row slab (kk <= 32 rows starting at global row row0, already reduced by every earlier
// pivot) searched the way rr_base searches (rankrev.hpp:40-57): the next pivot is the first row
// with a nonzero Schur entry, at its first nonzero column.  Earlier pivot columns are exact zeros
// here (the trailing updates zero them), so no column mask is needed.  The cluster's CTAs own
// column ranges [c0, c0 + w); every CTA publishes its first candidate (row, column) and that
// column's entries, and after one cluster barrier every CTA picks the same winner (lowest row,
// then lowest column) and eliminates it from its own columns fraction-free:
//     S_i <- piv * S_i - S_i[c*] * S_{i*}    (rows i > i*; nonzero scaling keeps the zero pattern)
// At the end the slab's pivot rows are brought to reduced echelon form V (V[t][c_t'] = delta_tt')
// by a column-parallel back substitution, so that any later row x is reduced by x - x[C] V.
__global__ void __launch_bounds__(RP_THREADS, 1)
    rp_slab_kernel(const uint32_t* __restrict__ W, uint64_t ldw, uint32_t row0, uint32_t kk, uint32_t n, uint32_t w,
                   uint32_t* __restrict__ prow_out, uint32_t* __restrict__ pcol_out, uint32_t* __restrict__ V,
                   uint64_t ldv, BaseInfo* __restrict__ info, uint32_t seq, uint32_t p, uint64_t mu) {
    extern __shared__ uint4 rp_dyn[];
    uint32_t* S = reinterpret_cast<uint32_t*>(rp_dyn);  // kk x w
    __shared__ RpPub pub[2];
    __shared__ uint32_t candmin[RP_KMAX];
    __shared__ uint32_t mneg[RP_KMAX], mnegsh[RP_KMAX];
    __shared__ uint32_t piv_row[RP_KMAX], piv_col[RP_KMAX];
    __shared__ uint32_t s_istar, s_piv, s_pivsh, s_done;
    __shared__ RpEnd rpend;

    const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint32_t cta = cluster_rank(), ncta = cluster_size();
    const uint32_t c0 = cta * w;
    const uint32_t wv = c0 < n ? min(w, n - c0) : 0u;  // valid columns of this CTA

    for (uint32_t i = 0; i < kk; ++i) {
        const uint32_t* src = W + (uint64_t)(row0 + i) * ldw + c0;
        for (uint32_t j = tid; j < w; j += RP_THREADS) S[i * w + j] = j < wv ? src[j] : 0u;
    }
    if (tid < RP_KMAX) candmin[tid] = NONE;
    __syncthreads();
    // first nonzero column of every row (warp ballots over 32-column groups)
    for (uint32_t i = 0; i < kk; ++i)
        for (uint32_t j0 = warp * 32; j0 < w; j0 += RP_THREADS) {
            const uint32_t b = __ballot_sync(0xffffffffu, S[i * w + j0 + lane] != 0u);
            if (lane == 0 && b) atomicMin(&candmin[i], c0 + j0 + __ffs(b) - 1);
        }
    __syncthreads();

    int iprev = -1;
    uint32_t par = 0, rho = 0;
    for (;;) {
        if (warp == 0) {  // this CTA's first candidate and its column's entries
            const uint32_t cm = (lane < kk && (int)lane > iprev) ? candmin[lane] : NONE;
            const uint32_t b = __ballot_sync(0xffffffffu, cm != NONE);
            const uint32_t fr = b ? (uint32_t)(__ffs(b) - 1) : NONE;
            const uint32_t fc = __shfl_sync(0xffffffffu, cm, b ? fr : 0);
            if (lane == 0) {
                pub[par].row = fr;
                pub[par].col = b ? fc : NONE;
            }
            if (b && lane < kk) pub[par].vals[lane] = S[lane * w + (fc - c0)];
        }
        cluster_sync_all();
        if (warp == 0) {  // the cluster-wide winner: lowest row, then lowest column
            uint64_t key = ~0ull;
            if (lane < ncta)
                key = ((uint64_t)ld_cluster(&pub[par].row, lane) << 32) | ld_cluster(&pub[par].col, lane);
            uint64_t kmin = key;
            for (int o = 16; o; o >>= 1) kmin = min(kmin, __shfl_xor_sync(0xffffffffu, kmin, o));
            const uint32_t istar = (uint32_t)(kmin >> 32), cstar = (uint32_t)kmin;
            if (istar == NONE) {
                if (lane == 0) s_done = 1;
            } else {
                const uint32_t owner = cstar / w;
                const uint32_t v = lane < kk ? ld_cluster(&pub[par].vals[lane], owner) : 0u;
                const uint32_t piv = __shfl_sync(0xffffffffu, v, istar);
                if (lane > istar && lane < kk) {
                    const uint32_t mn = v ? p - v : 0u;
                    mneg[lane] = mn;
                    mnegsh[lane] = shoup_pre(mn, p, mu);
                    if (mn) candmin[lane] = NONE;  // rows left unchanged keep their candidate
                }
                if (lane == 0) {
                    s_done = 0;
                    s_istar = istar;
                    s_piv = piv;
                    s_pivsh = shoup_pre(piv, p, mu);
                    piv_row[rho] = istar;
                    piv_col[rho] = cstar;
                }
            }
        }
        __syncthreads();
        if (s_done) break;
        const uint32_t istar = s_istar, piv = s_piv, pivsh = s_pivsh;
        ++rho;
        for (uint32_t i = istar + 1; i < kk; ++i) {
            const uint32_t mn = mneg[i];
            if (mn == 0) continue;
            const uint32_t mnsh = mnegsh[i];
            for (uint32_t j0 = warp * 32; j0 < w; j0 += RP_THREADS) {
                const uint32_t j = j0 + lane;
                uint32_t x = shoup_mul(S[i * w + j], piv, pivsh, p) + shoup_mul(S[istar * w + j], mn, mnsh, p);
                x = x >= p ? x - p : x;
                S[i * w + j] = x;
                const uint32_t b = __ballot_sync(0xffffffffu, x != 0u);
                if (lane == 0 && b) atomicMin(&candmin[i], c0 + j0 + __ffs(b) - 1);
            }
        }
        __syncthreads();
        iprev = (int)istar;
        par ^= 1u;
    }

    rp_finish(S, rpend, piv_row, piv_col, rho, w, wv, c0, cta, row0, prow_out, pcol_out, V, ldv, info, seq, p, mu);
    cluster_sync_all();  // no CTA leaves while another may still read its shared memory
}

// The same search with the slab in registers (w <= 512 * CPT columns per CTA, <= 32 rows): thread
// tid owns columns tid + 512 q (q < CPT) of every row, so an elimination step is thread-local --
// the pivot row's entry of a column sits in the column's own thread -- and needs only the rows'
// multipliers (shared memory, broadcast).  Per step:
//   * candidates only for the next RP_WIN rows after the last pivot (one ballot per row and
//     warp; a window without any nonzero row slides on without an elimination);
//   * every CTA PUSHES its candidate (row, column) and that column's 32 entries into its slot of
//     every CTA's inbox (st.shared::cluster) before the one cluster barrier of the step, so the
//     winner (lowest row, then lowest column) is picked from local shared memory;
//   * the winner is eliminated from every other row, above and below (fraction-free
//     Gauss-Jordan: S_i <- piv S_i - S_i[c*] S_i*), values kept lazily in [0, 2p): the pivot
//     rows end in reduced echelon form up to their diagonal entries, tracked by warp 0 and
//     divided out when the rows are stored -- no back substitution, no shared-memory slab;
//   * the slab's rank goes to the host mailbox as soon as the search ends, before the rows are
//     scaled and stored (the host enqueues the next launches meanwhile).
struct RpMsg {
    unsigned long long key;   // (row << 32) | column; ~0 = no candidate in the window
    uint32_t vals[RP_KMAX];   // the candidate column's entries (rows 0..31, in [0, 2p))
};
constexpr int RP_WIN = 8;

__device__ __forceinline__ uint32_t map_cluster(uint32_t local_addr, uint32_t cta) {
    uint32_t ra;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(local_addr), "r"(cta));
    return ra;
}
__device__ __forceinline__ void st_cluster_u32(uint32_t local_addr, uint32_t cta, uint32_t v) {
    asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(map_cluster(local_addr, cta)), "r"(v) : "memory");
}
__device__ __forceinline__ void st_cluster_u64(uint32_t local_addr, uint32_t cta, unsigned long long v) {
    asm volatile("st.shared::cluster.u64 [%0], %1;" ::"r"(map_cluster(local_addr, cta)), "l"(v) : "memory");
}
__device__ __forceinline__ void red_min_shared(uint32_t* a, uint32_t v) {
    asm volatile("red.shared::cta.min.u32 [%0], %1;" ::"r"(ptx::smem_u32(a)), "r"(v) : "memory");
}
// x * w mod p up to one p: in [0, 2p) for any 32-bit x (w < p, wp = shoup_pre(w))
__device__ __forceinline__ uint32_t shoup_lazy(uint32_t x, uint32_t w, uint32_t wp, uint32_t p) {
    return x * w - __umulhi(x, wp) * p;
}

template <int CPT>
__global__ void __launch_bounds__(RP_THREADS, 1)
    rp_slab_reg_kernel(const uint32_t* __restrict__ W, uint64_t ldw, uint32_t row0, uint32_t kk, uint32_t n, uint32_t w,
                       uint32_t* __restrict__ prow_out, uint32_t* __restrict__ pcol_out, uint32_t* __restrict__ V,
                       uint64_t ldv, BaseInfo* __restrict__ info, uint32_t seq, uint32_t p, uint64_t mu) {
    constexpr int KK = (int)RP_KMAX;
    __shared__ __align__(16) RpMsg inbox[2][16];
    __shared__ uint32_t cand[2][RP_WIN];
    __shared__ uint32_t stage[RP_KMAX];
    __shared__ __align__(16) uint32_t mneg[RP_KMAX], mnegsh[RP_KMAX];
    __shared__ uint32_t piv_row[RP_KMAX], piv_col[RP_KMAX];
    __shared__ uint32_t dinvs[RP_KMAX], dinvsh[RP_KMAX];
    __shared__ uint32_t s_mode, s_istar, s_piv, s_pivsh;

    const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint32_t cta = cluster_rank(), ncta = cluster_size();
    const uint32_t c0 = cta * w;
    const uint32_t wv = c0 < n ? min(w, n - c0) : 0u;  // valid columns of this CTA
    const uint32_t p2 = 2u * p;
#ifdef RP_TIMING
    unsigned long long rp_acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    unsigned long long rp_t0 = clock64();
#endif

    uint32_t s[KK][CPT];
#pragma unroll
    for (int i = 0; i < KK; ++i)
#pragma unroll
        for (int q = 0; q < CPT; ++q) {
            const uint32_t j = tid + RP_THREADS * q;
            s[i][q] = ((uint32_t)i < kk && j < wv) ? W[(uint64_t)(row0 + i) * ldw + c0 + j] : 0u;
        }
    uint32_t nz[CPT];  // bit i: s[i][q] is nonzero mod p
#pragma unroll
    for (int q = 0; q < CPT; ++q) {
        nz[q] = 0u;
#pragma unroll
        for (int i = 0; i < KK; ++i) nz[q] |= (s[i][q] != 0u ? 1u : 0u) << i;
    }
    if (tid < 2 * RP_WIN) (&cand[0][0])[tid] = NONE;
    __syncthreads();
    RP_T(0);

    int iprev = -1;
    uint32_t par = 0, rho = 0, pivmask = 0;
    uint32_t dg = 1;  // warp 0, lane i: row i's entry at its own pivot column
    for (;;) {
        // offers: this warp's first window row with a nonzero entry, at its first nonzero column
        // (the rows' nonzero patterns are kept as bit masks per column, so no register indexing)
        {
            const uint32_t sh = (uint32_t)(iprev + 1);
#pragma unroll
            for (int slot = 0; slot < RP_WIN; ++slot) {
                const uint32_t r = sh + slot;
                if (r >= (uint32_t)KK) break;
                uint32_t bq[CPT];
                uint32_t any = 0;
#pragma unroll
                for (int q = 0; q < CPT; ++q) {
                    bq[q] = __ballot_sync(0xffffffffu, (nz[q] >> r) & 1u);
                    any |= bq[q];
                }
                if (any) {
                    if (lane == 0) {
                        uint32_t first = 0;
#pragma unroll
                        for (int q = CPT - 1; q >= 0; --q)
                            if (bq[q]) first = RP_THREADS * q + warp * 32 + __ffs(bq[q]) - 1;
                        red_min_shared(&cand[par][slot], c0 + first);
                    }
                    break;  // the CTA's candidate row is this one or an earlier one
                }
            }
        }
        __syncthreads();
        {   // this CTA's candidate (every warp works it out); the owner's warp pushes it
            const uint32_t cm = lane < RP_WIN ? cand[par][lane] : NONE;
            const uint32_t b = __ballot_sync(0xffffffffu, cm != NONE);
            const uint32_t keyaddr = ptx::smem_u32(&inbox[par][cta].key);
            if (b) {
                const uint32_t slot = (uint32_t)(__ffs(b) - 1);
                const uint32_t fr = (uint32_t)(iprev + 1) + slot;
                const uint32_t fc = __shfl_sync(0xffffffffu, cm, slot);
                const uint32_t jl = fc - c0;
                if (warp == ((jl & (RP_THREADS - 1)) >> 5)) {
                    if (lane == (jl & 31u)) {
                        const uint32_t q = jl / RP_THREADS;
#pragma unroll
                        for (int i = 0; i < KK; ++i) {
                            uint32_t v = s[i][0];
#pragma unroll
                            for (int qq = 1; qq < CPT; ++qq) v = q == (uint32_t)qq ? s[i][qq] : v;
                            stage[i] = v;
                        }
                    }
                    __syncwarp();
                    const uint32_t myv = stage[lane];
                    const uint32_t vaddr = ptx::smem_u32(&inbox[par][cta].vals[lane]);
                    for (uint32_t d = 0; d < ncta; ++d) st_cluster_u32(vaddr, d, myv);
                    if (lane < ncta) st_cluster_u64(keyaddr, lane, ((unsigned long long)fr << 32) | fc);
                }
            } else if (warp == 0 && lane < ncta) {
                st_cluster_u64(keyaddr, lane, ~0ull);
            }
            if (tid < RP_WIN) cand[par ^ 1u][tid] = NONE;  // last read before the previous cluster barrier
        }
        RP_T(1);
        cluster_sync_all();
        RP_T(2);
        if (warp == 0) {  // the cluster-wide winner: lowest row, then lowest column
            const unsigned long long key = lane < ncta ? inbox[par][lane].key : ~0ull;
            const uint32_t rowk = (uint32_t)(key >> 32);
            const uint32_t rmin = __reduce_min_sync(0xffffffffu, rowk);
            if (rmin == NONE) {
                if (lane == 0) s_mode = (iprev + RP_WIN + 1 >= (int)kk) ? 2u : 1u;
            } else {
                const uint32_t colk = rowk == rmin ? (uint32_t)key : NONE;
                const uint32_t cmin = __reduce_min_sync(0xffffffffu, colk);
                const uint32_t owner = (uint32_t)(__ffs(__ballot_sync(0xffffffffu, colk == cmin && rowk == rmin)) - 1);
                uint32_t v = inbox[par][owner].vals[lane];
                v = v >= p ? v - p : v;
                const uint32_t istar = rmin;
                const uint32_t piv = __shfl_sync(0xffffffffu, v, istar);
                const uint32_t mn = (lane != istar && v) ? p - v : 0u;  // rows beyond the slab are zero
                mneg[lane] = mn;
                mnegsh[lane] = shoup_pre(mn, p, mu);
                if (lane == istar)
                    dg = piv;
                else if (mn)
                    dg = mul_mod(dg, piv, p, mu);
                if (lane == 0) {
                    s_mode = 0;
                    s_istar = istar;
                    s_piv = piv;
                    s_pivsh = shoup_pre(piv, p, mu);
                    piv_row[rho] = istar;
                    piv_col[rho] = cmin;
                }
            }
        }
        __syncthreads();
        RP_T(3);
        const uint32_t mode = s_mode;
        if (mode == 2u) break;
        par ^= 1u;
        if (mode == 1u) {  // no nonzero row in the window
            iprev += RP_WIN;
            continue;
        }
        const uint32_t istar = s_istar, piv = s_piv, pivsh = s_pivsh;
        uint32_t pr[CPT];
#pragma unroll
        for (int q = 0; q < CPT; ++q) pr[q] = 0u;
#pragma unroll
        for (int i = 0; i < KK; ++i)
            if ((uint32_t)i == istar) {
#pragma unroll
                for (int q = 0; q < CPT; ++q) pr[q] = s[i][q];
            }
#pragma unroll
        for (int g = 0; g < KK / 4; ++g) {
            const uint4 m4 = reinterpret_cast<const uint4*>(mneg)[g];
            const uint4 h4 = reinterpret_cast<const uint4*>(mnegsh)[g];
            const uint32_t mm[4] = {m4.x, m4.y, m4.z, m4.w}, hh[4] = {h4.x, h4.y, h4.z, h4.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                if (mm[e] == 0u) continue;  // the pivot row itself, rows with a zero entry
#pragma unroll
                for (int q = 0; q < CPT; ++q) {
                    const uint32_t x = shoup_lazy(s[4 * g + e][q], piv, pivsh, p) + shoup_lazy(pr[q], mm[e], hh[e], p);
                    const uint32_t y = x >= p2 ? x - p2 : x;
                    s[4 * g + e][q] = y;
                    const uint32_t BIT = 1u << (4 * g + e);
                    nz[q] = (y != 0u && y != p) ? (nz[q] | BIT) : (nz[q] & ~BIT);
                }
            }
        }
        iprev = (int)istar;
        ++rho;
        pivmask |= 1u << istar;
        RP_T(4);
    }
    if (cta == 0 && tid == 0) {  // the rank first: the host's next launches queue up behind this kernel
        __threadfence_system();
        *reinterpret_cast<volatile uint32_t*>(&info->rank) = rho;
        __threadfence_system();
        *reinterpret_cast<volatile uint32_t*>(&info->seq) = seq;
    }
    RP_T(5);
    if (warp == 0) {
        const uint32_t di = (pivmask >> lane) & 1u ? inv_mod32(dg, p) : 0u;
        dinvs[lane] = di;
        dinvsh[lane] = shoup_pre(di, p, mu);
    }
    __syncthreads();
    // pivot rows in discovery order = increasing row order: row i is pivot number popc(pivmask below i)
#pragma unroll
    for (int i = 0; i < KK; ++i) {
        if (!((pivmask >> i) & 1u)) continue;
        const uint32_t t = __popc(pivmask & ((1u << i) - 1u));
        const uint32_t di = dinvs[i], dish = dinvsh[i];
#pragma unroll
        for (int q = 0; q < CPT; ++q) {
            const uint32_t j = tid + RP_THREADS * q;
            if (j < wv) V[(uint64_t)t * ldv + c0 + j] = shoup_mul(s[i][q], di, dish, p);
        }
    }
    if (cta == 0 && tid < rho) {
        prow_out[tid] = row0 + piv_row[tid];
        pcol_out[tid] = piv_col[tid];
    }
    RP_T(6);
#ifdef RP_TIMING
    if (tid == 0 && cta == 0)
        for (int k = 0; k < 8; ++k) rp_clk[k] += rp_acc[k];
#endif
}

// X[i][t] = S[i][cols[t]]  (rows x nc)
__global__ void col_gather_kernel(const uint32_t* __restrict__ S, uint64_t lds, const uint32_t* __restrict__ cols,
                                  uint32_t rows, uint32_t nc, uint32_t* __restrict__ X, uint64_t ldx) {
    const uint64_t total = (uint64_t)rows * nc;
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < total; e += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t i = e / nc, t = e % nc;
        X[i * ldx + t] = S[i * lds + cols[t]];
    }
}

// W[i][j] = A[P[i]][Q[j]]: one row per CTA iteration, staged in shared memory
__global__ void __launch_bounds__(512) gather_pq_kernel(const uint32_t* __restrict__ A, uint64_t lda,
                                                        const uint32_t* __restrict__ P, const uint32_t* __restrict__ Q,
                                                        uint32_t m, uint32_t n, uint32_t* __restrict__ Wd, uint64_t ldw) {
    extern __shared__ uint4 gq_dyn[];
    uint32_t* row = reinterpret_cast<uint32_t*>(gq_dyn);
    for (uint32_t i = blockIdx.x; i < m; i += gridDim.x) {
        const uint32_t* src = A + (uint64_t)P[i] * lda;
        for (uint32_t j = threadIdx.x; j < n; j += blockDim.x) row[j] = src[j];
        __syncthreads();
        uint32_t* dst = Wd + (uint64_t)i * ldw;
        for (uint32_t j = threadIdx.x; j < n; j += blockDim.x) dst[j] = row[Q[j]];
        __syncthreads();
    }
}

int rp_cluster_ctas() {
    static const int c = (int)knob_int("FFG_RP_CLUSTER", 16);
    return std::max(1, std::min(16, c));
}

// device scratch freed on the owning stream on every exit path
struct DevBuf {
    uint32_t* d = nullptr;
    cudaStream_t st = nullptr;
    DevBuf(size_t words, cudaStream_t s) : st(s) {
        if (words) FFG_CUDA(cudaMallocAsync(&d, words * 4, st));
    }
    ~DevBuf() {
        if (d) cudaFreeAsync(d, st);
    }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
};

struct RankProfile {
    const Blas& b;
    DView W;            // working copy, reduced in place
    uint32_t* VB;       // reduced pivot rows, pivot order (rank x n, ld n)
    uint32_t* PR;       // pivot rows / columns, pivot order (device)
    uint32_t* PC;
    size_t total = 0;   // pivots found so far
    uint32_t kk = RP_KMAX, w = 0, ncta = 16;
    BaseInfo* info_host = nullptr;
    BaseInfo* info_dev = nullptr;
    cudaStream_t side = nullptr;
    size_t leaves = 0;
    bool reg_path = false;  // slab in registers (w <= 1024)

    RankProfile(const Blas& bb, DView w_, uint32_t* vb, uint32_t* pr, uint32_t* pc) : b(bb), W(w_), VB(vb), PR(pr), PC(pc) {}

    cudaEvent_t mark(cudaStream_t st) {
        cudaEvent_t e = b.ws.event();
        FFG_CUDA(cudaEventRecord(e, st));
        return e;
    }
    void wait(cudaStream_t st, cudaEvent_t& e) {
        if (e) FFG_CUDA(cudaStreamWaitEvent(st, e, 0));
        e = nullptr;
    }

    size_t leaf(size_t a, size_t rows) {
        const uint32_t seq = (b.ws.base_seq.fetch_add(1) + 1) & ~SPEC_BIT;
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(ncta);
        cfg.blockDim = dim3(RP_THREADS);
        cfg.dynamicSmemBytes = reg_path ? 0 : (size_t)kk * w * 4;
        cfg.stream = b.st;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = ncta;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        b.ws.prof.begin(b.st);
        auto kern = rp_slab_kernel;
        if (reg_path) kern = w <= RP_THREADS ? rp_slab_reg_kernel<1> : rp_slab_reg_kernel<2>;
        FFG_CUDA(cudaLaunchKernelEx(&cfg, kern, (const uint32_t*)W.d, (uint64_t)W.ld, (uint32_t)a,
                                    (uint32_t)rows, (uint32_t)W.cols, w, PR + total, PC + total,
                                    VB + total * W.cols, (uint64_t)W.cols, info_dev, seq, b.F.p, b.F.mu));
        b.ws.prof.end(b.st, PROF_BASE, 2.0 * rows * W.cols * 4, 0.0);
        b.count();
        ++leaves;
        // the slab's rank shapes the next update: spin on the mapped mailbox
        volatile uint32_t* s = &info_host->seq;
        for (uint64_t it = 0; *s != seq; ++it) {
            if (it > (1u << 22)) {
                FFG_CUDA(cudaStreamSynchronize(b.st));
                if (*s != seq) throw Error(FFG_ERR_INTERNAL, "rank profile slab did not report");
                break;
            }
#if defined(__x86_64__) || defined(__i386__)
            __builtin_ia32_pause();
#endif
        }
        std::atomic_thread_fence(std::memory_order_acquire);
        const size_t r = *reinterpret_cast<volatile uint32_t*>(&info_host->rank);
        total += r;
        return r;
    }

    // rows [a, e): the first kk rows are reduced by every earlier pivot, the rest once `pending`
    // (side-stream updates) completes.  Returns the pivots found; with need_v the node's pivot rows
    // VB[o, o + r) end in reduced echelon form over all of them.
    size_t rec(size_t a, size_t e, cudaEvent_t pending, bool need_v) {
        if (e - a <= kk) return leaf(a, e - a);
        const size_t nleaf = (e - a + kk - 1) / kk;
        const size_t mid = a + kk * ((nleaf + 1) / 2);
        const size_t o = total;
        const size_t r1 = rec(a, mid, pending, true);
        wait(b.st, pending);
        cudaEvent_t pend2 = nullptr;
        const size_t n = W.cols;
        if (r1 > 0) {
            // rows [mid, e) -= rows[mid, e)[:, C_top] * V_top; the next slab's rows on the critical
            // stream, the rest on the side stream
            const size_t rows = e - mid;
            DevBuf X(rows * r1, b.st);
            const uint64_t items = (uint64_t)rows * r1;
            col_gather_kernel<<<(unsigned)std::min<uint64_t>(ceil_div(items, 256), 148 * 8), 256, 0, b.st>>>(
                W.d + mid * W.ld, W.ld, PC + o, (uint32_t)rows, (uint32_t)r1, X.d, r1);
            FFG_CUDA(cudaGetLastError());
            b.count();
            const size_t first = std::min<size_t>(kk, rows);
            const DView Vt{VB + o * n, r1, n, n};
            b.gemm(b.F.p - 1, DView{X.d, first, r1, r1}, Vt, 1, W.sub(mid, 0, first, n));
            if (rows > first) {
                cudaEvent_t ready = mark(b.st);
                wait(side, ready);
                Blas sb = b;
                sb.st = side;
                sb.gemm(b.F.p - 1, DView{X.d + first * r1, rows - first, r1, r1}, Vt, 1,
                        W.sub(mid + first, 0, rows - first, n));
                pend2 = mark(side);
                X.st = side;  // freed after the side GEMM (the critical stream's uses precede `ready`)
            }
        }
        const size_t r2 = rec(mid, e, pend2, need_v);
        if (need_v && r1 > 0 && r2 > 0) {
            // V_top -= V_top[:, C_bottom] * V_bottom (reduced echelon over both halves)
            DevBuf Y(r1 * r2, b.st);
            col_gather_kernel<<<(unsigned)std::min<uint64_t>(ceil_div(r1 * r2, 256), 148 * 8), 256, 0, b.st>>>(
                VB + o * n, n, PC + o + r1, (uint32_t)r1, (uint32_t)r2, Y.d, r2);
            FFG_CUDA(cudaGetLastError());
            b.count();
            b.gemm(b.F.p - 1, DView{Y.d, r1, r2, r2}, DView{VB + (o + r1) * n, r2, n, n}, 1,
                   DView{VB + o * n, r1, n, n});
        }
        return r1 + r2;
    }
};

}  // namespace

size_t rank_profile_dev(const Blas& b, DView W, std::vector<uint32_t>& prow, std::vector<uint32_t>& pcol) {
    const size_t m = W.rows, n = W.cols;
    prow.clear();
    pcol.clear();
    if (m == 0 || n == 0) return 0;
    const uint32_t ncta = (uint32_t)std::min<size_t>(rp_cluster_ctas(), ceil_div(n, 32));
    const uint32_t w = (uint32_t)round_up(ceil_div(n, ncta), 32);
    const uint32_t kk = std::min<uint32_t>(RP_KMAX, RP_SMEM_WORDS / w);
    if (kk < 4) throw Error(FFG_ERR_INVALID_DIM, "rank profile: too many columns for the slab kernel");
    static PerDeviceOnce once;
    once([] {
        FFG_CUDA(cudaFuncSetAttribute(rp_slab_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)(RP_SMEM_WORDS * 4)));
        FFG_CUDA(cudaFuncSetAttribute(rp_slab_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
        FFG_CUDA(cudaFuncSetAttribute(rp_slab_reg_kernel<1>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
        FFG_CUDA(cudaFuncSetAttribute(rp_slab_reg_kernel<2>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    });
    const size_t rmax = std::min(m, n);
    DevBuf VB(rmax * n, b.st), PR(rmax, b.st), PC(rmax, b.st);
    RankProfile rp(b, W, VB.d, PR.d, PC.d);
    rp.kk = kk;
    rp.w = w;
    rp.ncta = ncta;
    // FFG_RP_SMEM=1: the shared-memory slab kernel at every width (diagnostics, parity tests)
    const bool smem_only = knob_on("FFG_RP_SMEM");  // per call: tests
    rp.reg_path = !smem_only && w <= 2 * RP_THREADS;
    const int slot = b.ws.acquire_slot();
    if (slot < 0) throw Error(FFG_ERR_INTERNAL, "rank profile: no free mailbox");
    struct SlotGuard {
        Workspace& ws;
        int s;
        ~SlotGuard() { ws.release_slot(s); }
    } guard{b.ws, slot};
    uint32_t* dptr = nullptr;
    rp.info_host = reinterpret_cast<BaseInfo*>(b.ws.mailbox(slot, &dptr));
    rp.info_dev = reinterpret_cast<BaseInfo*>(dptr);
    rp.side = b.ws.stream(400, 1);
    const size_t r = rp.rec(0, m, nullptr, false);
    prow.resize(r);
    pcol.resize(r);
    if (r) {
        FFG_CUDA(cudaMemcpyAsync(prow.data(), PR.d, r * 4, cudaMemcpyDeviceToHost, b.st));
        FFG_CUDA(cudaMemcpyAsync(pcol.data(), PC.d, r * 4, cudaMemcpyDeviceToHost, b.st));
    }
    FFG_CUDA(cudaStreamSynchronize(b.st));
#ifdef RP_TIMING
    {
        unsigned long long h[16];
        FFG_CUDA(cudaMemcpyFromSymbol(h, rp_clk, sizeof(h)));
        fprintf(stderr, "RP_TIMING slabs=%zu cycles/slab: load+offer %llu | publish %llu cluster_sync %llu winner %llu update %llu | dump %llu finish %llu exit %llu\n",
                rp.leaves, h[0] / rp.leaves, h[1] / rp.leaves, h[2] / rp.leaves, h[3] / rp.leaves, h[4] / rp.leaves,
                h[5] / rp.leaves, h[6] / rp.leaves, h[7] / rp.leaves);
        memset(h, 0, sizeof(h));
        FFG_CUDA(cudaMemcpyToSymbol(rp_clk, h, sizeof(h)));
    }
#endif
    static const bool log = knob_set("FFG_PROFILE_LOG");
    if (log) fprintf(stderr, "RANK_PROFILE m=%zu n=%zu rank=%zu slabs=%zu kk=%u ctas=%u\n", m, n, r, rp.leaves, kk, ncta);
    return r;
}

namespace {
thread_local int g_profile_depth = 0;
struct ProfileScope {
    ProfileScope() { ++g_profile_depth; }
    ~ProfileScope() { --g_profile_depth; }
};
}  // namespace
bool profile_first_active() { return g_profile_depth > 0; }

void pluq_from_profile_dev(const Blas& b, DView a, size_t threshold, size_t rank, const uint32_t* prow,
                           const uint32_t* pcol, uint32_t* P, uint32_t* Q, uint32_t* scratch) {
    ProfileScope scope;
    const size_t m = a.rows, n = a.cols;
    tile_rec_perms(m, n, threshold, rank, prow, pcol, P, Q);  // phase 2 (host)
    if (m == 0 || n == 0) return;
    // phase 3: B = A[P][:, Q] into the scratch (ld n)
    DevBuf Pd(m, b.st), Qd(n, b.st);
    FFG_CUDA(cudaMemcpyAsync(Pd.d, P, m * 4, cudaMemcpyHostToDevice, b.st));
    FFG_CUDA(cudaMemcpyAsync(Qd.d, Q, n * 4, cudaMemcpyHostToDevice, b.st));
    const DView B{scratch, m, n, n};
    const size_t smem = n * 4;
    if (smem <= 200 * 1024) {
        static PerDeviceOnce once;
        once([] { FFG_CUDA(cudaFuncSetAttribute(gather_pq_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024)); });
        gather_pq_kernel<<<(unsigned)std::min<size_t>(m, 148 * 2), 512, smem, b.st>>>(a.d, a.ld, Pd.d, Qd.d, (uint32_t)m,
                                                                                     (uint32_t)n, B.d, B.ld);
        FFG_CUDA(cudaGetLastError());
        b.count();
    } else {
        copy_block_dev(b, a, B);
        apply_perm_dev(b, B, 0, 0, Pd.d);
        apply_perm_dev(b, B, 1, 0, Qd.d);
    }
    const size_t r = rank;
    if (r > 0) {
        // leading r x r block: generic rank profile, so tile_rec = LU without pivoting; the
        // speculative schedule is forced (a rest after earlier failed guesses does not apply)
        std::vector<uint32_t> Pl(r), Ql(r);
        const int rest = b.ws.spec_rest;
        b.ws.spec_rest = 0;
        size_t rl = 0;
        try {
            rl = pluq_tile_recursive_dev(b, B.sub(0, 0, r, r), 64, Pl.data(), Ql.data());
        } catch (...) {
            b.ws.spec_rest = rest;
            throw;
        }
        b.ws.spec_rest = rest;
        bool ident = rl == r;
        for (size_t i = 0; ident && i < r; ++i) ident = Pl[i] == i && Ql[i] == i;
        if (!ident) throw Error(FFG_ERR_INTERNAL, "profile-first: the leading block is not in generic rank profile");
        if (n > r) ftrsm_dev(b, 0, 0, 0, B.sub(0, 0, r, r), B.sub(0, r, r, n - r), false);  // U2 = L1^-1 B12
        if (m > r) ftrsm_dev(b, 1, 1, 1, B.sub(0, 0, r, r), B.sub(r, 0, m - r, r), false);  // L2 = B21 U1^-1
    }
    if (m > r && n > r) FFG_CUDA(cudaMemset2DAsync(B.d + r * n + r, n * 4, 0, (n - r) * 4, m - r, b.st));
    copy_block_dev(b, B, a);
}

size_t pluq_profile_first_dev(const Blas& b, DView a, size_t threshold, uint32_t* P, uint32_t* Q) {
    const size_t m = a.rows, n = a.cols;
    ++b.ws.st_profile_first;
    if (m == 0 || n == 0) {
        tile_rec_perms(m, n, threshold, 0, nullptr, nullptr, P, Q);
        return 0;
    }
    DevBuf Wb(m * n, b.st);
    const DView W{Wb.d, m, n, n};
    copy_block_dev(b, a, W);
    std::vector<uint32_t> prow, pcol;
    static const bool log = knob_set("FFG_PROFILE_LOG");
    const auto t0 = std::chrono::steady_clock::now();
    const size_t r = rank_profile_dev(b, W, prow, pcol);  // phase 1 (reduces W)
    const auto t1 = std::chrono::steady_clock::now();
    pluq_from_profile_dev(b, a, threshold, r, prow.data(), pcol.data(), P, Q, Wb.d);
    FFG_CUDA(cudaStreamSynchronize(b.st));  // like every exit of the device entry: outputs final on return
    if (log) {
        const auto t2 = std::chrono::steady_clock::now();
        fprintf(stderr, "PROFILE_FIRST m=%zu n=%zu rank=%zu: rank profile %.2f ms, permutations + LU of the generic block %.2f ms\n",
                m, n, r, std::chrono::duration<double, std::milli>(t1 - t0).count(),
                std::chrono::duration<double, std::milli>(t2 - t1).count());
    }
    return r;
}

bool profile_first_fits(size_t n) {
    const size_t ncta = std::min<size_t>(rp_cluster_ctas(), ceil_div(n, 32));
    const size_t w = round_up(ceil_div(n, ncta), 32);
    return w && RP_SMEM_WORDS / w >= 4;
}

}  // namespace ffg
