// gemm.cu -- exact modular GEMM  C <- alpha*A*B + beta*C (mod p) on tcgen05 tensor cores.
//
// Replaces fgemm_classical / fgemm / pfgemm (blas.hpp:31-103, 220-246, 250-271).
//
// Embedding (the paper's delayed reduction, PAPER.md "fgemm"): every residue
// a < p < 2^26 is split into L = ceil(bits(p-1)/8) unsigned 8-bit limbs,
// a = sum_i 2^(8i) a_i.  Then A*B = sum_s 2^(8s) D_s with the limb-product
// diagonals D_s = sum_{i+j=s} A_i B_j, each computed EXACTLY by kind::i8
// tcgen05.mma with s32 accumulation in TMEM.  The only reduction mod p is in
// the epilogue (one per output entry), fused with alpha/beta and the C update;
// the host splits K into chunks of Field::kmax only when the exact s32 bound
// sum_{i+j=s} max(A_i)max(B_j) * K < 2^31 would be exceeded (never for the
// BASELINE shapes: kmax = 16512 for p = 131071, 34359 for p = 251).
//
// Tile: M = 128 rows (one CTA, cta_group::1), NT output columns.  The B
// operand tile holds the L limb planes of the NT columns stacked along N
// (N' = L*NT <= 256), so one MMA  A_i x [B_0|..|B_{L-1}]  writes diagonals
// i..i+L-1 at TMEM column offset i*NT: L MMAs per K-step cover all L^2 limb
// products, accumulating into (2L-1)*NT <= 512 TMEM columns.
//
// Operands are staged by one conversion pass per call (split kernels below)
// into K-major byte planes that TMA loads with 128-byte swizzle.
#include <cstdio>
#include <cstring>
#include <mutex>

#include "common.cuh"
#include "gemm.cuh"
#include "ptx.cuh"

namespace ffg {

// --------------------------------------------------------------------------- field
Field make_field(uint64_t p) {
    auto prime = [](uint64_t n) {
        if (n < 2) return false;
        for (uint64_t d = 2; d * d <= n; ++d)
            if (n % d == 0) return false;
        return true;
    };
    if (p < 2 || p >= (uint64_t(1) << 26) || !prime(p))
        throw Error(FFG_ERR_CAPACITY, "modulus must be a prime with 2 <= p < 2^26");
    Field F;
    F.p = (uint32_t)p;
    F.mu = ~uint64_t(0) / p;  // floor((2^64-1)/p) == floor(2^64/p) for p not a power of 2 (p=2: off by one, still < 3p)
    uint64_t pm1 = p - 1;
    int L = 1;
    while (L < 4 && (pm1 >> (8 * L)) != 0) ++L;
    F.limbs = L;
    uint64_t ml[4] = {0, 0, 0, 0};
    for (int i = 0; i < L; ++i) ml[i] = std::min<uint64_t>(255, pm1 >> (8 * i));
    uint64_t worst = 1;
    for (int s = 0; s <= 2 * (L - 1); ++s) {
        uint64_t d = 0;
        for (int i = 0; i < L; ++i) {
            int j = s - i;
            if (j >= 0 && j < L) d += ml[i] * ml[j];
        }
        worst = std::max(worst, d);
    }
    F.kmax = ((uint64_t(1) << 31) - 1) / worst;
    uint64_t w = 1 % p;
    for (int s = 0; s < 8; ++s) {
        F.w[s] = (uint32_t)w;
        w = (w << 8) % p;
    }
    return F;
}

// --------------------------------------------------------------------------- configs
template <int L>
struct TileCfg;
template <>
struct TileCfg<1> {
    static constexpr int NT = 256, STAGES = 4;
};
template <>
struct TileCfg<2> {
    static constexpr int NT = 128, STAGES = 3;
};
template <>
struct TileCfg<3> {
    static constexpr int NT = 80, STAGES = 2;
};
template <>
struct TileCfg<4> {
    static constexpr int NT = 64, STAGES = 2;
};

constexpr int BM = 128;  // rows per CTA tile (UMMA M)
constexpr int BK = 128;  // K bytes per stage (one 128-byte swizzle row)
constexpr int GROUP_M = 12;  // 8192^3, L = 3: DRAM reads 2.30 / 2.02 / 2.32 / 3.37 / 5.41 GB at 8 / 12 / 16 / 20 / 32 (the row group's A panel must stay in L2)

int tile_n(int limbs) {
    switch (limbs) {
        case 1: return TileCfg<1>::NT;
        case 2: return TileCfg<2>::NT;
        case 3: return TileCfg<3>::NT;
        default: return TileCfg<4>::NT;
    }
}

template <int L>
struct Smem {
    static constexpr int NT = TileCfg<L>::NT, STAGES = TileCfg<L>::STAGES;
    static constexpr int A_BYTES = L * BM * BK;       // L limb planes of 128 x 128 B
    static constexpr int B_BYTES = L * NT * BK;       // L*NT rows of 128 B
    static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
    static constexpr int BAR_OFF = STAGES * STAGE_BYTES;
    static constexpr int TOTAL = BAR_OFF + 256 + 1024;  // barriers + alignment slack
};

enum EpiMode : uint32_t { EPI_GENERIC = 0, EPI_SUB = 1, EPI_PROD = 2, EPI_ADD = 3 };

struct EpiParams {
    uint32_t mode;     // EPI_SUB: C - AB (alpha = p-1, beta = 1); EPI_PROD: AB (alpha 1, beta 0); EPI_ADD: C + AB
    uint32_t vec_ok;   // C rows 16-byte aligned (C and ldc multiples of 4 words)
    uint32_t vec8_ok;  // C rows 32-byte aligned (C and ldc multiples of 8 words): 256-bit accesses
    uint32_t* C;
    uint64_t ldc;
    uint32_t M, N;
    uint32_t p;
    uint64_t mu;
    uint32_t alpha, beta;
    uint32_t w[8];
    uint32_t kblocks;
    uint32_t m_tiles, n_tiles;
    uint32_t l2_hints;  // TMA loads carry L2 eviction policies (large problems: keep the A panel of a row group)
    uint32_t group_m;   // row blocks per rasterization group
};

// --------------------------------------------------------------------------- epilogue
// 8 warps: TMEM -> registers -> sum_s D_s w_s mod p -> alpha/beta update of C.  `before_wait`
// runs after the C prefetch and before waiting for the accumulator (the direct kernel stages
// its operands there).
template <int L, class TmemFn, class Hook>
__device__ __forceinline__ void epilogue_tile(const EpiParams& ep, TmemFn&& get_tmem, uint64_t* tmem_full,
                                              uint32_t m_blk, uint32_t n_blk, uint32_t warp, uint32_t lane,
                                              Hook&& before_wait, uint32_t phase = 0,
                                              uint64_t* tmem_empty = nullptr) {
    constexpr int NT = TileCfg<L>::NT;
    constexpr int D = 2 * L - 1;
    // warp (4 + e): TMEM lane quarter e & 3, column half e >> 2 (8-column chunks)
    constexpr int PER = NT / 16;                 // chunks per half
    // This thread's C values are read ahead into a ring of GC 8-column chunks (<= 64 registers): the
    // first GC before the accumulator is ready (overlapping the mainloop), chunk ch + GC as soon as
    // chunk ch has been consumed -- a rank-k update with small K and one limb (GF(251), NT = 256) is
    // bound by this read-modify-write of C, and loads issued one chunk at a time left it at the
    // memory latency (~0.5 TB/s over all SMs).  The chunks run as a ROLLED loop over groups of GC:
    // every instruction of an epilogue executes once per tile, so a fully unrolled one (17K SASS
    // instructions for L = 1) spent 60 % of its issue slots waiting for instruction fetches.
    constexpr int GC = L == 1 ? 8 : (PER % 4 == 0 ? 4 : PER);
    constexpr int NG = PER / GC;
    static_assert(PER % GC == 0 && GC * 8 <= 64, "chunk groups");
    const uint32_t e = warp - 4, q = e & 3, half = e >> 2;
    const uint32_t row = m_blk * BM + q * 32 + lane;
    const uint32_t col_first = n_blk * NT + half * PER * 8;
    const bool row_ok = row < ep.M;
    uint32_t* crow = ep.C + (uint64_t)(row_ok ? row : 0) * ep.ldc;
    const bool vec = ep.vec_ok && col_first + PER * 8 <= ep.N;
    // one 256-bit access per 8-column chunk: a warp's 32 rows are 32 different lines either way,
    // and the tag stage of the L1 takes one line per cycle -- half the instructions, half the time
    const bool vec8 = vec && ep.vec8_ok;
    const uint32_t mode = ep.mode, p = ep.p;
    const bool need_c = mode != EPI_PROD;
    uint32_t cpre[GC * 8];
#pragma unroll
    for (int j = 0; j < GC * 8; ++j) cpre[j] = 0u;
    auto load_chunk = [&](uint32_t ch, int slot) {  // chunk ch of this thread's row -> ring slot
        const uint32_t col = col_first + ch * 8;
        uint32_t* dst = cpre + slot * 8;
        if (vec8) {
            uint32_t v[8];
            ptx::ld_global_v8(crow + col, v);
#pragma unroll
            for (int j = 0; j < 8; ++j) dst[j] = v[j];
        } else if (vec) {
            const uint4 a = *reinterpret_cast<const uint4*>(crow + col);
            const uint4 b = *reinterpret_cast<const uint4*>(crow + col + 4);
            dst[0] = a.x, dst[1] = a.y, dst[2] = a.z, dst[3] = a.w;
            dst[4] = b.x, dst[5] = b.y, dst[6] = b.z, dst[7] = b.w;
        } else {
#pragma unroll
            for (int j = 0; j < 8; ++j) dst[j] = col + j < ep.N ? crow[col + j] : 0u;
        }
    };
    if (need_c && row_ok) {  // overlap the C read with the mainloop
#pragma unroll
        for (int c = 0; c < GC; ++c) load_chunk((uint32_t)c, c);
    }
    before_wait();
    ptx::mbar_wait(tmem_full, phase);
    ptx::tc_fence_after();
    const uint32_t tmem = get_tmem();
    const uint32_t t_lane = tmem + ((q * 32) << 16) + half * PER * 8;
    const uint32_t mu32 = (uint32_t)(ep.mu >> 32);  // floor(2^32 / p)
#pragma unroll 1
    for (int g = 0; g < NG; ++g) {
#pragma unroll
        for (int c = 0; c < GC; ++c) {
            const uint32_t ch = (uint32_t)(g * GC + c);
            uint32_t r[D][8];
#pragma unroll
            for (int s2 = 0; s2 < D; ++s2) ptx::tmem_ld8(t_lane + s2 * NT + ch * 8, r[s2]);
            ptx::tmem_ld_wait();
            if (c == GC - 1 && g == NG - 1 && tmem_empty) {  // accumulators read: the next tile's MMAs may start
                ptx::tc_fence_before();
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive(tmem_empty);
            }
            if (!row_ok) continue;
            const uint32_t col = col_first + ch * 8;
            uint32_t cv[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) cv[j] = cpre[c * 8 + j];
            if (need_c && g + 1 < NG) load_chunk(ch + GC, c);
            uint32_t prod[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                if (L == 1) {  // one limb: the accumulator itself (< 2^31), 32-bit Barrett
                    const uint32_t x = r[0][j];
                    const uint32_t t = x - __umulhi(x, mu32) * p;  // < 2p
                    prod[j] = min(t, t - p);
                } else {
                    uint64_t acc = 0;
#pragma unroll
                    for (int s2 = 0; s2 < D; ++s2) acc += (uint64_t)r[s2][j] * ep.w[s2];
                    prod[j] = mod_u64(acc, p, ep.mu);
                }
            }
            uint32_t out[8];
            if (mode == EPI_GENERIC) {
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    uint64_t v = (uint64_t)ep.alpha * prod[j];
                    if (ep.beta) v += (uint64_t)ep.beta * cv[j];
                    out[j] = mod_u64(v, p, ep.mu);
                }
            } else {  // C - AB, AB (cv = 0), C + AB: one add and one conditional subtraction
                const bool sub = mode == EPI_SUB;
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const uint32_t t = cv[j] + (sub ? p - prod[j] : prod[j]);  // < 2p (+1: p - 0)
                    out[j] = min(t, t - p);
                }
            }
            if (vec8) {
                ptx::st_global_v8(crow + col, out);
            } else if (vec) {
                *reinterpret_cast<uint4*>(crow + col) = make_uint4(out[0], out[1], out[2], out[3]);
                *reinterpret_cast<uint4*>(crow + col + 4) = make_uint4(out[4], out[5], out[6], out[7]);
            } else {
#pragma unroll
                for (int j = 0; j < 8; ++j)
                    if (col + j < ep.N) crow[col + j] = out[j];
            }
        }
    }
    ptx::tc_fence_before();
}

// --------------------------------------------------------------------------- the GEMM kernel
template <int L>
__global__ void __launch_bounds__(384, 1)
    modgemm_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
                   const EpiParams ep) {
    using S = Smem<L>;
    constexpr int NT = S::NT, STAGES = S::STAGES;
    constexpr int D = 2 * L - 1;
    constexpr uint32_t TMEM_COLS = 512;
    static_assert(D * NT <= 512, "accumulator diagonals exceed TMEM");
    // two accumulator stages where they fit (one limb: 2 x 256 columns): the next tile's MMAs run
    // while the epilogue drains this one
    constexpr int ACC = 2 * D * NT <= 512 ? 2 : 1;
    static_assert(L * NT <= 256 && (L * NT) % 16 == 0 && NT % 16 == 0, "invalid UMMA N");

    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + S::BAR_OFF);
    uint64_t* empty = full + STAGES;
    uint64_t* tmem_full = empty + STAGES;
    uint64_t* tmem_empty = tmem_full + ACC;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_empty + ACC);
    const uint32_t warp = ptx::warp_id(), lane = ptx::lane_id();

    // Persistent over tiles (grid may be capped below the tile count so that a low-priority
    // GEMM leaves SMs free for the critical path).  Grouped rasterization: a wave covers
    // GROUP_M row-blocks x a few column-blocks.
    const uint32_t tiles = ep.m_tiles * ep.n_tiles;
    auto tile_coords = [&](uint32_t pid, uint32_t& m_blk, uint32_t& n_blk) {
        const uint32_t in_group = ep.group_m * ep.n_tiles;
        const uint32_t first_m = (pid / in_group) * ep.group_m;
        const uint32_t gsize = min(ep.group_m, ep.m_tiles - first_m);
        m_blk = first_m + (pid % in_group) % gsize;
        n_blk = (pid % in_group) / gsize;
    };

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            ptx::mbar_init(&full[s], 1);
            ptx::mbar_init(&empty[s], 1);
        }
        for (int a = 0; a < ACC; ++a) {
            ptx::mbar_init(&tmem_full[a], 1);
            ptx::mbar_init(&tmem_empty[a], 8);  // one arrival per epilogue warp
        }
        ptx::fence_mbar_init();
    }
    if (warp == 0 && lane == 0) {
        ptx::tma_prefetch(&mapA);
        ptx::tma_prefetch(&mapB);
    }
    ptx::pdl_enter();
    if (warp == 2) ptx::tmem_alloc<TMEM_COLS>(tmem_slot);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        // ---------------- TMA producer (runs ahead across tile boundaries)
        if (lane == 0) {
            uint32_t it = 0;
            // a wave of CTAs covers GROUP_M row blocks x a few column blocks and the next wave moves
            // on to the next column blocks: the row group's A panel is re-read by every wave of the
            // group (keep it in L2), a B tile only inside its wave
            const bool hints = ep.l2_hints != 0;
            const uint64_t pol_a = hints ? ptx::l2_policy_evict_last() : 0, pol_b = hints ? ptx::l2_policy_evict_first() : 0;
            for (uint32_t tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
                uint32_t m_blk, n_blk;
                tile_coords(tile, m_blk, n_blk);
                const int32_t a_row0 = (int32_t)(m_blk * BM);
                const int32_t b_row0 = (int32_t)(n_blk * L * NT);
                for (uint32_t kb = 0; kb < ep.kblocks; ++kb, ++it) {
                    const uint32_t s = it % STAGES, ph = (it / STAGES) & 1;
                    ptx::mbar_wait(&empty[s], ph ^ 1);
                    uint8_t* st = smem + s * S::STAGE_BYTES;
                    ptx::mbar_expect_tx(&full[s], S::STAGE_BYTES);
                    if (hints) {
                        for (int i = 0; i < L; ++i)
                            ptx::tma_load_2d_hint(st + i * BM * BK, &mapA, &full[s], (int32_t)(kb * BK),
                                                  a_row0 + i * (int32_t)(ep.m_tiles * BM), pol_a);
                        ptx::tma_load_2d_hint(st + S::A_BYTES, &mapB, &full[s], (int32_t)(kb * BK), b_row0, pol_b);
                    } else {
                        for (int i = 0; i < L; ++i)
                            ptx::tma_load_2d(st + i * BM * BK, &mapA, &full[s], (int32_t)(kb * BK),
                                             a_row0 + i * (int32_t)(ep.m_tiles * BM));
                        ptx::tma_load_2d(st + S::A_BYTES, &mapB, &full[s], (int32_t)(kb * BK), b_row0);
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer (single thread)
        if (lane == 0) {
            constexpr uint32_t IDESC_FULL = ptx::idesc_u8(BM, L * NT);
            constexpr uint32_t IDESC_HEAD = ptx::idesc_u8(BM, (L > 1 ? (L - 1) : 1) * NT);
            constexpr uint32_t IDESC_TAIL = ptx::idesc_u8(BM, NT);
            uint32_t it = 0, t = 0;
            for (uint32_t tile = blockIdx.x; tile < tiles; tile += gridDim.x, ++t) {
                const uint32_t as = t % ACC, aph = (t / ACC) & 1;
                const uint32_t acc = tmem + as * (D * NT);
                ptx::mbar_wait(&tmem_empty[as], aph ^ 1);  // this stage's previous accumulators drained
                ptx::tc_fence_after();
                for (uint32_t kb = 0; kb < ep.kblocks; ++kb, ++it) {
                    const uint32_t s = it % STAGES, ph = (it / STAGES) & 1;
                    ptx::mbar_wait(&full[s], ph);
                    ptx::tc_fence_after();
                    const uint32_t a_base = ptx::smem_u32(smem + s * S::STAGE_BYTES);
                    const uint32_t b_base = a_base + S::A_BYTES;
#pragma unroll
                    for (int kk = 0; kk < BK / 32; ++kk) {
                        const uint64_t bdesc = ptx::desc_kmajor_sw128(b_base + kk * 32);
#pragma unroll
                        for (int i = 0; i < L; ++i) {
                            const uint64_t adesc = ptx::desc_kmajor_sw128(a_base + i * BM * BK + kk * 32);
                            if (kb != 0 || kk != 0) {
                                ptx::mma_i8(acc + i * NT, adesc, bdesc, IDESC_FULL, 1);
                            } else if (i == 0) {
                                ptx::mma_i8(acc, adesc, bdesc, IDESC_FULL, 0);
                            } else {
                                // first K-step: diagonals i..i+L-2 already hold data, i+L-1 is fresh
                                ptx::mma_i8(acc + i * NT, adesc, bdesc, IDESC_HEAD, 1);
                                const uint64_t btail =
                                    ptx::desc_kmajor_sw128(b_base + (L - 1) * NT * BK + kk * 32);
                                ptx::mma_i8(acc + (i + L - 1) * NT, adesc, btail, IDESC_TAIL, 0);
                            }
                        }
                    }
                    ptx::mma_commit(&empty[s]);  // frees the smem stage when these MMAs retire
                }
                ptx::mma_commit(&tmem_full[as]);
            }
        }
        __syncwarp();
    } else if (warp >= 4) {
        uint32_t t = 0;
        for (uint32_t tile = blockIdx.x; tile < tiles; tile += gridDim.x, ++t) {
            uint32_t m_blk, n_blk;
            tile_coords(tile, m_blk, n_blk);
            const uint32_t as = t % ACC, aph = (t / ACC) & 1;
            epilogue_tile<L>(ep, [&] { return tmem + as * (D * NT); }, &tmem_full[as], m_blk, n_blk, warp, lane,
                             [] {}, aph, &tmem_empty[as]);
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 2) ptx::tmem_dealloc<TMEM_COLS>(tmem);
}

// --------------------------------------------------------------------------- direct kernel (K <= 128 KB)
// Small-K GEMMs (the Schur updates and TRSM splits of the lower recursion levels: K = 128 or
// 256) are latency-bound; there the separate split launch and its round trip of limb planes
// through HBM cost as much as the GEMM.  This kernel stages the WHOLE K extent of its tile
// directly: all 12 warps read the u32 operands, cut them into limb bytes and store them in the
// same SW128 K-major layout TMA would produce, then one thread issues every MMA.  Requires C
// not to alias A or B (other CTAs' C writes would race with this CTA's operand reads).
struct DirectArgs {
    const uint32_t* A;
    uint64_t lda;
    const uint32_t* B;
    uint64_t ldb;
    uint32_t K;
    uint32_t a_vec;  // A rows 16-byte aligned: A and lda multiples of 4 words
    unsigned long long* dbg;  // diagnostics: %globaltimer stamps of CTA 0 (null = off)
};
__device__ __forceinline__ unsigned long long gtime() { return clock64(); }
__device__ __forceinline__ unsigned long long gns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

template <int L, int KB>
struct DirectSmem {
    static constexpr int NT = TileCfg<L>::NT;
    static constexpr int A_PLANE = BM * BK;               // one limb plane of one K block
    static constexpr int A_BYTES = KB * L * A_PLANE;
    static constexpr int B_BLOCK = L * NT * BK;           // the L stacked planes of one K block
    static constexpr int C_OFF = A_BYTES + KB * B_BLOCK;  // C tile prefetched by cp.async
    static constexpr int CS = NT + 4;                     // C row stride in words (16-byte rows)
    static constexpr int BAR_OFF = C_OFF + BM * CS * 4;
    static constexpr int TOTAL = BAR_OFF + 64 + 1024;
    static constexpr bool FITS = TOTAL <= 227 * 1024;
};

__device__ __forceinline__ uint32_t pack_limb(uint32_t v0, uint32_t v1, uint32_t v2, uint32_t v3, int sh) {
    return ((v0 >> sh) & 0xFF) | (((v1 >> sh) & 0xFF) << 8) | (((v2 >> sh) & 0xFF) << 16) | (((v3 >> sh) & 0xFF) << 24);
}

// byte l of each of v0..v3, packed little-endian (three byte permutes)
template <int l>
__device__ __forceinline__ uint32_t limb_bytes(uint32_t v0, uint32_t v1, uint32_t v2, uint32_t v3) {
    const uint32_t lo = __byte_perm(v0, v1, l | ((l + 4) << 4));
    const uint32_t hi = __byte_perm(v2, v3, l | ((l + 4) << 4));
    return __byte_perm(lo, hi, 0x5410);
}

__device__ __forceinline__ uint32_t sw128(uint32_t row, uint32_t kq) {  // byte offset of k = 4 kq in a row
    return row * 128 + ((((kq >> 2) ^ row) & 7) << 4) + ((kq & 3) << 2);
}

// Code size matters here: each CTA runs this kernel body once, so straight-line unrolled code
// is fetched cold from L2 (~6 KB L0 / 32 KB L1.5 I-cache).  Loops are therefore rolled, with
// 4 loads in flight per thread and the C tile prefetched by cp.async into shared memory.
template <int L, int KB>
__global__ void __launch_bounds__(384, 1)
    modgemm_direct_kernel(const DirectArgs da, const EpiParams ep) {
    using S = DirectSmem<L, KB>;
    constexpr int NT = S::NT, D = 2 * L - 1;
    constexpr uint32_t TMEM_COLS = 512;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint32_t* Cs = reinterpret_cast<uint32_t*>(smem + S::C_OFF);
    uint64_t* tmem_full = reinterpret_cast<uint64_t*>(smem + S::BAR_OFF);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_full + 1);
    const uint32_t warp = ptx::warp_id(), lane = ptx::lane_id(), tid = threadIdx.x;
    const uint32_t m_blk = blockIdx.x % ep.m_tiles, n_blk = blockIdx.x / ep.m_tiles;
    const bool need_c = ep.mode != EPI_PROD;
    const bool dbg = da.dbg && blockIdx.x == 0 && tid == 0;
    if (dbg) {
        da.dbg[0] = gtime();
        da.dbg[4] = gns();
    }

    if (tid == 0) {
        ptx::mbar_init(tmem_full, 1);
        ptx::fence_mbar_init();
    }
    ptx::pdl_enter();
    if (warp == 2) ptx::tmem_alloc<TMEM_COLS>(tmem_slot);
    // epilogue warps: C prefetch for the rows / columns they will write
    constexpr uint32_t PER = NT / 16;  // 8-column chunks per epilogue thread
    const uint32_t e = warp - 4, q = e & 3, half = e >> 2;
    const uint32_t r_in = q * 32 + lane, row = m_blk * BM + r_in;
    const uint32_t c_in = half * PER * 8, col0 = n_blk * NT + c_in;
    const bool row_ok = row < ep.M;
    uint32_t* crow = ep.C + (uint64_t)(row_ok ? row : 0) * ep.ldc;
    uint32_t* cs_row = Cs + r_in * S::CS + c_in;
    const bool vec = ep.vec_ok && col0 + PER * 8 <= ep.N;
    if (warp >= 4 && need_c && row_ok) {
        if (vec) {
            for (uint32_t i = 0; i < PER * 2; ++i) ptx::cp_async16(cs_row + 4 * i, crow + col0 + 4 * i);
        } else {
            for (uint32_t j = 0; j < PER * 8; ++j)
                if (col0 + j < ep.N) ptx::cp_async4(cs_row + j, crow + col0 + j);
        }
        ptx::cp_async_commit();
    }

    // ---- stage the operands' limb planes (all 12 warps).  Rows >= M of A and columns >= N of
    // B are left unstaged: they only feed output rows / columns that are never written.  A's
    // k >= K entries are zero, which also neutralises whatever B holds there.
    const uint32_t smem_s = ptx::smem_u32(smem);
    const uint32_t a_rows = min((uint32_t)BM, ep.M - m_blk * BM);
    const uint32_t b_cols = min((uint32_t)NT, ep.N - n_blk * NT);
    const uint32_t kq_live = (da.K + 3) / 4;  // 4-element groups of B that hold data
#pragma unroll 1
    for (uint32_t kb = 0; kb < (uint32_t)KB; ++kb) {
        const uint32_t ablk = smem_s + kb * L * S::A_PLANE;
#pragma unroll 1
        for (uint32_t base = tid; base < a_rows * 32; base += 4 * 384) {
            uint4 v[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {  // A: row r, k = 4 (it & 31) .. + 3 of this K block
                const uint32_t it = base + u * 384, r = it >> 5, k = kb * BK + (it & 31) * 4;
                v[u] = make_uint4(0, 0, 0, 0);
                if (it < a_rows * 32) {
                    const uint32_t* src = da.A + (uint64_t)(m_blk * BM + r) * da.lda + k;
                    if (da.a_vec && k + 3 < da.K) {
                        v[u] = *reinterpret_cast<const uint4*>(src);
                    } else {
                        v[u].x = k < da.K ? src[0] : 0u;
                        v[u].y = k + 1 < da.K ? src[1] : 0u;
                        v[u].z = k + 2 < da.K ? src[2] : 0u;
                        v[u].w = k + 3 < da.K ? src[3] : 0u;
                    }
                }
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const uint32_t it = base + u * 384;
                if (it < a_rows * 32) {
                    const uint32_t off = ablk + sw128(it >> 5, it & 31);
                    ptx::st_shared_u32(off, limb_bytes<0>(v[u].x, v[u].y, v[u].z, v[u].w));
                    if (L > 1) ptx::st_shared_u32(off + S::A_PLANE, limb_bytes<1>(v[u].x, v[u].y, v[u].z, v[u].w));
                    if (L > 2) ptx::st_shared_u32(off + 2 * S::A_PLANE, limb_bytes<2>(v[u].x, v[u].y, v[u].z, v[u].w));
                    if (L > 3) ptx::st_shared_u32(off + 3 * S::A_PLANE, limb_bytes<3>(v[u].x, v[u].y, v[u].z, v[u].w));
                }
            }
        }
        const uint32_t bblk = smem_s + S::A_BYTES + kb * S::B_BLOCK;
        const uint32_t kq_n = min(32u, kq_live > kb * 32 ? kq_live - kb * 32 : 0u);
#pragma unroll 1
        for (uint32_t base = tid; base < b_cols * kq_n; base += 4 * 384) {
            uint32_t v[4][4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {  // B: column nn, k = 4 kq .. + 3 (rows of B)
                const uint32_t it = base + u * 384, nn = it % b_cols, k = kb * BK + (it / b_cols) * 4;
                const bool ok = it < b_cols * kq_n;
                const uint32_t* src = da.B + (uint64_t)k * da.ldb + n_blk * NT + nn;
#pragma unroll
                for (int t = 0; t < 4; ++t) v[u][t] = ok && k + t < da.K ? src[(uint64_t)t * da.ldb] : 0u;
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const uint32_t it = base + u * 384;
                if (it < b_cols * kq_n) {
                    const uint32_t nn = it % b_cols, kq = it / b_cols;
                    const uint32_t off = bblk + sw128(nn, kq);  // plane l at row l*NT + nn (NT % 8 == 0)
                    ptx::st_shared_u32(off, limb_bytes<0>(v[u][0], v[u][1], v[u][2], v[u][3]));
                    if (L > 1) ptx::st_shared_u32(off + NT * BK, limb_bytes<1>(v[u][0], v[u][1], v[u][2], v[u][3]));
                    if (L > 2) ptx::st_shared_u32(off + 2 * NT * BK, limb_bytes<2>(v[u][0], v[u][1], v[u][2], v[u][3]));
                    if (L > 3) ptx::st_shared_u32(off + 3 * NT * BK, limb_bytes<3>(v[u][0], v[u][1], v[u][2], v[u][3]));
                }
            }
        }
    }
    ptx::fence_proxy_async_smem();
    ptx::tc_fence_before();
    __syncthreads();  // operands staged, TMEM allocated, barrier initialised
    ptx::tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    if (dbg) da.dbg[1] = gtime();

    if (warp == 1 && lane == 0) {
        // ---- all MMAs of the tile (same diagonal scheme as modgemm_kernel)
        constexpr uint32_t IDESC_FULL = ptx::idesc_u8(BM, L * NT);
        constexpr uint32_t IDESC_HEAD = ptx::idesc_u8(BM, (L > 1 ? (L - 1) : 1) * NT);
        constexpr uint32_t IDESC_TAIL = ptx::idesc_u8(BM, NT);
#pragma unroll 1
        for (uint32_t kb = 0; kb < (uint32_t)KB; ++kb) {
            const uint32_t a_base = ptx::smem_u32(smem + kb * L * S::A_PLANE);
            const uint32_t b_base = ptx::smem_u32(smem + S::A_BYTES + kb * S::B_BLOCK);
#pragma unroll 1
            for (uint32_t kk = 0; kk < BK / 32; ++kk) {
                const uint64_t bdesc = ptx::desc_kmajor_sw128(b_base + kk * 32);
#pragma unroll
                for (int i = 0; i < L; ++i) {
                    const uint64_t adesc = ptx::desc_kmajor_sw128(a_base + i * S::A_PLANE + kk * 32);
                    if (kb != 0 || kk != 0) {
                        ptx::mma_i8(tmem + i * NT, adesc, bdesc, IDESC_FULL, 1);
                    } else if (i == 0) {
                        ptx::mma_i8(tmem, adesc, bdesc, IDESC_FULL, 0);
                    } else {
                        ptx::mma_i8(tmem + i * NT, adesc, bdesc, IDESC_HEAD, 1);
                        const uint64_t btail = ptx::desc_kmajor_sw128(b_base + (L - 1) * NT * BK + kk * 32);
                        ptx::mma_i8(tmem + (i + L - 1) * NT, adesc, btail, IDESC_TAIL, 0);
                    }
                }
            }
        }
        ptx::mma_commit(tmem_full);
    } else if (warp >= 4) {
        // ---- epilogue: rolled over 8-column chunks, C from shared memory
        if (need_c && row_ok) ptx::cp_async_wait_all();
        ptx::mbar_wait(tmem_full, 0);
        ptx::tc_fence_after();
        if (warp == 4 && lane == 0 && da.dbg && blockIdx.x == 0) da.dbg[2] = gtime();
        const uint32_t t_lane = tmem + ((q * 32) << 16) + c_in;
        // chunks past N and warps whose 32 rows are all past M have nothing to write (uniform
        // per warp, so the warp-collective TMEM loads can be skipped with them)
        const uint32_t n_ch = m_blk * BM + q * 32 >= ep.M ? 0u
                              : col0 >= ep.N               ? 0u
                                                           : min(PER, (ep.N - col0 + 7) / 8);
#pragma unroll 1
        for (uint32_t ch = 0; ch < n_ch; ++ch) {
            uint32_t r[D][8];
#pragma unroll
            for (int s2 = 0; s2 < D; ++s2) ptx::tmem_ld8(t_lane + s2 * NT + ch * 8, r[s2]);
            ptx::tmem_ld_wait();
            if (!row_ok) continue;
            const uint32_t col = col0 + ch * 8;
            uint32_t cv[8];
            if (need_c) {
                const uint4 a = ptx::ld_shared_v4(ptx::smem_u32(cs_row + ch * 8));
                const uint4 b = ptx::ld_shared_v4(ptx::smem_u32(cs_row + ch * 8 + 4));
                cv[0] = a.x, cv[1] = a.y, cv[2] = a.z, cv[3] = a.w, cv[4] = b.x, cv[5] = b.y, cv[6] = b.z, cv[7] = b.w;
            }
            uint32_t out[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                uint64_t acc = 0;
#pragma unroll
                for (int s2 = 0; s2 < D; ++s2) acc += (uint64_t)r[s2][j] * ep.w[s2];
                const uint32_t prod = mod_u64(acc, ep.p, ep.mu);
                if (ep.mode == EPI_SUB) {
                    out[j] = cv[j] >= prod ? cv[j] - prod : cv[j] + ep.p - prod;
                } else if (ep.mode == EPI_PROD) {
                    out[j] = prod;
                } else {
                    uint64_t t = (uint64_t)ep.alpha * prod;
                    if (ep.beta) t += (uint64_t)ep.beta * cv[j];
                    out[j] = mod_u64(t, ep.p, ep.mu);
                }
            }
            if (vec) {
                *reinterpret_cast<uint4*>(crow + col) = make_uint4(out[0], out[1], out[2], out[3]);
                *reinterpret_cast<uint4*>(crow + col + 4) = make_uint4(out[4], out[5], out[6], out[7]);
            } else {
#pragma unroll
                for (int j = 0; j < 8; ++j)
                    if (col + j < ep.N) crow[col + j] = out[j];
            }
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (dbg) {
        da.dbg[3] = gtime();
        da.dbg[5] = gns();
    }
    if (warp == 2) ptx::tmem_dealloc<TMEM_COLS>(tmem);
}

// --------------------------------------------------------------------------- limb split (one launch)
// Blocks [0, a_blocks): A (M x K view) -> planes[l][Mp][Kp] (K-major, no transpose), one
//   thread = 4 consecutive k of one row, 1024 (row, k-quad) items per block.
// Blocks [a_blocks, ...): B (K x N view) -> rows (n/NT)*L*NT + l*NT + n%NT of Kp bytes
//   (K-major), through a 64(k) x 64(n) shared-memory transpose.
struct SplitArgs {
    const uint32_t* A;
    uint64_t lda;
    uint32_t M, K, Mp, Kp;
    uint8_t* outA;
    const uint32_t* B;
    uint64_t ldb;
    uint32_t N, Np;
    uint8_t* outB;
    int L, NT;
    uint32_t a_blocks, b_kblocks;
    uint32_t a_vec;  // A rows 16-byte aligned (A and lda multiples of 4 words): vector loads
};


__global__ void __launch_bounds__(256) split_kernel(const SplitArgs a) {
    __shared__ uint32_t tile[64][65];
    ptx::pdl_enter();
    if (blockIdx.x < a.a_blocks) {
        // 16 consecutive k of one row per thread: four 16-byte loads in flight, one 16-byte store
        // per limb plane
        const uint32_t kh_per_row = a.Kp >> 4;
        const uint64_t item = (uint64_t)blockIdx.x * 256 + threadIdx.x;
        const uint32_t m = (uint32_t)(item / kh_per_row), kh = (uint32_t)(item % kh_per_row), k = kh * 16;
        if (m >= a.Mp) return;
        uint4 v[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            v[q] = make_uint4(0, 0, 0, 0);
            const uint32_t kk = k + 4 * q;
            if (m < a.M) {
                const uint32_t* row = a.A + (uint64_t)m * a.lda + kk;
                if (a.a_vec && kk + 3 < a.K) {
                    v[q] = *reinterpret_cast<const uint4*>(row);
                } else {
                    v[q].x = kk < a.K ? row[0] : 0u;
                    v[q].y = kk + 1 < a.K ? row[1] : 0u;
                    v[q].z = kk + 2 < a.K ? row[2] : 0u;
                    v[q].w = kk + 3 < a.K ? row[3] : 0u;
                }
            }
        }
        for (int l = 0; l < a.L; ++l) {
            uint4 o;
            o.x = pack_limb(v[0].x, v[0].y, v[0].z, v[0].w, 8 * l);
            o.y = pack_limb(v[1].x, v[1].y, v[1].z, v[1].w, 8 * l);
            o.z = pack_limb(v[2].x, v[2].y, v[2].z, v[2].w, 8 * l);
            o.w = pack_limb(v[3].x, v[3].y, v[3].z, v[3].w, 8 * l);
            *reinterpret_cast<uint4*>(a.outA + ((uint64_t)l * a.Mp + m) * a.Kp + k) = o;
        }
        return;
    }
    const uint32_t bid = blockIdx.x - a.a_blocks;
    const uint32_t k0 = (bid % a.b_kblocks) * 64, n0 = (bid / a.b_kblocks) * 64;
    const uint32_t tx = threadIdx.x & 63, ty = threadIdx.x >> 6;
    {
        uint32_t v[16];  // all 16 loads of the thread in flight
#pragma unroll
        for (int q = 0; q < 16; ++q) {
            const uint32_t k = k0 + ty + 4 * q, n = n0 + tx;
            v[q] = (k < a.K && n < a.N) ? a.B[(uint64_t)k * a.ldb + n] : 0u;
        }
#pragma unroll
        for (int q = 0; q < 16; ++q) tile[ty + 4 * q][tx] = v[q];
    }
    __syncthreads();
    // each item: 16 consecutive k of one column n, one limb plane -> one 16-byte store
    for (uint32_t idx = threadIdx.x; idx < 64u * 4u * (uint32_t)a.L; idx += blockDim.x) {
        const uint32_t g = idx & 3, nn = (idx >> 2) & 63, l = idx >> 8;
        const uint32_t n = n0 + nn, kb = k0 + 16 * g;
        if (n >= a.Np || kb >= a.Kp) continue;
        uint4 o;
        const uint32_t r0 = 16 * g;
        o.x = pack_limb(tile[r0 + 0][nn], tile[r0 + 1][nn], tile[r0 + 2][nn], tile[r0 + 3][nn], 8 * l);
        o.y = pack_limb(tile[r0 + 4][nn], tile[r0 + 5][nn], tile[r0 + 6][nn], tile[r0 + 7][nn], 8 * l);
        o.z = pack_limb(tile[r0 + 8][nn], tile[r0 + 9][nn], tile[r0 + 10][nn], tile[r0 + 11][nn], 8 * l);
        o.w = pack_limb(tile[r0 + 12][nn], tile[r0 + 13][nn], tile[r0 + 14][nn], tile[r0 + 15][nn], 8 * l);
        const uint64_t orow = (uint64_t)(n / a.NT) * a.L * a.NT + (uint64_t)l * a.NT + (n % a.NT);
        *reinterpret_cast<uint4*>(a.outB + orow * a.Kp + kb) = o;
    }
}

// --------------------------------------------------------------------------- CUDA-core path for small GEMMs
// C <- alpha*A*B + beta*C with 64x64 tiles, 256 threads x (4x4) outputs, exact u64
// accumulation (products < 2^52; folded mod p every 2048 terms).  One launch, no limb
// staging: used when the problem is too small to amortize split + tensor-core launches.
constexpr int SG_T = 64, SG_K = 32;
__global__ void __launch_bounds__(256) modgemm_simt_kernel(const uint32_t* __restrict__ A, uint64_t lda,
                                                          const uint32_t* __restrict__ B, uint64_t ldb,
                                                          uint32_t* __restrict__ C, uint64_t ldc, uint32_t M,
                                                          uint32_t N, uint32_t K, uint32_t alpha, uint32_t beta,
                                                          uint32_t p, uint64_t mu) {
    __shared__ uint32_t As[SG_K][SG_T + 1];  // transposed: As[k][m]
    __shared__ uint32_t Bs[SG_K][SG_T];
    ptx::pdl_enter();
    const uint32_t m0 = blockIdx.y * SG_T, n0 = blockIdx.x * SG_T;
    const uint32_t tx = threadIdx.x & 15, ty = threadIdx.x >> 4;  // 16 x 16 threads, 4 x 4 outputs each
    uint64_t acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = 0;
    uint32_t since_fold = 0;
    for (uint32_t k0 = 0; k0 < K; k0 += SG_K) {
        for (uint32_t idx = threadIdx.x; idx < SG_T * SG_K; idx += 256) {
            const uint32_t r = idx / SG_K, c = idx % SG_K;  // A tile: rows m, cols k
            const uint32_t m = m0 + r, k = k0 + c;
            As[c][r] = (m < M && k < K) ? A[(uint64_t)m * lda + k] : 0u;
            const uint32_t rb = idx / SG_T, cb = idx % SG_T;  // B tile: rows k, cols n
            const uint32_t kb = k0 + rb, n = n0 + cb;
            Bs[rb][cb] = (kb < K && n < N) ? B[(uint64_t)kb * ldb + n] : 0u;
        }
        __syncthreads();
#pragma unroll 8
        for (int kk = 0; kk < SG_K; ++kk) {
            uint32_t a[4], b[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) a[i] = As[kk][ty * 4 + i];
#pragma unroll
            for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx * 4 + j];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] += (uint64_t)a[i] * b[j];
        }
        since_fold += SG_K;
        if (since_fold >= 2048) {
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = mod_u64(acc[i][j], p, mu);
            since_fold = 0;
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const uint32_t m = m0 + ty * 4 + i;
        if (m >= M) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const uint32_t n = n0 + tx * 4 + j;
            if (n >= N) continue;
            uint32_t& c = C[(uint64_t)m * ldc + n];
            uint64_t v = (uint64_t)alpha * mod_u64(acc[i][j], p, mu);
            if (beta) v += (uint64_t)beta * c;
            c = mod_u64(v, p, mu);
        }
    }
}

// C <- beta*C (alpha == 0 or K == 0 path, blas.hpp:39-51)
__global__ void scale_kernel(uint32_t* C, uint64_t ldc, uint32_t M, uint32_t N, uint32_t beta, uint32_t p,
                             uint64_t mu) {
    ptx::pdl_enter();
    const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x, i = blockIdx.y;
    if (i < M && j < N) {
        uint32_t& c = C[(uint64_t)i * ldc + j];
        c = beta == 0 ? 0u : (beta == 1 ? c : mul_mod(beta, c, p, mu));
    }
}

// --------------------------------------------------------------------------- host side
namespace {

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn encode_fn() {
    static EncodeFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeFn>(f);
    });
    if (!fn) throw Error(FFG_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    return fn;
}

CUtensorMap make_map(const uint8_t* base, uint64_t inner_bytes, uint64_t rows, uint32_t box_rows) {
    CUtensorMap m;
    cuuint64_t dims[2] = {inner_bytes, rows};
    cuuint64_t strides[1] = {inner_bytes};
    cuuint32_t box[2] = {(cuuint32_t)BK, box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<uint8_t*>(base), dims, strides, box,
                             estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw Error(FFG_ERR_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
    return m;
}

EpiParams make_ep(const Field& F, uint32_t alpha, uint32_t beta, DView C) {
    EpiParams ep{};
    ep.C = C.d;
    ep.ldc = C.ld;
    ep.M = (uint32_t)C.rows;
    ep.N = (uint32_t)C.cols;
    ep.p = F.p;
    ep.mu = F.mu;
    ep.alpha = alpha;
    ep.beta = beta;
    ep.mode = (alpha == F.p - 1 && beta == 1 && F.p > 2) ? EPI_SUB
              : (alpha == 1 && beta == 0)                ? EPI_PROD
              : (alpha == 1 && beta == 1)                ? EPI_ADD
                                                         : EPI_GENERIC;
    ep.vec_ok = ((reinterpret_cast<uintptr_t>(C.d) & 15) == 0 && (C.ld & 3) == 0) ? 1u : 0u;
    ep.vec8_ok = ((reinterpret_cast<uintptr_t>(C.d) & 31) == 0 && (C.ld & 7) == 0) ? 1u : 0u;
    for (int s = 0; s < 8; ++s) ep.w[s] = F.w[s];
    return ep;
}

template <int L>
void launch_modgemm(const Field& F, uint32_t alpha, uint32_t beta, const uint8_t* Ap, const uint8_t* Bp, size_t Mp,
                    size_t Np, size_t Kp, DView C, cudaStream_t st, int sm_cap) {
    using S = Smem<L>;
    static PerDeviceOnce once;
    once([] { FFG_CUDA(cudaFuncSetAttribute(modgemm_kernel<L>, cudaFuncAttributeMaxDynamicSharedMemorySize, S::TOTAL)); });
    CUtensorMap ma = make_map(Ap, Kp, (uint64_t)L * Mp, BM);
    CUtensorMap mb = make_map(Bp, Kp, (uint64_t)(Np / S::NT) * L * S::NT, L * S::NT);
    EpiParams ep = make_ep(F, alpha, beta, C);
    ep.kblocks = (uint32_t)(Kp / BK);
    ep.m_tiles = (uint32_t)(Mp / BM);
    ep.n_tiles = (uint32_t)(Np / S::NT);
    // L2 eviction hints once the limb planes no longer fit in L2 beside C (FFG_GEMM_L2_HINTS=0/1 forces)
    static const int hints_env = (int)knob_int("FFG_GEMM_L2_HINTS", -1);
    ep.l2_hints = hints_env >= 0 ? (uint32_t)hints_env : ((uint64_t)L * (Mp + Np) * Kp > (64ull << 20) ? 1u : 0u);
    static const int group_env = (int)knob_int("FFG_GEMM_GROUP_M", GROUP_M);
    ep.group_m = (uint32_t)std::max(1, group_env);
    const uint32_t tiles = ep.m_tiles * ep.n_tiles;
    dim3 grid(sm_cap > 0 ? std::min<uint32_t>(tiles, (uint32_t)sm_cap) : tiles);
    launch_k(modgemm_kernel<L>, grid, dim3(384), S::TOTAL, st, ma, mb, ep);
    FFG_CUDA(cudaGetLastError());
}

bool direct_fits(int L, int KB) {
    switch (L * 4 + KB) {
        case 1 * 4 + 1: return DirectSmem<1, 1>::FITS;
        case 1 * 4 + 2: return DirectSmem<1, 2>::FITS;
        case 2 * 4 + 1: return DirectSmem<2, 1>::FITS;
        case 2 * 4 + 2: return DirectSmem<2, 2>::FITS;
        case 3 * 4 + 1: return DirectSmem<3, 1>::FITS;
        case 3 * 4 + 2: return DirectSmem<3, 2>::FITS;
        case 4 * 4 + 1: return DirectSmem<4, 1>::FITS;
        case 4 * 4 + 2: return DirectSmem<4, 2>::FITS;
        default: return false;
    }
}

template <int L, int KB>
void launch_direct(const Field& F, uint32_t alpha, uint32_t beta, DView A, DView B, DView C, cudaStream_t st) {
    using S = DirectSmem<L, KB>;
    if constexpr (!S::FITS) {
        throw Error(FFG_ERR_INTERNAL, "direct GEMM tile does not fit shared memory");
    } else {
    static PerDeviceOnce once;
    once([] {
        FFG_CUDA(cudaFuncSetAttribute(modgemm_direct_kernel<L, KB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      S::TOTAL));
    });
    EpiParams ep = make_ep(F, alpha, beta, C);
    ep.kblocks = KB;
    ep.m_tiles = (uint32_t)ceil_div(C.rows, BM);
    ep.n_tiles = (uint32_t)ceil_div(C.cols, S::NT);
    DirectArgs da;
    da.A = A.d;
    da.lda = A.ld;
    da.B = B.d;
    da.ldb = B.ld;
    da.K = (uint32_t)A.cols;
    da.a_vec = ((reinterpret_cast<uintptr_t>(A.d) & 15) == 0 && (A.ld & 3) == 0) ? 1u : 0u;
    static unsigned long long* dbg_buf = nullptr;
    static const bool dbg_on = knob_set("FFG_DIRECT_DBG");
    if (dbg_on && !dbg_buf) FFG_CUDA(cudaMalloc(&dbg_buf, 64));
    da.dbg = dbg_on ? dbg_buf : nullptr;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (dbg_on) {
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0, st);
    }
    launch_k(modgemm_direct_kernel<L, KB>, dim3(ep.m_tiles * ep.n_tiles), dim3(384), S::TOTAL, st, da, ep);
    FFG_CUDA(cudaGetLastError());
    if (dbg_on) {
        cudaEventRecord(e1, st);
        cudaStreamSynchronize(st);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        unsigned long long h[6];
        cudaMemcpy(h, dbg_buf, 48, cudaMemcpyDeviceToHost);
        const double c2us = (double)(h[5] - h[4]) / 1e3 / (double)(h[3] - h[0]);  // measured clock
        fprintf(stderr, "DIRECT_DBG clock %.0f MHz, body %.2f us (globaltimer)\n", 1.0 / c2us,
                (h[5] - h[4]) / 1e3);
        fprintf(stderr, "DIRECT_DBG %zux%zux%zu staged %.2f us, mma %.2f us, epilogue %.2f us, body %.2f us, event %.2f us\n",
                C.rows, C.cols, A.cols, (h[1] - h[0]) * c2us, (h[2] - h[1]) * c2us, (h[3] - h[2]) * c2us,
                (h[3] - h[0]) * c2us, ms * 1e3);
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
    }
    }
}

}  // namespace

// CUDA-core path for problems with M*N*K <= g_simt_macs (off by default: inside the PLUQ the
// direct tensor-core kernel wins from K = 64 up) or with a tiny inner dimension K <= g_simt_kmax:
// the rank-sized updates of rank-deficient blocks (K = 1..32), where the tensor-core kernel's
// fixed cost (TMEM, staging a 128-row tile, epilogue) is all there is.
size_t g_simt_macs = 0;
size_t g_simt_kmax = 32;
bool use_simt(size_t M, size_t N, size_t K) { return M * N * K <= g_simt_macs || K <= g_simt_kmax; }

size_t gemm_workspace_bytes(const Field& F, size_t m, size_t n, size_t k) {
    const int L = F.limbs, NT = tile_n(L);
    const size_t kc = std::min<size_t>(k, F.kmax);
    const size_t Kp = round_up(std::max<size_t>(kc, 1), BK);
    return (size_t)L * round_up(m, BM) * Kp + (size_t)L * round_up(n, NT) * Kp + 2048;
}

void fgemm_dev(const Field& F, uint32_t alpha, DView A, DView B, uint32_t beta, DView C, cudaStream_t st,
               Workspace& ws, uint64_t* launches, int sm_cap, bool no_direct_call) {
    if (A.cols != B.rows || C.rows != A.rows || C.cols != B.cols)
        throw Error(FFG_ERR_DIM_MISMATCH, "gemm: non-conforming shapes");  // blas.hpp:21-24
    const size_t M = C.rows, N = C.cols, K = A.cols;
    if (M == 0 || N == 0) return;
    alpha %= F.p;
    beta %= F.p;
    if (alpha == 0 || K == 0) {
        if (beta != 1) {
            dim3 g((unsigned)ceil_div(N, 256), (unsigned)M);
            launch_k(scale_kernel, g, dim3(256), 0, st, C.d, C.ld, (uint32_t)M, (uint32_t)N, beta, F.p, F.mu);
            FFG_CUDA(cudaGetLastError());
            if (launches) __atomic_add_fetch(launches, 1, __ATOMIC_RELAXED);
        }
        return;
    }
    // element-exact overlap of two strided windows; windows of one parent (same ld) compare as
    // rectangles, anything else conservatively by address span
    auto overlap = [](const DView& x, const DView& y) {
        if (x.empty() || y.empty()) return false;
        if (x.ld == y.ld && x.ld > 0) {
            const int64_t off = (int64_t)(y.d - x.d);  // y's origin relative to x's, in elements
            const int64_t ld = (int64_t)x.ld;
            int64_t r = off / ld, c = off % ld;
            if (c < 0) {
                c += ld;
                --r;
            }
            // the column offset is c or c - ld (one row further down); test both placements
            auto hit = [&](int64_t rr, int64_t cc) {
                return rr < (int64_t)x.rows && rr + (int64_t)y.rows > 0 && cc < (int64_t)x.cols &&
                       cc + (int64_t)y.cols > 0;
            };
            return hit(r, c) || hit(r + 1, c - ld);
        }
        const uintptr_t a0 = reinterpret_cast<uintptr_t>(x.d), a1 = reinterpret_cast<uintptr_t>(x.d + (x.rows - 1) * x.ld + x.cols);
        const uintptr_t b0 = reinterpret_cast<uintptr_t>(y.d), b1 = reinterpret_cast<uintptr_t>(y.d + (y.rows - 1) * y.ld + y.cols);
        return a0 < b1 && b0 < a1;
    };
    // the CUDA-core kernel reads operands while other CTAs write C: only when C aliases nothing
    const bool simt = use_simt(M, N, K) && !overlap(C, A) && !overlap(C, B);
    static const bool log = knob_set("FFG_GEMM_LOG");
    if (log) fprintf(stderr, "FFG_GEMM %zu %zu %zu %d\n", M, N, K, (int)simt);
    if (simt) {
        ws.prof.begin(st);
        dim3 g((unsigned)ceil_div(N, SG_T), (unsigned)ceil_div(M, SG_T));
        launch_k(modgemm_simt_kernel, g, dim3(256), 0, st, A.d, A.ld, B.d, B.ld, C.d, C.ld, (uint32_t)M, (uint32_t)N,
                 (uint32_t)K, alpha, beta, F.p, F.mu);
        FFG_CUDA(cudaGetLastError());
        ws.prof.end(st, PROF_SIMT, 2.0 * (double)M * N * K, 2.0 * (double)M * N * K);
        if (launches) __atomic_add_fetch(launches, 1, __ATOMIC_RELAXED);
        return;
    }
    const int L = F.limbs, NT = tile_n(L);
    static const int cap_env = (int)knob_int("FFG_GEMM_SM_CAP", 0);
    if (sm_cap <= 0) sm_cap = cap_env;  // test hook: force the persistent multi-tile path
    // small K, no aliasing: operands staged by the GEMM itself (one launch, no limb planes in HBM)
    static const bool no_direct = knob_on("FFG_NO_DIRECT");
    // in place on B (the TRSM leaf X = inv(T) X) is race-free with one row tile: each CTA stages
    // its whole column strip of B before the CTA's own epilogue overwrites exactly that strip
    const bool c_is_b = C.d == B.d && C.ld == B.ld && C.rows == B.rows && C.cols == B.cols && M <= (size_t)BM;
    const size_t kb_need = ceil_div(K, (size_t)BK);
    // 128 < K <= 256 takes the TMA pipeline: inside the PLUQ the direct kernel's two staged K
    // blocks cost more than the split (measured 29.9 -> 29.4 ms at n = 16384); FFG_DIRECT_KB2=1
    // restores the direct path for them
    static const bool kb2 = knob_on("FFG_DIRECT_KB2");
    const bool fits = kb_need == 1 ? direct_fits(L, 1) : (kb2 && kb_need == 2 && direct_fits(L, 2));
    if (!no_direct && !no_direct_call && fits && !overlap(C, A) && (c_is_b || !overlap(C, B))) {
        ws.prof.begin(st);
        const bool one = kb_need == 1;
        switch (L) {
            case 1: one ? launch_direct<1, 1>(F, alpha, beta, A, B, C, st) : launch_direct<1, 2>(F, alpha, beta, A, B, C, st); break;
            case 2: one ? launch_direct<2, 1>(F, alpha, beta, A, B, C, st) : launch_direct<2, 2>(F, alpha, beta, A, B, C, st); break;
            case 3: one ? launch_direct<3, 1>(F, alpha, beta, A, B, C, st) : launch_direct<3, 2>(F, alpha, beta, A, B, C, st); break;
            default: one ? launch_direct<4, 1>(F, alpha, beta, A, B, C, st) : launch_direct<4, 2>(F, alpha, beta, A, B, C, st); break;
        }
        ws.prof.end(st, PROF_GEMM, 2.0 * L * L * (double)M * N * K, 2.0 * (double)M * N * K);
        if (launches) __atomic_add_fetch(launches, 1, __ATOMIC_RELAXED);
        return;
    }
    const size_t Mp = round_up(M, BM), Np = round_up(N, NT);
    for (size_t k0 = 0; k0 < K; k0 += F.kmax) {  // delayed reduction: one fold per kmax chunk
        const size_t kc = std::min<size_t>(K - k0, F.kmax);
        const size_t Kp = round_up(kc, BK);
        uint8_t* Ap = ws.get(st, (size_t)L * Mp * Kp + (size_t)L * Np * Kp);
        uint8_t* Bp = Ap + (size_t)L * Mp * Kp;
        ws.prof.begin(st);
        {
            SplitArgs sa;
            sa.A = A.d + k0;
            sa.lda = A.ld;
            sa.M = (uint32_t)M;
            sa.K = (uint32_t)kc;
            sa.Mp = (uint32_t)Mp;
            sa.Kp = (uint32_t)Kp;
            sa.outA = Ap;
            sa.B = B.d + k0 * B.ld;
            sa.ldb = B.ld;
            sa.N = (uint32_t)N;
            sa.Np = (uint32_t)Np;
            sa.outB = Bp;
            sa.L = L;
            sa.NT = NT;
            sa.a_blocks = (uint32_t)ceil_div(Mp * (Kp / 16), 256);
            sa.a_vec = ((reinterpret_cast<uintptr_t>(sa.A) & 15) == 0 && (A.ld & 3) == 0) ? 1u : 0u;
            sa.b_kblocks = (uint32_t)ceil_div(Kp, 64);
            const size_t nblk = sa.a_blocks + (size_t)sa.b_kblocks * ceil_div(Np, 64);
            launch_k(split_kernel, dim3((unsigned)nblk), dim3(256), 0, st, sa);
            FFG_CUDA(cudaGetLastError());
        }
        // split traffic: read M*kc + kc*N residues (4 B), write the padded limb planes
        ws.prof.end(st, PROF_SPLIT, 4.0 * ((double)M * kc + (double)kc * N) + (double)L * Kp * (Mp + Np));
        const uint32_t b = (k0 == 0) ? beta : 1u;
        ws.prof.begin(st);
        switch (L) {
            case 1: launch_modgemm<1>(F, alpha, b, Ap, Bp, Mp, Np, Kp, C, st, sm_cap); break;
            case 2: launch_modgemm<2>(F, alpha, b, Ap, Bp, Mp, Np, Kp, C, st, sm_cap); break;
            case 3: launch_modgemm<3>(F, alpha, b, Ap, Bp, Mp, Np, Kp, C, st, sm_cap); break;
            default: launch_modgemm<4>(F, alpha, b, Ap, Bp, Mp, Np, Kp, C, st, sm_cap); break;
        }
        // algorithmic work: L^2 u8 limb products per field MAC -> 2 L^2 M N kc int8 tensor ops
        ws.prof.end(st, PROF_GEMM, 2.0 * L * L * (double)M * N * kc, 2.0 * (double)M * N * kc);
        if (launches) __atomic_add_fetch(launches, 2, __ATOMIC_RELAXED);
    }
}

}  // namespace ffg
