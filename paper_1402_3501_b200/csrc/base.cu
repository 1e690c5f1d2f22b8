// base.cu -- the rank-profile revealing base case (rr_base, rankrev.hpp:29-78) as one CTA.
//
// The reference eliminates Crout-lazily and physically rotates rows and
// columns after each pivot.  Its output is fully determined by the pivot
// sequence: pivot k is the first remaining row (original order) whose Schur
// row is nonzero, at the first nonzero non-pivot column (original order) --
// rotations keep non-pivot rows/columns in original relative order
// (perm.hpp:11-13).  Given the pivot sequence, P A Q = L U has unique packed
// factors, so this kernel uses eager right-looking elimination on the block
// held in shared memory, keeps rows/columns in place, and applies the final
// permutations once when writing the block back:
//     P = [pivot rows in discovery order, non-pivot rows ascending]
//     Q = [pivot cols in discovery order, non-pivot cols ascending]
//     out[t][u] = S[P[t]][Q[u]]
// Exhausted rows (no nonzero left, rankrev.hpp:54-57) keep their computed
// zeros; their L entries for later pivots are those zeros, as in the
// reference.  Values are exact residues, so the bits match rr_base.
#include "pluq.cuh"

namespace ffg {

constexpr int BASE_THREADS = 512;
constexpr size_t BASE_SMEM_LIMIT = 200 * 1024;

__device__ __forceinline__ uint32_t sub_mod(uint32_t a, uint32_t b, uint32_t p) { return a >= b ? a - b : a + p - b; }

template <bool IN_SMEM>
__global__ void __launch_bounds__(BASE_THREADS)
    rr_base_kernel(uint32_t* __restrict__ A, uint64_t lda, uint32_t m, uint32_t n, uint32_t* __restrict__ scratch,
                   uint32_t* __restrict__ Pd, uint32_t* __restrict__ Qd, BaseInfo* __restrict__ info, uint32_t p,
                   uint64_t mu) {
    extern __shared__ uint32_t sm[];
    // shared layout: [flags: rowpiv m bytes | colpiv n bytes] [prow | pcol] [block if IN_SMEM]
    uint8_t* rowpiv = reinterpret_cast<uint8_t*>(sm);
    uint8_t* colpiv = rowpiv + m;
    const uint32_t flag_words = (m + n + 3) / 4;
    uint32_t* prow = sm + flag_words;
    const uint32_t rmax = min(m, n);
    uint32_t* pcol = prow + rmax;
    uint32_t* S = IN_SMEM ? (pcol + rmax) : scratch;
    __shared__ uint32_t s_pi, s_pj, s_inv;

    const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, nwarps = BASE_THREADS / 32;
    for (uint32_t i = tid; i < m + n; i += BASE_THREADS) rowpiv[i] = 0;
    for (uint32_t idx = tid; idx < m * n; idx += BASE_THREADS) {
        const uint32_t r = idx / n, c = idx % n;
        S[idx] = A[(uint64_t)r * lda + c];
    }
    __syncthreads();

    uint32_t r = 0, cur = 0;
    while (cur < m && r < n) {
        if (warp == 0) {  // row-major pivot search (rankrev.hpp:40-57)
            uint32_t pi = m, pj = n;
            for (uint32_t i = cur; i < m && pi == m; ++i) {
                const uint32_t* row = S + (uint64_t)i * n;
                for (uint32_t jc = 0; jc < n; jc += 32) {
                    const uint32_t j = jc + lane;
                    const bool nz = j < n && !colpiv[j] && row[j] != 0;
                    const uint32_t bal = __ballot_sync(0xffffffffu, nz);
                    if (bal) {
                        pi = i;
                        pj = jc + __ffs(bal) - 1;
                        break;
                    }
                }
            }
            if (lane == 0) {
                s_pi = pi;
                s_pj = pj;
                if (pi < m) {
                    s_inv = inv_mod(S[(uint64_t)pi * n + pj], p);
                    prow[r] = pi;
                    pcol[r] = pj;
                    rowpiv[pi] = 1;
                    colpiv[pj] = 1;
                }
            }
        }
        __syncthreads();
        const uint32_t pi = s_pi, pj = s_pj;
        if (pi >= m) break;
        const uint32_t inv = s_inv;
        const uint32_t* prw = S + (uint64_t)pi * n;
        // eager update of the rows after the pivot row; rows before it are pivots or exhausted
        for (uint32_t i = pi + 1 + warp; i < m; i += nwarps) {
            uint32_t* row = S + (uint64_t)i * n;
            const uint32_t l = mul_mod(row[pj], inv, p, mu);
            __syncwarp();
            if (lane == 0) row[pj] = l;  // L entry (rankrev.hpp:68-72)
            if (l) {
                for (uint32_t j = lane; j < n; j += 32)
                    if (!colpiv[j]) row[j] = sub_mod(row[j], mul_mod(l, prw[j], p, mu), p);
            }
        }
        ++r;
        cur = pi + 1;
        __syncthreads();
    }

    // permutations: pivots in discovery order, then the rest ascending
    if (tid == 0) {
        uint32_t t = r;
        for (uint32_t i = 0; i < m; ++i)
            if (!rowpiv[i]) Pd[t++] = i;
        for (uint32_t k = 0; k < r; ++k) Pd[k] = prow[k];
        t = r;
        for (uint32_t j = 0; j < n; ++j)
            if (!colpiv[j]) Qd[t++] = j;
        for (uint32_t k = 0; k < r; ++k) Qd[k] = pcol[k];
        uint32_t lo = m, hi = 0;
        for (uint32_t i = 0; i < m; ++i)
            if (Pd[i] != i) {
                lo = min(lo, i);
                hi = i + 1;
            }
        info->rank = r;
        info->plo = lo < hi ? lo : 0;
        info->phi = lo < hi ? hi : 0;
        lo = n;
        hi = 0;
        for (uint32_t j = 0; j < n; ++j)
            if (Qd[j] != j) {
                lo = min(lo, j);
                hi = j + 1;
            }
        info->qlo = lo < hi ? lo : 0;
        info->qhi = lo < hi ? hi : 0;
    }
    __syncthreads();
    for (uint32_t idx = tid; idx < m * n; idx += BASE_THREADS) {
        const uint32_t t = idx / n, u = idx % n;
        A[(uint64_t)t * lda + u] = S[(uint64_t)Pd[t] * n + Qd[u]];
    }
}

void rr_base_launch(const Blas& b, DView a, uint32_t* Pd, uint32_t* Qd, void* info_dev) {
    const uint32_t m = (uint32_t)a.rows, n = (uint32_t)a.cols;
    const size_t fixed = (((size_t)m + n + 3) / 4 + 2 * std::min(m, n)) * 4;
    const size_t blk = (size_t)m * n * 4;
    BaseInfo* info = static_cast<BaseInfo*>(info_dev);
    b.ws.prof.begin(b.st);
    if (fixed + blk <= BASE_SMEM_LIMIT) {
        static bool set = false;
        if (!set) {
            FFG_CUDA(cudaFuncSetAttribute(rr_base_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)BASE_SMEM_LIMIT));
            set = true;
        }
        rr_base_kernel<true><<<1, BASE_THREADS, fixed + blk, b.st>>>(a.d, a.ld, m, n, nullptr, Pd, Qd, info, b.F.p,
                                                                     b.F.mu);
    } else {
        if (fixed > BASE_SMEM_LIMIT) throw Error(FFG_ERR_INVALID_BLOCK, "base case block too large");
        static bool set = false;
        if (!set) {
            FFG_CUDA(cudaFuncSetAttribute(rr_base_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)BASE_SMEM_LIMIT));
            set = true;
        }
        uint32_t* scratch = nullptr;
        FFG_CUDA(cudaMallocAsync(&scratch, blk, b.st));
        rr_base_kernel<false><<<1, BASE_THREADS, fixed, b.st>>>(a.d, a.ld, m, n, scratch, Pd, Qd, info, b.F.p, b.F.mu);
        FFG_CUDA(cudaFreeAsync(scratch, b.st));
    }
    FFG_CUDA(cudaGetLastError());
    b.ws.prof.end(b.st, PROF_BASE, 2.0 * blk, 2.0 * std::min(m, n) * (double)m * n);
    b.count();
}

}  // namespace ffg
