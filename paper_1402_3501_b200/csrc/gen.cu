// gen.cu -- seeded input generators on the device (same bits as the CPU definitions).
//
// random_mat (test_util.hpp:22-28): entry (i, j) is output number i*n + j of
// SplitMix64(seed) mod p.  SplitMix64 (generate.hpp:10-24) is counter-based,
// so every entry is computed independently.
// L*R*U (config 4): L unit lower / U unit upper with
// SplitMix64 entries, R with r ones at Fisher-Yates positions; M is formed as
// the n x r by r x n product L[:, rows] * U[cols, :] on the tensor-core GEMM.
#include <vector>

#include "pluq.cuh"

namespace ffg {

__host__ __device__ __forceinline__ uint64_t splitmix_at(uint64_t seed, uint64_t k) {
    uint64_t z = seed + (k + 1) * 0x9e3779b97f4a7c15ull;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

__global__ void random_mat_kernel(uint32_t* A, uint64_t lda, uint32_t m, uint32_t n, uint32_t p, uint64_t seed) {
    const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x, i = blockIdx.y;
    if (i < m && j < n) A[(uint64_t)i * lda + j] = (uint32_t)(splitmix_at(seed, (uint64_t)i * n + j) % p);
}

// Lr[i][t] = L[i][rows[t]]  (n x r),  Uc[t][j] = U[cols[t]][j]  (r x n)
__global__ void lru_factor_kernel(uint32_t* Lr, uint32_t* Uc, const uint32_t* rows, const uint32_t* cols, uint32_t n,
                                  uint32_t r, uint32_t p, uint64_t sL, uint64_t sU) {
    const uint32_t x = blockIdx.x * blockDim.x + threadIdx.x, y = blockIdx.y;
    if (blockIdx.z == 0) {  // Lr: row y, column x
        if (y < n && x < r) {
            const uint32_t j = rows[x];
            const uint64_t idx = (uint64_t)y * n + j;
            Lr[(uint64_t)y * r + x] = j < y ? (uint32_t)(splitmix_at(sL, idx) % p) : (j == y ? 1u : 0u);
        }
    } else {  // Uc: row y (< r), column x (< n)
        if (y < r && x < n) {
            const uint32_t i = cols[y];
            const uint64_t idx = (uint64_t)i * n + x;
            Uc[(uint64_t)y * n + x] = x > i ? (uint32_t)(splitmix_at(sU, idx) % p) : (x == i ? 1u : 0u);
        }
    }
}

void random_mat_dev(const Blas& b, DView A, uint64_t seed) {
    if (A.empty()) return;
    dim3 g((unsigned)ceil_div(A.cols, 256), (unsigned)A.rows);
    random_mat_kernel<<<g, 256, 0, b.st>>>(A.d, A.ld, (uint32_t)A.rows, (uint32_t)A.cols, b.F.p, seed);
    FFG_CUDA(cudaGetLastError());
    b.count();
}

void lru_positions(size_t n, size_t r, uint64_t seed, std::vector<uint32_t>& rows, std::vector<uint32_t>& cols) {
    const uint64_t sR = splitmix_at(seed, 2);
    std::vector<uint32_t> pr(n), pc(n);
    for (size_t i = 0; i < n; ++i) pr[i] = pc[i] = (uint32_t)i;
    uint64_t k = 0;
    for (size_t i = n; i > 1; --i) std::swap(pr[i - 1], pr[splitmix_at(sR, k++) % i]);
    for (size_t i = n; i > 1; --i) std::swap(pc[i - 1], pc[splitmix_at(sR, k++) % i]);
    rows.assign(pr.begin(), pr.begin() + r);
    cols.assign(pc.begin(), pc.begin() + r);
}

void lru_matrix_dev(const Blas& b, DView M, size_t r, uint64_t seed, uint32_t* rows_out, uint32_t* cols_out) {
    const size_t n = M.rows;
    if (M.cols != n) throw Error(FFG_ERR_DIM_MISMATCH, "lru: square output required");
    if (r > n) throw Error(FFG_ERR_INVALID_RANK, "lru: rank exceeds n");
    std::vector<uint32_t> rows, cols;
    lru_positions(n, r, seed, rows, cols);
    if (rows_out) std::copy(rows.begin(), rows.end(), rows_out);
    if (cols_out) std::copy(cols.begin(), cols.end(), cols_out);
    if (n == 0) return;
    if (r == 0) {
        FFG_CUDA(cudaMemset2DAsync(M.d, M.ld * 4, 0, n * 4, n, b.st));
        return;
    }
    uint32_t *Lr = nullptr, *Uc = nullptr, *dpos = nullptr;
    FFG_CUDA(cudaMallocAsync(&Lr, n * r * 4, b.st));
    FFG_CUDA(cudaMallocAsync(&Uc, n * r * 4, b.st));
    FFG_CUDA(cudaMallocAsync(&dpos, 2 * r * 4, b.st));
    FFG_CUDA(cudaMemcpyAsync(dpos, rows.data(), r * 4, cudaMemcpyHostToDevice, b.st));
    FFG_CUDA(cudaMemcpyAsync(dpos + r, cols.data(), r * 4, cudaMemcpyHostToDevice, b.st));
    dim3 g((unsigned)ceil_div(std::max(n, r), 256), (unsigned)std::max(n, r), 2);
    lru_factor_kernel<<<g, 256, 0, b.st>>>(Lr, Uc, dpos, dpos + r, (uint32_t)n, (uint32_t)r, b.F.p,
                                           splitmix_at(seed, 0), splitmix_at(seed, 1));
    FFG_CUDA(cudaGetLastError());
    b.count();
    b.gemm(1, DView{Lr, n, r, r}, DView{Uc, r, n, n}, 0, M);
    FFG_CUDA(cudaFreeAsync(Lr, b.st));
    FFG_CUDA(cudaFreeAsync(Uc, b.st));
    FFG_CUDA(cudaFreeAsync(dpos, b.st));
    // the pinned/pageable host vectors above are consumed by the async copies before return
    FFG_CUDA(cudaStreamSynchronize(b.st));
}

}  // namespace ffg
