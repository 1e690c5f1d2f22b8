// pluq.cuh -- internal API of the triangular solves, base case, permutations and the
// tile-recursive driver.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include "common.cuh"
#include "gemm.cuh"

namespace ffg {

// Everything a BLAS-level call needs: field, scratch, stream, launch counter.
struct Blas {
    const Field& F;
    Workspace& ws;
    cudaStream_t st;
    uint64_t* launches;
    int sm_cap = 0;          // > 0: tensor-core GEMMs on this stream use at most this many SMs
    bool no_direct = false;  // skip the one-launch direct kernel (throughput over latency)
    void gemm(uint32_t alpha, DView A, DView B, uint32_t beta, DView C) const {
        fgemm_dev(F, alpha, A, B, beta, C, st, ws, launches, sm_cap, no_direct);
    }
    void count(uint64_t n = 1) const {
        if (launches) __atomic_add_fetch(launches, n, __ATOMIC_RELAXED);
    }
};

// B <- op(A)^-1 B (side 0) or B op(A)^-1 (side 1); blas.hpp:389-398.  check_diag
// scans the diagonal first (nonunit) and throws SingularDiagonal(i) like blas.hpp:291-297.
void ftrsm_dev(const Blas& b, int side, int uplo, int diag, DView A, DView B, bool check_diag);

// panel schedule: both factor inverses of a packed square block (<= 64) into inv (2 t^2 words),
// then B <- inv(L) B (side 0) or B <- B inv(U) (side 1) over any number of strips
void panel_inverses_dev(const Blas& b, DView T, uint32_t* inv);
void panel_apply_dev(const Blas& b, int side, const uint32_t* inv, size_t t, DView B, const uint32_t* qperm = nullptr);

// a leaf's next-block panels in one launch: X <- inv(L) X (t x w), Y <- Y[:, q] inv(U) (h x t)
void panel_mini_dev(const Blas& b, const uint32_t* inv, size_t t, DView X, DView Y, const uint32_t* qperm);

// C -= Y X for blocks <= 64 (small CTAs, 16 columns each)
void panel_update_dev(const Blas& b, DView Y, DView X, DView C);


// pluq_tile_recursive on a HOST matrix (ld lda), pipelined: the recursion's top-left spine
// starts while the rest uploads, the root's finished top rows download while its trailing
// block recurses.  Same outputs as the device entry.
size_t pluq_tile_recursive_host(const Blas& b, uint32_t* host, size_t m, size_t n, size_t lda, size_t threshold,
                                uint32_t* P, uint32_t* Q);

// The same on a host matrix of bytes (p <= 256; entries taken mod p): bytes cross PCIe in row
// chunks, widened to u32 in HBM, factored, narrowed back.
size_t pluq_tile_recursive_host_u8(const Blas& b, uint8_t* host, size_t m, size_t n, size_t lda, size_t threshold,
                                   uint32_t* P, uint32_t* Q);
void widen_u8_dev(const Blas& b, const uint8_t* src, size_t lds, DView dst);
void narrow_u8_dev(const Blas& b, DView src, uint8_t* dst, size_t ldd);

// rr_base (rankrev.hpp:29-78) on a device block; P/Q host arrays (to_array semantics).
size_t rr_base_dev(const Blas& b, DView a, uint32_t* P, uint32_t* Q);

// pluq_tile_recursive (rankrev.hpp:229-233); P/Q host arrays.
size_t pluq_tile_recursive_dev(const Blas& b, DView a, size_t threshold, uint32_t* P, uint32_t* Q);

// rank + moved ranges of a base-case result (device -> pinned host)
struct BaseInfo {
    uint32_t rank, plo, phi, qlo, qhi;
    uint32_t cached;     // 1 when inv_out received inv(L_r), inv(U_r) (r x r each, ld r)
    uint32_t seq;        // written last: the launch's sequence number (host spins on it)
    uint32_t spec_fail;  // sticky: a speculative launch (seq & SPEC_BIT) did not see full rank +
                         // identity permutations
    uint32_t fail_seq;   // the sequence number of the first launch that raised spec_fail
};
constexpr uint32_t SPEC_BIT = 0x80000000u;
// one-CTA rr_base kernel: writes the permuted packed block, P/Q index arrays and info; with
// inv_out != nullptr also the inverses of the leading r x r L and U factors (r <= 64)
// returns whether inverses were requested (the kernel still reports info->cached)
// allow_q (speculative launches on square blocks): the guess is full rank only, column pivots
// allowed (Qd receives them; P is then the identity)
bool rr_base_launch(const Blas& b, DView a, uint32_t* Pd, uint32_t* Qd, void* info_dev,
                    uint32_t* inv_out = nullptr, uint32_t seq = 0, bool allow_q = false);
// speculative square block (t <= 64) of the panel schedule + both factor inverses in one launch
// (baseinv.cu): inv[0, t^2) = inv(L), inv[t^2, 2 t^2) = inv(U), row-major ld t
void rr_base_inv_launch(const Blas& b, DView a, uint32_t* Pd, uint32_t* Qd, void* info_dev, uint32_t* inv,
                        uint32_t seq, bool allow_q);


// permutation kernels (perm.cu)
void perm_apply_range(const Blas& b, DView a, int axis, const uint32_t* perm, size_t lo, size_t hi);
void rotate_block_dev(const Blas& b, DView a, int axis, size_t first, size_t mid, size_t len);
void perm_compose_dev(const Blas& b, uint32_t* dst, size_t off, const uint32_t* child, size_t lo, size_t hi);
void perm_rot_dev(const Blas& b, uint32_t* arr, size_t first, size_t mid, size_t len);
void perm_iota_dev(const Blas& b, uint32_t* arr, size_t len);

// seeded generators (gen.cu)
void random_mat_dev(const Blas& b, DView A, uint64_t seed);
void lru_matrix_dev(const Blas& b, DView M, size_t r, uint64_t seed, uint32_t* rows_out, uint32_t* cols_out);

// row (axis 0) / column (axis 1) gather by a device index array
void apply_perm_dev(const Blas& b, DView a, int axis, int inverse, const uint32_t* perm);

// a[i][t] <- a[i][q[t]] for t < a.cols <= 64 (q: device, local indices)
void block_cols_perm_dev(const Blas& b, DView a, const uint32_t* q);

// dst <- src, same shape (device copy kernel: far faster HBM to HBM than the DMA engines)
void copy_block_dev(const Blas& b, DView src, DView dst);

}  // namespace ffg
