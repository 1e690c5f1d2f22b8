/*
 * ffg.h -- C ABI of the B200-native ffpluq hot path (libffg_b200.so).
 *
 * Drop-in boundary for the reference's tile-recursive PLUQ over GF(p) and the
 * two kernels under it.  Plain pointers and sizes only.  Matrices are row-major
 * uint32 canonical residues in [0, p) with an explicit leading dimension, the
 * layout of the reference's MatView (proj/include/ffpluq/matrix.hpp:13-43).
 *
 * Every entry point exists in two forms:
 *   ffg_X(...)      host buffers: the drop-in for the reference call on a
 *                   host MatView (copies in, computes on the GPU, copies out)
 *   ffg_X_dev(...)  device buffers, enqueued on the context's stream
 *
 * Permutations are returned as index arrays with the meaning of
 * PermSeq::to_array() (perm.hpp:88-95): entry t = original index now at
 * position t.  Status codes mirror the reference exception types
 * (proj/include/ffpluq/errors.hpp:9-59).
 */
#ifndef FFG_H
#define FFG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (errors.hpp:9-59) ----------------------------------- */
#define FFG_OK 0
#define FFG_ERR_ZERO_DIVISION 1     /* ZeroDivision      errors.hpp:9-11  */
#define FFG_ERR_CAPACITY 2          /* CapacityError     errors.hpp:13-15 (bad modulus) */
#define FFG_ERR_DIM_MISMATCH 3      /* DimMismatch       errors.hpp:17-19 */
#define FFG_ERR_EMPTY_MATRIX 4      /* EmptyMatrix       errors.hpp:21-23 */
#define FFG_ERR_ZERO_PIVOT 5        /* ZeroPivot         errors.hpp:27-31 */
#define FFG_ERR_SINGULAR_DIAGONAL 6 /* SingularDiagonal  errors.hpp:33-38, index via ffg_last_error_index() */
#define FFG_ERR_NOT_RANK_REVEALING 7
#define FFG_ERR_INVALID_BLOCK 8
#define FFG_ERR_INVALID_DIM 9
#define FFG_ERR_INVALID_RANK 10
#define FFG_ERR_NO_MEMORY 12
#define FFG_ERR_CUDA 100            /* CUDA runtime failure (message via ffg_last_error()) */
#define FFG_ERR_NO_DEVICE 101       /* no sm_100 device: there is no CPU fallback */
#define FFG_ERR_INVALID_ARG 102     /* null context / pointer */
#define FFG_ERR_INTERNAL 103

typedef struct ffg_ctx ffg_ctx;

/* Context: one CUDA device, one stream, device workspace.  Fails with
 * FFG_ERR_NO_DEVICE when the device is not a compute-capability 10.x GPU. */
int ffg_create(ffg_ctx **out, int device);
void ffg_destroy(ffg_ctx *ctx);
/* cudaStream_t passed as void* so the header stays CUDA-free; NULL = the context's own */
int ffg_set_stream(ffg_ctx *ctx, void *stream);
void *ffg_get_stream(ffg_ctx *ctx);
int ffg_synchronize(ffg_ctx *ctx);

const char *ffg_last_error(void);     /* thread-local message of the last failure */
size_t ffg_last_error_index(void);    /* SingularDiagonal::index (errors.hpp:33-38) */
const char *ffg_version(void);
/* The library snapshots its FFG_* environment switches (tuning values, test
 * hooks, diagnostics) once, at first use, and never
 * reads the environment on a call path.  This takes a fresh snapshot (tests
 * that change a switch between calls; not needed otherwise). */
void ffg_knobs_reload(void);

/* ---- modular GEMM ------------------------------------------------------
 * C <- alpha*A*B + beta*C mod p, A m x k, B k x n, C m x n.
 * Replaces fgemm / fgemm_classical / pfgemm (blas.hpp:31-103, 220-246, 250-271):
 * same arguments and values, any alpha, beta in [0, p).  2 <= p < 2^26 prime
 * (PrimeField, field.hpp:47-54), else FFG_ERR_CAPACITY. */
int ffg_fgemm(ffg_ctx *ctx, uint64_t p, uint32_t alpha, const uint32_t *A, size_t lda, const uint32_t *B,
              size_t ldb, uint32_t beta, uint32_t *C, size_t ldc, size_t m, size_t n, size_t k);
int ffg_fgemm_dev(ffg_ctx *ctx, uint64_t p, uint32_t alpha, const uint32_t *A, size_t lda, const uint32_t *B,
                  size_t ldb, uint32_t beta, uint32_t *C, size_t ldc, size_t m, size_t n, size_t k);

/* ---- triangular solve --------------------------------------------------
 * B (m x n) <- op(A)^-1 B (side 0 = left) or B op(A)^-1 (side 1 = right), in place.
 * uplo 0 = lower, 1 = upper; diag 0 = unit, 1 = nonunit.  A is t x t with
 * t = m (left) or n (right); only the selected triangle (and the diagonal if
 * nonunit) is read, so A may be a packed L\U square like in tile_rec.
 * Replaces ftrsm / pftrsm (blas.hpp:389-398, 402-419).  A zero diagonal entry
 * with diag = nonunit gives FFG_ERR_SINGULAR_DIAGONAL with the smallest index. */
int ffg_ftrsm(ffg_ctx *ctx, uint64_t p, int side, int uplo, int diag, const uint32_t *A, size_t lda,
              uint32_t *B, size_t ldb, size_t m, size_t n);
int ffg_ftrsm_dev(ffg_ctx *ctx, uint64_t p, int side, int uplo, int diag, const uint32_t *A, size_t lda,
                  uint32_t *B, size_t ldb, size_t m, size_t n);

/* ---- rank-profile revealing PLUQ ---------------------------------------
 * In place: A (m x n) receives the packed L\U factors exactly as the reference
 * leaves them; P (m entries) and Q (n entries) receive PermSeq::to_array() of
 * the row / column permutations; *rank the rank.
 * ffg_pluq_tile_recursive replaces pluq_tile_recursive (rankrev.hpp:229-233,
 * recursion rankrev.hpp:85-183, threshold clamped to >= 1).
 * ffg_rr_base replaces the base case rr_base (rankrev.hpp:29-78). */
int ffg_pluq_tile_recursive(ffg_ctx *ctx, uint64_t p, uint32_t *A, size_t m, size_t n, size_t lda,
                            size_t threshold, uint32_t *P, uint32_t *Q, size_t *rank);
int ffg_pluq_tile_recursive_dev(ffg_ctx *ctx, uint64_t p, uint32_t *A, size_t m, size_t n, size_t lda,
                                size_t threshold, uint32_t *P, uint32_t *Q, size_t *rank);
/* Byte storage for small fields (p <= 256, BASELINE config 5 "stored as uint8"): the same
 * factorisation on a host matrix of uint8 residues (entries taken mod p; the packed L\U factors
 * come back as bytes).  Not in the reference, whose storage is u32 only (field.hpp:15-17):
 * PCIe traffic is a quarter of the u32 entry's.  FFG_ERR_CAPACITY when p > 256. */
int ffg_pluq_tile_recursive_u8(ffg_ctx *ctx, uint64_t p, uint8_t *A, size_t m, size_t n, size_t lda,
                               size_t threshold, uint32_t *P, uint32_t *Q, size_t *rank);
int ffg_rr_base(ffg_ctx *ctx, uint64_t p, uint32_t *A, size_t m, size_t n, size_t lda, uint32_t *P, uint32_t *Q,
                size_t *rank);

/* ---- permutations (perm.hpp:167-215) -----------------------------------
 * Row (axis 0) or column (axis 1) gather of a device matrix by an index array
 * perm (device pointer, dim entries): out position t <- in position perm[t]
 * (forward, = apply_perm of a PermSeq whose to_array() is perm), or the
 * inverse scatter when inverse != 0. */
int ffg_apply_perm_dev(ffg_ctx *ctx, uint32_t *A, size_t m, size_t n, size_t lda, int axis, int inverse,
                       const uint32_t *perm);

/* ---- field embedding (introspection) ----------------------------------
 * For modulus p: *limbs = 8-bit limbs per residue on the tensor cores,
 * *kmax = inner-dimension chunk of one exact s32 accumulation (the GEMM reduces
 * mod p once per kmax products -- the delayed-reduction bound, field.hpp:26-35
 * restated for the limb embedding), *nt = output columns per GEMM tile.
 * Pure host function (no device needed). */
int ffg_field_info(uint64_t p, int *limbs, uint64_t *kmax, int *nt);

/* ---- rank profile matrix -> tile_rec permutations (host) ---------------
 * tile_rec's P and Q depend only on the rank profile matrix R_A (the pivots
 * (prow[k], pcol[k]), k < rank, in any order), m, n and the threshold: this
 * evaluates pluq_tile_recursive's permutation logic (rankrev.hpp:85-183) on
 * R_A itself, where every TRSM/GEMM is a no-op.  P (m words) and Q (n words)
 * receive the to_array() forms.  Pure host function (no device needed); the
 * profile-first exact path of ffg_pluq_tile_recursive[_dev] uses it. */
int ffg_tile_rec_perms(size_t m, size_t n, size_t threshold, size_t rank, const uint32_t *prow,
                       const uint32_t *pcol, uint32_t *P, uint32_t *Q);

/* ---- rank profile (device) --------------------------------------------
 * ffg_rank_profile_dev: the rank profile matrix of a device matrix A (not
 * modified): prow/pcol (host, min(m, n) words) receive the pivots in rr_base's
 * discovery order -- rr_base's P[k], Q[k] for k < rank (rankrev.hpp:29-78) --
 * computed by the blocked slab search of the profile-first path.
 * ffg_pluq_from_profile_dev: pluq_tile_recursive's outputs on A (in place)
 * given its rank profile (phases 2 and 3 of the profile-first path; the
 * profile must be A's, e.g. from ffg_rank_profile_dev). */
int ffg_rank_profile_dev(ffg_ctx *ctx, uint64_t p, const uint32_t *A, size_t m, size_t n, size_t lda,
                         uint32_t *prow, uint32_t *pcol, size_t *rank);
int ffg_pluq_from_profile_dev(ffg_ctx *ctx, uint64_t p, uint32_t *A, size_t m, size_t n, size_t lda,
                              size_t threshold, size_t rank, const uint32_t *prow, const uint32_t *pcol,
                              uint32_t *P, uint32_t *Q);

/* ---- seeded inputs on the device (generate.hpp / test_util.hpp) --------
 * ffg_random_mat_dev: A[i][j] = output i*n+j of SplitMix64(seed) mod p -- the
 *   reference's random_mat (test_util.hpp:22-28), bit for bit.
 * ffg_lru_matrix_dev: the BASELINE config-4 input M = L*R*U (n x n, rank r;
 *   definition in DESIGN.md); rows/cols (host, r entries each, may be NULL)
 *   receive the positions of R's ones, i.e. the rank profile matrix. */
int ffg_random_mat_dev(ffg_ctx *ctx, uint64_t p, uint64_t seed, uint32_t *A, size_t m, size_t n, size_t lda);
int ffg_lru_matrix_dev(ffg_ctx *ctx, uint64_t p, uint64_t seed, uint32_t *M, size_t n, size_t ldm, size_t r,
                       uint32_t *rows, uint32_t *cols);

/* ---- instrumentation ----------------------------------------------------
 * Kernel launches issued by this context since creation (all kernels of this
 * library; used for the bench's gpu_launches claim). */
uint64_t ffg_launch_count(ffg_ctx *ctx);
/* Outcomes of the speculative full-rank guesses since the context was created
 * (the GPU schedule's own bookkeeping, no reference counterpart): out[0..4] =
 * whole-matrix guesses tried, of those failed (resumed at the failed block or
 * rerun profile-first), node-level guesses tried, of those failed, profile-first
 * factorisations run. */
int ffg_spec_stats(ffg_ctx *ctx, uint64_t *out);
/* Per-kernel-class timing with CUDA events on the launching stream (off by
 * default).  Classes: 0 tensor-core GEMM, 1 limb split, 2 base case,
 * 3 triangle inverse, 4 permutation gathers, 5 CUDA-core small GEMM.  ffg_profile_read fills
 * out[4*c + {0,1,2,3}] = {milliseconds, launches, work, field ops} per class c
 * (work = int8 tensor ops for class 0, bytes moved otherwise) and clears.
 * on = 1: events around every launch; on = 2: count launches and work only (no
 * events, ms stays 0 -- pair with an external kernel timeline such as CUPTI). */
int ffg_profile_enable(ffg_ctx *ctx, int on);
int ffg_profile_read(ffg_ctx *ctx, double *out, int nclasses);

/* ---- multi-GPU: partitioned PLUQ, one process per GPU ---------------------
 * No reference counterpart (the reference parallelises over threads of one
 * host: pool.hpp, pfgemm/pftrsm in blas.hpp:117-153, 401-419); this is the
 * north_star's "trailing update partitioned across the GPUs of one box".
 * After ffg_dist_init on every rank (same world, distinct ranks, the same id
 * from ffg_dist_unique_id on one rank), ffg_pluq_tile_recursive[_dev] called
 * by all ranks on identical inputs returns identical outputs on every rank:
 * each Schur GEMM/TRSM of at least min_work MACs is split into per-rank
 * output slices, exchanged with one NCCL all-gather; everything smaller runs
 * replicated.  NCCL (libnccl.so.2) is loaded on first use.
 * ffg_dist_init_virtual: one process computes every slice of a world of that
 * size on its own GPU (no exchange) -- the single-GPU check of the partition;
 * loopback != 0 also routes every slice through the exchange's pack/unpack.
 * ffg_dist_partition: slice [lo, hi) of `total` for rank (pure host function). */
int ffg_dist_unique_id(unsigned char id[128]);
int ffg_dist_init(ffg_ctx *ctx, int world, int rank, const unsigned char id[128]);
int ffg_dist_init_virtual(ffg_ctx *ctx, int world, int loopback);
int ffg_dist_set_min_work(ffg_ctx *ctx, uint64_t macs);
int ffg_dist_info(ffg_ctx *ctx, int *world, int *rank, int *is_virtual, uint64_t *exchanges, uint64_t *bytes);
int ffg_dist_finalize(ffg_ctx *ctx);
int ffg_dist_partition(size_t total, int world, int rank, size_t align, size_t *lo, size_t *hi);

#ifdef __cplusplus
}
#endif
#endif
