/*
 * oracle.h -- CPU restatement of the reference ffpluq hot path (TEST INFRASTRUCTURE ONLY).
 *
 * This is the parity checker for the B200 implementation.  Only tests/, the
 * smoke() check in __graft_entry__.py and bench.py's cpu_baseline / reference
 * legs may load it.  The product library (paper_1402_3501_b200/) never links
 * or calls anything in here.
 *
 * Every function cites the reference file:line it restates (paths relative to
 * the reference checkout, proj/include/ffpluq/...).  Pinned against the
 * reference itself: tests/golden/ holds vectors produced by oracle/_ref (the
 * reference headers compiled unchanged) and tests/test_oracle_pins.py checks
 * this restatement against them.
 */
#ifndef FFG_ORACLE_H
#define FFG_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes: same numbering as include/ffg.h (errors.hpp:9-59) */
enum {
    ORC_OK = 0,
    ORC_ZERO_DIVISION = 1,
    ORC_CAPACITY = 2,
    ORC_DIM_MISMATCH = 3,
    ORC_EMPTY_MATRIX = 4,
    ORC_ZERO_PIVOT = 5,
    ORC_SINGULAR_DIAGONAL = 6,
    ORC_NOT_RANK_REVEALING = 7,
    ORC_INVALID_BLOCK = 8,
    ORC_INVALID_DIM = 9,
    ORC_INVALID_RANK = 10,
    ORC_NO_MEMORY = 12
};

/* field.hpp:39-54 */
typedef struct {
    uint64_t p;
    int acc_bits;
    uint64_t n_star;
    uint64_t n_star_seeded;
} orc_field;

int orc_field_init(orc_field *F, uint64_t p, int acc_bits);
uint32_t orc_inv(const orc_field *F, uint32_t a); /* field.hpp:91-107; a != 0 */

/* SplitMix64 (generate.hpp:10-24) */
uint64_t orc_splitmix_at(uint64_t seed, uint64_t k); /* k-th output (0-based) of SplitMix64(seed) */
/* test_util.hpp:22-28 random_mat: row-major, entry t = next() % p */
void orc_random_mat(uint32_t *a, size_t m, size_t n, size_t lda, uint64_t p, uint64_t seed);

/* blas.hpp:31-103: C <- alpha*A*B + beta*C (m x n, inner k) */
int orc_fgemm(const orc_field *F, uint32_t alpha, const uint32_t *A, size_t lda,
              const uint32_t *B, size_t ldb, uint32_t beta, uint32_t *C, size_t ldc,
              size_t m, size_t n, size_t k);

/* blas.hpp:389-398: side 0=left 1=right, uplo 0=lower 1=upper, diag 0=unit 1=nonunit.
 * A is t x t (lda), B is m x n (ldb).  On SingularDiagonal *bad_index gets the index. */
int orc_ftrsm(const orc_field *F, int side, int uplo, int diag, const uint32_t *A, size_t lda,
              uint32_t *B, size_t ldb, size_t m, size_t n, size_t *bad_index);

/* perm.hpp:167-193 applied through an explicit move list (type 0=Swap 1=Rot) */
int orc_apply_moves(uint32_t *a, size_t rows, size_t cols, size_t lda, int axis_cols,
                    int inverse, const uint32_t *mv_type, const uint32_t *mv_i,
                    const uint32_t *mv_j, size_t nmoves);
/* perm.hpp:90-95 */
void orc_moves_to_array(size_t n, const uint32_t *mv_type, const uint32_t *mv_i,
                        const uint32_t *mv_j, size_t nmoves, uint32_t *out);

/* rankrev.hpp:29-78: in place; P (m), Q (n) receive PermSeq::to_array() */
int orc_rr_base(const orc_field *F, uint32_t *a, size_t m, size_t n, size_t lda, uint32_t *P,
                uint32_t *Q, size_t *rank);

/* rankrev.hpp:85-183 + 229-233.  fix_j != 0 keeps block I and solves J into a
 * temporary (the fix of rankrev.hpp:146); fix_j == 0 reproduces the reference
 * as written.  threshold is clamped to >= 1 like rankrev.hpp:232. */
int orc_pluq_tile_recursive(const orc_field *F, uint32_t *a, size_t m, size_t n, size_t lda,
                            size_t threshold, int fix_j, uint32_t *P, uint32_t *Q,
                            size_t *rank);

/* rankrev.hpp:244-282 (slab iterative) -- used to pin the GPU base-case strategy */
int orc_pluq_slab_iterative(const orc_field *F, uint32_t *a, size_t m, size_t n, size_t lda,
                            size_t k, uint32_t *P, uint32_t *Q, size_t *rank);

/* matrix.hpp:53-68 FNV-1a checksum over (rows, cols, p, entries) */
uint64_t orc_checksum(const uint32_t *a, size_t m, size_t n, size_t lda, uint64_t p);

/* oracle.hpp:198-215: expand packed L\U, multiply, undo P/Q given as arrays.
 * out is m x n (ld n). */
int orc_reconstruct(const orc_field *F, const uint32_t *packed, size_t m, size_t n, size_t lda,
                    const uint32_t *P, const uint32_t *Q, size_t rank, uint32_t *out);

/* generate.hpp:52-96: n x m matrix of the given rank with intended profiles */
int orc_generate_matrix(size_t n, size_t m, size_t rank, uint64_t p, uint64_t seed, uint32_t *out,
                        uint32_t *rows, uint32_t *cols);

/* config-4 generator (this repo's definition):
 * M = L * R * U mod p, L unit lower / U unit upper with SplitMix64 entries,
 * R an n x n 0/1 matrix with r ones at seeded positions (no shared row/col).
 * rows[k], cols[k] (k < r) receive the positions of R's ones. */
int orc_lru_factors(size_t n, size_t r, uint64_t p, uint64_t seed, uint32_t *L, uint32_t *U,
                    uint32_t *rows, uint32_t *cols);
int orc_lru_matrix(size_t n, size_t r, uint64_t p, uint64_t seed, uint32_t *M, uint32_t *rows,
                   uint32_t *cols);

#ifdef __cplusplus
}
#endif
#endif
