/*
 * oracle.c -- CPU restatement of the reference ffpluq hot path.
 *
 * TEST INFRASTRUCTURE ONLY: the parity checker for the B200 library, never
 * part of the product path (see oracle.h).  Plain C11, scalar, single thread.
 *
 * References (file:line) are into the reference checkout,
 * proj/include/ffpluq/*.hpp unless stated otherwise.
 */
#include "oracle.h"

#include <stdlib.h>
#include <string.h>
#include <stdio.h>

typedef uint32_t u32;
typedef uint64_t u64;
typedef int64_t i64;

/* ------------------------------------------------------------------------ */
/* field.hpp                                                                 */

static int is_prime_u64(u64 n) /* field.hpp:19-24 */
{
    if (n < 2) return 0;
    for (u64 d = 2; d * d <= n; ++d)
        if (n % d == 0) return 0;
    return 1;
}

int orc_field_init(orc_field *F, u64 p, int acc_bits) /* field.hpp:28-54 */
{
    if (p < 2 || p >= ((u64)1 << 26)) return ORC_CAPACITY;
    if (!is_prime_u64(p)) return ORC_CAPACITY;
    if (acc_bits < 2 || acc_bits > 62) return ORC_CAPACITY;
    const u64 cap = ((u64)1 << acc_bits) - 1;
    const u64 d = (p - 1) * (p - 1);
    if (d > cap) return ORC_CAPACITY;
    F->p = p;
    F->acc_bits = acc_bits;
    F->n_star = cap / d;
    F->n_star_seeded = (cap - (p - 1)) / d;
    return ORC_OK;
}

static inline u32 residue(const orc_field *F, i64 acc) /* field.hpp:85-89 */
{
    i64 r = acc % (i64)F->p;
    if (r < 0) r += (i64)F->p;
    return (u32)r;
}

static inline u32 fmul(const orc_field *F, u32 a, u32 b) { return (u32)(((u64)a * b) % F->p); }
static inline u32 fadd(const orc_field *F, u32 a, u32 b)
{
    u64 s = (u64)a + b;
    if (s >= F->p) s -= F->p;
    return (u32)s;
}

u32 orc_inv(const orc_field *F, u32 a) /* field.hpp:91-107 extended Euclid */
{
    i64 t = 0, newt = 1, r = (i64)F->p, newr = (i64)a;
    while (newr != 0) {
        i64 q = r / newr, tmp = t - q * newt;
        t = newt;
        newt = tmp;
        tmp = r - q * newr;
        r = newr;
        newr = tmp;
    }
    if (t < 0) t += (i64)F->p;
    return (u32)t;
}

/* ------------------------------------------------------------------------ */
/* generate.hpp:10-24 SplitMix64; test_util.hpp:22-28                        */

static inline u64 mix64(u64 z)
{
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

u64 orc_splitmix_at(u64 seed, u64 k) { return mix64(seed + (k + 1) * 0x9e3779b97f4a7c15ull); }

void orc_random_mat(u32 *a, size_t m, size_t n, size_t lda, u64 p, u64 seed)
{
    u64 k = 0;
    for (size_t i = 0; i < m; ++i)
        for (size_t j = 0; j < n; ++j) a[i * lda + j] = (u32)(orc_splitmix_at(seed, k++) % p);
}

/* ------------------------------------------------------------------------ */
/* blas.hpp:31-103 fgemm_classical                                           */

int orc_fgemm(const orc_field *F, u32 alpha, const u32 *A, size_t lda, const u32 *B, size_t ldb,
              u32 beta, u32 *C, size_t ldc, size_t m, size_t n, size_t kk)
{
    if (m == 0 || n == 0) return ORC_OK;
    if (beta != 0 && beta != 1) { /* :39-45 */
        for (size_t i = 0; i < m; ++i)
            for (size_t j = 0; j < n; ++j) C[i * ldc + j] = fmul(F, beta, C[i * ldc + j]);
        beta = 1;
    }
    if (alpha == 0 || kk == 0) { /* :46-51 */
        if (beta == 0)
            for (size_t i = 0; i < m; ++i)
                for (size_t j = 0; j < n; ++j) C[i * ldc + j] = 0;
        return ORC_OK;
    }
    const int negate = (alpha == F->p - 1 && F->p > 2); /* :53-55 */
    const int plain = (alpha == 1) || negate;
    const u64 chunk = F->n_star < 1 ? 1 : F->n_star;
    i64 *acc = (i64 *)malloc(n * sizeof(i64));
    if (!acc) return ORC_NO_MEMORY;
    for (size_t i = 0; i < m; ++i) {
        const u32 *arow = A + i * lda;
        u32 *crow = C + i * ldc;
        for (size_t j = 0; j < n; ++j) acc[j] = (plain && beta == 1) ? (i64)crow[j] : 0;
        size_t t0 = 0;
        while (t0 < kk) { /* :66-89 chunks of n_star products, intermediate folds */
            size_t t1 = (kk - t0 > chunk) ? t0 + (size_t)chunk : kk;
            for (size_t t = t0; t < t1; ++t) {
                const u64 av = arow[t];
                if (!av) continue;
                const u32 *brow = B + t * ldb;
                if (negate)
                    for (size_t j = 0; j < n; ++j) acc[j] -= (i64)(av * brow[j]);
                else
                    for (size_t j = 0; j < n; ++j) acc[j] += (i64)(av * brow[j]);
            }
            t0 = t1;
            if (t0 < kk)
                for (size_t j = 0; j < n; ++j) acc[j] = (i64)residue(F, acc[j]);
        }
        if (plain) { /* :91-101 */
            for (size_t j = 0; j < n; ++j) crow[j] = residue(F, acc[j]);
        } else {
            for (size_t j = 0; j < n; ++j) {
                u32 v = fmul(F, alpha, residue(F, acc[j]));
                crow[j] = (beta == 1) ? fadd(F, crow[j], v) : v;
            }
        }
    }
    free(acc);
    return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* blas.hpp:285-398 ftrsm                                                    */

static int trsm_left(const orc_field *F, int upper, int nonunit, const u32 *A, size_t lda, u32 *B,
                     size_t ldb, size_t t, size_t n) /* blas.hpp:285-338 */
{
    u32 *dinv = NULL;
    if (nonunit) {
        dinv = (u32 *)malloc(t * sizeof(u32));
        for (size_t i = 0; i < t; ++i) dinv[i] = orc_inv(F, A[i * lda + i]);
    }
    i64 *acc = (i64 *)malloc((n ? n : 1) * sizeof(i64));
    const u64 budget = F->n_star_seeded < 1 ? 1 : F->n_star_seeded;
    for (size_t step = 0; step < t; ++step) {
        const size_t r = upper ? t - 1 - step : step;
        const u32 *arow = A + r * lda;
        u32 *xr = B + r * ldb;
        if (step == 0) {
            if (nonunit)
                for (size_t j = 0; j < n; ++j) xr[j] = fmul(F, xr[j], dinv[r]);
            continue;
        }
        for (size_t j = 0; j < n; ++j) acc[j] = (i64)xr[j];
        u64 folded = 0;
        size_t s0 = upper ? r + 1 : 0, s1 = upper ? t : r;
        for (size_t s = s0; s < s1; ++s) {
            const u64 av = arow[s];
            if (av) {
                const u32 *xs = B + s * ldb;
                for (size_t j = 0; j < n; ++j) acc[j] -= (i64)(av * xs[j]);
            }
            if (++folded == budget) {
                for (size_t j = 0; j < n; ++j) acc[j] = (i64)residue(F, acc[j]);
                folded = 0;
            }
        }
        for (size_t j = 0; j < n; ++j) {
            u32 v = residue(F, acc[j]);
            xr[j] = nonunit ? fmul(F, v, dinv[r]) : v;
        }
    }
    free(acc);
    free(dinv);
    return ORC_OK;
}

static int trsm_right(const orc_field *F, int upper, int nonunit, const u32 *A, size_t lda, u32 *B,
                      size_t ldb, size_t m, size_t t) /* blas.hpp:342-384 */
{
    u32 *dinv = NULL;
    if (nonunit) {
        dinv = (u32 *)malloc(t * sizeof(u32));
        for (size_t i = 0; i < t; ++i) dinv[i] = orc_inv(F, A[i * lda + i]);
    }
    i64 *acc = (i64 *)malloc((t ? t : 1) * sizeof(i64));
    for (size_t r = 0; r < m; ++r) {
        u32 *xr = B + r * ldb;
        for (size_t c = 0; c < t; ++c) acc[c] = (i64)xr[c];
        for (size_t step = 0; step < t; ++step) {
            const size_t c = upper ? step : t - 1 - step;
            u32 v = (step == 0) ? xr[c] : residue(F, acc[c]);
            if (nonunit) v = fmul(F, v, dinv[c]);
            xr[c] = v;
            if (v) {
                const u32 *arow = A + c * lda;
                for (size_t j = step + 1; j < t; ++j) {
                    size_t cc = upper ? j : t - 1 - j;
                    acc[cc] -= (i64)((u64)v * arow[cc]);
                }
            }
        }
    }
    free(acc);
    free(dinv);
    return ORC_OK;
}

int orc_ftrsm(const orc_field *F, int side, int uplo, int diag, const u32 *A, size_t lda, u32 *B,
              size_t ldb, size_t m, size_t n, size_t *bad_index)
{
    /* blas.hpp:389-398: the triangle is t x t with t = B's solved dimension */
    const size_t t = (side == 0) ? m : n;
    if (m == 0 || n == 0 || t == 0) return ORC_OK;
    if (diag == 1) /* blas.hpp:291-297 / 347-353: first zero diagonal wins */
        for (size_t i = 0; i < t; ++i)
            if (A[i * lda + i] % F->p == 0) {
                if (bad_index) *bad_index = i;
                return ORC_SINGULAR_DIAGONAL;
            }
    if (side == 0) return trsm_left(F, uplo == 1, diag == 1, A, lda, B, ldb, t, n);
    return trsm_right(F, uplo == 1, diag == 1, A, lda, B, ldb, m, t);
}

/* ------------------------------------------------------------------------ */
/* perm.hpp: move lists                                                      */

typedef struct {
    u32 type; /* 0 Swap, 1 Rot (perm.hpp:14-18) */
    u32 i, j;
} move_t;

typedef struct {
    size_t n;
    size_t len, cap;
    move_t *mv;
} perm_t;

static void perm_init(perm_t *p, size_t n)
{
    p->n = n;
    p->len = p->cap = 0;
    p->mv = NULL;
}
static void perm_free(perm_t *p)
{
    free(p->mv);
    p->mv = NULL;
    p->len = p->cap = 0;
}
static void perm_push(perm_t *p, u32 type, size_t i, size_t j)
{
    if (i == j) return; /* perm.hpp:34-39 */
    if (p->len == p->cap) {
        p->cap = p->cap ? 2 * p->cap : 16;
        p->mv = (move_t *)realloc(p->mv, p->cap * sizeof(move_t));
    }
    p->mv[p->len].type = type;
    p->mv[p->len].i = (u32)i;
    p->mv[p->len].j = (u32)j;
    p->len++;
}
static void perm_push_rot_block(perm_t *p, size_t first, size_t mid, size_t len) /* :44-46 */
{
    for (size_t t = 0; t < len; ++t) perm_push(p, 1, first + t, mid + t);
}
static void perm_append_embedded(perm_t *p, const perm_t *in, size_t at) /* :49-53 */
{
    for (size_t k = 0; k < in->len; ++k) perm_push(p, in->mv[k].type, in->mv[k].i + at, in->mv[k].j + at);
}
static void perm_to_array(const perm_t *p, u32 *out) /* :60-95 */
{
    for (size_t t = 0; t < p->n; ++t) out[t] = (u32)t;
    for (size_t k = 0; k < p->len; ++k) {
        size_t i = p->mv[k].i, j = p->mv[k].j;
        if (p->mv[k].type == 0) {
            u32 tmp = out[i];
            out[i] = out[j];
            out[j] = tmp;
        } else {
            u32 tmp = out[j];
            for (size_t t = j; t > i; --t) out[t] = out[t - 1];
            out[i] = tmp;
        }
    }
}

typedef struct {
    u32 *d;
    size_t rows, cols, ld;
} view_t;

static view_t sub(view_t a, size_t r0, size_t c0, size_t h, size_t w) /* matrix.hpp:28-36 */
{
    view_t v = {a.d + r0 * a.ld + c0, h, w, a.ld};
    return v;
}

/* perm.hpp:123-161 + 167-193 */
static void apply_move(view_t a, int cols, move_t m, int fwd)
{
    size_t i = m.i, j = m.j;
    if (!cols) {
        if (m.type == 0) {
            for (size_t c = 0; c < a.cols; ++c) {
                u32 t = a.d[i * a.ld + c];
                a.d[i * a.ld + c] = a.d[j * a.ld + c];
                a.d[j * a.ld + c] = t;
            }
        } else if (fwd) {
            u32 *tmp = (u32 *)malloc((a.cols ? a.cols : 1) * sizeof(u32));
            memcpy(tmp, a.d + j * a.ld, a.cols * sizeof(u32));
            for (size_t t = j; t > i; --t) memcpy(a.d + t * a.ld, a.d + (t - 1) * a.ld, a.cols * sizeof(u32));
            memcpy(a.d + i * a.ld, tmp, a.cols * sizeof(u32));
            free(tmp);
        } else {
            u32 *tmp = (u32 *)malloc((a.cols ? a.cols : 1) * sizeof(u32));
            memcpy(tmp, a.d + i * a.ld, a.cols * sizeof(u32));
            for (size_t t = i; t < j; ++t) memcpy(a.d + t * a.ld, a.d + (t + 1) * a.ld, a.cols * sizeof(u32));
            memcpy(a.d + j * a.ld, tmp, a.cols * sizeof(u32));
            free(tmp);
        }
    } else {
        for (size_t r = 0; r < a.rows; ++r) {
            u32 *row = a.d + r * a.ld;
            if (m.type == 0) {
                u32 t = row[i];
                row[i] = row[j];
                row[j] = t;
            } else if (fwd) {
                u32 t = row[j];
                for (size_t q = j; q > i; --q) row[q] = row[q - 1];
                row[i] = t;
            } else {
                u32 t = row[i];
                for (size_t q = i; q < j; ++q) row[q] = row[q + 1];
                row[j] = t;
            }
        }
    }
}

static void apply_perm(const perm_t *p, view_t a, int cols) /* perm.hpp:167-193, forward */
{
    if (a.rows == 0 || a.cols == 0) return;
    for (size_t k = 0; k < p->len; ++k) apply_move(a, cols, p->mv[k], 1);
}

int orc_apply_moves(u32 *a, size_t rows, size_t cols, size_t lda, int axis_cols, int inverse,
                    const u32 *mv_type, const u32 *mv_i, const u32 *mv_j, size_t nmoves)
{
    view_t v = {a, rows, cols, lda};
    for (size_t k = 0; k < nmoves; ++k) {
        size_t idx = inverse ? nmoves - 1 - k : k;
        move_t m = {mv_type[idx], mv_i[idx], mv_j[idx]};
        size_t dim = axis_cols ? cols : rows;
        if (m.i >= dim || m.j >= dim) return ORC_DIM_MISMATCH;
        apply_move(v, axis_cols, m, !inverse);
    }
    return ORC_OK;
}

void orc_moves_to_array(size_t n, const u32 *mv_type, const u32 *mv_i, const u32 *mv_j,
                        size_t nmoves, u32 *out)
{
    perm_t p;
    perm_init(&p, n);
    for (size_t k = 0; k < nmoves; ++k) perm_push(&p, mv_type[k], mv_i[k], mv_j[k]);
    perm_to_array(&p, out);
    perm_free(&p);
}

static void rotate_rows_block(view_t a, size_t first, size_t mid, size_t len) /* perm.hpp:197-207 */
{
    if (len == 0 || mid == first) return;
    const size_t span = mid - first;
    u32 *tmp = (u32 *)malloc((span * a.cols ? span * a.cols : 1) * sizeof(u32));
    for (size_t t = 0; t < span; ++t) memcpy(tmp + t * a.cols, a.d + (first + t) * a.ld, a.cols * sizeof(u32));
    for (size_t t = 0; t < len; ++t) memcpy(a.d + (first + t) * a.ld, a.d + (mid + t) * a.ld, a.cols * sizeof(u32));
    for (size_t t = 0; t < span; ++t) memcpy(a.d + (first + len + t) * a.ld, tmp + t * a.cols, a.cols * sizeof(u32));
    free(tmp);
}

static void rotate_cols_block(view_t a, size_t first, size_t mid, size_t len) /* perm.hpp:209-215 */
{
    if (len == 0 || mid == first) return;
    const size_t span = mid - first;
    u32 *tmp = (u32 *)malloc(span * sizeof(u32));
    for (size_t r = 0; r < a.rows; ++r) {
        u32 *row = a.d + r * a.ld;
        memcpy(tmp, row + first, span * sizeof(u32));
        memmove(row + first, row + mid, len * sizeof(u32));
        memcpy(row + first + len, tmp, span * sizeof(u32));
    }
    free(tmp);
}

/* ------------------------------------------------------------------------ */
/* rankrev.hpp:29-78 rr_base                                                 */

typedef struct {
    perm_t P, Q;
    size_t rank;
} res_t;

static void res_init(res_t *r, size_t m, size_t n)
{
    perm_init(&r->P, m);
    perm_init(&r->Q, n);
    r->rank = 0;
}
static void res_free(res_t *r)
{
    perm_free(&r->P);
    perm_free(&r->Q);
}

/* seed - sum_{t<r} x[t]*y[t*ld] folded to [0,p): the FoldAcc value (pluq.hpp:50-85);
 * the intermediate budget folds never change the residue. */
static u32 crout_entry(const orc_field *F, u32 seed, const u32 *x, const u32 *y, size_t ldy, size_t r)
{
    i64 acc = (i64)seed;
    const u64 budget = F->n_star_seeded < 1 ? 1 : F->n_star_seeded;
    u64 terms = 0;
    for (size_t t = 0; t < r; ++t) {
        acc -= (i64)((u64)x[t] * y[t * ldy]);
        if (++terms == budget) {
            acc = (i64)residue(F, acc);
            terms = 0;
        }
    }
    return residue(F, acc);
}

static void rr_base(const orc_field *F, view_t a, res_t *res)
{
    const size_t m = a.rows, n = a.cols;
    res_init(res, m, n);
    if (m == 0 || n == 0) return;
    size_t r = 0, row = 0;
    while (row < m && r < n) { /* :40 */
        size_t pivcol = n;
        u32 pivval = 0;
        for (size_t j = r; j < n; ++j) { /* :43-53 */
            u32 v = crout_entry(F, a.d[row * a.ld + j], a.d + row * a.ld, a.d + j, a.ld, r);
            a.d[row * a.ld + j] = v;
            if (v) {
                pivcol = j;
                pivval = v;
                break;
            }
        }
        if (pivcol == n) { /* :54-57 */
            ++row;
            continue;
        }
        perm_push(&res->P, 1, r, row); /* :58-61 */
        if (row != r) {
            move_t mv = {1, (u32)r, (u32)row};
            apply_move(a, 0, mv, 1);
        }
        perm_push(&res->Q, 1, r, pivcol);
        if (pivcol != r) {
            move_t mv = {1, (u32)r, (u32)pivcol};
            apply_move(a, 1, mv, 1);
        }
        const u32 ipiv = orc_inv(F, pivval); /* :62 */
        for (size_t j = pivcol + 1; j < n; ++j) /* :63-67 U row */
            a.d[r * a.ld + j] = crout_entry(F, a.d[r * a.ld + j], a.d + r * a.ld, a.d + j, a.ld, r);
        for (size_t i = row + 1; i < m; ++i) /* :68-72 L column */
            a.d[i * a.ld + r] =
                fmul(F, crout_entry(F, a.d[i * a.ld + r], a.d + i * a.ld, a.d + r, a.ld, r), ipiv);
        ++r;
        ++row;
    }
    res->rank = r;
}

int orc_rr_base(const orc_field *F, u32 *a, size_t m, size_t n, size_t lda, u32 *P, u32 *Q, size_t *rank)
{
    view_t v = {a, m, n, lda};
    res_t res;
    rr_base(F, v, &res);
    if (P) perm_to_array(&res.P, P);
    if (Q) perm_to_array(&res.Q, Q);
    if (rank) *rank = res.rank;
    res_free(&res);
    return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* view-level BLAS wrappers used by the recursion                            */

static int empty(view_t v) { return v.rows == 0 || v.cols == 0; }

static void gemm_sub(const orc_field *F, view_t A, view_t B, view_t C) /* C -= A*B */
{
    orc_fgemm(F, (u32)(F->p - 1), A.d, A.ld, B.d, B.ld, 1, C.d, C.ld, C.rows, C.cols, A.cols);
}

static void trsm_left_lower_unit(const orc_field *F, view_t L, view_t B)
{
    trsm_left(F, 0, 0, L.d, L.ld, B.d, B.ld, B.rows, B.cols);
}

static void trsm_right_upper_nonunit(const orc_field *F, view_t U, view_t B)
{
    size_t bad;
    orc_ftrsm(F, 1, 1, 1, U.d, U.ld, B.d, B.ld, B.rows, B.cols, &bad);
}

/* ------------------------------------------------------------------------ */
/* rankrev.hpp:85-183 tile_rec                                               */

static void tile_rec(const orc_field *F, view_t a, size_t thr, int fix_j, res_t *res)
{
    const size_t m = a.rows, n = a.cols;
    if (m == 0 || n == 0) {
        res_init(res, m, n);
        return;
    }
    if ((m < n ? m : n) <= thr) { /* :92 */
        if (getenv("ORC_TRACE")) fprintf(stderr, "base %zu %zu\n", m, n);
        rr_base(F, a, res);
        return;
    }
    res_init(res, m, n);
    const size_t m1 = (m + 1) / 2, n1 = (n + 1) / 2; /* :95 */

    res_t r1s;
    tile_rec(F, sub(a, 0, 0, m1, n1), thr, fix_j, &r1s); /* :97 */
    const size_t r1 = r1s.rank;
    apply_perm(&r1s.P, sub(a, 0, n1, m1, n - n1), 0); /* :99-100 */
    apply_perm(&r1s.Q, sub(a, m1, 0, m - m1, n1), 1);

    view_t L1 = sub(a, 0, 0, r1, r1); /* :102-109 */
    view_t V1 = sub(a, 0, r1, r1, n1 - r1);
    view_t M1 = sub(a, r1, 0, m1 - r1, r1);
    view_t D = sub(a, 0, n1, r1, n - n1);
    view_t E = sub(a, r1, n1, m1 - r1, n - n1);
    view_t Fb = sub(a, m1, 0, m - m1, r1);
    view_t G = sub(a, m1, r1, m - m1, n1 - r1);
    view_t H = sub(a, m1, n1, m - m1, n - n1);

    if (r1 > 0) { /* :111-117 */
        if (!empty(D)) trsm_left_lower_unit(F, L1, D);
        if (!empty(E)) gemm_sub(F, M1, D, E);
        if (!empty(Fb)) trsm_right_upper_nonunit(F, L1, Fb);
        if (!empty(G) && !empty(V1)) gemm_sub(F, Fb, V1, G);
        if (!empty(H)) gemm_sub(F, Fb, D, H);
    }

    res_t r2s, r3s; /* :119-125 (E || G; independent, order irrelevant) */
    tile_rec(F, E, thr, fix_j, &r2s);
    tile_rec(F, G, thr, fix_j, &r3s);
    const size_t r2 = r2s.rank, r3 = r3s.rank;

    apply_perm(&r2s.P, sub(a, r1, 0, m1 - r1, r1), 0); /* :128-133 */
    apply_perm(&r2s.Q, sub(a, 0, n1, r1, n - n1), 1);
    apply_perm(&r2s.Q, sub(a, m1, n1, m - m1, n - n1), 1);
    apply_perm(&r3s.P, sub(a, m1, 0, m - m1, r1), 0);
    apply_perm(&r3s.P, sub(a, m1, n1, m - m1, n - n1), 0);
    apply_perm(&r3s.Q, sub(a, 0, r1, r1, n1 - r1), 1);

    view_t U2 = sub(a, r1, n1, r2, r2); /* :135-142 */
    view_t V2 = sub(a, r1, n1 + r2, r2, n - n1 - r2);
    view_t L3 = sub(a, m1, r1, r3, r3);
    view_t M3 = sub(a, m1 + r3, r1, m - m1 - r3, r3);
    view_t I = sub(a, m1, n1, r3, r2);
    view_t K = sub(a, m1 + r3, n1, m - m1 - r3, r2);
    view_t N = sub(a, m1, n1 + r2, r3, n - n1 - r2);
    view_t R = sub(a, m1 + r3, n1 + r2, m - m1 - r3, n - n1 - r2);

    if (r2 > 0 && !empty(I)) trsm_right_upper_nonunit(F, U2, I); /* :144-145 */
    if (r2 > 0 && !empty(K)) trsm_right_upper_nonunit(F, U2, K);
    u32 *jbuf = NULL;
    view_t J = I;
    if (fix_j && !empty(I)) { /* fix of :146 -- J = L3^-1 I lives in a temporary */
        jbuf = (u32 *)malloc(I.rows * I.cols * sizeof(u32));
        for (size_t i = 0; i < I.rows; ++i) memcpy(jbuf + i * I.cols, I.d + i * I.ld, I.cols * sizeof(u32));
        J.d = jbuf;
        J.ld = I.cols;
    }
    if (r3 > 0 && !empty(J)) trsm_left_lower_unit(F, L3, J); /* :146 */
    if (r3 > 0 && !empty(N)) trsm_left_lower_unit(F, L3, N); /* :147 */
    if (!empty(N) && !empty(J)) gemm_sub(F, J, V2, N);        /* :148 O = N - J*V2 */
    if (!empty(R)) {                                          /* :149-152 */
        if (!empty(K) && !empty(V2)) gemm_sub(F, K, V2, R);
        if (!empty(N)) gemm_sub(F, M3, N, R);
    }
    free(jbuf);

    res_t r4s;
    tile_rec(F, R, thr, fix_j, &r4s); /* :154 */
    const size_t r4 = r4s.rank;
    apply_perm(&r4s.P, sub(a, m1 + r3, 0, m - m1 - r3, r1 + r3), 0); /* :156-161 */
    if (r2 > 0) apply_perm(&r4s.P, sub(a, m1 + r3, n1, m - m1 - r3, r2), 0);
    apply_perm(&r4s.Q, sub(a, 0, n1 + r2, r1, n - n1 - r2), 1);
    if (r2 > 0) apply_perm(&r4s.Q, sub(a, r1, n1 + r2, r2, n - n1 - r2), 1);
    if (r3 > 0) apply_perm(&r4s.Q, sub(a, m1, n1 + r2, r3, n - n1 - r2), 1);

    perm_append_embedded(&res->P, &r1s.P, 0); /* :163-170 */
    perm_append_embedded(&res->P, &r2s.P, r1);
    perm_append_embedded(&res->P, &r3s.P, m1);
    perm_append_embedded(&res->P, &r4s.P, m1 + r3);
    perm_append_embedded(&res->Q, &r1s.Q, 0);
    perm_append_embedded(&res->Q, &r3s.Q, r1);
    perm_append_embedded(&res->Q, &r2s.Q, n1);
    perm_append_embedded(&res->Q, &r4s.Q, n1 + r2);

    perm_push_rot_block(&res->P, r1 + r2, m1, r3 + r4); /* :174-179 pivot gather */
    rotate_rows_block(a, r1 + r2, m1, r3 + r4);
    perm_push_rot_block(&res->Q, r1, n1, r2);
    rotate_cols_block(a, r1, n1, r2);
    perm_push_rot_block(&res->Q, r1 + r2 + r3, n1 + r2, r4);
    rotate_cols_block(a, r1 + r2 + r3, n1 + r2, r4);

    res->rank = r1 + r2 + r3 + r4;
    res_free(&r1s);
    res_free(&r2s);
    res_free(&r3s);
    res_free(&r4s);
}

int orc_pluq_tile_recursive(const orc_field *F, u32 *a, size_t m, size_t n, size_t lda,
                            size_t threshold, int fix_j, u32 *P, u32 *Q, size_t *rank)
{
    view_t v = {a, m, n, lda};
    res_t res;
    tile_rec(F, v, threshold < 1 ? 1 : threshold, fix_j, &res); /* rankrev.hpp:232 */
    if (P) perm_to_array(&res.P, P);
    if (Q) perm_to_array(&res.Q, Q);
    if (rank) *rank = res.rank;
    res_free(&res);
    return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* rankrev.hpp:244-282 slab iterative                                        */

int orc_pluq_slab_iterative(const orc_field *F, u32 *a, size_t m, size_t n, size_t lda, size_t k,
                            u32 *P, u32 *Q, size_t *rank)
{
    view_t A = {a, m, n, lda};
    res_t res;
    res_init(&res, m, n);
    if (k < 1) k = 1;
    size_t R = 0;
    for (size_t s0 = 0; s0 < m && m && n; s0 += k) {
        const size_t kb = (k < m - s0) ? k : m - s0;
        view_t slab = sub(A, s0, 0, kb, n);
        apply_perm(&res.Q, slab, 1);
        if (R > 0) {
            view_t X = sub(A, s0, 0, kb, R);
            trsm_right_upper_nonunit(F, sub(A, 0, 0, R, R), X);
            if (n > R) gemm_sub(F, X, sub(A, 0, R, R, n - R), sub(A, s0, R, kb, n - R));
        }
        res_t s;
        rr_base(F, sub(A, s0, R, kb, n - R), &s);
        apply_perm(&s.P, sub(A, s0, 0, kb, R), 0);
        if (R > 0) apply_perm(&s.Q, sub(A, 0, R, R, n - R), 1);
        perm_append_embedded(&res.P, &s.P, s0);
        perm_append_embedded(&res.Q, &s.Q, R);
        const size_t rs = s.rank;
        if (rs > 0 && s0 > R) {
            perm_push_rot_block(&res.P, R, s0, rs);
            rotate_rows_block(A, R, s0, rs);
        }
        R += rs;
        res_free(&s);
    }
    res.rank = R;
    if (P) perm_to_array(&res.P, P);
    if (Q) perm_to_array(&res.Q, Q);
    if (rank) *rank = R;
    res_free(&res);
    return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* matrix.hpp:53-68                                                          */

uint64_t orc_checksum(const u32 *a, size_t m, size_t n, size_t lda, u64 p)
{
    u64 h = 14695981039346656037ull;
#define MIX(x)                                                                                     \
    do {                                                                                           \
        u64 _x = (x);                                                                              \
        for (int s = 0; s < 64; s += 8) {                                                          \
            h ^= (_x >> s) & 0xff;                                                                 \
            h *= 1099511628211ull;                                                                 \
        }                                                                                          \
    } while (0)
    MIX(m);
    MIX(n);
    MIX(p);
    for (size_t i = 0; i < m; ++i)
        for (size_t j = 0; j < n; ++j) MIX(a[i * lda + j]);
#undef MIX
    return h;
}

/* ------------------------------------------------------------------------ */
/* oracle.hpp:198-215 with P/Q given as to_array() index arrays              */

int orc_reconstruct(const orc_field *F, const u32 *packed, size_t m, size_t n, size_t lda,
                    const u32 *P, const u32 *Q, size_t r, u32 *out)
{
    /* prod = L*U (m x n) in the permuted frame; then out[P[i]][Q[j]] = prod[i][j]
     * (undoing P/Q, perm.hpp:90-95: entry t of the array = original index at position t) */
    const u64 p = F->p;
    for (size_t i = 0; i < m; ++i)
        for (size_t j = 0; j < n; ++j) {
            u64 v = 0;
            size_t kmax = r;
            if (i < kmax) kmax = i + 1; /* L is unit lower: L[i][k]=0 for k>i */
            if (j + 1 < kmax) kmax = j + 1; /* U is upper: U[k][j]=0 for k>j */
            for (size_t k = 0; k < kmax; ++k) {
                u64 l = (k == i) ? 1 : packed[i * lda + k];
                u64 u = packed[k * lda + j];
                v = (v + l * u) % p;
            }
            out[(size_t)P[i] * n + Q[j]] = (u32)v;
        }
    return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* config-4 generator (repo definition)                        */

int orc_lru_factors(size_t n, size_t r, u64 p, u64 seed, u32 *L, u32 *U, u32 *rows, u32 *cols)
{
    if (r > n) return ORC_INVALID_RANK;
    const u64 sL = orc_splitmix_at(seed, 0), sU = orc_splitmix_at(seed, 1), sR = orc_splitmix_at(seed, 2);
    for (size_t i = 0; i < n; ++i)
        for (size_t j = 0; j < n; ++j) {
            const u64 idx = (u64)i * n + j;
            if (L) L[idx] = (j < i) ? (u32)(orc_splitmix_at(sL, idx) % p) : (j == i ? 1u : 0u);
            if (U) U[idx] = (j > i) ? (u32)(orc_splitmix_at(sU, idx) % p) : (j == i ? 1u : 0u);
        }
    /* two Fisher-Yates shuffles from one SplitMix64(sR) stream (generate.hpp:33-40 style),
     * first r entries of each, paired in shuffled order */
    u32 *pr = (u32 *)malloc(n * sizeof(u32)), *pc = (u32 *)malloc(n * sizeof(u32));
    u64 k = 0;
    for (size_t i = 0; i < n; ++i) pr[i] = pc[i] = (u32)i;
    for (size_t i = n; i > 1; --i) {
        size_t s = (size_t)(orc_splitmix_at(sR, k++) % i);
        u32 t = pr[i - 1];
        pr[i - 1] = pr[s];
        pr[s] = t;
    }
    for (size_t i = n; i > 1; --i) {
        size_t s = (size_t)(orc_splitmix_at(sR, k++) % i);
        u32 t = pc[i - 1];
        pc[i - 1] = pc[s];
        pc[s] = t;
    }
    for (size_t t = 0; t < r; ++t) {
        rows[t] = pr[t];
        cols[t] = pc[t];
    }
    free(pr);
    free(pc);
    return ORC_OK;
}

int orc_lru_matrix(size_t n, size_t r, u64 p, u64 seed, u32 *M, u32 *rows, u32 *cols)
{
    u32 *L = (u32 *)malloc(n * n * sizeof(u32)), *U = (u32 *)malloc(n * n * sizeof(u32));
    if (!L || !U) return ORC_NO_MEMORY;
    orc_lru_factors(n, r, p, seed, L, U, rows, cols);
    /* M = sum_t L[:, rows[t]] (x) U[cols[t], :] */
    u64 *acc = (u64 *)calloc(n, sizeof(u64));
    for (size_t i = 0; i < n; ++i) {
        memset(acc, 0, n * sizeof(u64));
        for (size_t t = 0; t < r; ++t) {
            const u64 l = L[(u64)i * n + rows[t]];
            if (!l) continue;
            const u32 *urow = U + (u64)cols[t] * n;
            for (size_t j = 0; j < n; ++j) acc[j] = (acc[j] + l * urow[j]) % p;
        }
        for (size_t j = 0; j < n; ++j) M[(u64)i * n + j] = (u32)acc[j];
    }
    free(acc);
    free(L);
    free(U);
    return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* generate.hpp:33-96 generate_matrix (restated; rows/cols get the intended  */
/* profiles).  n x m output, ld m.                                           */

static void sorted_subset(u64 seed, u64 *k, size_t dim, size_t count, u32 *out) /* generate.hpp:33-40 */
{
    u32 *all = (u32 *)malloc((dim ? dim : 1) * sizeof(u32));
    for (size_t i = 0; i < dim; ++i) all[i] = (u32)i;
    for (size_t i = dim; i > 1; --i) {
        size_t s = (size_t)(orc_splitmix_at(seed, (*k)++) % i);
        u32 t = all[i - 1];
        all[i - 1] = all[s];
        all[s] = t;
    }
    /* sort the first count entries (insertion sort; small) */
    for (size_t i = 1; i < count; ++i) {
        u32 v = all[i];
        size_t j = i;
        while (j > 0 && all[j - 1] > v) {
            all[j] = all[j - 1];
            --j;
        }
        all[j] = v;
    }
    memcpy(out, all, count * sizeof(u32));
    free(all);
}

int orc_generate_matrix(size_t n, size_t m, size_t rank, u64 p, u64 seed, u32 *out, u32 *rows, u32 *cols)
{
    if (rank > (n < m ? n : m)) return ORC_INVALID_RANK;
    u64 k = 0; /* position in the SplitMix64(seed) stream */
    u32 *R = (u32 *)malloc((rank ? rank : 1) * sizeof(u32)), *Cc = (u32 *)malloc((rank ? rank : 1) * sizeof(u32));
    sorted_subset(seed, &k, n, rank, R);
    sorted_subset(seed, &k, m, rank, Cc);
    u32 *X = (u32 *)calloc(n * (rank ? rank : 1), sizeof(u32)), *Y = (u32 *)calloc((rank ? rank : 1) * m, sizeof(u32));
    size_t t = 0;
    for (size_t i = 0; i < n; ++i) { /* :61-71 */
        const int is_pivot = t < rank && R[t] == i;
        for (size_t u = 0; u < t; ++u) X[i * rank + u] = (u32)(orc_splitmix_at(seed, k++) % p);
        if (is_pivot) {
            X[i * rank + t] = 1;
            ++t;
        }
    }
    t = 0;
    for (size_t j = 0; j < m; ++j) { /* :72-82 */
        const int is_pivot = t < rank && Cc[t] == j;
        for (size_t u = 0; u < t; ++u) Y[u * m + j] = (u32)(orc_splitmix_at(seed, k++) % p);
        if (is_pivot) {
            Y[t * m + j] = (u32)(1 + orc_splitmix_at(seed, k++) % (p - 1));
            ++t;
        }
    }
    for (size_t i = 0; i < n; ++i) /* :85-91 */
        for (size_t j = 0; j < m; ++j) {
            u64 v = 0;
            for (size_t u = 0; u < rank; ++u) v = (v + (u64)X[i * rank + u] * Y[u * m + j]) % p;
            out[i * m + j] = (u32)v;
        }
    if (rows) memcpy(rows, R, rank * sizeof(u32));
    if (cols) memcpy(cols, Cc, rank * sizeof(u32));
    free(R);
    free(Cc);
    free(X);
    free(Y);
    return ORC_OK;
}
