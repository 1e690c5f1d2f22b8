// ref_driver.cpp -- extern "C" shim over the UNMODIFIED reference headers
// (proj/include/ffpluq/*.hpp).  TEST INFRASTRUCTURE ONLY.
//
// Built by oracle/build_ref.py into oracle/_ref/ (git-ignored) twice:
//   libffref.so        -- the reference headers exactly as checked in
//   libffref_fixed.so  -- same, with the rankrev.hpp:146 temp-J fix and the
//                         pool.hpp:112-118 notify-under-lock fix applied to a
//                         copy under oracle/_ref/include_fixed/ 
// Used to pin oracle/oracle.c (tests/golden/) and as the CPU baseline / the
// `bench.py --impl reference` arm.  Never linked by the product library.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <vector>

#include "ffpluq/ffpluq.hpp"

using namespace ffpluq;

namespace {

int code_of(const std::exception_ptr& e, size_t* bad) {
    try {
        std::rethrow_exception(e);
    } catch (const ZeroDivision&) {
        return 1;
    } catch (const CapacityError&) {
        return 2;
    } catch (const DimMismatch&) {
        return 3;
    } catch (const EmptyMatrix&) {
        return 4;
    } catch (const ZeroPivot&) {
        return 5;
    } catch (const SingularDiagonal& s) {
        if (bad) *bad = s.index;
        return 6;
    } catch (const NotRankRevealing&) {
        return 7;
    } catch (const InvalidBlock&) {
        return 8;
    } catch (const InvalidDim&) {
        return 9;
    } catch (const InvalidRank&) {
        return 10;
    } catch (...) {
        return 99;
    }
}

Mat load(const PrimeField& F, const uint32_t* a, size_t m, size_t n, size_t lda) {
    Mat M(m, n, F);
    for (size_t i = 0; i < m; ++i) std::memcpy(M.row(i), a + i * lda, n * sizeof(uint32_t));
    return M;
}

void store(const Mat& M, uint32_t* a, size_t lda) {
    for (size_t i = 0; i < M.rows(); ++i) std::memcpy(a + i * lda, M.row(i), M.cols() * sizeof(uint32_t));
}

void out_arrays(const PluqResult& res, uint32_t* P, uint32_t* Q, size_t* rank) {
    if (P) {
        auto v = res.P.to_array();
        std::memcpy(P, v.data(), v.size() * sizeof(uint32_t));
    }
    if (Q) {
        auto v = res.Q.to_array();
        std::memcpy(Q, v.data(), v.size() * sizeof(uint32_t));
    }
    if (rank) *rank = res.rank;
}

}  // namespace

extern "C" {

int ref_set_workers(unsigned w) {
    set_workers(w);
    return 0;
}

int ref_random_mat(uint64_t p, size_t m, size_t n, uint64_t seed, uint32_t* out) {
    try {
        PrimeField F(p);
        SplitMix64 rng(seed);  // test_util.hpp:22-28
        for (size_t i = 0; i < m * n; ++i) out[i] = elem(rng.below(F.p));
        return 0;
    } catch (...) {
        return code_of(std::current_exception(), nullptr);
    }
}

int ref_generate_matrix(uint64_t p, size_t n, size_t m, size_t rank, uint64_t seed, uint32_t* out,
                        uint32_t* rows, uint32_t* cols) {
    try {
        PrimeField F(p);
        auto g = generate_matrix(n, m, rank, F, seed);
        store(g.A, out, m);
        if (rows) std::memcpy(rows, g.intended.rows.data(), rank * sizeof(uint32_t));
        if (cols) std::memcpy(cols, g.intended.cols.data(), rank * sizeof(uint32_t));
        return 0;
    } catch (...) {
        return code_of(std::current_exception(), nullptr);
    }
}

int ref_fgemm(uint64_t p, int acc_bits, uint32_t alpha, const uint32_t* A, size_t lda, const uint32_t* B,
              size_t ldb, uint32_t beta, uint32_t* C, size_t ldc, size_t m, size_t n, size_t k) {
    try {
        PrimeField F(p, acc_bits);
        Mat a = load(F, A, m, k, lda), b = load(F, B, k, n, ldb), c = load(F, C, m, n, ldc);
        fgemm_classical(alpha, a.view(), b.view(), beta, c.view());
        store(c, C, ldc);
        return 0;
    } catch (...) {
        return code_of(std::current_exception(), nullptr);
    }
}

int ref_ftrsm(uint64_t p, int side, int uplo, int diag, const uint32_t* A, size_t lda, size_t t,
              uint32_t* B, size_t ldb, size_t m, size_t n, size_t* bad_index) {
    try {
        PrimeField F(p);
        Mat a = load(F, A, t, t, lda), b = load(F, B, m, n, ldb);
        ftrsm(side ? Side::right : Side::left, uplo ? UpLo::upper : UpLo::lower,
              diag ? Diag::nonunit : Diag::unit, a.view(), b.view());
        store(b, B, ldb);
        return 0;
    } catch (...) {
        return code_of(std::current_exception(), bad_index);
    }
}

int ref_rr_base(uint64_t p, uint32_t* a, size_t m, size_t n, size_t lda, uint32_t* P, uint32_t* Q,
                size_t* rank) {
    try {
        PrimeField F(p);
        Mat M = load(F, a, m, n, lda);
        auto res = rr_base(M.view());
        store(M, a, lda);
        out_arrays(res, P, Q, rank);
        return 0;
    } catch (...) {
        return code_of(std::current_exception(), nullptr);
    }
}

// pluq_tile_recursive (rankrev.hpp:229-233); seconds receives the wall time of
// the factorization call alone, timed like proj/tools/ffpluq.cpp:182-189.
int ref_pluq_tile_recursive(uint64_t p, uint32_t* a, size_t m, size_t n, size_t lda, size_t thr,
                            unsigned workers, uint32_t* P, uint32_t* Q, size_t* rank, double* seconds) {
    try {
        PrimeField F(p);
        Mat M = load(F, a, m, n, lda);
        const auto t0 = std::chrono::steady_clock::now();
        auto res = pluq_tile_recursive(M.view(), thr, {}, workers);
        const auto t1 = std::chrono::steady_clock::now();
        if (seconds) *seconds = std::chrono::duration<double>(t1 - t0).count();
        store(M, a, lda);
        out_arrays(res, P, Q, rank);
        return 0;
    } catch (...) {
        return code_of(std::current_exception(), nullptr);
    }
}

int ref_pluq_slab_iterative(uint64_t p, uint32_t* a, size_t m, size_t n, size_t lda, size_t k,
                            uint32_t* P, uint32_t* Q, size_t* rank) {
    try {
        PrimeField F(p);
        Mat M = load(F, a, m, n, lda);
        auto res = pluq_slab_iterative(M.view(), k, {}, 1);
        store(M, a, lda);
        out_arrays(res, P, Q, rank);
        return 0;
    } catch (...) {
        return code_of(std::current_exception(), nullptr);
    }
}

// pfgemm timing leg for the fgemm metric (blas.hpp:250-271)
int ref_pfgemm_timed(uint64_t p, uint32_t alpha, const uint32_t* A, const uint32_t* B, uint32_t beta,
                     uint32_t* C, size_t m, size_t n, size_t k, unsigned workers, double* seconds) {
    try {
        PrimeField F(p);
        Mat a = load(F, A, m, k, k), b = load(F, B, k, n, n), c = load(F, C, m, n, n);
        set_workers(workers);
        const auto t0 = std::chrono::steady_clock::now();
        pfgemm(alpha, a.view(), b.view(), beta, c.view(), {}, workers);
        const auto t1 = std::chrono::steady_clock::now();
        if (seconds) *seconds = std::chrono::duration<double>(t1 - t0).count();
        store(c, C, n);
        return 0;
    } catch (...) {
        return code_of(std::current_exception(), nullptr);
    }
}

uint64_t ref_checksum(uint64_t p, const uint32_t* a, size_t m, size_t n, size_t lda) {
    PrimeField F(p);
    Mat M = load(F, a, m, n, lda);
    return checksum(M.view());
}

int ref_naive_rank_profiles(uint64_t p, const uint32_t* a, size_t m, size_t n, uint32_t* rows,
                            uint32_t* cols, size_t* rank) {
    try {
        PrimeField F(p);
        Mat M = load(F, a, m, n, n);
        auto prof = naive_rank_profiles(M.view());
        std::memcpy(rows, prof.rows.data(), prof.rows.size() * sizeof(uint32_t));
        std::memcpy(cols, prof.cols.data(), prof.cols.size() * sizeof(uint32_t));
        *rank = prof.rank;
        return 0;
    } catch (...) {
        return code_of(std::current_exception(), nullptr);
    }
}

}  // extern "C"
