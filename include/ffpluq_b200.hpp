// ffpluq_b200.hpp -- header-only C++ mirror of the reference API over the C ABI (ffg.h).
//
// A user of the reference (proj/include/ffpluq/*.hpp) replaces
//     #include "ffpluq/ffpluq.hpp"            ffpluq::pluq_tile_recursive(a.view(), thr)
// with
//     #include "ffpluq_b200.hpp"              ffpluq_b200::pluq_tile_recursive(view, thr)
// Same argument meaning, same in-place packed output, same P/Q (as PermSeq-style Rot moves whose
// to_array() equals the reference's), same exception names (errors.hpp:9-59).  Link with
// -lffg_b200 (paper_1402_3501_b200/libffg_b200.so).
#pragma once

#include <cstddef>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "ffg.h"

namespace ffpluq_b200 {

using u32 = std::uint32_t;
using usize = std::size_t;

struct ZeroDivision : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct CapacityError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct DimMismatch : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct EmptyMatrix : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct SingularDiagonal : std::runtime_error {
    std::size_t index;
    SingularDiagonal(const std::string& w, std::size_t i) : std::runtime_error(w), index(i) {}
};
struct DeviceError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

inline void check(int rc) {
    if (rc == FFG_OK) return;
    const std::string msg = ffg_last_error();
    switch (rc) {
        case FFG_ERR_ZERO_DIVISION: throw ZeroDivision(msg);
        case FFG_ERR_CAPACITY: throw CapacityError(msg);
        case FFG_ERR_DIM_MISMATCH: throw DimMismatch(msg);
        case FFG_ERR_EMPTY_MATRIX: throw EmptyMatrix(msg);
        case FFG_ERR_SINGULAR_DIAGONAL: throw SingularDiagonal(msg, ffg_last_error_index());
        default: throw DeviceError(msg);
    }
}

// matrix.hpp:13-43 MatView (host memory, row-major u32 residues); the modulus travels with it
struct MatView {
    u32* data = nullptr;
    usize rows = 0, cols = 0, stride = 0;
    std::uint64_t p = 2;
};

// perm.hpp:14-119, reduced to what a PLUQ result needs: Rot moves and to_array()
struct PermMove {
    enum Type : u32 { Swap, Rot } type;
    u32 i, j;
};
class PermSeq {
public:
    PermSeq() = default;
    explicit PermSeq(usize n) : size_(n) {}
    // the order-preserving rotations realizing an array whose first `r` entries are pivots
    // and whose remaining entries ascend (every PLUQ result has that shape)
    static PermSeq from_pivot_array(const std::vector<u32>& arr) {
        PermSeq s(arr.size());
        std::vector<u32> cur(arr.size());
        for (usize t = 0; t < cur.size(); ++t) cur[t] = (u32)t;
        for (usize t = 0; t < arr.size(); ++t) {
            usize j = t;
            while (cur[j] != arr[t]) ++j;
            if (j != t) {
                s.moves_.push_back({PermMove::Rot, (u32)t, (u32)j});
                const u32 v = cur[j];
                for (usize q = j; q > t; --q) cur[q] = cur[q - 1];
                cur[t] = v;
            }
        }
        return s;
    }
    usize size() const { return size_; }
    bool is_identity() const { return moves_.empty(); }
    const std::vector<PermMove>& moves() const { return moves_; }
    std::vector<u32> to_array() const {
        std::vector<u32> v(size_);
        for (usize t = 0; t < size_; ++t) v[t] = (u32)t;
        for (const auto& m : moves_) {
            if (m.type == PermMove::Swap) {
                std::swap(v[m.i], v[m.j]);
            } else {
                const u32 tmp = v[m.j];
                for (usize t = m.j; t > m.i; --t) v[t] = v[t - 1];
                v[m.i] = tmp;
            }
        }
        return v;
    }

private:
    usize size_ = 0;
    std::vector<PermMove> moves_;
};

// pluq.hpp:12-19
struct PluqResult {
    PermSeq P, Q;
    usize rank = 0;
    bool rank_revealing = true;
};

class Context {
public:
    explicit Context(int device = 0) { check(ffg_create(&h_, device)); }
    ~Context() { ffg_destroy(h_); }
    Context(const Context&) = delete;
    Context& operator=(const Context&) = delete;
    ffg_ctx* get() const { return h_; }
    static Context& global() {
        static Context c(0);
        return c;
    }

private:
    ffg_ctx* h_ = nullptr;
};

// rankrev.hpp:229-233 (threshold clamped to >= 1 inside the library)
inline PluqResult pluq_tile_recursive(MatView a, usize threshold = 8, Context& ctx = Context::global()) {
    std::vector<u32> P(a.rows ? a.rows : 1), Q(a.cols ? a.cols : 1);
    usize r = 0;
    check(ffg_pluq_tile_recursive(ctx.get(), a.p, a.data, a.rows, a.cols, a.stride, threshold, P.data(), Q.data(), &r));
    P.resize(a.rows);
    Q.resize(a.cols);
    return PluqResult{PermSeq::from_pivot_array(P), PermSeq::from_pivot_array(Q), r, true};
}

// Byte storage for p <= 256 (BASELINE config 5; an extension -- the reference stores u32 only)
inline PluqResult pluq_tile_recursive_u8(std::uint8_t* data, usize rows, usize cols, usize stride, u32 p,
                                         usize threshold = 8, Context& ctx = Context::global()) {
    std::vector<u32> P(rows ? rows : 1), Q(cols ? cols : 1);
    usize r = 0;
    check(ffg_pluq_tile_recursive_u8(ctx.get(), p, data, rows, cols, stride, threshold, P.data(), Q.data(), &r));
    P.resize(rows);
    Q.resize(cols);
    return PluqResult{PermSeq::from_pivot_array(P), PermSeq::from_pivot_array(Q), r, true};
}

// rankrev.hpp:29-78
inline PluqResult rr_base(MatView a, Context& ctx = Context::global()) {
    std::vector<u32> P(a.rows ? a.rows : 1), Q(a.cols ? a.cols : 1);
    usize r = 0;
    check(ffg_rr_base(ctx.get(), a.p, a.data, a.rows, a.cols, a.stride, P.data(), Q.data(), &r));
    P.resize(a.rows);
    Q.resize(a.cols);
    return PluqResult{PermSeq::from_pivot_array(P), PermSeq::from_pivot_array(Q), r, true};
}

// blas.hpp:220-246 fgemm / 31-103 fgemm_classical: C <- alpha*A*B + beta*C
inline void fgemm(u32 alpha, const MatView& A, const MatView& B, u32 beta, MatView C,
                  Context& ctx = Context::global()) {
    if (A.cols != B.rows || C.rows != A.rows || C.cols != B.cols) throw DimMismatch("gemm: non-conforming shapes");
    check(ffg_fgemm(ctx.get(), C.p, alpha, A.data, A.stride, B.data, B.stride, beta, C.data, C.stride, C.rows, C.cols,
                    A.cols));
}

enum class Side { left, right };
enum class UpLo { lower, upper };
enum class Diag { unit, nonunit };

// blas.hpp:389-398 ftrsm
inline void ftrsm(Side side, UpLo uplo, Diag diag, const MatView& A, MatView B, Context& ctx = Context::global()) {
    check(ffg_ftrsm(ctx.get(), B.p, side == Side::right, uplo == UpLo::upper, diag == Diag::nonunit, A.data, A.stride,
                    B.data, B.stride, B.rows, B.cols));
}

}  // namespace ffpluq_b200
