// rpsim.cu -- tile_rec's permutations from the rank profile matrix alone (host code).
//
// tile_rec (rankrev.hpp:85-183) decides every block shape and every permutation move from the
// zero pattern of the Schur complements it visits, and those patterns are fixed by the rank
// profile matrix R_A (the 0/1 matrix with a one at each pivot (P[k], Q[k]), k < rank; Dumas,
// Pernet, Sultan -- every rank-profile-revealing elimination reveals the same R_A).  So tile_rec
// run on R_A itself produces the same P, Q arrays as on A (tests/test_profile.py checks this
// against the reference on random, rank-deficient and small-field inputs).  On a partial
// permutation matrix the recursion is pure index work: a pivot's row and column hold no other
// one, so every TRSM / GEMM of tile_rec is a no-op, each Schur complement is the input with the
// pivot rows and columns removed, and only the ones (points) still live in E, G and R move.
//
// sim() restates tile_rec on the points of a node: the split m1 = ceil(m/2), n1 = ceil(n/2)
// (:95), the base case iff min(m, n) <= thr (:92) as rr_base's outcome (rankrev.hpp:29-78:
// pivot rows in row order, each at its only point; P = [pivot rows, the other rows ascending],
// Q = [pivot columns in pivot order, the other columns ascending]), the children's permutations
// applied to the blocks that still hold points (:99-100, :128-133), the PermSeq compositions
// (append_embedded, :163-170) and the pivot gathers (push_rot_block, :174-179), all on
// PermSeq::to_array() index arrays (perm.hpp:88-95).  A node without points is rank 0 with
// identity permutations and is never visited, so the work is O(rank * depth) plus the arrays of
// the nodes that hold points.
#include <algorithm>
#include <cstdint>
#include <numeric>
#include <vector>

#include "common.cuh"
#include "profile.cuh"

namespace ffg {
namespace {

struct Pt {
    uint32_t i, j;
};

struct Sim {
    size_t thr;
    std::vector<uint32_t> inv;  // scratch: inverse of a child's array

    // P (m words) and Q (n words) receive the node's to_array() forms; pts is non-empty
    size_t node(std::vector<Pt>& pts, size_t m, size_t n, uint32_t* P, uint32_t* Q) {
        if (std::min(m, n) <= thr) return base(pts, m, n, P, Q);
        const size_t m1 = (m + 1) / 2, n1 = (n + 1) / 2;
        std::vector<Pt> a1, tr, bl, br;
        for (const Pt& t : pts) {
            if (t.i < m1)
                (t.j < n1 ? a1 : tr).push_back(t);
            else
                (t.j < n1 ? bl : br).push_back(t);
        }
        std::vector<Pt>().swap(pts);
        // A1 (:97) and the row / column moves it sends to its right and lower neighbours (:99-100)
        std::vector<uint32_t> P1, Q1;
        size_t r1 = 0;
        if (!a1.empty()) {
            P1.resize(m1);
            Q1.resize(n1);
            r1 = node(a1, m1, n1, P1.data(), Q1.data());
            if (!tr.empty()) {
                invert(P1.data(), m1);
                for (Pt& t : tr) t.i = inv[t.i];
            }
            if (!bl.empty()) {
                invert(Q1.data(), n1);
                for (Pt& t : bl) t.j = inv[t.j];
            }
        }
        // E = rows r1.. of the top-right block, G = columns r1.. of the bottom-left one (:102-109);
        // the rows above E are A1's pivot rows and the columns left of G its pivot columns
        for (Pt& t : tr) {
            if (t.i < r1) throw Error(FFG_ERR_INTERNAL, "rank profile: a point in D");
            t.i -= (uint32_t)r1;
            t.j -= (uint32_t)n1;
        }
        for (Pt& t : bl) {
            if (t.j < r1) throw Error(FFG_ERR_INTERNAL, "rank profile: a point in Fb");
            t.i -= (uint32_t)m1;
            t.j -= (uint32_t)r1;
        }
        const size_t em = m1 - r1, en = n - n1, gm = m - m1, gn = n1 - r1;
        std::vector<uint32_t> P2, Q2, P3, Q3;
        size_t r2 = 0, r3 = 0;
        if (!tr.empty()) {  // :121
            P2.resize(em);
            Q2.resize(en);
            r2 = node(tr, em, en, P2.data(), Q2.data());
        }
        if (!bl.empty()) {  // :122
            P3.resize(gm);
            Q3.resize(gn);
            r3 = node(bl, gm, gn, P3.data(), Q3.data());
        }
        // E's column moves and G's row moves reach H (:130-132); R = H minus the rows of G's
        // pivots and the columns of E's pivots (:142)
        if (!br.empty() && r2) {
            invert(Q2.data(), en);
            for (Pt& t : br) t.j = (uint32_t)n1 + inv[t.j - n1];
        }
        if (!br.empty() && r3) {
            invert(P3.data(), gm);
            for (Pt& t : br) t.i = (uint32_t)m1 + inv[t.i - m1];
        }
        for (Pt& t : br) {
            if (t.i < m1 + r3 || t.j < n1 + r2) throw Error(FFG_ERR_INTERNAL, "rank profile: a point in I, K or N");
            t.i -= (uint32_t)(m1 + r3);
            t.j -= (uint32_t)(n1 + r2);
        }
        const size_t rm = m - m1 - r3, rn = n - n1 - r2;
        std::vector<uint32_t> P4, Q4;
        size_t r4 = 0;
        if (!br.empty()) {  // :154
            P4.resize(rm);
            Q4.resize(rn);
            r4 = node(br, rm, rn, P4.data(), Q4.data());
        }
        // res.P / res.Q = the children's moves embedded in order (:163-170), then the gathers
        std::iota(P, P + m, 0u);
        if (!P1.empty()) std::copy(P1.begin(), P1.end(), P);
        embed(P, r1, P2);
        embed(P, m1, P3);
        embed(P, m1 + r3, P4);
        std::rotate(P + r1 + r2, P + m1, P + m1 + r3 + r4);  // :174
        std::iota(Q, Q + n, 0u);
        if (!Q1.empty()) std::copy(Q1.begin(), Q1.end(), Q);
        embed(Q, r1, Q3);
        embed(Q, n1, Q2);
        embed(Q, n1 + r2, Q4);
        std::rotate(Q + r1, Q + n1, Q + n1 + r2);                  // :176
        std::rotate(Q + r1 + r2 + r3, Q + n1 + r2, Q + n1 + r2 + r4);  // :178
        return r1 + r2 + r3 + r4;
    }

    // rr_base on a partial permutation matrix (rankrev.hpp:40-75): rows in order, the pivot of a
    // row is its only point; rotations keep the other rows / columns in ascending order
    size_t base(std::vector<Pt>& pts, size_t m, size_t n, uint32_t* P, uint32_t* Q) {
        std::sort(pts.begin(), pts.end(), [](const Pt& a, const Pt& b) { return a.i < b.i; });
        std::vector<uint8_t> rused(m, 0), cused(n, 0);
        size_t r = 0;
        for (const Pt& t : pts) {
            if (t.i >= m || t.j >= n || rused[t.i] || cused[t.j])
                throw Error(FFG_ERR_INTERNAL, "rank profile: not a partial permutation");
            rused[t.i] = cused[t.j] = 1;
            P[r] = t.i;
            Q[r] = t.j;
            ++r;
        }
        size_t k = r;
        for (size_t i = 0; i < m; ++i)
            if (!rused[i]) P[k++] = (uint32_t)i;
        k = r;
        for (size_t j = 0; j < n; ++j)
            if (!cused[j]) Q[k++] = (uint32_t)j;
        return r;
    }

    void invert(const uint32_t* a, size_t len) {
        if (inv.size() < len) inv.resize(len);
        for (size_t t = 0; t < len; ++t) inv[a[t]] = (uint32_t)t;
    }
    // moves of a child acting on [at, at + c.size()) after the earlier ones: v[at + t] = v[at + c[t]]
    void embed(uint32_t* v, size_t at, const std::vector<uint32_t>& c) {
        if (c.empty()) return;
        tmp.assign(v + at, v + at + c.size());
        for (size_t t = 0; t < c.size(); ++t) v[at + t] = tmp[c[t]];
    }
    std::vector<uint32_t> tmp;
};

}  // namespace

size_t tile_rec_perms(size_t m, size_t n, size_t thr, size_t rank, const uint32_t* prow, const uint32_t* pcol,
                      uint32_t* P, uint32_t* Q) {
    if (rank > std::min(m, n)) throw Error(FFG_ERR_INVALID_RANK, "rank profile: rank exceeds min(m, n)");
    std::vector<Pt> pts(rank);
    for (size_t k = 0; k < rank; ++k) pts[k] = Pt{prow[k], pcol[k]};
    if (m) std::iota(P, P + m, 0u);
    if (n) std::iota(Q, Q + n, 0u);
    if (rank == 0) return 0;
    Sim s;
    s.thr = std::max<size_t>(1, thr);
    return s.node(pts, m, n, P, Q);
}

}  // namespace ffg
