// pluq.cu -- host driver of the tile-recursive PLUQ (rankrev.hpp:85-183, 229-233).
//
// The recursion is copied exactly -- split m1 = ceil(m/2), n1 = ceil(n/2)
// (:95), base case iff min(m, n) <= threshold (:92), the same Schur updates in
// the same order, the same pivot-gather (A1, E, G, R) -- because on rank
// deficient inputs the P/Q arrays depend on that structure.  What changes:
//   * every block operation is a device kernel on the matrix resident in HBM
//     (GEMM/TRSM on tcgen05, permutations as range-limited gathers);
//   * permutations are index arrays in a device LIFO arena; the host only
//     tracks each node's rank and the [lo, hi) range its P/Q actually move,
//     so identity permutations (all of them on generic full-rank input) cost
//     no launch at all;
//   * the one unavoidable device->host sync is the rank of each base case,
//     which decides every later block shape.
// Deliberate deviation: rankrev.hpp:146 overwrites block I with J = L3^-1 I,
// which corrupts the L factor whenever r2 > 0 and r3 > 0;
// here J lives in a temporary, which is what the reference's own comment
// "O = N - J*V2" describes.  Outputs equal the fixed reference everywhere and
// the unmodified reference wherever r2 == 0 or r3 == 0 (all full-rank input).
#include <algorithm>
#include <cstring>
#include <deque>
#include <vector>

#include "pluq.cuh"

namespace ffg {

namespace {

struct Range {
    size_t lo = 0, hi = 0;
    bool empty() const { return hi <= lo; }
    void add(size_t l, size_t h) {
        if (h <= l) return;
        if (empty()) {
            lo = l;
            hi = h;
        } else {
            lo = std::min(lo, l);
            hi = std::max(hi, h);
        }
    }
};

struct NodeRes {
    size_t rank = 0;
    uint32_t* P = nullptr;  // device index arrays (valid inside pr / qr)
    uint32_t* Q = nullptr;
    Range pr, qr;
    Factor* fac = nullptr;  // structure of the leading r x r factor (for TRSMs that use it)
};

// device LIFO arena for permutation index arrays
class PermArena {
public:
    PermArena(size_t words, cudaStream_t st) : st_(st), cap_(words) {
        if (cap_) FFG_CUDA(cudaMallocAsync(&base_, cap_ * 4, st_));
    }
    ~PermArena() {
        if (base_) cudaFreeAsync(base_, st_);
    }
    uint32_t* alloc(size_t words) {
        if (top_ + words > cap_) throw Error(FFG_ERR_INTERNAL, "permutation arena exhausted");
        uint32_t* p = base_ + top_;
        top_ += (words + 31) & ~size_t(31);
        return p;
    }
    size_t mark() const { return top_; }
    void reset(size_t m) { top_ = m; }

private:
    cudaStream_t st_;
    uint32_t* base_ = nullptr;
    size_t cap_ = 0, top_ = 0;
};

struct Driver {
    const Blas& b;
    size_t thr;
    PermArena arena;
    BaseInfo* info_dev = nullptr;
    BaseInfo* info_host = nullptr;
    cudaEvent_t ev = nullptr;
    uint64_t base_cases = 0;
    // factor tree + the base cases' cached factor inverses (live for the whole call)
    std::deque<Factor> factors;
    uint32_t* inv_arena = nullptr;
    size_t inv_cap = 0, inv_top = 0;
    bool use_factors = true;

    Driver(const Blas& bl, size_t t, size_t m, size_t n)
        : b(bl), thr(std::max<size_t>(1, t)), arena(8 * (m + n) + 4096, bl.st) {
        uint32_t* dev = nullptr;
        // the base kernel writes rank + moved ranges straight into host-mapped memory
        info_host = reinterpret_cast<BaseInfo*>(b.ws.mapped_host(sizeof(BaseInfo) / 4 + 2, &dev));
        info_dev = reinterpret_cast<BaseInfo*>(dev);
        ev = b.ws.sync_event();
        // factor-tree TRSM (cached base-case inverses): opt-in, slower than blocked inverses today
        static const bool on = getenv("FFG_FACTOR_TRSM") && atoi(getenv("FFG_FACTOR_TRSM")) != 0;
        use_factors = on;
        if (use_factors) {
            // sum of r^2 over base cases <= min(m, n) * 64; two triangles each, plus one slot of slack
            inv_cap = 2 * (std::min(m, n) * 64 + 64 * 64) + 64;
            FFG_CUDA(cudaMallocAsync(&inv_arena, inv_cap * 4, b.st));
        }
    }
    ~Driver() {
        if (inv_arena) cudaFreeAsync(inv_arena, b.st);
    }

    Factor* new_factor(size_t rank) {
        factors.emplace_back();
        factors.back().rank = rank;
        return &factors.back();
    }

    NodeRes base(DView a, NodeRes res) {
        const size_t rmax = std::min(a.rows, a.cols);
        uint32_t* slot = nullptr;
        if (use_factors && rmax <= 64 && inv_top + 2 * rmax * rmax <= inv_cap) slot = inv_arena + inv_top;
        const bool asked = rr_base_launch(b, a, res.P, res.Q, info_dev, slot);
        FFG_CUDA(cudaEventRecord(ev, b.st));
        FFG_CUDA(cudaEventSynchronize(ev));  // the rank decides every later shape
        ++base_cases;
        res.rank = info_host->rank;
        res.pr = Range{info_host->plo, info_host->phi};
        res.qr = Range{info_host->qlo, info_host->qhi};
        res.fac = new_factor(res.rank);
        if (asked && info_host->cached && res.rank > 0) {
            res.fac->invL = slot;
            res.fac->invU = slot + res.rank * res.rank;
            inv_top += 2 * res.rank * res.rank;
        }
        return res;
    }

    // TRSMs of tile_rec always use a child's leading factor: walk its factor tree when every
    // leaf has cached inverses, else the generic blocked-inverse TRSM
    void trsm_lower_unit(const NodeRes& c, DView L, DView B) {
        if (c.fac && c.fac->complete())
            trsm_factor(b, 0, *c.fac, L, B);
        else
            ftrsm_dev(b, 0, 0, 0, L, B, false);
    }
    void trsm_upper_nonunit(const NodeRes& c, DView U, DView B) {
        if (c.fac && c.fac->complete())
            trsm_factor(b, 1, *c.fac, U, B);
        else
            ftrsm_dev(b, 1, 1, 1, U, B, false);
    }

    void apply(const NodeRes& c, int axis, DView v) {
        const Range& r = axis == 0 ? c.pr : c.qr;
        if (r.empty() || v.empty()) return;
        perm_apply_range(b, v, axis, axis == 0 ? c.P : c.Q, r.lo, r.hi);
    }

    void gemm_sub(DView A, DView B, DView C) { b.gemm(b.F.p - 1, A, B, 1, C); }

    // compose a child's permutation into this node's array at offset off
    void compose(uint32_t* arr, bool& init, size_t len, Range& acc, size_t off, const uint32_t* child,
                 const Range& cr) {
        if (cr.empty()) return;
        if (!init) {
            perm_iota_dev(b, arr, len);
            init = true;
        }
        perm_compose_dev(b, arr, off, child, cr.lo, cr.hi);
        acc.add(off + cr.lo, off + cr.hi);
    }
    void rot(uint32_t* arr, bool& init, size_t len, Range& acc, size_t first, size_t mid, size_t cnt) {
        if (cnt == 0 || mid == first) return;
        if (!init) {
            perm_iota_dev(b, arr, len);
            init = true;
        }
        perm_rot_dev(b, arr, first, mid, cnt);
        acc.add(first, mid + cnt);
    }

    NodeRes rec(DView a) {
        const size_t m = a.rows, n = a.cols;
        NodeRes res;
        res.P = arena.alloc(std::max<size_t>(m, 1));
        res.Q = arena.alloc(std::max<size_t>(n, 1));
        if (m == 0 || n == 0) return res;                        // rankrev.hpp:91
        if (std::min(m, n) <= thr) return base(a, res);          // :92
        const size_t mark = arena.mark();
        const size_t m1 = (m + 1) / 2, n1 = (n + 1) / 2;         // :95

        NodeRes r1s = rec(a.sub(0, 0, m1, n1));                  // :97
        const size_t r1 = r1s.rank;
        apply(r1s, 0, a.sub(0, n1, m1, n - n1));                 // :99
        apply(r1s, 1, a.sub(m1, 0, m - m1, n1));                 // :100

        DView L1 = a.sub(0, 0, r1, r1);                          // :102-109
        DView V1 = a.sub(0, r1, r1, n1 - r1);
        DView M1 = a.sub(r1, 0, m1 - r1, r1);
        DView D = a.sub(0, n1, r1, n - n1);
        DView E = a.sub(r1, n1, m1 - r1, n - n1);
        DView Fb = a.sub(m1, 0, m - m1, r1);
        DView G = a.sub(m1, r1, m - m1, n1 - r1);
        DView H = a.sub(m1, n1, m - m1, n - n1);
        if (r1 > 0) {                                            // :111-117
            if (!D.empty()) trsm_lower_unit(r1s, L1, D);
            if (!E.empty()) gemm_sub(M1, D, E);
            if (!Fb.empty()) trsm_upper_nonunit(r1s, L1, Fb);
            if (!G.empty() && !V1.empty()) gemm_sub(Fb, V1, G);
            if (!H.empty()) gemm_sub(Fb, D, H);
        }

        NodeRes r2s = rec(E);                                    // :119-125 (E, G independent)
        NodeRes r3s = rec(G);
        const size_t r2 = r2s.rank, r3 = r3s.rank;

        apply(r2s, 0, a.sub(r1, 0, m1 - r1, r1));                // :128-133
        apply(r2s, 1, a.sub(0, n1, r1, n - n1));
        apply(r2s, 1, a.sub(m1, n1, m - m1, n - n1));
        apply(r3s, 0, a.sub(m1, 0, m - m1, r1));
        apply(r3s, 0, a.sub(m1, n1, m - m1, n - n1));
        apply(r3s, 1, a.sub(0, r1, r1, n1 - r1));

        DView U2 = a.sub(r1, n1, r2, r2);                        // :135-142
        DView V2 = a.sub(r1, n1 + r2, r2, n - n1 - r2);
        DView L3 = a.sub(m1, r1, r3, r3);
        DView M3 = a.sub(m1 + r3, r1, m - m1 - r3, r3);
        DView I = a.sub(m1, n1, r3, r2);
        DView K = a.sub(m1 + r3, n1, m - m1 - r3, r2);
        DView N = a.sub(m1, n1 + r2, r3, n - n1 - r2);
        DView R = a.sub(m1 + r3, n1 + r2, m - m1 - r3, n - n1 - r2);

        if (r2 > 0 && !I.empty()) trsm_upper_nonunit(r2s, U2, I);    // :144
        if (r2 > 0 && !K.empty()) trsm_upper_nonunit(r2s, U2, K);    // :145
        uint32_t* jbuf = nullptr;
        DView J = I;
        if (r3 > 0 && !I.empty()) {                              // :146, J = L3^-1 I into a temporary
            FFG_CUDA(cudaMallocAsync(&jbuf, I.rows * I.cols * 4, b.st));
            FFG_CUDA(cudaMemcpy2DAsync(jbuf, I.cols * 4, I.d, I.ld * 4, I.cols * 4, I.rows, cudaMemcpyDeviceToDevice,
                                       b.st));
            J = DView{jbuf, I.rows, I.cols, I.cols};
            trsm_lower_unit(r3s, L3, J);
        }
        if (r3 > 0 && !N.empty()) trsm_lower_unit(r3s, L3, N);       // :147
        if (!N.empty() && !J.empty()) gemm_sub(J, V2, N);        // :148  O = N - J*V2
        if (!R.empty()) {                                        // :149-152
            if (!K.empty() && !V2.empty()) gemm_sub(K, V2, R);
            if (!N.empty()) gemm_sub(M3, N, R);
        }
        if (jbuf) FFG_CUDA(cudaFreeAsync(jbuf, b.st));

        NodeRes r4s = rec(R);                                    // :154
        const size_t r4 = r4s.rank;
        apply(r4s, 0, a.sub(m1 + r3, 0, m - m1 - r3, r1 + r3));  // :156-161
        if (r2 > 0) apply(r4s, 0, a.sub(m1 + r3, n1, m - m1 - r3, r2));
        apply(r4s, 1, a.sub(0, n1 + r2, r1, n - n1 - r2));
        if (r2 > 0) apply(r4s, 1, a.sub(r1, n1 + r2, r2, n - n1 - r2));
        if (r3 > 0) apply(r4s, 1, a.sub(m1, n1 + r2, r3, n - n1 - r2));

        bool pinit = false, qinit = false;                       // :163-170
        compose(res.P, pinit, m, res.pr, 0, r1s.P, r1s.pr);
        compose(res.P, pinit, m, res.pr, r1, r2s.P, r2s.pr);
        compose(res.P, pinit, m, res.pr, m1, r3s.P, r3s.pr);
        compose(res.P, pinit, m, res.pr, m1 + r3, r4s.P, r4s.pr);
        compose(res.Q, qinit, n, res.qr, 0, r1s.Q, r1s.qr);
        compose(res.Q, qinit, n, res.qr, r1, r3s.Q, r3s.qr);
        compose(res.Q, qinit, n, res.qr, n1, r2s.Q, r2s.qr);
        compose(res.Q, qinit, n, res.qr, n1 + r2, r4s.Q, r4s.qr);

        rot(res.P, pinit, m, res.pr, r1 + r2, m1, r3 + r4);       // :174-179 pivot gather
        rotate_block_dev(b, a, 0, r1 + r2, m1, r3 + r4);
        rot(res.Q, qinit, n, res.qr, r1, n1, r2);
        rotate_block_dev(b, a, 1, r1, n1, r2);
        rot(res.Q, qinit, n, res.qr, r1 + r2 + r3, n1 + r2, r4);
        rotate_block_dev(b, a, 1, r1 + r2 + r3, n1 + r2, r4);

        res.rank = r1 + r2 + r3 + r4;
        res.fac = new_factor(res.rank);  // leading factor = children's factors in gather order
        for (const NodeRes* c : {&r1s, &r2s, &r3s, &r4s})
            if (c->rank > 0) res.fac->kids.push_back(c->fac);
        arena.reset(mark);  // children consumed (stream order protects the pending kernels)
        return res;
    }

    void download(const NodeRes& res, size_t m, size_t n, uint32_t* P, uint32_t* Q) {
        if (P) {
            for (size_t i = 0; i < m; ++i) P[i] = (uint32_t)i;
            if (!res.pr.empty())
                FFG_CUDA(cudaMemcpyAsync(P + res.pr.lo, res.P + res.pr.lo, (res.pr.hi - res.pr.lo) * 4,
                                         cudaMemcpyDeviceToHost, b.st));
        }
        if (Q) {
            for (size_t j = 0; j < n; ++j) Q[j] = (uint32_t)j;
            if (!res.qr.empty())
                FFG_CUDA(cudaMemcpyAsync(Q + res.qr.lo, res.Q + res.qr.lo, (res.qr.hi - res.qr.lo) * 4,
                                         cudaMemcpyDeviceToHost, b.st));
        }
        FFG_CUDA(cudaStreamSynchronize(b.st));
    }
};

}  // namespace

size_t pluq_tile_recursive_dev(const Blas& b, DView a, size_t threshold, uint32_t* P, uint32_t* Q) {
    Driver drv(b, threshold, a.rows, a.cols);
    NodeRes res = drv.rec(a);
    drv.download(res, a.rows, a.cols, P, Q);
    return res.rank;
}

size_t rr_base_dev(const Blas& b, DView a, uint32_t* P, uint32_t* Q) {
    Driver drv(b, SIZE_MAX, a.rows, a.cols);
    NodeRes res = drv.rec(a);
    drv.download(res, a.rows, a.cols, P, Q);
    return res.rank;
}

}  // namespace ffg
