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
#include <chrono>
#include <cstdio>
#include <atomic>
#include <cstring>
#include <deque>
#include <future>
#include <thread>
#include <memory>
#include <vector>

#include "pluq.cuh"
#include "profile.cuh"

namespace ffg {

// Stream-ordered buffers of one call: freed on every exit path (an exception escaping a call --
// out of memory in a workspace, a CUDA error -- must not leak a matrix-sized backup in a
// long-lived context).  free_async frees early and disarms the guard.
template <class T>
struct AsyncFreeGuard {
    T*& p;
    cudaStream_t st;
    ~AsyncFreeGuard() {
        if (p) cudaFreeAsync(p, st);
    }
};
template <class T>
static void free_async(T*& p, cudaStream_t st) {
    if (!p) return;
    T* q = p;
    p = nullptr;
    FFG_CUDA(cudaFreeAsync(q, st));
}

static bool panel_no_direct();

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
    void free_on(cudaStream_t st) { st_ = st; }  // the stream whose later work reads these arrays
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
    const Blas& user;  // caller's stream: forked into `b` (high priority) and joined back at the end
    Blas b;
    size_t thr;
    PermArena arena;
    BaseInfo* info_dev = nullptr;
    BaseInfo* info_host = nullptr;
    cudaEvent_t ev = nullptr;
    uint64_t base_cases = 0;
    bool use_streams = true;     // exact recursion: side streams (off when partitioned)
    bool panel_streams = true;   // panel schedule: side streams (collectives stay on the critical one)
    int lookahead_sms = 0;  // SM cap of the look-ahead GEMMs (FFG_LOOKAHEAD_SMS, default SMs - 32)

    // host-pipelined entry (pluq_tile_recursive_host): the top-left spine of the recursion
    // (the chain of first children from the root) starts on data already uploaded; spine[d]
    // marks the upload of the depth-d spine block minus its first child's block
    const uint32_t* spine_root = nullptr;
    std::vector<cudaEvent_t> spine;
    // Early download (host entry only).  On the recursion's right spine (root, its R, R's R, ...)
    // a node whose E and G are empty has finished everything outside R when R's recursion
    // starts: its top rows and its left block (L1\U1, D, Fb) go to the host on the copy stream
    // while R recurses, and only the last spine node's R is left for the end.  A region that a
    // later permutation touches (R's P/Q, or a rank-deficient A1's pivot gather) is re-copied.
    struct EarlyTop {
        struct Reg {
            size_t r0 = 0, c0 = 0, rows = 0, cols = 0;
        };
        bool armed = false, spine_ok = true;
        cudaStream_t cs = nullptr;
        uint32_t* host = nullptr;
        size_t ldh = 0;
        const uint32_t* root = nullptr;
        size_t ld = 0;
        Reg tail;               // still to copy after the recursion
        std::vector<Reg> redo;  // early copies made stale by later permutations
    } early;
    void early_copy(const EarlyTop::Reg& g, cudaStream_t st) {
        if (g.rows && g.cols)
            FFG_CUDA(cudaMemcpy2DAsync(early.host + g.r0 * early.ldh + g.c0, early.ldh * 4,
                                       early.root + g.r0 * early.ld + g.c0, early.ld * 4, g.cols * 4, g.rows,
                                       cudaMemcpyDeviceToHost, st));
    }

    // slot: 0 for the root driver of a call; a concurrent subtree (E || G) gets its own slot =
    // its own streams (ids slot*1000 + ...) and base-case mailbox
    int slot = 0;
    bool owns_slot = true;  // false for a node-level speculative sub-driver sharing its parent's slot
    int device = 0;
    static int sid(int slot, int k) { return slot * 1000 + k; }

    Driver(const Blas& bl, size_t t, size_t m, size_t n, bool keep_events = false, int slot_ = 0)
        : user(bl),
          b(Blas{bl.F, bl.ws, bl.ws.stream(sid(slot_, 0), 0), bl.launches}),
          thr(std::max<size_t>(1, t)),
          arena(8 * (m + n) + 4096, bl.ws.stream(sid(slot_, 0), 0)),
          slot(slot_) {
        if (!keep_events) b.ws.reset_events();
        FFG_CUDA(cudaGetDevice(&device));
        cudaEvent_t e = b.ws.event();  // critical stream starts after the caller's pending work
        FFG_CUDA(cudaEventRecord(e, user.st));
        FFG_CUDA(cudaStreamWaitEvent(b.st, e, 0));
        static const bool no_streams = knob_on("FFG_NO_STREAMS");
        // partitioned (multi-GPU) runs keep their side streams: every split operation (the only ones
        // with a collective) is moved onto the critical stream (pgemm_sub / ptrsm), so all ranks issue
        // their collectives in one stream and one order
        use_streams = !no_streams;
        panel_streams = !no_streams;
        {
            static int sms = -1;
            if (sms < 0) {
                int dev = 0;
                FFG_CUDA(cudaGetDevice(&dev));
                FFG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
            }
            static const char* env = knob_str("FFG_LOOKAHEAD_SMS");
            lookahead_sms = env ? atoi(env) : std::max(1, sms - 32);
            static const char* ed = knob_str("FFG_DEFER_SMS");
            static const char* es = knob_str("FFG_SIDE_SMS");
            defer_sms = ed ? atoi(ed) : std::max(1, sms - 4);
            side_sms = es ? atoi(es) : std::max(1, sms - 4);
        }
        uint32_t* dev = nullptr;
        // the base kernel writes rank + moved ranges straight into host-mapped memory
        static_assert(sizeof(BaseInfo) <= Workspace::MAILBOX_WORDS * 4, "mailbox too small");
        info_host = reinterpret_cast<BaseInfo*>(b.ws.mailbox(slot, &dev));
        info_dev = reinterpret_cast<BaseInfo*>(dev);
        ev = b.ws.event();
    }
    void alloc_panel_inv() {
        static const bool off = knob_on("FFG_PANEL_FUSED_TRSM");
        static const bool no_q = knob_on("FFG_SPEC_NO_Q");
        if (!off && !panel_inv) FFG_CUDA(cudaMallocAsync(&panel_inv, 2 * 2 * 64 * 64 * 4, b.st));
        // column pivots need the inverse-apply path (it gathers the bottom panel through Q)
        if (panel_inv && !no_q && !gq && pcols) {
            FFG_CUDA(cudaMallocAsync(&gq, pcols * 4, b.st));
            allow_q = true;
        }
    }
    // End of a speculative panel run whose guess held: Q = the base cases' column pivots (P is the
    // identity), and each base case's pivots applied to the rows above its block -- what tile_rec's
    // ancestors do with R's Q (rankrev.hpp:158-161).  Synchronizes.  `fixed` receives the regions
    // rewritten here (the host entry re-downloads them).
    void panel_finish(uint32_t* P, uint32_t* Q, std::vector<std::pair<size_t, size_t>>* fixed) {
        std::vector<uint32_t> ql(gq ? pcols : 0);
        if (gq) FFG_CUDA(cudaMemcpyAsync(ql.data(), gq, pcols * 4, cudaMemcpyDeviceToHost, b.st));
        FFG_CUDA(cudaStreamSynchronize(b.st));
        if (P)
            for (size_t i = 0; i < prows; ++i) P[i] = (uint32_t)i;
        if (Q)
            for (size_t j = 0; j < pcols; ++j) Q[j] = (uint32_t)j;
        if (!gq || *reinterpret_cast<volatile uint32_t*>(&info_host->spec_fail)) return;
        bool any = false;
        for (const auto& lf : leaves) {
            const size_t o = lf.first, sz = lf.second;
            bool id = true;
            for (size_t t = 0; t < sz; ++t) {
                if (Q) Q[o + t] = (uint32_t)(o + ql[o + t]);
                id = id && ql[o + t] == t;
            }
            if (!id && o > 0) {
                block_cols_perm_dev(b, at(0, o, o, sz), gq + o);
                if (fixed) fixed->push_back(lf);
                any = true;
            }
        }
        if (any) FFG_CUDA(cudaStreamSynchronize(b.st));
    }
    ~Driver() {
        if (gq) cudaFreeAsync(gq, b.st);
        if (panel_inv) cudaFreeAsync(panel_inv, b.st);
        if (owns_slot) b.ws.release_slot(slot);
    }
    // join the critical stream back into the caller's stream
    void finish() {
        cudaEvent_t e = b.ws.event();
        FFG_CUDA(cudaEventRecord(e, b.st));
        FFG_CUDA(cudaStreamWaitEvent(user.st, e, 0));
    }
    Blas on(cudaStream_t st) const {
        Blas r{b.F, b.ws, st, b.launches};
        r.no_direct = b.no_direct;
        return r;
    }
    // a second critical-path stream per recursion depth (the node's independent TRSM), and a
    // low-priority stream per depth for the look-ahead part of the trailing update
    // (one stream when partitioned: every rank must issue its collectives in the same order)
    bool multi() const { return use_streams || (panel && panel_streams); }
    cudaStream_t twin(int depth) { return multi() ? b.ws.stream(sid(slot, 100 + depth), 0) : b.st; }
    cudaStream_t lookahead(int depth) { return multi() ? b.ws.stream(sid(slot, 200 + depth), 1) : b.st; }

    // ---- concurrent subtrees: G's recursion (rankrev.hpp:123) is independent of E's (:119) --
    // disjoint blocks, results combined only afterwards -- so a large G runs in a child driver
    // on its own host thread, streams and mailbox while this thread recurses into E.  The
    // per-base-case rank round trip is what bounds rank-deficient inputs (4-way recursion), so
    // this overlaps exactly that latency.
    static std::atomic<int>& active_children() {
        static std::atomic<int> n{0};
        return n;
    }
    bool can_fork(const DView& E, const DView& G) const {
        // each child thread spins on its mailbox: keep them within the host's cores
        const int max_threads =  // read per call (tests switch it)
            (int)knob_int("FFG_SUBTREE_THREADS", std::max(0, std::min(15, (int)std::thread::hardware_concurrency() - 2)));
        static const size_t gmin = (size_t)knob_int("FFG_FORK_MIN", 0);
        const size_t gm = gmin ? gmin : 2 * thr;  // smallest G worth a host thread
        return max_threads > 0 && !spec && use_streams && !b.ws.dist.active() && b.ws.prof.mode != 1 &&
               !E.empty() && !G.empty() &&
               std::min(G.rows, G.cols) > gm && std::min(E.rows, E.cols) > thr &&
               active_children().load() < max_threads;
    }
    cudaEvent_t mark_event(cudaStream_t st) {
        cudaEvent_t e = b.ws.event();
        FFG_CUDA(cudaEventRecord(e, st));
        return e;
    }
    void wait(cudaStream_t st, cudaEvent_t e) {
        if (e) FFG_CUDA(cudaStreamWaitEvent(st, e, 0));
    }

    // The base kernel writes its result into host-mapped memory and then the launch's sequence
    // number; spinning on it returns within a few microseconds of the kernel's end (an event
    // wait costs tens).  A slow or failed kernel falls back to the blocking event wait, which
    // also reports launch errors.
    void wait_mailbox(uint32_t seq) {
        volatile uint32_t* s = &info_host->seq;
        for (int it = 0; it < (1 << 18); ++it) {
            if (*s == seq) {
                std::atomic_thread_fence(std::memory_order_acquire);
                return;
            }
#if defined(__x86_64__) || defined(__i386__)
            __builtin_ia32_pause();
#endif
        }
        FFG_CUDA(cudaEventRecord(ev, b.st));
        FFG_CUDA(cudaEventSynchronize(ev));
        if (*s != seq) throw Error(FFG_ERR_INTERNAL, "base case did not report its rank");
        std::atomic_thread_fence(std::memory_order_acquire);
    }

    // ---- speculative full-rank mode: every base case is assumed to return full rank with identity
    // permutations -- what i.i.d. input does with probability ~1 - m/p per block -- so the host never
    // waits for a rank and the whole recursion is enqueued at once.  Each base kernel compares and
    // raises the sticky spec_fail flag in its mailbox; the caller keeps a backup of the input and
    // reruns without speculation when the flag is seen (the outputs are then those of the exact
    // path, so correctness never depends on the guess).
    struct SpecAbort {};
    bool spec = false;
    bool allow_q = false;  // panel schedule: the guess is full rank only (column pivots allowed)
    // the host stays at most spec_window base cases ahead of the device, so a failed guess is
    // noticed (and the queue drained) within a few steps instead of after the whole recursion
    size_t spec_window = 32;
    std::vector<uint32_t> spec_seqs;
    std::vector<size_t> spec_pos;  // panel schedule: diagonal offset of each speculative base case
    // the offset of the base case whose guess failed first (after a drain); false if unknown
    bool failed_at(size_t& off) const {
        if (!*reinterpret_cast<volatile uint32_t*>(&info_host->spec_fail)) return false;
        const uint32_t fs = *reinterpret_cast<volatile uint32_t*>(&info_host->fail_seq);
        for (size_t i = 0; i < spec_seqs.size(); ++i)
            if (spec_seqs[i] == fs && spec_pos[i] != SIZE_MAX) {
                off = spec_pos[i];
                return true;
            }
        return false;
    }
    // the schedule's prefix before `off`: block-local column pivots and base cases (call after a drain)
    void prefix_of(size_t off, std::vector<uint32_t>& gqh, std::vector<std::pair<size_t, size_t>>& lv) const {
        gqh.assign(off, 0u);
        lv.clear();
        for (const auto& lf : leaves)
            if (lf.first + lf.second <= off) lv.push_back(lf);
        if (gq && off) {
            FFG_CUDA(cudaMemcpy(gqh.data(), gq, off * 4, cudaMemcpyDeviceToHost));
        } else {
            for (const auto& lf : lv)
                for (size_t i = 0; i < lf.second; ++i) gqh[lf.first + i] = (uint32_t)i;  // no column pivots
        }
    }
    // diagnostics (FFG_SPEC_LOG): throttle calls, and those that found the device behind (the host
    // had to wait: the device, not the host's enqueue rate, bounds the run)
    uint64_t throttle_calls = 0, throttle_waits = 0;
    void spec_throttle() {
        if (spec_seqs.size() < spec_window) return;
        const uint32_t target = spec_seqs[spec_seqs.size() - spec_window] & ~SPEC_BIT;
        volatile uint32_t* sq = &info_host->seq;
        volatile uint32_t* sf = &info_host->spec_fail;
        ++throttle_calls;
        for (uint64_t it = 0;; ++it) {
            if (*sf) throw SpecAbort{};
            const uint32_t cur = *sq & ~SPEC_BIT;
            if (it == 1) ++throttle_waits;
            if (((cur - target) & ~SPEC_BIT) < 0x40000000u) return;  // cur at or after target (mod 2^31)
            if (it > (1u << 24)) {  // slow or failed kernel: block on the stream (reports errors)
                FFG_CUDA(cudaStreamSynchronize(b.st));
                if (*sf) throw SpecAbort{};
                return;
            }
#if defined(__x86_64__) || defined(__i386__)
            __builtin_ia32_pause();
#endif
        }
    }

    // Partitioned runs abort a failed guess only at deterministic points: wait for the base case
    // spec_window launches back to complete and abort iff the FIRST failure (its sequence number,
    // which every rank computes identically) is at or before it -- whatever else any rank's device
    // has reached by then -- so every rank stops after the same launch and issues the same
    // collectives.
    void spec_throttle_det() {
        if (spec_seqs.size() < spec_window) return;
        const uint32_t target = spec_seqs[spec_seqs.size() - spec_window] & ~SPEC_BIT;
        volatile uint32_t* sq = &info_host->seq;
        auto at_or_after = [](uint32_t x, uint32_t y) { return ((x - y) & ~SPEC_BIT) < 0x40000000u; };
        for (uint64_t it = 0;; ++it) {
            const uint32_t cur = *sq & ~SPEC_BIT;
            if (at_or_after(cur, target)) break;
            if (it > (1u << 24)) {
                FFG_CUDA(cudaStreamSynchronize(b.st));
                break;
            }
#if defined(__x86_64__) || defined(__i386__)
            __builtin_ia32_pause();
#endif
        }
        std::atomic_thread_fence(std::memory_order_acquire);
        if (*reinterpret_cast<volatile uint32_t*>(&info_host->spec_fail)) {
            const uint32_t fs = *reinterpret_cast<volatile uint32_t*>(&info_host->fail_seq) & ~SPEC_BIT;
            if (at_or_after(target, fs)) throw SpecAbort{};
        }
    }

    bool base_wrote_inv = false;  // the last speculative base case also wrote its factor inverses
    NodeRes base(DView a, NodeRes res, uint32_t* inv_out = nullptr) {
        if (spec) {
            if (a.rows > 64 || a.cols > 64) throw SpecAbort{};  // only the slab kernel checks
            if (!b.ws.dist.active()) {
                if (*reinterpret_cast<volatile uint32_t*>(&info_host->spec_fail)) throw SpecAbort{};
                spec_throttle();
            } else {
                spec_throttle_det();  // partitioned: abort at the same point on every rank
            }
            const uint32_t seq = ((b.ws.base_seq.fetch_add(1) + 1) & ~SPEC_BIT) | SPEC_BIT;
            // (inverses inside the base kernel by substitution measured slower than the separate
            // log-depth kernel: 38 -> 90 us per base case; the spec kernel ignores inv_out)
            base_wrote_inv = rr_base_launch(b, a, res.P, res.Q, info_dev, inv_out, seq, allow_q && a.rows == a.cols);
            spec_seqs.push_back(seq);
            spec_pos.push_back(proot ? (size_t)(a.d - proot) / pld : SIZE_MAX);
            ++base_cases;
            res.rank = std::min(a.rows, a.cols);
            res.pr = Range{};
            res.qr = Range{};
            return res;
        }
        const uint32_t seq = (b.ws.base_seq.fetch_add(1) + 1) & ~SPEC_BIT;
        rr_base_launch(b, a, res.P, res.Q, info_dev, nullptr, seq);
        wait_mailbox(seq);  // the rank decides every later shape
        ++base_cases;
        res.rank = info_host->rank;
        res.pr = Range{info_host->plo, info_host->phi};
        res.qr = Range{info_host->qlo, info_host->qhi};
        return res;
    }

    // TRSMs of tile_rec against a child's leading factor: the blocked-inverse TRSM
    void trsm_lower_unit(const Blas& bb, const NodeRes&, DView L, DView B) { ftrsm_dev(bb, 0, 0, 0, L, B, false); }
    void trsm_upper_nonunit(const Blas& bb, const NodeRes&, DView U, DView B) { ftrsm_dev(bb, 1, 1, 1, U, B, false); }

    void apply(const NodeRes& c, int axis, DView v) {
        const Range& r = axis == 0 ? c.pr : c.qr;
        if (r.empty() || v.empty()) return;
        perm_apply_range(b, v, axis, axis == 0 ? c.P : c.Q, r.lo, r.hi);
    }

    void gemm_sub(DView A, DView B, DView C) { b.gemm(b.F.p - 1, A, B, 1, C); }
    void gemm_sub(const Blas& bb, DView A, DView B, DView C) { bb.gemm(bb.F.p - 1, A, B, 1, C); }

    // ---- partitioned execution (dist.cuh): large operations split into per-rank output
    // slices + one all-gather; small ones replicated.  Single-GPU runs take the plain calls.
    static constexpr size_t kAlign = 128;  // slice granularity = the GEMM's M tile
    bool split(double macs) const { return b.ws.dist.active() && macs >= (double)b.ws.dist.min_work; }
    template <class Fn>
    void slices(size_t total, Fn&& fn) {
        const Dist& d = b.ws.dist;
        for (int r = 0; r < d.world; ++r) {
            if (!d.virt && r != d.rank) continue;
            const Slice s = partition(total, d.world, r, kAlign);
            if (s.hi > s.lo) fn(s.lo, s.hi - s.lo);
        }
    }
    // C -= A B, split along C's longer side
    // a split operation requested on a side stream runs on the critical stream (joined both ways)
    template <class Fn>
    void on_critical(const Blas& bb, Fn&& fn) {
        if (bb.st == b.st) {
            fn(b);
            return;
        }
        wait(b.st, mark_event(bb.st));
        fn(b);
        wait(bb.st, mark_event(b.st));
    }
    void pgemm_sub(const Blas& bb, DView A, DView B, DView C) {
        if (!split((double)C.rows * C.cols * A.cols)) {
            gemm_sub(bb, A, B, C);
            return;
        }
        if (bb.st != b.st) {
            on_critical(bb, [&](const Blas& c) { pgemm_sub(c, A, B, C); });
            return;
        }
        const int axis = C.rows >= C.cols ? 0 : 1;
        if (axis == 0)
            slices(C.rows, [&](size_t lo, size_t len) {
                gemm_sub(bb, A.sub(lo, 0, len, A.cols), B, C.sub(lo, 0, len, C.cols));
            });
        else
            slices(C.cols, [&](size_t lo, size_t len) {
                gemm_sub(bb, A, B.sub(0, lo, B.rows, len), C.sub(0, lo, C.rows, len));
            });
        dist_allgather(b.ws.dist, C.d, C.rows, C.cols, C.ld, axis, kAlign, bb.st);
    }
    // side 0: B <- L^-1 B (B's columns independent); side 1: B <- B U^-1 (B's rows independent)
    void ptrsm(const Blas& bb, int side, const NodeRes& c, DView T, DView B) {
        auto one = [&](DView X) {
            if (side == 0)
                trsm_lower_unit(bb, c, T, X);
            else
                trsm_upper_nonunit(bb, c, T, X);
        };
        const double w = side == 0 ? (double)B.cols : (double)B.rows;
        if (!split(0.5 * (double)T.rows * T.rows * w)) {
            one(B);
            return;
        }
        if (bb.st != b.st) {
            on_critical(bb, [&](const Blas& cb) { ptrsm(cb, side, c, T, B); });
            return;
        }
        if (side == 0)
            slices(B.cols, [&](size_t lo, size_t len) { one(B.sub(0, lo, B.rows, len)); });
        else
            slices(B.rows, [&](size_t lo, size_t len) { one(B.sub(lo, 0, len, B.cols)); });
        dist_allgather(b.ws.dist, B.d, B.rows, B.cols, B.ld, side == 0 ? 1 : 0, kAlign, bb.st);
    }

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

    // `pending`: work on the side streams that everything outside the top-left quadrant A1
    // of `a` still depends on (the look-ahead part of the parent's trailing update)
    // ---- diagnostics (FFG_LEVEL_TIMING, root driver): critical-stream time per recursion depth,
    // split into a node's own work (between its children) and its base cases
    struct LevelRec {
        int depth;
        bool leaf;
        cudaEvent_t e[4];
    };
    bool level_timing = false;
    std::vector<LevelRec> levels;
    cudaEvent_t tev() {
        cudaEvent_t e;
        FFG_CUDA(cudaEventCreate(&e));
        FFG_CUDA(cudaEventRecord(e, b.st));
        return e;
    }
    void level_report() {
        if (levels.empty()) return;
        FFG_CUDA(cudaStreamSynchronize(b.st));
        std::vector<double> self(64, 0.0), leaf(64, 0.0);
        std::vector<int> cnt(64, 0), lcnt(64, 0);
        for (auto& L : levels) {
            float a = 0, c = 0;
            if (L.leaf) {
                cudaEventElapsedTime(&a, L.e[0], L.e[1]);
                leaf[L.depth] += a;
                ++lcnt[L.depth];
            } else {
                cudaEventElapsedTime(&a, L.e[0], L.e[1]);  // after A1 -> before R
                cudaEventElapsedTime(&c, L.e[2], L.e[3]);  // after R -> end
                self[L.depth] += a + c;
                ++cnt[L.depth];
            }
            for (auto e : L.e)
                if (e) cudaEventDestroy(e);
        }
        for (int d = 0; d < 64; ++d)
            if (cnt[d] || lcnt[d])
                fprintf(stderr, "LEVEL depth %2d: %5d nodes  own %8.3f ms (%.1f us/node) | %5d base cases %8.3f ms (%.1f us each)\n",
                        d, cnt[d], self[d], cnt[d] ? 1e3 * self[d] / cnt[d] : 0.0, lcnt[d], leaf[d],
                        lcnt[d] ? 1e3 * leaf[d] / lcnt[d] : 0.0);
        levels.clear();
    }

    // ---- panel mode (speculative runs on square input): with full rank and identity
    // permutations the TRSMs of tile_rec (:111-114) need not wait for a whole child: every base
    // case solves its entire right panel (its rows, all later columns) with its L and its entire
    // bottom panel with its U right after it is factored, and every internal node, once its A1
    // child is done, updates [H | right panel of R's rows] and the bottom panel of R's columns
    // with two wide GEMMs.  This is tile_rec's arithmetic evaluated right-looking inside the same
    // recursion; L, U (unique for full rank without pivoting) come out identical, and no TRSM
    // chain remains above the base cases.  Any failed guess reruns the exact path anyway.
    bool panel = false;
    uint32_t* panel_inv = nullptr;  // 2 slots x (2 x 64 x 64): factor inverses of the last two base cases
    uint32_t* inv_slot() const { return panel_inv + (leaves.size() & 1) * 2 * 64 * 64; }  // current leaf's
    uint32_t* gq = nullptr;         // base cases' column pivots (local indices) at their columns
    std::vector<std::pair<size_t, size_t>> leaves;  // (offset, size) of every base case
    const uint32_t* proot = nullptr;
    size_t pld = 0, prows = 0, pcols = 0;

    // ---- streamed host entry (panel mode on host buffers).  Panel mode touches the matrix in
    // L-shaped bands of increasing index -- band [a, e) = rows [a, e) x cols [a, n) plus rows
    // [e, n) x cols [a, e) -- and a band is final once its last base case has solved its panels,
    // so band c uploads while earlier bands factor and downloads as soon as it is done.  Band
    // ends sit on node boundaries of the recursion (band_bounds).
    struct Bands {
        bool on = false;
        std::vector<size_t> end;                              // band c = [end[c-1], end[c])
        std::vector<cudaEvent_t> uploaded;                    // band c is in HBM
        std::vector<cudaEvent_t> ready;                       // ... and backed up (enqueued lazily)
        uint32_t* backup = nullptr;
        cudaStream_t bks = nullptr;
        std::vector<std::pair<cudaStream_t, size_t>> waited;  // per stream: bands already waited for
        cudaStream_t down = nullptr;                          // D2H copy stream
        uint32_t* host = nullptr;
        size_t ldh = 0, next_down = 0;
    } bands;
    void band_copy(size_t c, bool to_host, cudaStream_t st) {
        const size_t a0 = c ? bands.end[c - 1] : 0, e = bands.end[c], n = pcols, m = prows;
        auto rect = [&](size_t r0, size_t c0, size_t rows, size_t cols) {
            if (!rows || !cols) return;
            uint32_t* dv = const_cast<uint32_t*>(proot) + r0 * pld + c0;
            uint32_t* hv = bands.host + r0 * bands.ldh + c0;
            if (to_host)
                FFG_CUDA(cudaMemcpy2DAsync(hv, bands.ldh * 4, dv, pld * 4, cols * 4, rows, cudaMemcpyDeviceToHost, st));
            else
                FFG_CUDA(cudaMemcpy2DAsync(dv, pld * 4, hv, bands.ldh * 4, cols * 4, rows, cudaMemcpyHostToDevice, st));
        };
        rect(a0, a0, e - a0, n - a0);
        rect(e, a0, m - e, e - a0);
    }
    // ---- look-ahead pieces (panel mode): a node of size >= la_min does not update its whole
    // trailing region [H | right panel] + bottom panel before R's recursion.  The update is cut
    // into R's L-shaped bands of doubling width (64, 64, 128, 256, ...): the first band on the
    // critical stream, the rest on a low-priority look-ahead stream (SM-capped), each band's
    // completion event waited for by the first operation of R's recursion that reaches it.
    struct Piece {
        size_t a;  // band [a, e): operations touching rows / columns >= a must wait
        cudaEvent_t ev;
    };
    std::vector<Piece> pieces;
    size_t la_min = 0;  // 0: off
    size_t la_end = SIZE_MAX;  // ... and only for nodes ending at or before la_end
    bool la_here(size_t r0, size_t m, size_t m1) const {
        return la_min && m >= la_min && m - m1 > thr && r0 + m <= la_end;
    }
    DView at(size_t r, size_t c, size_t rows, size_t cols) const {
        return DView{const_cast<uint32_t*>(proot) + r * pld + c, rows, cols, pld};
    }
    // band [x, e) of the trailing update of node (o, m) whose first half [o, o + h) is factored:
    // rows [x, e) x cols [x, N) and rows [e, M) x cols [x, e), both -= L(., A1 cols) U(A1 rows, .)
    void piece(const Blas& rows_bl, const Blas& cols_bl, size_t o, size_t h, size_t x, size_t e) {
        if (pcols > x) gemm_sub(rows_bl, at(x, o, e - x, h), at(o, x, h, pcols - x), at(x, x, e - x, pcols - x));
        if (prows > e) gemm_sub(cols_bl, at(e, o, prows - e, h), at(o, x, h, e - x), at(e, x, prows - e, e - x));
    }

    // every later operation on `st` may touch rows / columns < hi
    void need(cudaStream_t st, size_t hi) {
        for (size_t i = 0; i < pieces.size();) {
            if (pieces[i].a < hi) {
                wait(st, pieces[i].ev);
                if (st == b.st) {  // every other stream forks from the critical one
                    pieces.erase(pieces.begin() + (long)i);
                    continue;
                }
            }
            ++i;
        }
        if (!bands.on) return;
        const size_t c = (size_t)(std::lower_bound(bands.end.begin(), bands.end.end(), hi) - bands.end.begin());
        if (c >= bands.uploaded.size()) return;
        // Backups are enqueued only when a band is first needed: a stream waiting on a late
        // upload at the head of a shared hardware queue would stall every later launch behind it.
        while (bands.ready.size() <= c) {
            const size_t k = bands.ready.size();
            const size_t a0 = k ? bands.end[k - 1] : 0, e = bands.end[k], n = pcols, m = prows;
            uint32_t* d = const_cast<uint32_t*>(proot);
            const Blas bb = on(bands.bks);
            wait(bands.bks, bands.uploaded[k]);
            copy_block_dev(bb, DView{d + a0 * pld + a0, e - a0, n - a0, pld},
                           DView{bands.backup + a0 * pld + a0, e - a0, n - a0, pld});
            copy_block_dev(bb, DView{d + e * pld + a0, m - e, e - a0, pld},
                           DView{bands.backup + e * pld + a0, m - e, e - a0, pld});
            bands.ready.push_back(mark_event(bands.bks));
        }
        size_t* w = nullptr;
        for (auto& pr : bands.waited)
            if (pr.first == st) w = &pr.second;
        if (!w) {
            bands.waited.push_back({st, 0});
            w = &bands.waited.back().second;
        }
        if (*w < c + 1) {
            wait(st, bands.ready[c]);
            *w = c + 1;
        }
    }
    // every operation on rows / columns < hi is enqueued (and joined into the critical stream)
    void band_done(size_t hi) {
        if (!bands.on || !bands.host) return;  // the device entry uses bands for lazy backups only
        while (bands.next_down < bands.end.size() && bands.end[bands.next_down] <= hi) {
            wait(bands.down, mark_event(b.st));
            for (cudaEvent_t e : deferred) wait(bands.down, e);
            band_copy(bands.next_down++, true, bands.down);
        }
    }

    // ---- progressive trailing updates (panel schedule): a node Y of size >= prog_min does not
    // wait for its whole first half A1 before its trailing update H -= L(., A1) U(A1, .): the
    // update is applied in K-chunks, each as soon as the chunk's sub-nodes of A1 are done, on a
    // low-priority SM-capped stream while A1's chain goes on.  Y's [H | right panel] and bottom
    // panel of R's columns are untouched by A1's processing, and chunks commute (exact
    // arithmetic), so only the last chunk is left when A1 finishes.
    struct Prog {
        size_t o, m, m1, next_k, chunk;
        int depth;
        cudaEvent_t last;
    };
    std::vector<Prog> progs;
    size_t prog_min = 0, prog_nchunks = 4;
    int prog_sms = 0;
    void prog_update(Prog& g, size_t k0, size_t k1) {
        Blas la = on(lookahead(g.depth));
        la.sm_cap = prog_sms;
        const size_t A = g.o + g.m1, E = g.o + g.m;  // R's rows / columns
        need(la.st, E);
        wait(la.st, mark_event(b.st));
        for (cudaEvent_t e : deferred) wait(la.st, e);
        if (E > A && pcols > A) gemm_sub(la, at(A, k0, E - A, k1 - k0), at(k0, A, k1 - k0, pcols - A), at(A, A, E - A, pcols - A));
        if (prows > E) gemm_sub(la, at(E, k0, prows - E, k1 - k0), at(k0, A, k1 - k0, E - A), at(E, A, prows - E, E - A));
        g.last = mark_event(la.st);
        g.next_k = k1;
    }
    // every operation on rows / columns < done is enqueued: start the chunks that became ready
    void prog_progress(size_t done) {
        for (auto& g : progs) {
            const size_t lim = std::min(done, g.o + g.m1);
            if (lim > g.next_k && lim - g.next_k >= g.chunk) prog_update(g, g.next_k, lim);
        }
    }

    // ---- deferred wide work (panel schedule): the last leaf of a subtree solves only the next
    // thr columns / rows of its panels on the critical stream and leaves the rest, and a node of
    // size <= corner_max updates only the first block of R on the critical stream (the corner) and
    // leaves its wide GEMMs -- on side streams.  Their events are waited for right after the next
    // base case and its inverses (flush_deferred), before anything that reads wide regions.
    std::vector<cudaEvent_t> deferred;
    // SM caps of the side streams' tensor-core GEMMs (persistent grids): the corner nodes'
    // deferred GEMMs (FFG_DEFER_SMS) and a two-leaf node's wide updates (FFG_SIDE_SMS); 0 = none
    // (persistent grids leaving 4 SMs free measured 28.7 -> 28.1 ms at n = 16384; 8 or 28 free: 28.2 / 29.2)
    int defer_sms = -1, side_sms = -1;  // resolved in the constructor
    size_t corner_max = 0;
    void flush_deferred() {
        for (cudaEvent_t e : deferred) wait(b.st, e);
        deferred.clear();
    }
    cudaStream_t side_stream(int k) { return multi() ? b.ws.stream(sid(slot, 400 + k), 0) : b.st; }
    // the leaf's right panel (rows of blk, columns beyond `beyond_c`) and bottom panel (rows beyond
    // `beyond_r`, columns of blk): the first thr columns / rows on the critical stream, the rest
    // on the side streams sa / sb (deferred)
    void leaf_panels_split(DView blk, size_t r0, size_t c0, size_t beyond_r, size_t beyond_c, const uint32_t* inv,
                           const uint32_t* q, int depth, const Blas& sa, const Blas& sb) {
        const size_t t = blk.rows;
        const size_t wr = pcols - beyond_c, hb = prows - beyond_r;
        const size_t mr = std::min(thr, wr), mb = std::min(thr, hb);
        DView rmini = at(r0, beyond_c, t, mr), bmini = at(beyond_r, c0, mb, t);
        DView rrest = at(r0, beyond_c + mr, t, wr - mr), brest = at(beyond_r + mb, c0, hb - mb, t);
        const cudaEvent_t f = mark_event(b.st);
        panel_mini_dev(b, inv, t, rmini, bmini, q);  // one launch of small CTAs
        if (!rrest.empty()) {
            wait(sa.st, f);
            panel_apply_dev(sa, 0, inv, t, rrest);
            deferred.push_back(mark_event(sa.st));
        }
        if (!brest.empty()) {
            wait(sb.st, f);
            panel_apply_dev(sb, 1, inv, t, brest, q);
            deferred.push_back(mark_event(sb.st));
        }
    }
    // size of the first base case of a node of size s
    size_t first_leaf(size_t s) const {
        while (s > thr) s = (s + 1) / 2;
        return s;
    }

    // Two-leaf node (A1, R both base cases): R's base case waits only for a one-CTA corner update
    // (A1's panel blocks inside the node and A(R, R) -= L(R, A1) U(A1, R)); A1's wide panels beyond
    // the node and their updates of R's rows / columns run on two side streams meanwhile, and R's
    // own panels wait for them.  Same arithmetic as the generic node, reordered.
    void two_leaf(DView a, int depth, NodeRes& res) {
        const size_t m = a.rows, t1 = (m + 1) / 2, t2 = m - t1;
        const size_t off = (size_t)(a.d - proot), r0 = off / pld, c0 = off % pld;
        need(b.st, r0 + m);
        const uint32_t* q1 = gq ? gq + c0 : nullptr;
        // A1
        NodeRes r1;
        r1.P = arena.alloc(t1);
        r1.Q = gq ? gq + c0 : arena.alloc(t1);
        uint32_t* inv1 = inv_slot();
        base(a.sub(0, 0, t1, t1), r1, inv1);
        leaves.push_back({c0, t1});
        if (!base_wrote_inv) panel_inverses_dev(b, a.sub(0, 0, t1, t1), inv1);
        flush_deferred();  // the node's rows / columns carry every earlier update
        // A1's wide panels beyond the node need only A1's inverses: they fork here, before the
        // corner kernels (disjoint regions); their GEMMs read the corner's L(R, A1) / U(A1, R)
        // blocks and wait for the second event
        static const bool early_apply = knob_int("FFG_EARLY_APPLY", 1) != 0;
        const cudaEvent_t f0 = early_apply ? mark_event(b.st) : nullptr;
        // A1's panel blocks inside the node, then R's update, each in small CTAs
        panel_mini_dev(b, inv1, t1, a.sub(0, t1, t1, t2), a.sub(t1, 0, t2, t1), q1);
        panel_update_dev(b, a.sub(t1, 0, t2, t1), a.sub(0, t1, t1, t2), a.sub(t1, t1, t2, t2));
        const cudaEvent_t f = mark_event(b.st);
        Blas sa = on(side_stream(0)), sb = on(side_stream(1));
        sa.sm_cap = sb.sm_cap = side_sms;
        static const bool side_direct = knob_on("FFG_SIDE_DIRECT");
        if (side_direct) sa.no_direct = sb.no_direct = false;
        wait(sa.st, early_apply ? f0 : f);
        wait(sb.st, early_apply ? f0 : f);
        DView rightA{a.d + m, t1, pcols - (c0 + m), pld};       // A1 rows, columns beyond the node
        DView bottomA{a.d + m * pld, prows - (r0 + m), t1, pld};  // rows beyond the node, A1 columns
        panel_apply_dev(sa, 0, inv1, t1, rightA);
        panel_apply_dev(sb, 1, inv1, t1, bottomA, q1);
        if (early_apply) {
            wait(sa.st, f);
            wait(sb.st, f);
        }
        DView HRp{a.d + t1 * pld + m, t2, pcols - (c0 + m), pld};  // R rows beyond the node
        DView BPp{a.d + m * pld + t1, prows - (r0 + m), t2, pld};  // beyond the node, R columns
        if (!HRp.empty()) gemm_sub(sa, a.sub(t1, 0, t2, t1), rightA, HRp);
        if (!BPp.empty()) gemm_sub(sb, bottomA, a.sub(0, t1, t1, t2), BPp);
        const cudaEvent_t ea = mark_event(sa.st), eb = mark_event(sb.st);
        // R
        DView Rb = a.sub(t1, t1, t2, t2);
        NodeRes r2;
        r2.P = arena.alloc(t2);
        r2.Q = gq ? gq + c0 + t1 : arena.alloc(t2);
        uint32_t* inv2 = inv_slot();
        base(Rb, r2, inv2);
        leaves.push_back({c0 + t1, t2});
        if (!base_wrote_inv) panel_inverses_dev(b, Rb, inv2);
        wait(b.st, ea);
        wait(b.st, eb);
        if (corner_max) {
            leaf_panels_split(Rb, r0 + t1, c0 + t1, r0 + m, c0 + m, inv2, gq ? gq + c0 + t1 : nullptr, depth, sa, sb);
        } else {
            DView rightR{Rb.d + t2, t2, pcols - (c0 + m), pld};
            DView bottomR{Rb.d + t2 * pld, prows - (r0 + m), t2, pld};
            const bool both = !rightR.empty() && !bottomR.empty();
            const Blas side = both ? on(twin(depth)) : b;
            if (both) wait(side.st, mark_event(b.st));
            panel_apply_dev(b, 0, inv2, t2, rightR);
            panel_apply_dev(side, 1, inv2, t2, bottomR, gq ? gq + c0 + t1 : nullptr);
            if (both) wait(b.st, mark_event(side.st));
        }
        band_done(r0 + m);
        prog_progress(r0 + m);
        res.rank = m;
        res.pr = Range{};
        res.qr = Range{};
    }

    NodeRes rec_panel(DView a, int depth) {
        const size_t m = a.rows, n = a.cols;  // square
        NodeRes res;
        res.P = arena.alloc(std::max<size_t>(m, 1));
        res.Q = arena.alloc(std::max<size_t>(n, 1));
        if (m == 0 || n == 0) return res;
        const size_t off = (size_t)(a.d - proot), r0 = off / pld, c0 = off % pld;
        if (std::min(m, n) <= thr) {
            need(b.st, r0 + m);
            if (gq) res.Q = gq + c0;
            res = base(a, res, panel_inv && m == n && m <= 64 ? inv_slot() : nullptr);  // speculative: no wait
            // whole right panel (L^-1, left) and bottom panel (U^-1, right) of this block
            DView right{a.d + n, m, pcols - (c0 + n), pld};
            DView bottom{a.d + m * pld, prows - (r0 + m), n, pld};
            const bool both = !right.empty() && !bottom.empty();
            const Blas side = both ? on(twin(depth)) : b;
            if (panel_inv && m == n && m <= 64) {
                // inverses once, then every strip of both panels only applies them
                uint32_t* inv = inv_slot();
                if (!base_wrote_inv) panel_inverses_dev(b, a, inv);
                flush_deferred();
                if (both) wait(side.st, mark_event(b.st));
                panel_apply_dev(b, 0, inv, m, right);
                panel_apply_dev(side, 1, inv, m, bottom, gq ? gq + c0 : nullptr);
            } else {
                flush_deferred();
                if (both) wait(side.st, mark_event(b.st));
                if (!right.empty()) ftrsm_dev(b, 0, 0, 0, a, right, false);
                if (!bottom.empty()) ftrsm_dev(side, 1, 1, 1, a, bottom, false);
            }
            if (both) wait(b.st, mark_event(side.st));
            leaves.push_back({c0, n});
            band_done(r0 + m);
            prog_progress(r0 + m);
            return res;
        }
        const size_t mark = arena.mark();
        const size_t m1 = (m + 1) / 2, n1 = (n + 1) / 2;
        const bool no_corner = knob_on("FFG_NO_CORNER");  // per call: tests
        if (!no_corner && panel_inv && m == n && m1 <= thr && m1 <= 64 && m - m1 > 0) {
            two_leaf(a, depth, res);
            arena.reset(mark);
            return res;
        }
        const bool prog = prog_min && m >= prog_min && use_streams && m == n && m - m1 > thr;
        if (prog) progs.push_back(Prog{r0, m, m1, r0, std::max(thr, m1 / prog_nchunks), depth, nullptr});
        rec_panel(a.sub(0, 0, m1, n1), depth + 1);
        // A1's panels solved D and Fb (and the parts of A1's rows / columns beyond this node)
        DView Fb = a.sub(m1, 0, m - m1, n1);                                  // rows of R, cols of A1
        DView Dx{a.d + n1, m1, pcols - (c0 + n1), pld};                       // A1 rows, cols >= n1
        DView HR{a.d + m1 * pld + n1, m - m1, pcols - (c0 + n1), pld};        // [H | right panel]
        DView Fbelow{a.d + m * pld, prows - (r0 + m), n1, pld};               // below the node, A1 cols
        DView Dn = a.sub(0, n1, m1, n - n1);                                  // D
        DView BP{a.d + m * pld + n1, prows - (r0 + m), n - n1, pld};          // below the node, R cols
        const bool both = !BP.empty();
        const Blas side = both ? on(twin(depth)) : b;
        if (prog) {
            Prog g = progs.back();
            progs.pop_back();
            if (g.next_k < r0 + m1) prog_update(g, g.next_k, r0 + m1);  // the last chunk
            need(b.st, r0 + m);
            flush_deferred();
            wait(b.st, g.last);  // [H | right panel] and the bottom panel are complete
        } else if (corner_max && m <= corner_max && m - m1 > thr && !la_here(r0, m, m1)) {
            // corner: R's first base block gets its update now; the wide GEMMs of the node are
            // deferred to side streams (after the last leaf's deferred panels)
            const size_t A = r0 + m1, f = first_leaf(m - m1), E = r0 + m;
            need(b.st, E);
            const cudaEvent_t forked = mark_event(b.st);
            static const bool tc_corner = knob_on("FFG_CORNER_TC");
            if (tc_corner)
                gemm_sub(b, at(A, c0, f, n1), at(r0, A, m1, f), at(A, A, f, f));
            else  // f x f x m1 in small CUDA-core CTAs: shorter than a tensor-core launch at this size
                panel_update_dev(b, at(A, c0, f, n1), at(r0, A, m1, f), at(A, A, f, f));
            Blas sc = on(side_stream(2)), sd = on(side_stream(3));
            sc.sm_cap = sd.sm_cap = defer_sms;  // leave SMs for the critical stream's small kernels
            // these GEMMs gate the next two-leaf node (flush_deferred): FFG_DEFER_DIRECT=1 lets the
            // single-launch direct kernel take the ones with K <= 128 (no limb split round trip)
            static const bool defer_direct = knob_on("FFG_DEFER_DIRECT");
            if (defer_direct) sc.no_direct = sd.no_direct = false;
            for (const Blas* sx : {&sc, &sd}) {
                wait(sx->st, forked);
                for (cudaEvent_t e : deferred) wait(sx->st, e);
            }
            deferred.clear();
            // (replicated when partitioned: only the critical stream issues collectives)
            // R's rows right of the corner in one GEMM (full row tiles), then the block below the
            // corner (rows A+f..E, columns A..A+f)
            static const bool split_hr = knob_on("FFG_SPLIT_HR");
            if (split_hr) {
                if (pcols > A + f) gemm_sub(sc, at(A, c0, f, n1), at(r0, A + f, m1, pcols - (A + f)), at(A, A + f, f, pcols - (A + f)));
                if (E > A + f) gemm_sub(sc, at(A + f, c0, E - (A + f), n1), at(r0, A, m1, pcols - A), at(A + f, A, E - (A + f), pcols - A));
            } else {
                if (pcols > A + f) gemm_sub(sc, at(A, c0, E - A, n1), at(r0, A + f, m1, pcols - (A + f)), at(A, A + f, E - A, pcols - (A + f)));
                if (E > A + f) {
                    if (E - (A + f) <= 64)
                        panel_update_dev(sc, at(A + f, c0, E - (A + f), n1), at(r0, A, m1, f), at(A + f, A, E - (A + f), f));
                    else
                        gemm_sub(sc, at(A + f, c0, E - (A + f), n1), at(r0, A, m1, f), at(A + f, A, E - (A + f), f));
                }
            }
            if (prows > E) gemm_sub(sd, at(E, c0, prows - E, n1), at(r0, A, m1, E - A), at(E, A, prows - E, E - A));
            deferred.push_back(mark_event(sc.st));
            deferred.push_back(mark_event(sd.st));
        } else if (la_here(r0, m, m1)) {
            flush_deferred();
            const size_t A = r0 + m1, E = r0 + m;  // R's rows / columns
            const size_t e1 = A + thr;
            need(b.st, e1);
            cudaEvent_t forked = mark_event(b.st);
            Blas la = on(lookahead(depth));
            la.sm_cap = lookahead_sms;  // keep SMs free for the critical path
            wait(la.st, forked);
            wait(side.st, forked);
            piece(b, side, r0, m1, A, e1);
            wait(b.st, mark_event(side.st));
            for (size_t x = e1; x < E;) {
                const size_t e = std::min(E, x + std::max(thr, x - A));
                // the bands and older pieces this piece touches only: in the host entry later
                // bands are still on their way over PCIe
                need(la.st, e);
                piece(la, la, r0, m1, x, e);
                pieces.push_back(Piece{x, mark_event(la.st)});
                x = e;
            }
        } else {
            need(b.st, r0 + m);
            flush_deferred();
            // partitioned: both split over the ranks, on the critical stream (one collective order)
            const Blas bside = b.ws.dist.active() ? b : side;
            if (both) wait(bside.st, mark_event(b.st));
            if (!HR.empty()) pgemm_sub(b, Fb, Dx, HR);
            if (both) pgemm_sub(bside, Fbelow, Dn, BP);
            if (both) wait(b.st, mark_event(bside.st));
        }
        rec_panel(a.sub(m1, n1, m - m1, n - n1), depth + 1);
        band_done(r0 + m);
        prog_progress(r0 + m);
        res.rank = std::min(m, n);
        res.pr = Range{};
        res.qr = Range{};
        arena.reset(mark);
        return res;
    }

    // ---- node-level speculation (exact recursion on small fields): where a whole-matrix guess
    // is likely to fail (config 5: GF(251), ~2 rank-deficient blocks per matrix), a square node
    // of <= node_spec_max is still likely full rank; it runs the speculative panel schedule
    // restricted to itself (a sub-driver whose "matrix" is the node), backed up in HBM and
    // rerun exactly when its guess fails.  A full-rank node's result is the unique one (P the
    // identity, Q its blocks' column pivots), so the exact parent continues unchanged.
    size_t node_spec_max = 0;
    int node_spec_fails = 0;  // consecutive failures at a node's first block: stop trying after 3
    const uint32_t* spec_dead = nullptr;  // origin of the last node whose first block failed
    static double host_ms() {
        return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
    }
    static inline const uint32_t* g_log_root = nullptr;  // FFG_NODE_LOG: offsets relative to the entry's matrix
    static inline size_t g_log_ld = 1;
    bool try_node_spec(DView a, int depth, NodeRes& res) {
        const size_t m = a.rows;
        static const bool nlog = knob_set("FFG_NODE_LOG");
        const double t0 = nlog ? host_ms() : 0.0;
        uint32_t* bk = nullptr;
        AsyncFreeGuard<uint32_t> bk_guard{bk, b.st};
        FFG_CUDA(cudaMallocAsync(&bk, m * m * 4, b.st));
        copy_block_dev(b, a, DView{bk, m, m, m});
        std::vector<uint32_t> qh(m);
        bool ok = false, resumable = false;
        size_t fail_off = 0;
        Prefix px;
        {
            Driver sub(b, thr, m, m, /*keep_events=*/true, slot);
            sub.owns_slot = false;
            sub.spec = true;
            *reinterpret_cast<volatile uint32_t*>(&sub.info_host->spec_fail) = 0u;
            sub.panel = true;
            sub.proot = a.d;
            sub.pld = a.ld;
            sub.prows = m;
            sub.pcols = m;
            sub.corner_max = corner_max;
            sub.b.no_direct = panel_no_direct();  // throughput GEMMs, as the whole-matrix schedule
            sub.alloc_panel_inv();
            try {
                sub.rec_panel(a, depth);
                sub.flush_deferred();
                sub.finish();
                sub.panel_finish(nullptr, qh.data(), nullptr);  // synchronizes
                ok = *reinterpret_cast<volatile uint32_t*>(&sub.info_host->spec_fail) == 0u;
            } catch (const SpecAbort&) {
                ok = false;
            }
            if (!ok) {
                FFG_CUDA(cudaDeviceSynchronize());
                if (sub.failed_at(fail_off)) {
                    sub.prefix_of(fail_off, px.gq, px.leaves);
                    resumable = true;
                }
            }
        }
        ++b.ws.st_node;
        if (!ok) ++b.ws.st_node_failed;
        if (nlog)
            fprintf(stderr, "[node] depth %d m %zu at %td: %s fail_off %zu, %.2f ms host\n", depth, m,
                    g_log_root ? (a.d - g_log_root) / (ptrdiff_t)g_log_ld : -1, ok ? "ok" : (resumable ? "resume" : "fail"), fail_off, host_ms() - t0);
        if (!ok && resumable && fail_off > 0) {
            // keep the prefix the schedule finished; recompute the rest of the node from its backup
            node_spec_fails = 0;
            px.root = a.d;
            px.ld = a.ld;
            res = recover(a, depth, fail_off, bk, m, px);
            free_async(bk, b.st);
            return true;
        }
        if (!ok) {
            // the node's first block is deficient: every node on its left spine would fail there
            // too, so the exact recursion descends that spine without guessing (spec_dead)
            copy_block_dev(b, DView{bk, m, m, m}, a);
            free_async(bk, b.st);
            ++node_spec_fails;
            spec_dead = a.d;
            return false;
        }
        free_async(bk, b.st);
        node_spec_fails = 0;
        size_t lo = m, hi = 0;
        for (size_t j = 0; j < m; ++j)
            if (qh[j] != j) {
                lo = std::min(lo, j);
                hi = j + 1;
            }
        res.rank = m;
        res.pr = Range{};
        res.qr = Range{};
        if (hi > lo) {
            FFG_CUDA(cudaMemcpyAsync(res.Q + lo, qh.data() + lo, (hi - lo) * 4, cudaMemcpyHostToDevice, b.st));
            FFG_CUDA(cudaStreamSynchronize(b.st));  // qh is a local buffer
            res.qr = Range{lo, hi};
        }
        return true;
    }

    NodeRes rec(DView a, int depth = 0, cudaEvent_t pending = nullptr, bool rspine = false) {
        const size_t m = a.rows, n = a.cols;
        NodeRes res;
        res.P = arena.alloc(std::max<size_t>(m, 1));
        res.Q = arena.alloc(std::max<size_t>(n, 1));
        if (m == 0 || n == 0) return res;                        // rankrev.hpp:91
        if (node_spec_max && m == n && m > thr && m <= node_spec_max && node_spec_fails < 3 && thr <= 64 &&
            !spine_root && !early.armed && a.d != spec_dead) {
            wait(b.st, pending);
            if (try_node_spec(a, depth, res)) return res;
        }
        if (std::min(m, n) <= thr) {                             // :92
            wait(b.st, pending);
            if (level_timing) {
                LevelRec L{depth, true, {tev(), nullptr, nullptr, nullptr}};
                NodeRes r = base(a, res);
                L.e[1] = tev();
                levels.push_back(L);
                return r;
            }
            return base(a, res);
        }
        LevelRec LR{depth, false, {nullptr, nullptr, nullptr, nullptr}};
        const size_t mark = arena.mark();
        const size_t m1 = (m + 1) / 2, n1 = (n + 1) / 2;         // :95

        cudaEvent_t spine_next = (spine_root && a.d == spine_root && (size_t)depth + 1 < spine.size())
                                     ? spine[depth + 1] : nullptr;
        NodeRes r1s = rec(a.sub(0, 0, m1, n1), depth + 1, spine_next);  // :97
        if (level_timing) LR.e[0] = tev();
        wait(b.st, pending);
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
        cudaEvent_t pending_r = nullptr;
        if (r1 > 0) {                                            // :111-117
            // D = L1^-1 D and Fb = Fb U1^-1 are independent: Fb's chain runs on a twin stream
            const bool fork = use_streams && !D.empty() && !Fb.empty();
            const Blas side = fork ? on(twin(depth)) : b;
            if (fork) wait(side.st, mark_event(b.st));
            if (!D.empty()) ptrsm(b, 0, r1s, L1, D);
            if (!E.empty()) pgemm_sub(b, M1, D, E);
            if (!Fb.empty()) ptrsm(side, 1, r1s, L1, Fb);
            if (!G.empty() && !V1.empty()) pgemm_sub(side, Fb, V1, G);
            if (fork) wait(b.st, mark_event(side.st));
            if (!H.empty()) {
                // look-ahead: with E and G empty, R == H and R's recursion starts with its
                // top-left quadrant; update that first on the critical stream, the rest on a
                // low-priority stream that R waits for only after its first child
                const size_t hm1 = (H.rows + 1) / 2, hn1 = (H.cols + 1) / 2;
                if (use_streams && !b.ws.dist.active() && E.empty() && G.empty() && std::min(H.rows, H.cols) > thr) {
                    gemm_sub(b, Fb.sub(0, 0, hm1, r1), D.sub(0, 0, r1, hn1), H.sub(0, 0, hm1, hn1));
                    Blas la = on(lookahead(depth));
                    la.sm_cap = lookahead_sms;  // keep SMs free for the critical path
                    wait(la.st, mark_event(b.st));
                    gemm_sub(la, Fb.sub(0, 0, hm1, r1), D.sub(0, hn1, r1, H.cols - hn1),
                             H.sub(0, hn1, hm1, H.cols - hn1));
                    gemm_sub(la, Fb.sub(hm1, 0, H.rows - hm1, r1), D, H.sub(hm1, 0, H.rows - hm1, H.cols));
                    pending_r = mark_event(la.st);
                } else {
                    pgemm_sub(b, Fb, D, H);
                }
            }
        }

        return rec_tail(a, depth, res, mark, r1s, pending_r, rspine, LR);
    }

    // tile_rec after its first child and the Schur updates that child feeds (rankrev.hpp:119-183):
    // E and G, the I / K / N / R updates, R, the permutations and the pivot gather
    NodeRes rec_tail(DView a, int depth, NodeRes& res, size_t mark, const NodeRes& r1s, cudaEvent_t pending_r,
                     bool rspine, LevelRec& LR) {
        const size_t m = a.rows, n = a.cols;
        const size_t m1 = (m + 1) / 2, n1 = (n + 1) / 2;
        const size_t r1 = r1s.rank;
        DView E = a.sub(r1, n1, m1 - r1, n - n1);
        DView G = a.sub(m1, r1, m - m1, n1 - r1);
        NodeRes r2s, r3s;                                        // :119-125 (E, G independent)
        std::unique_ptr<Driver> child;
        int cslot = can_fork(E, G) ? b.ws.acquire_slot() : -1;
        if (cslot > 0) {
            active_children().fetch_add(1);
            // the child's streams start after everything enqueued so far (G's updates included)
            child.reset(new Driver(b, thr, G.rows, G.cols, /*keep_events=*/true, cslot));
            Driver* c = child.get();
            std::future<NodeRes> fut = std::async(std::launch::async, [c, G, depth] {
                FFG_CUDA(cudaSetDevice(c->device));
                return c->rec(G, depth + 1);
            });
            try {
                r2s = rec(E, depth + 1);
            } catch (...) {
                fut.wait();
                active_children().fetch_sub(1);
                throw;
            }
            r3s = fut.get();  // rethrows the child's failure
            active_children().fetch_sub(1);
            child->finish();                  // this driver's stream waits for the subtree
            child->arena.free_on(b.st);       // r3s's index arrays are read on this stream
        } else {
            r2s = rec(E, depth + 1);
            r3s = rec(G, depth + 1);
        }
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

        if (r2 > 0 && !I.empty()) ptrsm(b, 1, r2s, U2, I);      // :144
        if (r2 > 0 && !K.empty()) ptrsm(b, 1, r2s, U2, K);      // :145
        uint32_t* jbuf = nullptr;
        AsyncFreeGuard<uint32_t> jbuf_guard{jbuf, b.st};
        DView J = I;
        if (r3 > 0 && !I.empty()) {                              // :146, J = L3^-1 I into a temporary
            FFG_CUDA(cudaMallocAsync(&jbuf, I.rows * I.cols * 4, b.st));
            copy_block_dev(b, I, DView{jbuf, I.rows, I.cols, I.cols});  // kernel: a DMA copy costs more latency
            J = DView{jbuf, I.rows, I.cols, I.cols};
            ptrsm(b, 0, r3s, L3, J);
        }
        if (r3 > 0 && !N.empty()) ptrsm(b, 0, r3s, L3, N);      // :147
        if (!N.empty() && !J.empty()) pgemm_sub(b, J, V2, N);   // :148  O = N - J*V2
        if (!R.empty()) {                                        // :149-152
            if (!K.empty() && !V2.empty()) pgemm_sub(b, K, V2, R);
            if (!N.empty()) pgemm_sub(b, M3, N, R);
        }
        free_async(jbuf, b.st);

        bool early_here = false;
        EarlyTop::Reg reg_top, reg_left;
        if (rspine && early.armed && early.spine_ok) {
            if (r2 == 0 && r3 == 0) {
                // everything that writes outside R before R's recursion is enqueued on b.st
                const size_t off = (size_t)(a.d - early.root);
                const size_t r0 = off / early.ld, c0 = off % early.ld;
                reg_top = EarlyTop::Reg{r0, c0, m1, n};
                reg_left = EarlyTop::Reg{r0 + m1, c0, m - m1, n1};
                wait(early.cs, mark_event(b.st));
                early_copy(reg_top, early.cs);
                early_copy(reg_left, early.cs);
                early.tail = EarlyTop::Reg{r0 + m1, c0 + n1, m - m1, n - n1};  // = R when r2 = r3 = 0
                early_here = true;
            } else {
                early.spine_ok = false;  // this node's whole region stays in the tail
            }
        }
        if (level_timing) LR.e[1] = tev();
        NodeRes r4s = rec(R, depth + 1, pending_r, rspine);      // :154
        if (level_timing) LR.e[2] = tev();
        const size_t r4 = r4s.rank;
        if (early_here && (!r4s.pr.empty() || !r4s.qr.empty() || r1 != m1 || r1 != n1)) {
            // R's permutations or this node's pivot gather move rows/columns of the early copies --
            // its own and, through the gather rotations, those of every spine node below: re-copy
            // the whole node region at the end
            early.redo.push_back(EarlyTop::Reg{reg_top.r0, reg_top.c0, m, n});
        }
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
        arena.reset(mark);  // children consumed (stream order protects the pending kernels)
        if (level_timing) {
            LR.e[3] = tev();
            levels.push_back(LR);
        }
        return res;
    }

    // ---- resume after a failed whole-matrix guess.  The speculative panel
    // schedule failed at the base case starting at global offset pre_a; every pivot before it is
    // final (the schedule solved its row panel, its column panel and -- recomputed from the backup by
    // the caller -- its whole contribution to the trailing square).  resume(node, pre) evaluates
    // tile_rec (rankrev.hpp:85-183) on a square node whose first `pre` rows / columns are that
    // prefix: a first child wholly inside the prefix is taken as factored (full rank, P the identity,
    // Q its blocks' column pivots); otherwise the path to the failed block recurses, and the node's
    // TRSMs / GEMMs after it touch only the non-prefix parts (the prefix parts of D, Fb, E, G, H
    // were applied by the schedule).  The prefix's column pivots reach the rows above their blocks
    // once, at the end (block_cols_perm, as panel_finish does), never through the recursion.
    struct Prefix {
        const uint32_t* root = nullptr;                 // the matrix the offsets refer to
        size_t ld = 0;
        std::vector<uint32_t> gq;                       // block-local column pivot of each prefix column
        std::vector<std::pair<size_t, size_t>> leaves;  // prefix base cases (offset, size)
    };
    NodeRes prefix_res(size_t o, size_t s, const Prefix& px) {
        NodeRes r;
        r.P = arena.alloc(std::max<size_t>(s, 1));
        r.Q = arena.alloc(std::max<size_t>(s, 1));
        r.rank = s;
        std::vector<uint32_t> q(s);
        for (size_t t = 0; t < s; ++t) q[t] = (uint32_t)t;
        size_t lo = s, hi = 0;
        for (const auto& lf : px.leaves) {
            if (lf.first < o || lf.first + lf.second > o + s) continue;
            for (size_t i = 0; i < lf.second; ++i) {
                const size_t t = lf.first - o + i;
                q[t] = (uint32_t)(lf.first - o + px.gq[lf.first + i]);
                if (q[t] != t) {
                    lo = std::min(lo, t);
                    hi = std::max(hi, t + 1);
                }
            }
        }
        if (hi > lo) {
            FFG_CUDA(cudaMemcpyAsync(r.Q + lo, q.data() + lo, (hi - lo) * 4, cudaMemcpyHostToDevice, b.st));
            FFG_CUDA(cudaStreamSynchronize(b.st));  // q is a local buffer
            r.qr = Range{lo, hi};
        }
        return r;
    }
    // a child's column permutation applied only past the prefix (its prefix part is applied later)
    void apply_cols_from(const NodeRes& c, DView v, size_t from) {
        Range r = c.qr;
        r.lo = std::max(r.lo, from);
        if (r.empty() || v.empty()) return;
        perm_apply_range(b, v, 1, c.Q, r.lo, r.hi);
    }
    // After a failed guess on the square region a (speculative schedule drained): restore its
    // trailing square [off, s) x [off, s) from the backup bk (ld ldb, same shape as a) and subtract
    // the prefix pivots' whole contribution, L(rows >= off, prefix) U(prefix, cols >= off) -- the
    // schedule's row and column panels of the prefix are final -- then resume tile_rec on a and
    // apply the prefix blocks' column pivots to the rows above them inside a.
    NodeRes recover(DView a, int depth, size_t off, const uint32_t* bk, size_t ldb, const Prefix& px) {
        const size_t s = a.rows;
        copy_block_dev(b, DView{const_cast<uint32_t*>(bk) + off * ldb + off, s - off, s - off, ldb},
                       a.sub(off, off, s - off, s - off));
        if (off > 0) pgemm_sub(b, a.sub(off, 0, s - off, off), a.sub(0, off, off, s - off), a.sub(off, off, s - off, s - off));
        NodeRes res = resume(a, depth, off, px);
        // prefix column pivots -> the rows above each block (panel_finish's block_cols_perm)
        uint32_t* dq = nullptr;
        for (const auto& lf : px.leaves) {
            bool id = true;
            for (size_t i = 0; i < lf.second; ++i) id = id && px.gq[lf.first + i] == i;
            if (id || lf.first == 0) continue;
            if (!dq) {
                dq = arena.alloc(std::max<size_t>(off, 1));
                FFG_CUDA(cudaMemcpyAsync(dq, px.gq.data(), off * 4, cudaMemcpyHostToDevice, b.st));
                FFG_CUDA(cudaStreamSynchronize(b.st));
            }
            block_cols_perm_dev(b, a.sub(0, lf.first, lf.first, lf.second), dq + lf.first);
        }
        return res;
    }

    NodeRes resume(DView a, int depth, size_t pre, const Prefix& px) {
        const size_t m = a.rows, n = a.cols;  // square, diagonal
        if (pre == 0) return rec(a, depth);
        if (m <= thr || pre >= m) throw Error(FFG_ERR_INTERNAL, "resume: prefix does not end at a base case");
        NodeRes res;
        res.P = arena.alloc(m);
        res.Q = arena.alloc(n);
        LevelRec LR{depth, false, {nullptr, nullptr, nullptr, nullptr}};
        const size_t mark = arena.mark();
        const size_t m1 = (m + 1) / 2, n1 = (n + 1) / 2;
        if (pre >= m1) {  // the failed block lies in R: A1 is a full-rank prefix node
            const NodeRes r1s = prefix_res((size_t)(a.d - px.root) / px.ld, m1, px);
            const size_t r1 = m1;
            // D, Fb solved, E and G empty, H updated: the schedule did all of it
            NodeRes r4s = resume(a.sub(m1, n1, m - m1, n - n1), depth + 1, pre - m1, px);
            const size_t r4 = r4s.rank;
            apply(r4s, 0, a.sub(m1, 0, m - m1, r1));                      // rankrev.hpp:156
            apply_cols_from(r4s, a.sub(0, n1, r1, n - n1), pre - m1);     // :158
            bool pinit = false, qinit = false;                            // :163-170 (r2 = r3 = 0)
            compose(res.P, pinit, m, res.pr, 0, r1s.P, r1s.pr);
            compose(res.P, pinit, m, res.pr, m1, r4s.P, r4s.pr);
            compose(res.Q, qinit, n, res.qr, 0, r1s.Q, r1s.qr);
            compose(res.Q, qinit, n, res.qr, n1, r4s.Q, r4s.qr);
            // :174-179: every gather rotation is empty (r1 = m1 = n1, r2 = r3 = 0)
            res.rank = r1 + r4;
            arena.reset(mark);
            return res;
        }
        // the failed block lies in A1
        NodeRes r1s = resume(a.sub(0, 0, m1, n1), depth + 1, pre, px);  // :97
        const size_t r1 = r1s.rank;
        apply(r1s, 0, a.sub(0, n1, m1, n - n1));                        // :99 (never moves prefix rows)
        apply_cols_from(r1s, a.sub(m1, 0, m - m1, n1), pre);            // :100
        if (r1 > pre) {                                                 // :111-117, past the prefix
            const size_t q = r1 - pre;
            DView Lr = a.sub(pre, pre, q, q);  // trailing part of L1 \ U1
            DView Dr = a.sub(pre, n1, q, n - n1);
            DView M1r = a.sub(r1, pre, m1 - r1, q);
            DView E = a.sub(r1, n1, m1 - r1, n - n1);
            DView Fbr = a.sub(m1, pre, m - m1, q);
            DView V1r = a.sub(pre, r1, q, n1 - r1);
            DView G = a.sub(m1, r1, m - m1, n1 - r1);
            DView H = a.sub(m1, n1, m - m1, n - n1);
            if (!Dr.empty()) ptrsm(b, 0, r1s, Lr, Dr);
            if (!E.empty() && !M1r.empty()) pgemm_sub(b, M1r, Dr, E);
            if (!Fbr.empty()) ptrsm(b, 1, r1s, Lr, Fbr);
            if (!G.empty() && !V1r.empty()) pgemm_sub(b, Fbr, V1r, G);
            if (!H.empty()) pgemm_sub(b, Fbr, Dr, H);
        }
        return rec_tail(a, depth, res, mark, r1s, nullptr, false, LR);
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

void base_dbg_dump();

// Speculation is tried unless disabled (FFG_NO_SPEC), partitioned, profiled, or recently failed in
// this context (then it rests for a few calls: rank-deficient workloads pay one failed try).
static bool spec_allowed(const Blas& b, const DView& a, size_t thr) {
    static const bool off = knob_set("FFG_NO_SPEC") || knob_set("FFG_LEVEL_TIMING");
    if (off || a.rows == 0 || a.cols == 0) return false;
    // A base block of i.i.d. residues is rank deficient with probability ~1/p (config 5's GF(251)
    // at n = 32768: ~2 such blocks per matrix).  A failed guess costs little on square input: the
    // schedule's prefix is kept and tile_rec resumes at the failed block (Driver::recover).
    // Non-square input reruns from scratch: skip the guess there when it is likely to fail.
    const double blocks = (double)std::min(a.rows, a.cols) / (double)std::max<size_t>(thr, 1);
    if (a.rows != a.cols && blocks > 0.25 * (double)b.F.p) return false;
    if (b.ws.spec_rest > 0) {
        --b.ws.spec_rest;
        return false;
    }
    return true;
}

// panel-mode nodes of at least this size cut their trailing update into look-ahead pieces
// (FFG_PANEL_LA, read per call so tests can sweep it; 0 = off)
// the whole-matrix panel schedule issues its tensor-core GEMMs through the split + TMA pipeline:
// off the critical path, throughput beats the direct kernel's latency (n = 16384: 29.4 -> 29.0
// ms); the exact recursion (configs 4 / 5) keeps the direct kernel.  FFG_PANEL_DIRECT=1 reverts.
static bool panel_no_direct() {
    static const bool keep = knob_on("FFG_PANEL_DIRECT");
    return !keep;
}

// panel-mode nodes up to this size update only R's first block on the critical stream and defer
// their wide GEMMs (FFG_CORNER_MAX, read per call; 0 = off)
static size_t panel_corner_max() {
    const char* e = knob_str("FFG_CORNER_MAX");
    return e ? (size_t)atoll(e) : 4096;  // 1024 / 2048 / 4096 / 8192: 29.1 / 28.7 / 28.7 / 28.7 ms
}
// partitioned runs split the generic nodes' GEMMs over the ranks and keep the corner nodes'
// deferred GEMMs replicated: keep more nodes generic there
static size_t panel_corner_max(const Blas& b) {
    const size_t c = panel_corner_max();
    return (b.ws.dist.active() && !knob_set("FFG_CORNER_MAX")) ? std::min<size_t>(c, 1024) : c;
}

// panel-mode nodes of at least this size apply their trailing update progressively in K-chunks
// (FFG_PROG_MIN, read per call; 0 = off); FFG_PROG_CHUNKS chunks per node, FFG_PROG_SMS SM cap
static size_t panel_prog_min() {
    const char* e = knob_str("FFG_PROG_MIN");
    return e ? (size_t)atoll(e) : 0;
}
static size_t prog_chunks() {
    const char* e = knob_str("FFG_PROG_CHUNKS");
    return e ? std::max<size_t>(1, (size_t)atoll(e)) : 4;
}

static size_t panel_lookahead_min() {
    const char* e = knob_str("FFG_PANEL_LA");
    return e ? (size_t)atoll(e) : 0;
}

// Node-level speculation of the exact recursion (FFG_NODE_SPEC = largest node, 0 = off): only
// where the whole-matrix guess was skipped for a small field, nodes whose guess holds with
// probability >= ~90% (blocks per node <= p / 10), single stream drivers excluded.
static size_t node_spec_max(const Blas& b, const DView& a, size_t thr, const Driver& drv) {
    static const bool off = knob_set("FFG_NO_SPEC") || knob_set("FFG_LEVEL_TIMING");
    const char* e = knob_str("FFG_NODE_SPEC");
    size_t s = e ? (size_t)atoll(e) : 1024;
    if (off || s == 0 || !drv.use_streams || thr > 64) return 0;
    const double blocks_all = (double)std::min(a.rows, a.cols) / (double)std::max<size_t>(thr, 1);
    if (blocks_all <= 0.25 * (double)b.F.p) return 0;  // the whole-matrix guess was tried instead
    static const double risk = knob_num("FFG_NODE_SPEC_RISK", 0.1);
    while (s > thr && (double)s / (double)thr > risk * (double)b.F.p) s /= 2;
    return s > 2 * thr ? s : 0;
}

// band ends for the streamed host entry: the recursion's nodes of size <= min(T, max(Tmin, o)) in
// order -- finer at the start, where the factorisation waits for each band
static void band_bounds(size_t o, size_t s, size_t thr, size_t T, size_t Tmin, std::vector<size_t>& out) {
    if (s <= thr || s <= std::min(T, std::max(Tmin, o))) {
        out.push_back(o + s);
        return;
    }
    const size_t h = (s + 1) / 2;
    band_bounds(o, h, thr, T, Tmin, out);
    band_bounds(o + h, s - h, thr, T, Tmin, out);
}

// The profile-first exact path (profile.cu) replaces the exact recursion for rank-deficient input
// of order >= 512: FFG_PROFILE_FIRST (read per call) 0 = never, 2 = always (whenever the slab kernel
// takes the width; tests), default: when the whole-matrix guess failed in its first eighth -- the
// matrix is deficient throughout -- or was not tried, on single-GPU runs (partitioned runs keep
// the recursion, whose large operations split over the ranks).
static int profile_first_mode() {
    const char* e = knob_str("FFG_PROFILE_FIRST");
    return e ? atoi(e) : 1;
}
static bool profile_first_ok(const Blas& b, size_t m, size_t n) {
    const int mode = profile_first_mode();
    // (the path factors its generic leading block through pluq_tile_recursive_dev: never nested)
    if (mode == 0 || profile_first_active() || b.ws.dist.active() || b.ws.prof.mode == 1 || !profile_first_fits(n)) return false;
    return mode == 2 || std::min(m, n) >= 512;
}
// after a failed whole-matrix guess at diagonal offset fail_off: the matrix counts as deficient
// throughout when its very first block failed, or when it failed in the first eighth over a field
// where a random singular block is not expected (blocks / p < 0.05; GF(251) at n = 32768 expects
// two such blocks per matrix, and resuming there costs less than a second elimination)
static bool profile_first_after_failure(const Blas& b, size_t fail_off, size_t m, size_t n, size_t thr) {
    if (!profile_first_ok(b, m, n)) return false;
    if (fail_off == 0) return true;
    const double blocks = (double)std::min(m, n) / (double)std::max<size_t>(thr, 1);
    return fail_off < std::min(m, n) / 8 && blocks < 0.05 * (double)b.F.p;
}

// Streamed speculative attempt of the host entry (square input, panel mode): band c uploads on
// one copy engine, is backed up in HBM by a copy kernel, factors, and downloads on the other copy
// engine as soon as its last base case is done -- PCIe in both directions overlaps the
// factorisation.  false: the guess failed (or was abandoned); d then holds the input again.
static bool host_streamed_spec(const Blas& b, uint32_t* host, size_t n, size_t lda, size_t thr, uint32_t* d,
                               uint32_t* P, uint32_t* Q, size_t& rank) {
    uint32_t* bk = nullptr;
    AsyncFreeGuard<uint32_t> bk_guard{bk, b.st};
    FFG_CUDA(cudaMallocAsync(&bk, n * n * 4, b.st));
    bool ok = false, resumable = false;
    size_t fail_off = 0;
    Driver::Prefix px;
    {
        Driver drv(b, thr, n, n);
        drv.spec = true;
        *reinterpret_cast<volatile uint32_t*>(&drv.info_host->spec_fail) = 0u;
        drv.panel = true;
        drv.b.no_direct = panel_no_direct();
        drv.la_min = panel_lookahead_min();
        {
            // look-ahead pieces in the first half of the matrix, where the factorisation waits for
            // the bands still crossing PCIe: R's first band starts as soon as it has arrived
            // (n = 16384: e2e 42.4 -> 39.6 ms with nodes >= n/4 ending in the first half; the root
            // included: 40.3 ms)
            const char* e = knob_str("FFG_HOST_LA");
            const char* ee = knob_str("FFG_HOST_LA_END");
            const size_t hl = e ? (size_t)atoll(e) : (n / 4 >= 2048 ? n / 4 : 0);
            if (hl && !drv.la_min) {  // an explicit FFG_PANEL_LA wins
                drv.la_min = hl;
                drv.la_end = ee ? (size_t)(atof(ee) * (double)n) : n / 2;
            }
        }
        drv.corner_max = panel_corner_max(b);
        drv.prog_min = panel_prog_min();
        drv.prog_nchunks = prog_chunks();
        drv.prog_sms = (int)knob_int("FFG_PROG_SMS", drv.lookahead_sms);
        drv.proot = d;
        drv.pld = n;
        drv.prows = n;
        drv.pcols = n;
        drv.alloc_panel_inv();
        cudaStream_t up = b.ws.stream(300, 0), down = b.ws.stream(301, 0), bks = b.ws.stream(302, 0);
        cudaEvent_t start = drv.b.ws.event();  // d and bk are allocated on the caller's stream
        FFG_CUDA(cudaEventRecord(start, b.st));
        for (cudaStream_t st : {up, down, bks}) drv.wait(st, start);
        const size_t T_env = (size_t)knob_int("FFG_BAND_MAX", 0);
        const size_t Tmin_env = (size_t)knob_int("FFG_BAND_MIN", 256);
        const size_t T = T_env ? T_env : std::max<size_t>(256, n / 16);
        // bands of 256 rows first (a narrower band's column strip is a 2-D copy of short rows,
        // which the copy engines move slowly: 128-row bands measured slower)
        band_bounds(0, n, thr, T, Tmin_env, drv.bands.end);
        drv.bands.on = true;
        drv.bands.host = host;
        drv.bands.ldh = lda;
        drv.bands.down = down;
        drv.bands.backup = bk;
        drv.bands.bks = bks;
        for (size_t c = 0; c < drv.bands.end.size(); ++c) {
            drv.band_copy(c, false, up);
            drv.bands.uploaded.push_back(drv.mark_event(up));
        }
        try {
            NodeRes res = drv.rec_panel(DView{d, n, n, n}, 0);
            drv.flush_deferred();
            drv.need(drv.b.st, n);  // every band backed up before the call returns
            drv.finish();
            FFG_CUDA(cudaStreamSynchronize(down));
            std::vector<std::pair<size_t, size_t>> fixed;
            drv.panel_finish(P, Q, &fixed);  // synchronizes the critical stream
            ok = *reinterpret_cast<volatile uint32_t*>(&drv.info_host->spec_fail) == 0u;
            if (ok && !fixed.empty()) {  // rows above a pivoted block changed after their band left
                for (const auto& f : fixed)
                    FFG_CUDA(cudaMemcpy2DAsync(host + f.first, lda * 4, d + f.first, n * 4, f.second * 4, f.first,
                                               cudaMemcpyDeviceToHost, drv.b.st));
                FFG_CUDA(cudaStreamSynchronize(drv.b.st));
            }
            rank = res.rank;
        } catch (const Driver::SpecAbort&) {
            ok = false;
            drv.need(drv.b.st, n);  // bands no operation touched yet are still pristine: back them up too
        }
        if (!ok) {
            FFG_CUDA(cudaDeviceSynchronize());  // every speculative kernel and copy retired
            if (drv.failed_at(fail_off)) {
                drv.prefix_of(fail_off, px.gq, px.leaves);
                resumable = true;
            }
        }
    }
    ++b.ws.st_guess;
    if (!ok) ++b.ws.st_guess_failed;
    if (!ok && resumable && profile_first_after_failure(b, fail_off, n, n, thr)) resumable = false;  // profile-first
    if (!ok && resumable) {
        // resume tile_rec at the failed block on the device copy (every band is uploaded and backed
        // up by now), then bring the whole matrix back
        Driver rdrv(b, thr, n, n);
        rdrv.node_spec_max = n;
        px.root = d;
        px.ld = n;
        NodeRes res = rdrv.recover(DView{d, n, n, n}, 0, fail_off, bk, n, px);
        rdrv.finish();
        FFG_CUDA(cudaMemcpy2DAsync(host, lda * 4, d, n * 4, n * 4, n, cudaMemcpyDeviceToHost, rdrv.b.st));
        rdrv.download(res, n, n, P, Q);  // synchronizes
        rank = res.rank;
        if (fail_off == 0)
            b.ws.spec_failed();
        else
            b.ws.spec_fails = 0;
        free_async(bk, b.st);
        return true;
    }
    if (!ok) {
        copy_block_dev(b, DView{bk, n, n, n}, DView{d, n, n, n});
        b.ws.spec_failed();
    } else {
        b.ws.spec_fails = 0;
    }
    free_async(bk, b.st);
    return ok;
}

size_t pluq_tile_recursive_dev(const Blas& b, DView a, size_t threshold, uint32_t* P, uint32_t* Q) {
    if (profile_first_mode() == 2 && profile_first_ok(b, a.rows, a.cols))
        return pluq_profile_first_dev(b, a, threshold, P, Q);
    if (threshold <= 64 && spec_allowed(b, a, threshold)) {
        const size_t m = a.rows, n = a.cols;
        const bool no_panel = knob_on("FFG_NO_PANEL");
        const bool panel = !no_panel && m == n;
        // backup of the input for a failed guess: the panel schedule backs each band up lazily
        // on a side stream right before its first use (bands, as the host entry); otherwise
        // one copy up front
        uint32_t* bk = nullptr;
        AsyncFreeGuard<uint32_t> bk_guard{bk, b.st};
        const size_t ldb = panel ? a.ld : n;
        FFG_CUDA(cudaMallocAsync(&bk, m * ldb * 4, b.st));
        if (!panel) copy_block_dev(b, a, DView{bk, m, n, ldb});
        bool ok = false, resumable = false;
        size_t rank = 0, fail_off = 0;
        Driver::Prefix px;
        {
            Driver drv(b, threshold, m, n);
            drv.spec = true;
            *reinterpret_cast<volatile uint32_t*>(&drv.info_host->spec_fail) = 0u;
            drv.panel = panel;
            drv.la_min = panel_lookahead_min();
            drv.corner_max = panel_corner_max(b);
            drv.prog_min = panel_prog_min();
            drv.prog_nchunks = prog_chunks();
            drv.prog_sms = (int)knob_int("FFG_PROG_SMS", drv.lookahead_sms);
            drv.proot = a.d;
            drv.pld = a.ld;
            drv.prows = m;
            drv.pcols = n;
            if (drv.panel) {
                drv.b.no_direct = panel_no_direct();  // the panel schedule's GEMMs are throughput work
                drv.alloc_panel_inv();
                const size_t T = std::max<size_t>(256, n / 16);
                band_bounds(0, n, drv.thr, T, 256, drv.bands.end);
                const cudaEvent_t start = drv.mark_event(b.st);  // the input is in place
                drv.bands.uploaded.assign(drv.bands.end.size(), start);
                drv.bands.backup = bk;
                drv.bands.bks = b.ws.stream(302, 0);
                drv.bands.on = true;
            }
            try {
                NodeRes res = drv.panel ? drv.rec_panel(a, 0) : drv.rec(a);
                drv.flush_deferred();
                drv.finish();
                if (drv.panel)
                    drv.panel_finish(P, Q, nullptr);  // synchronizes: every base kernel has reported
                else
                    drv.download(res, m, n, P, Q);
                ok = *reinterpret_cast<volatile uint32_t*>(&drv.info_host->spec_fail) == 0u;
                rank = res.rank;
            } catch (const Driver::SpecAbort&) {
                ok = false;
            }
            if (!ok && drv.panel) drv.need(drv.b.st, n);  // bands nothing touched yet are still pristine
            if (!ok) FFG_CUDA(cudaDeviceSynchronize());  // all speculative work retired
            if (!ok && drv.panel && drv.failed_at(fail_off)) {
                drv.prefix_of(fail_off, px.gq, px.leaves);
                resumable = true;
            }
            static const bool tlog = knob_set("FFG_SPEC_LOG");
            if (tlog)
                fprintf(stderr, "SPEC host run-ahead: %llu throttle points, the host waited for the device at %llu\n",
                        (unsigned long long)drv.throttle_calls, (unsigned long long)drv.throttle_waits);
        }
        ++b.ws.st_guess;
        if (!ok) ++b.ws.st_guess_failed;
        static const bool log = knob_set("FFG_SPEC_LOG");
        if (log) fprintf(stderr, "SPEC %s (panel %d, %zu base cases enqueued)\n", ok ? "ok" : "failed", (int)(m == n), (size_t)b.ws.base_seq.load());
        if (ok) {
            b.ws.spec_fails = 0;
            free_async(bk, b.st);
            return rank;
        }
        if (resumable && profile_first_after_failure(b, fail_off, m, n, threshold)) {
            // deficient from the start: the profile-first path on the restored input
            copy_block_dev(b, DView{bk, m, n, ldb}, a);
            free_async(bk, b.st);
            if (fail_off == 0) b.ws.spec_failed();
            return pluq_profile_first_dev(b, a, threshold, P, Q);
        }
        if (resumable) {
            // the pivots before the failed block are final: resume tile_rec from there (the rest of
            // the matrix is recomputed from the backup), node-level guesses again on fresh subproblems
            Driver rdrv(b, threshold, m, n);
            rdrv.node_spec_max = std::min(m, n);
            Driver::Prefix& rx = px;
            Driver::g_log_root = a.d;
            Driver::g_log_ld = a.ld;
            rx.root = a.d;
            rx.ld = a.ld;
            NodeRes res = rdrv.recover(a, 0, fail_off, bk, ldb, rx);
            rdrv.finish();
            rdrv.download(res, m, n, P, Q);
            free_async(bk, b.st);
            if (fail_off == 0)
                b.ws.spec_failed();  // the very first block: likely deficient everywhere, rest a few calls
            else
                b.ws.spec_fails = 0;
            static const bool log2 = knob_set("FFG_SPEC_LOG");
            if (log2) fprintf(stderr, "SPEC resumed at offset %zu of %zu\n", fail_off, m);
            return res.rank;
        }
        copy_block_dev(b, DView{bk, m, n, ldb}, a);  // a copy kernel: the DMA engines are far slower HBM to HBM
        free_async(bk, b.st);
        b.ws.spec_failed();
    }
    if (profile_first_ok(b, a.rows, a.cols)) return pluq_profile_first_dev(b, a, threshold, P, Q);
    Driver drv(b, threshold, a.rows, a.cols);
    drv.level_timing = knob_set("FFG_LEVEL_TIMING");
    drv.node_spec_max = node_spec_max(b, a, threshold, drv);
    NodeRes res = drv.rec(a);
    drv.level_report();
    drv.finish();
    drv.download(res, a.rows, a.cols, P, Q);
    base_dbg_dump();
    return res.rank;
}

size_t pluq_tile_recursive_host(const Blas& b, uint32_t* host, size_t m, size_t n, size_t lda, size_t threshold,
                                uint32_t* P, uint32_t* Q) {
    if (m == 0 || n == 0) {
        Driver drv(b, threshold, m, n);
        NodeRes res = drv.rec(DView{nullptr, m, n, n});
        drv.finish();
        drv.download(res, m, n, P, Q);
        return 0;
    }
    const size_t thr = std::max<size_t>(1, threshold);
    cudaStream_t cs = b.ws.stream(300, 0);  // copy stream
    uint32_t* d = nullptr;
    AsyncFreeGuard<uint32_t> d_guard{d, b.st};
    FFG_CUDA(cudaMallocAsync(&d, m * n * 4, b.st));
    static const bool no_stream_spec = knob_set("FFG_NO_HOST_SPEC");
    static const bool no_streams = knob_on("FFG_NO_STREAMS");
    static const bool no_panel = knob_on("FFG_NO_PANEL");
    bool restored = false;  // d already holds the input (a failed speculative attempt restored it)
    if (m == n && thr <= 64 && !no_stream_spec && !no_streams && !no_panel && spec_allowed(b, DView{host, m, n, lda}, thr)) {
        size_t rank = 0;
        if (host_streamed_spec(b, host, n, lda, thr, d, P, Q, rank)) {
            free_async(d, b.st);
            FFG_CUDA(cudaStreamSynchronize(b.st));
            return rank;
        }
        restored = true;
    }
    if (profile_first_ok(b, m, n)) {  // rank-deficient input: upload, profile-first, download
        if (!restored)
            FFG_CUDA(cudaMemcpy2DAsync(d, n * 4, host, lda * 4, n * 4, m, cudaMemcpyHostToDevice, b.st));
        const size_t rank = pluq_profile_first_dev(b, DView{d, m, n, n}, thr, P, Q);
        FFG_CUDA(cudaMemcpy2DAsync(host, lda * 4, d, n * 4, n * 4, m, cudaMemcpyDeviceToHost, b.st));
        free_async(d, b.st);
        FFG_CUDA(cudaStreamSynchronize(b.st));
        return rank;
    }
    // speculative full rank (see Driver::spec) is off here: its device backup would share the copy
    // stream with the spine uploads and delay them more than the saved rank round trips gain
    // (measured: e2e 75 ms with, 63 ms without).  The machinery below stays ready for it.
    const bool spec = false;
    uint32_t* bk = nullptr;
    AsyncFreeGuard<uint32_t> bk_guard{bk, b.st};
    if (spec) FFG_CUDA(cudaMallocAsync(&bk, m * n * 4, b.st));
    b.ws.reset_events();
    auto record = [&](cudaStream_t st) {
        cudaEvent_t e = b.ws.event();
        FFG_CUDA(cudaEventRecord(e, st));
        return e;
    };
    FFG_CUDA(cudaStreamWaitEvent(cs, record(b.st), 0));
    auto up = [&](size_t r0, size_t c0, size_t rows, size_t cols) {
        if (!rows || !cols) return;
        FFG_CUDA(cudaMemcpy2DAsync(d + r0 * n + c0, n * 4, host + r0 * lda + c0, lda * 4, cols * 4, rows,
                                   cudaMemcpyHostToDevice, cs));
        if (bk)
            FFG_CUDA(cudaMemcpy2DAsync(bk + r0 * n + c0, n * 4, d + r0 * n + c0, n * 4, cols * 4, rows,
                                       cudaMemcpyDeviceToDevice, cs));
    };
    // spine blocks S_0 = whole matrix, S_{d+1} = top-left ceil-halves, down to ~16 MB or a leaf
    std::vector<std::pair<size_t, size_t>> sp{{m, n}};
    static const bool no_spine = knob_set("FFG_NO_SPINE");  // diagnostics: upload all first
    while (!restored && !no_spine && std::min(sp.back().first, sp.back().second) > thr &&
           sp.back().first * sp.back().second > (size_t(1) << 22))
        sp.push_back({(sp.back().first + 1) / 2, (sp.back().second + 1) / 2});
    const size_t K = sp.size() - 1;
    if (!restored) up(0, 0, sp[K].first, sp[K].second);
    FFG_CUDA(cudaStreamWaitEvent(b.st, record(cs), 0));  // the deepest spine block is in place
    std::vector<cudaEvent_t> spine(K, nullptr);
    for (size_t lv = K; lv-- > 0;) {  // S_lv minus S_{lv+1}: right strip, then the rows below
        up(0, sp[lv + 1].second, sp[lv + 1].first, sp[lv].second - sp[lv + 1].second);
        up(sp[lv + 1].first, 0, sp[lv].first - sp[lv + 1].first, sp[lv].second);
        spine[lv] = record(cs);
    }
    // one factorisation of d with early downloads; false when a speculative guess failed
    auto run = [&](bool speculative, bool upload_pending, size_t& rank) -> bool {
        // the Driver resets the event cursor: keep the events above alive by recording after it
        Driver drv(b, thr, m, n, /*keep_events=*/true);
        drv.spec = speculative;
        if (speculative) *reinterpret_cast<volatile uint32_t*>(&drv.info_host->spec_fail) = 0u;
        if (upload_pending) {
            drv.spine_root = d;
            drv.spine = spine;
        }
        drv.early.armed = !knob_set("FFG_NO_EARLY");  // diagnostics: download all at the end
        drv.early.cs = cs;
        drv.early.host = host;
        drv.early.ldh = lda;
        drv.early.root = d;
        drv.early.ld = n;
        drv.early.tail = Driver::EarlyTop::Reg{0, 0, m, n};
        try {
            NodeRes res = drv.rec(DView{d, m, n, n}, 0, upload_pending && K > 0 ? spine[0] : nullptr,
                                  /*rspine=*/true);
            drv.finish();
            // after the early copies (same host buffer, same D2H engine): the tail and stale regions
            FFG_CUDA(cudaStreamWaitEvent(b.st, record(cs), 0));
            drv.early.cs = b.st;
            drv.early_copy(drv.early.tail, b.st);
            for (const auto& g : drv.early.redo) drv.early_copy(g, b.st);
            drv.download(res, m, n, P, Q);  // synchronizes the critical stream
            FFG_CUDA(cudaStreamSynchronize(cs));
            FFG_CUDA(cudaStreamSynchronize(b.st));
            rank = res.rank;
        } catch (const Driver::SpecAbort&) {
            FFG_CUDA(cudaDeviceSynchronize());
            return false;
        }
        return !speculative || *reinterpret_cast<volatile uint32_t*>(&drv.info_host->spec_fail) == 0u;
    };
    size_t rank = 0;
    if (restored) {
        run(false, false, rank);
    } else if (!run(spec, true, rank)) {
        FFG_CUDA(cudaDeviceSynchronize());  // every speculative kernel and copy retired
        FFG_CUDA(cudaMemcpy2DAsync(d, n * 4, bk, n * 4, n * 4, m, cudaMemcpyDeviceToDevice, b.st));
        b.ws.spec_failed();
        run(false, false, rank);
    }
    free_async(bk, b.st);
    free_async(d, b.st);
    return rank;
}

size_t pluq_tile_recursive_host_u8(const Blas& b, uint8_t* host, size_t m, size_t n, size_t lda, size_t threshold,
                                   uint32_t* P, uint32_t* Q) {
    if (b.F.p > 256) throw Error(FFG_ERR_CAPACITY, "byte storage needs p <= 256");
    if (m == 0 || n == 0) return pluq_tile_recursive_dev(b, DView{nullptr, m, n, std::max<size_t>(n, 1)}, threshold, P, Q);
    cudaStream_t cs = b.ws.stream(300, 0);  // copy stream
    uint32_t* d = nullptr;
    uint8_t* s8 = nullptr;
    AsyncFreeGuard<uint32_t> d_guard{d, b.st};
    AsyncFreeGuard<uint8_t> s8_guard{s8, b.st};
    FFG_CUDA(cudaMallocAsync(&d, m * n * 4, b.st));
    FFG_CUDA(cudaMallocAsync(&s8, m * n, b.st));
    b.ws.reset_events();
    auto mark = [&](cudaStream_t st) {
        cudaEvent_t e = b.ws.event();
        FFG_CUDA(cudaEventRecord(e, st));
        return e;
    };
    FFG_CUDA(cudaStreamWaitEvent(cs, mark(b.st), 0));
    const size_t chunk = std::max<size_t>(1, (size_t(32) << 20) / n);  // ~32 MB of bytes per copy
    for (size_t r0 = 0; r0 < m; r0 += chunk) {  // upload chunk i while chunk i-1 widens
        const size_t rows = std::min(chunk, m - r0);
        FFG_CUDA(cudaMemcpy2DAsync(s8 + r0 * n, n, host + r0 * lda, lda, n, rows, cudaMemcpyHostToDevice, cs));
        FFG_CUDA(cudaStreamWaitEvent(b.st, mark(cs), 0));
        widen_u8_dev(b, s8 + r0 * n, n, DView{d + r0 * n, rows, n, n});
    }
    const size_t rank = pluq_tile_recursive_dev(b, DView{d, m, n, n}, threshold, P, Q);
    for (size_t r0 = 0; r0 < m; r0 += chunk) {  // narrow chunk i while chunk i-1 downloads
        const size_t rows = std::min(chunk, m - r0);
        narrow_u8_dev(b, DView{d + r0 * n, rows, n, n}, s8 + r0 * n, n);
        FFG_CUDA(cudaStreamWaitEvent(cs, mark(b.st), 0));
        FFG_CUDA(cudaMemcpy2DAsync(host + r0 * lda, lda, s8 + r0 * n, n, n, rows, cudaMemcpyDeviceToHost, cs));
    }
    FFG_CUDA(cudaStreamWaitEvent(b.st, mark(cs), 0));
    free_async(s8, b.st);
    free_async(d, b.st);
    FFG_CUDA(cudaStreamSynchronize(b.st));
    return rank;
}

size_t rr_base_dev(const Blas& b, DView a, uint32_t* P, uint32_t* Q) {
    Driver drv(b, SIZE_MAX, a.rows, a.cols);
    NodeRes res = drv.rec(a);
    drv.finish();
    drv.download(res, a.rows, a.cols, P, Q);
    return res.rank;
}

}  // namespace ffg
