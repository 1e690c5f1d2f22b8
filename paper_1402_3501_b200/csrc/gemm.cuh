// gemm.cuh -- internal API of the modular BLAS layer (GEMM, TRSM) and device workspace.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstring>
#include <mutex>
#include <unordered_map>
#include <vector>

#include "common.cuh"
#include "dist.cuh"

namespace ffg {

// Optional per-kernel timing: CUDA events recorded on the launching stream
// around each kernel of a class, summed on read.  Off unless a caller enables
// it (bench.py's roofline), so the product path pays nothing by default.
enum ProfKind {
    PROF_GEMM = 0,
    PROF_SPLIT = 1,
    PROF_BASE = 2,
    PROF_TRINV = 3,
    PROF_PERM = 4,
    PROF_SIMT = 5,
    PROF_NKINDS = 6
};

class Profiler {
public:
    // 0 off, 1 CUDA events around every launch, 2 count launches and work only (no events: the
    // schedule is not perturbed; bench.py pairs it with CUPTI kernel durations)
    int mode = 0;
    ~Profiler() { clear(true); }
    void begin(cudaStream_t st) {
        if (mode != 1) return;
        std::lock_guard<std::mutex> g(mu_);
        cur_a_ = take();
        cudaEventRecord(cur_a_, st);
    }
    // work = algorithmic units of this launch (int8 tensor ops for GEMM, bytes for others)
    void end(cudaStream_t st, int kind, double work, double field_ops = 0) {
        if (mode == 0) return;
        std::lock_guard<std::mutex> g(mu_);
        cudaEvent_t b = nullptr;
        if (mode == 1) {
            b = take();
            cudaEventRecord(b, st);
        }
        recs_.push_back(Rec{mode == 1 ? cur_a_ : nullptr, b, kind, work, field_ops});
    }
    // totals per kind: ms, launches, work, field_ops (synchronizes the recorded events)
    void read(double* ms, double* launches, double* work, double* field_ops) {
        std::lock_guard<std::mutex> g(mu_);
        for (int k = 0; k < PROF_NKINDS; ++k) ms[k] = launches[k] = work[k] = field_ops[k] = 0;
        for (auto& r : recs_) {
            float t = 0;
            if (r.a && r.b) {
                cudaEventSynchronize(r.b);
                cudaEventElapsedTime(&t, r.a, r.b);
            }
            ms[r.kind] += t;
            launches[r.kind] += 1;
            work[r.kind] += r.work;
            field_ops[r.kind] += r.field_ops;
        }
    }
    void clear(bool destroy = false) {
        std::lock_guard<std::mutex> g(mu_);
        for (auto& r : recs_) {
            if (r.a) free_.push_back(r.a);
            if (r.b) free_.push_back(r.b);
        }
        recs_.clear();
        if (destroy) {
            for (auto e : free_) cudaEventDestroy(e);
            free_.clear();
        }
    }

private:
    struct Rec {
        cudaEvent_t a, b;
        int kind;
        double work, field_ops;
    };
    cudaEvent_t take() {
        if (!free_.empty()) {
            cudaEvent_t e = free_.back();
            free_.pop_back();
            return e;
        }
        cudaEvent_t e;
        cudaEventCreate(&e);
        return e;
    }
    std::mutex mu_;
    cudaEvent_t cur_a_ = nullptr;
    std::vector<Rec> recs_;
    std::vector<cudaEvent_t> free_;
};

// Per-stream scratch arena (the limb planes of the operands, temporaries of the
// recursion).  Growth synchronizes the owning stream, so kernels already
// enqueued on it never see their scratch freed.  Allocation is a bump pointer
// reset by mark/release around each top-level call.
class Workspace {
public:
    Profiler prof;
    std::atomic<uint32_t> base_seq{0};  // sequence numbers of base-case completion mailboxes
    // outcomes of the full-rank guesses since the context was created (ffg_spec_stats):
    // whole-matrix guesses tried / failed, node-level guesses tried / failed, profile-first runs
    std::atomic<uint64_t> st_guess{0}, st_guess_failed{0}, st_node{0}, st_node_failed{0}, st_profile_first{0};
    int spec_rest = 0;                   // calls left before speculative full rank is tried again
    int spec_fails = 0;                  // consecutive failed guesses (the rest doubles with them)
    void spec_failed() {
        ++spec_fails;
        spec_rest = (1 << std::min(spec_fails - 1, 3)) - 1;  // 0, 1, 3, 7 calls
    }
    Dist dist;  // multi-GPU partitioning of the recursion's large operations (dist.cuh)
    ~Workspace() {
        for (auto& kv : bufs_)
            if (kv.second.ptr) cudaFree(kv.second.ptr);
        if (mapped_) cudaFreeHost(mapped_);
        if (ev_) cudaEventDestroy(ev_);
        for (auto e : ev_pool_) cudaEventDestroy(e);
        for (auto& kv : streams_) {
            cudaStreamSynchronize(kv.second);
            cudaStreamDestroy(kv.second);
        }
    }
    // host-mapped pinned mailboxes the device writes directly (base-case rank + moved ranges),
    // one per concurrently running recursion driver; allocated once per context
    static constexpr int MAILBOXES = 64, MAILBOX_WORDS = 16;
    uint32_t* mailbox(int slot, uint32_t** dev_ptr) {
        std::lock_guard<std::mutex> lk(mu_);
        if (!mapped_) {
            FFG_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&mapped_), MAILBOXES * MAILBOX_WORDS * 4,
                                   cudaHostAllocMapped));
            FFG_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&mapped_dev_), mapped_, 0));
            std::memset(mapped_, 0, MAILBOXES * MAILBOX_WORDS * 4);
        }
        *dev_ptr = mapped_dev_ + slot * MAILBOX_WORDS;
        return mapped_ + slot * MAILBOX_WORDS;
    }
    // driver slots (mailbox + stream-id range) for concurrent subtrees; slot 0 is the root's
    int acquire_slot() {
        std::lock_guard<std::mutex> lk(mu_);
        for (int s = 1; s < MAILBOXES; ++s)
            if (!slot_busy_[s]) {
                slot_busy_[s] = true;
                return s;
            }
        return -1;
    }
    void release_slot(int s) {
        std::lock_guard<std::mutex> lk(mu_);
        if (s > 0) slot_busy_[s] = false;
    }
    cudaEvent_t sync_event() {
        std::lock_guard<std::mutex> lk(mu_);
        if (!ev_) FFG_CUDA(cudaEventCreateWithFlags(&ev_, cudaEventDisableTiming));
        return ev_;
    }
    // streams owned by the context for the recursion's concurrency: id -> stream, created on
    // first use with the given priority class (0 = highest, 1 = lowest)
    cudaStream_t stream(int id, int low_priority) {
        std::lock_guard<std::mutex> lk(mu_);
        auto it = streams_.find(id);
        if (it != streams_.end()) return it->second;
        int least = 0, greatest = 0;
        FFG_CUDA(cudaDeviceGetStreamPriorityRange(&least, &greatest));
        cudaStream_t s;
        FFG_CUDA(cudaStreamCreateWithPriority(&s, cudaStreamNonBlocking, low_priority ? least : greatest));
        streams_[id] = s;
        return s;
    }
    // events for fork/join within one call: recycled across calls (reset_events at call start)
    void reset_events() {
        std::lock_guard<std::mutex> lk(mu_);
        ev_cursor_ = 0;
    }
    cudaEvent_t event() {
        std::lock_guard<std::mutex> lk(mu_);
        if (ev_cursor_ == ev_pool_.size()) {
            cudaEvent_t e;
            FFG_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            ev_pool_.push_back(e);
        }
        return ev_pool_[ev_cursor_++];
    }
    // scratch valid until the next get() on the same stream
    uint8_t* get(cudaStream_t st, size_t bytes) {
        std::lock_guard<std::mutex> lk(mu_);
        auto& b = bufs_[st];
        if (b.cap < bytes) {
            if (b.ptr) {
                FFG_CUDA(cudaStreamSynchronize(st));
                FFG_CUDA(cudaFree(b.ptr));
                b.ptr = nullptr;
            }
            size_t cap = bytes + bytes / 4 + (1 << 20);
            cudaError_t e = cudaMalloc(&b.ptr, cap);
            if (e != cudaSuccess) {
                (void)cudaGetLastError();
                b.ptr = nullptr;
                b.cap = 0;
                throw Error(FFG_ERR_NO_MEMORY, "workspace allocation failed");
            }
            b.cap = cap;
        }
        return static_cast<uint8_t*>(b.ptr);
    }

private:
    struct Buf {
        void* ptr = nullptr;
        size_t cap = 0;
    };
    std::mutex mu_;
    std::unordered_map<cudaStream_t, Buf> bufs_;
    uint32_t* mapped_ = nullptr;
    uint32_t* mapped_dev_ = nullptr;
    bool slot_busy_[MAILBOXES] = {};
    cudaEvent_t ev_ = nullptr;
    std::unordered_map<int, cudaStream_t> streams_;
    std::vector<cudaEvent_t> ev_pool_;
    size_t ev_cursor_ = 0;
};

// C <- alpha*A*B + beta*C mod p (blas.hpp:31-103 semantics), enqueued on st.
// sm_cap > 0: the tensor-core GEMM runs persistent on at most sm_cap CTAs (one per SM), leaving
// the other SMs to kernels of higher-priority streams.
// no_direct: take the split + TMA pipeline even where the one-launch direct kernel applies
void fgemm_dev(const Field& F, uint32_t alpha, DView A, DView B, uint32_t beta, DView C, cudaStream_t st,
               Workspace& ws, uint64_t* launches, int sm_cap = 0, bool no_direct = false);
size_t gemm_workspace_bytes(const Field& F, size_t m, size_t n, size_t k);
int tile_n(int limbs);
extern size_t g_simt_macs;  // problems with M*N*K <= this use the CUDA-core kernel
extern size_t g_simt_kmax;  // ... and so do problems with K <= this
bool use_simt(size_t M, size_t N, size_t K);

}  // namespace ffg
