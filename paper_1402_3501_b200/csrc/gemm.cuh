// gemm.cuh -- internal API of the modular BLAS layer (GEMM, TRSM) and device workspace.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <mutex>
#include <unordered_map>

#include "common.cuh"

namespace ffg {

// Per-stream scratch arena (the limb planes of the operands, temporaries of the
// recursion).  Growth synchronizes the owning stream, so kernels already
// enqueued on it never see their scratch freed.  Allocation is a bump pointer
// reset by mark/release around each top-level call.
class Workspace {
public:
    ~Workspace() {
        for (auto& kv : bufs_)
            if (kv.second.ptr) cudaFree(kv.second.ptr);
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
};

// C <- alpha*A*B + beta*C mod p (blas.hpp:31-103 semantics), enqueued on st.
void fgemm_dev(const Field& F, uint32_t alpha, DView A, DView B, uint32_t beta, DView C, cudaStream_t st,
               Workspace& ws, uint64_t* launches);
size_t gemm_workspace_bytes(const Field& F, size_t m, size_t n, size_t k);
int tile_n(int limbs);

}  // namespace ffg
