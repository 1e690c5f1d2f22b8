// dist.cuh -- multi-GPU state of a context: one process per GPU, NCCL over NVLink/NVSwitch.
//
// Partitioned PLUQ (north_star: "tiles of the trailing update are partitioned across the
// GPUs of one box, with NCCL ... over NVLink for the panel and pivot blocks"):
//   * every rank holds the whole matrix (16384^2 u32 = 1 GiB of 180 GB) and runs the same
//     recursion; the kernels are exact and deterministic, so every rank discovers the same
//     base-case ranks and takes the same branches without exchanging them;
//   * the panel work (base cases, small TRSMs/GEMMs, permutations) is replicated -- it is
//     latency-bound, a broadcast would cost more than recomputing it;
//   * each large Schur GEMM / TRSM (>= min_work MACs) is split into `world` slices of its
//     output (rows or columns, 128-aligned); a rank computes its own slice, then one NCCL
//     all-gather brings every slice to every rank, so the replicas stay identical.
// "virtual" mode runs all slices of a world in one process on one GPU, through the same
// partition code, with no exchange: the single-GPU parity tests of the partitioning.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

namespace ffg {

// rows x cols u32 copy between device buffers with leading dimensions (perm.cu: a copy kernel)
void copy_2d_dev(const uint32_t* src, size_t lds, uint32_t* dst, size_t ldd, size_t rows, size_t cols,
                 cudaStream_t st);

struct Slice {
    size_t lo = 0, hi = 0;
};

// [lo, hi) of `total` for rank r of w: chunks of ceil(total / w) rounded up to `align`
// (the GEMM's 128-row tile), trailing ranks possibly empty.  Pure function, exported for tests.
Slice partition(size_t total, int world, int rank, size_t align);

struct Dist {
    int world = 1;
    int rank = 0;
    bool virt = false;        // all slices computed locally (single-GPU validation mode)
    bool loopback = false;    // virtual mode: route every slice through the staging pack/unpack
    void* comm = nullptr;     // ncclComm_t
    size_t min_work = size_t(1) << 28;  // MACs: smaller operations stay replicated
    uint32_t* stage = nullptr;          // all-gather staging buffer (device)
    size_t stage_words = 0;
    uint64_t exchanges = 0;   // all-gathers issued (diagnostics)
    uint64_t bytes = 0;       // bytes received by this rank over all all-gathers
    bool active() const { return world > 1; }
    ~Dist();
    void reset();
};

// NCCL, loaded on first use (dlopen), so single-GPU users need no NCCL at all
bool nccl_available();
void nccl_unique_id(unsigned char out[128]);
void dist_init_nccl(Dist& d, int world, int rank, const unsigned char id[128], int device);

// All-gather of the output slices of one partitioned operation on C (rows x cols window,
// leading dimension ld): axis 0 = row slices, 1 = column slices of `align`-aligned chunks.
// On return (stream order) every rank's C holds all slices.  Virtual mode: no-op, or with
// loopback every slice goes through the same pack -> stage -> unpack path (window wiped between).
void dist_allgather(Dist& d, uint32_t* C, size_t rows, size_t cols, size_t ld, int axis, size_t align,
                    cudaStream_t st);

}  // namespace ffg
