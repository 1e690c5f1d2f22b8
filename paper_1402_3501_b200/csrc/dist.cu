// dist.cu -- partitioning and the NCCL exchange of the partitioned PLUQ (see dist.cuh).
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <mutex>
#include <string>

#include "common.cuh"
#include "dist.cuh"

namespace ffg {

Slice partition(size_t total, int world, int rank, size_t align) {
    if (world <= 1) return Slice{0, total};
    if (align == 0) align = 1;
    const size_t chunk = round_up(ceil_div(total, (size_t)world), align);
    const size_t lo = std::min(total, (size_t)rank * chunk);
    return Slice{lo, std::min(total, lo + chunk)};
}

namespace {

struct Nccl {
    bool ok = false;
    std::string why;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

Nccl& nccl() {
    static Nccl n;
    static std::once_flag once;
    std::call_once(once, [] {
        // FFG_NCCL_LIB names the exact library (the Python mirror points it at the NCCL that
        // torch bundles, so both share one copy); otherwise the process's / system libnccl.so.2
        void* h = nullptr;
        if (const char* path = getenv("FFG_NCCL_LIB")) h = dlopen(path, RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            n.why = std::string("cannot load libnccl.so.2: ") + dlerror();
            return;
        }
        n.GetUniqueId = reinterpret_cast<decltype(n.GetUniqueId)>(dlsym(h, "ncclGetUniqueId"));
        n.CommInitRank = reinterpret_cast<decltype(n.CommInitRank)>(dlsym(h, "ncclCommInitRank"));
        n.CommDestroy = reinterpret_cast<decltype(n.CommDestroy)>(dlsym(h, "ncclCommDestroy"));
        n.AllGather = reinterpret_cast<decltype(n.AllGather)>(dlsym(h, "ncclAllGather"));
        n.GetErrorString = reinterpret_cast<decltype(n.GetErrorString)>(dlsym(h, "ncclGetErrorString"));
        n.ok = n.GetUniqueId && n.CommInitRank && n.CommDestroy && n.AllGather && n.GetErrorString;
        if (!n.ok) n.why = "libnccl.so.2 lacks a required symbol";
    });
    return n;
}

void check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess)
        throw Error(FFG_ERR_CUDA, std::string("NCCL ") + what + ": " + nccl().GetErrorString(r));
}

Nccl& need() {
    Nccl& n = nccl();
    if (!n.ok) throw Error(FFG_ERR_NO_DEVICE, n.why);
    return n;
}

}  // namespace

bool nccl_available() { return nccl().ok; }

void nccl_unique_id(unsigned char out[128]) {
    static_assert(sizeof(ncclUniqueId) == 128, "NCCL unique id size");
    ncclUniqueId id;
    check(need().GetUniqueId(&id), "GetUniqueId");
    std::memcpy(out, &id, sizeof(id));
}

void Dist::reset() {
    if (comm) nccl().CommDestroy(static_cast<ncclComm_t>(comm));
    comm = nullptr;
    if (stage) cudaFree(stage);
    stage = nullptr;
    stage_words = 0;
    world = 1;
    rank = 0;
    virt = false;
    loopback = false;
    exchanges = bytes = 0;
}

Dist::~Dist() { reset(); }

void dist_init_nccl(Dist& d, int world, int rank, const unsigned char id[128], int device) {
    if (world < 1 || rank < 0 || rank >= world) throw Error(FFG_ERR_INVALID_ARG, "dist: bad world/rank");
    d.reset();
    if (world == 1) return;
    Nccl& n = need();
    ncclUniqueId uid;
    std::memcpy(&uid, id, sizeof(uid));
    FFG_CUDA(cudaSetDevice(device));
    ncclComm_t c = nullptr;
    check(n.CommInitRank(&c, world, uid, rank), "CommInitRank");
    d.comm = c;
    d.world = world;
    d.rank = rank;
}

void dist_allgather(Dist& d, uint32_t* C, size_t rows, size_t cols, size_t ld, int axis, size_t align,
                    cudaStream_t st) {
    if (!d.active() || (d.virt && !d.loopback) || rows == 0 || cols == 0) return;
    const size_t total = axis == 0 ? rows : cols;
    const size_t chunk = round_up(ceil_div(total, (size_t)d.world), align ? align : 1);
    const size_t S = axis == 0 ? chunk * cols : rows * chunk;  // words per rank in the stage
    if (d.stage_words < S * d.world) {
        if (d.stage) {
            FFG_CUDA(cudaStreamSynchronize(st));
            FFG_CUDA(cudaFree(d.stage));
            d.stage = nullptr;
        }
        const size_t want = S * d.world + S * d.world / 4;
        if (cudaMalloc(&d.stage, want * 4) != cudaSuccess) {
            (void)cudaGetLastError();
            d.stage_words = 0;
            throw Error(FFG_ERR_NO_MEMORY, "dist: staging allocation failed");
        }
        d.stage_words = want;
    }
    // packed slice layouts: row slices (hi-lo) x cols at pitch cols; column slices rows x (hi-lo)
    // at pitch chunk
    auto copy = [&](int r, bool pack) {
        const Slice s = partition(total, d.world, r, align);
        if (s.hi <= s.lo) return;
        uint32_t* buf = d.stage + (size_t)r * S;
        uint32_t* win = axis == 0 ? C + s.lo * ld : C + s.lo;
        const size_t w = axis == 0 ? cols : s.hi - s.lo, h = axis == 0 ? s.hi - s.lo : rows;
        const size_t pitch = axis == 0 ? cols : chunk;
        if (pack)
            copy_2d_dev(win, ld, buf, pitch, h, w, st);
        else
            copy_2d_dev(buf, pitch, win, ld, h, w, st);
    };
    if (d.virt) {
        // loopback: the same pack / unpack through the stage with the window wiped in between,
        // so a wrong slice layout shows up as corrupted output on one GPU
        for (int r = 0; r < d.world; ++r) copy(r, true);
        FFG_CUDA(cudaMemset2DAsync(C, ld * 4, 0, cols * 4, rows, st));
        for (int r = 0; r < d.world; ++r) copy(r, false);
    } else {
        copy(d.rank, true);
        check(need().AllGather(d.stage + (size_t)d.rank * S, d.stage, S, ncclUint32, static_cast<ncclComm_t>(d.comm),
                               st),
              "AllGather");
        for (int r = 0; r < d.world; ++r)
            if (r != d.rank) copy(r, false);
    }
    ++d.exchanges;
    d.bytes += (uint64_t)S * (d.world - 1) * 4;
}

}  // namespace ffg
