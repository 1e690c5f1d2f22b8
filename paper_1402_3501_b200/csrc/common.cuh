// common.cuh -- shared host/device definitions of the B200 ffpluq library.
#pragma once

#include <cstddef>
#include <atomic>
#include <cstdint>
#include <mutex>
#include <cstdlib>
#include <utility>
#include <cuda_runtime.h>
#include <stdexcept>
#include <string>

#include "../../include/ffg.h"
#include "knobs.cuh"

namespace ffg {

// One-time per-device setup (cudaFuncSetAttribute is a per-device property: a process with
// contexts on several GPUs must set it on each).  Thread-safe; devices 0..63.
class PerDeviceOnce {
public:
    template <class Fn>
    void operator()(Fn&& fn) {
        int dev = 0;
        cudaGetDevice(&dev);
        const uint64_t bit = 1ull << (dev & 63);
        if (mask_.load(std::memory_order_acquire) & bit) return;
        std::lock_guard<std::mutex> g(mu_);
        if (mask_.load(std::memory_order_relaxed) & bit) return;
        fn();
        mask_.fetch_or(bit, std::memory_order_release);
    }

private:
    std::atomic<uint64_t> mask_{0};
    std::mutex mu_;
};


// A non-owning row-major window of u32 residues in device memory (the
// device-side twin of MatView, matrix.hpp:13-43).
struct DView {
    uint32_t* d = nullptr;
    size_t rows = 0, cols = 0, ld = 0;
    bool empty() const { return rows == 0 || cols == 0; }
    DView sub(size_t r0, size_t c0, size_t h, size_t w) const { return DView{d + r0 * ld + c0, h, w, ld}; }
};

// Library error carrying an ffg status code (include/ffg.h, mirrors errors.hpp).
struct Error : std::runtime_error {
    int code;
    size_t index;
    Error(int c, const std::string& what, size_t idx = 0) : std::runtime_error(what), code(c), index(idx) {}
};

#define FFG_CUDA(x)                                                                                       \
    do {                                                                                                  \
        cudaError_t e_ = (x);                                                                             \
        if (e_ != cudaSuccess)                                                                            \
            throw ::ffg::Error(FFG_ERR_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_));            \
    } while (0)

// Prime-field context shared by every kernel (field.hpp:39-54 semantics plus the
// tensor-core embedding parameters).
struct Field {
    uint32_t p = 2;
    uint64_t mu = 0;      // floor(2^64 / p), Barrett constant
    int limbs = 1;        // 8-bit limbs per residue
    uint64_t kmax = 0;    // inner-dimension chunk that keeps every s32 limb accumulator exact
    uint32_t w[8] = {};   // w[s] = 2^(8s) mod p, weights of the limb-product diagonals
};

Field make_field(uint64_t p);  // throws Error(FFG_ERR_CAPACITY) like PrimeField (field.hpp:47-54)

// ---------------------------------------------------------------- device arithmetic
__host__ __device__ __forceinline__ uint32_t mod_u64(uint64_t x, uint32_t p, uint64_t mu) {
#ifdef __CUDA_ARCH__
    uint64_t q = __umul64hi(x, mu);
#else
    uint64_t q = (uint64_t)(((unsigned __int128)x * mu) >> 64);
#endif
    uint64_t r = x - q * p;
    if (r >= p) r -= p;
    if (r >= p) r -= p;
    return (uint32_t)r;
}

// binary extended Euclid for odd p (no divisions): a^-1 mod p for a != 0 mod p; p == 2 -> 1
#ifdef __CUDACC__
__device__ __forceinline__ uint32_t inv_mod_bin(uint32_t a, uint32_t p) {
    if (p == 2) return 1;
    a %= p;
    if (a == 0) return 0;  // no inverse; callers on a failed speculative path get garbage, not a hang
    uint32_t u = a, v = p, x1 = 1, x2 = 0;  // a*x1 = u, a*x2 = v (mod p)
    while (u != 1 && v != 1) {
        while ((u & 1) == 0) {
            u >>= 1;
            x1 = (x1 & 1) ? (x1 + p) >> 1 : x1 >> 1;
        }
        while ((v & 1) == 0) {
            v >>= 1;
            x2 = (x2 & 1) ? (x2 + p) >> 1 : x2 >> 1;
        }
        if (u >= v) {
            u -= v;
            x1 = x1 >= x2 ? x1 - x2 : x1 + p - x2;
        } else {
            v -= u;
            x2 = x2 >= x1 ? x2 - x1 : x2 + p - x1;
        }
    }
    return u == 1 ? x1 : x2;
}
#endif

__host__ __device__ __forceinline__ uint32_t mul_mod(uint32_t a, uint32_t b, uint32_t p, uint64_t mu) {
    return mod_u64((uint64_t)a * b, p, mu);
}

// extended Euclid (field.hpp:91-107); a != 0
__host__ __device__ __forceinline__ uint32_t inv_mod(uint32_t a, uint32_t p) {
    int64_t t = 0, nt = 1, r = p, nr = a;
    while (nr != 0) {
        int64_t q = r / nr, tmp = t - q * nt;
        t = nt;
        nt = tmp;
        tmp = r - q * nr;
        r = nr;
        nr = tmp;
    }
    if (t < 0) t += p;
    return (uint32_t)t;
}

// extended Euclid in 32-bit arithmetic (p < 2^26 keeps every quantity in range); a != 0
__host__ __device__ __forceinline__ uint32_t inv_mod32(uint32_t a, uint32_t p) {
    int32_t t = 0, nt = 1;
    uint32_t r = p, nr = a;
    while (nr != 0) {
        const uint32_t q = r / nr;
        const int32_t tmp = t - (int32_t)q * nt;
        t = nt;
        nt = tmp;
        const uint32_t r2 = r - q * nr;
        r = nr;
        nr = r2;
    }
    return t < 0 ? (uint32_t)(t + (int32_t)p) : (uint32_t)t;
}

// Shoup multiplication by a fixed factor w: wp = floor(w * 2^32 / p); x*w mod p in 32-bit ops
// Branch-free: for x = w * 2^32, hi64(x * mu) = w * mu_hi + hi32(w * mu_lo) (two products), and
// the Barrett estimate with mu = floor((2^64 - 1) / p) is short by at most 2.
__host__ __device__ __forceinline__ uint32_t shoup_pre(uint32_t w, uint32_t p, uint64_t mu) {
    const uint64_t x = (uint64_t)w << 32;
#ifdef __CUDA_ARCH__
    uint64_t q = (uint64_t)w * (uint32_t)(mu >> 32) + __umulhi(w, (uint32_t)mu);
#else
    uint64_t q = (uint64_t)(((unsigned __int128)x * mu) >> 64);
#endif
    uint32_t r = (uint32_t)(x - q * p);  // in [0, 3p): exact in 32 bits
    const uint32_t c1 = r >= p;
    r -= c1 * p;
    const uint32_t c2 = r >= p;
    return (uint32_t)q + c1 + c2;
}
__device__ __forceinline__ uint32_t shoup_mul(uint32_t x, uint32_t w, uint32_t wp, uint32_t p) {
    const uint32_t q = __umulhi(x, wp);
    uint32_t t = x * w - q * p;  // exact in [0, 2p) modulo 2^32
    return t >= p ? t - p : t;
}

inline size_t round_up(size_t x, size_t m) { return (x + m - 1) / m * m; }

// Kernel launch with programmatic stream serialization (PDL): the kernel may start while its
// predecessor on the stream finishes; every kernel launched this way calls ptx::pdl_wait()
// before its first global-memory access.  FFG_NO_PDL=1 launches plainly.
inline bool pdl_enabled() {
    static const bool on = !(knob_on("FFG_NO_PDL"));
    return on;
}
template <typename... KArgs, typename... Args>
inline void launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    FFG_CUDA(cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...));
}
inline size_t ceil_div(size_t x, size_t m) { return (x + m - 1) / m; }

}  // namespace ffg
