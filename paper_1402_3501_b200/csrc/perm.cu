// perm.cu -- permutation kernels: index-array compositions and row/column gathers.
//
// Replaces apply_perm / rotate_rows_block / rotate_cols_block / PermSeq
// composition (perm.hpp:44-53, 167-215).  The reference replays Rot/Swap
// moves one at a time (each a memmove of whole rows); here a permutation is
// an index array (PermSeq::to_array() semantics) and every application is one
// gather over the moved range only: HBM traffic = 2 reads + 2 writes of the
// rows/columns that actually move, nothing for the rest.
#include <algorithm>
#include <mutex>

#include "pluq.cuh"
#include "ptx.cuh"

namespace ffg {

// position t (relative to the range start) takes source position src(t)
struct PermSrc {
    const uint32_t* arr;  // if non-null: src(t) = arr[t + base] - base... see at()
    uint32_t base;        // arr is indexed at t + base and returns absolute positions
    uint32_t span, len;   // rotation: [0,len) <- [span, span+len), [len, len+span) <- [0, span)
    __device__ __forceinline__ uint32_t at(uint32_t t) const {
        if (arr) return arr[t + base] - base;
        return t < len ? span + t : t - len;
    }
};

__global__ void rows_gather_kernel(const uint32_t* __restrict__ A, uint64_t lda, uint32_t nrows, uint32_t ncols,
                                   PermSrc src, uint32_t* __restrict__ tmp) {
    ptx::pdl_enter();
    const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x, t = blockIdx.y;
    if (c < ncols && t < nrows) tmp[(uint64_t)t * ncols + c] = A[(uint64_t)src.at(t) * lda + c];
}
__global__ void rows_store_kernel(uint32_t* __restrict__ A, uint64_t lda, uint32_t nrows, uint32_t ncols,
                                  const uint32_t* __restrict__ tmp) {
    ptx::pdl_enter();
    const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x, t = blockIdx.y;
    if (c < ncols && t < nrows) A[(uint64_t)t * lda + c] = tmp[(uint64_t)t * ncols + c];
}
__global__ void cols_gather_kernel(const uint32_t* __restrict__ A, uint64_t lda, uint32_t nrows, uint32_t ncols,
                                   PermSrc src, uint32_t* __restrict__ tmp) {
    ptx::pdl_enter();
    const uint32_t u = blockIdx.x * blockDim.x + threadIdx.x, r = blockIdx.y;
    if (u < ncols && r < nrows) tmp[(uint64_t)r * ncols + u] = A[(uint64_t)r * lda + src.at(u)];
}

// in-place gather of an index array range through shared memory: a[t] = old[src(t)]
__global__ void array_gather_kernel(uint32_t* __restrict__ a, uint32_t len, PermSrc src) {
    extern __shared__ uint32_t s[];
    ptx::pdl_enter();
    for (uint32_t t = threadIdx.x; t < len; t += blockDim.x) s[t] = a[t];
    __syncthreads();
    for (uint32_t t = threadIdx.x; t < len; t += blockDim.x) a[t] = s[src.at(t)];
}
__global__ void array_gather_global_kernel(const uint32_t* __restrict__ a, uint32_t len, PermSrc src,
                                          uint32_t* __restrict__ out) {
    ptx::pdl_enter();
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t < len) out[t] = a[src.at(t)];
}
__global__ void iota_kernel(uint32_t* a, uint32_t len) {
    ptx::pdl_enter();
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t < len) a[t] = t;
}

// In-place gathers in one launch for the common small ranges (every permutation of the
// rank-deficient recursion): a CTA stages its slice of the moved block in shared memory and
// writes it back permuted -- rows: a column slice of all moved rows; columns: a row slice of all
// moved columns.  Larger ranges take the two-pass gather through a temporary.
constexpr size_t PERM_SMEM = 96 * 1024;
__global__ void __launch_bounds__(256) rows_perm_inplace_kernel(uint32_t* __restrict__ A, uint64_t lda, uint32_t nrows,
                                                                uint32_t ncols, uint32_t w, PermSrc src) {
    extern __shared__ uint32_t sbuf[];
    ptx::pdl_enter();
    const uint32_t c0 = blockIdx.x * w, cw = min(w, ncols - c0), tot = nrows * cw;
    for (uint32_t idx = threadIdx.x; idx < tot; idx += blockDim.x) {
        const uint32_t r = idx / cw, c = idx % cw;
        sbuf[idx] = A[(uint64_t)r * lda + c0 + c];
    }
    __syncthreads();
    for (uint32_t idx = threadIdx.x; idx < tot; idx += blockDim.x) {
        const uint32_t t = idx / cw, c = idx % cw;
        A[(uint64_t)t * lda + c0 + c] = sbuf[src.at(t) * cw + c];
    }
}
__global__ void __launch_bounds__(256) cols_perm_inplace_kernel(uint32_t* __restrict__ A, uint64_t lda, uint32_t nrows,
                                                                uint32_t ncols, uint32_t h, PermSrc src) {
    extern __shared__ uint32_t sbuf[];
    uint32_t* sidx = sbuf + (size_t)h * ncols;  // src.at(u) for every column
    ptx::pdl_enter();
    const uint32_t r0 = blockIdx.x * h, rh = min(h, nrows - r0), tot = rh * ncols;
    for (uint32_t u = threadIdx.x; u < ncols; u += blockDim.x) sidx[u] = src.at(u);
    for (uint32_t idx = threadIdx.x; idx < tot; idx += blockDim.x) {
        const uint32_t r = idx / ncols, c = idx % ncols;
        sbuf[idx] = A[(uint64_t)(r0 + r) * lda + c];
    }
    __syncthreads();
    for (uint32_t idx = threadIdx.x; idx < tot; idx += blockDim.x) {
        const uint32_t r = idx / ncols, u = idx % ncols;
        A[(uint64_t)(r0 + r) * lda + u] = sbuf[r * ncols + sidx[u]];
    }
}

namespace {
void perm_smem_attr() {
    static PerDeviceOnce once;
    once([] {
        FFG_CUDA(cudaFuncSetAttribute(rows_perm_inplace_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)PERM_SMEM));
        FFG_CUDA(cudaFuncSetAttribute(cols_perm_inplace_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)PERM_SMEM));
    });
}
void gather_rows(const Blas& b, DView a, PermSrc src) {
    if (a.empty()) return;
    if (a.rows * 4 * 32 <= PERM_SMEM) {  // at least 32 columns per CTA
        perm_smem_attr();
        const size_t w = std::min<size_t>(a.cols, std::min<size_t>(512, PERM_SMEM / (a.rows * 4)));
        b.ws.prof.begin(b.st);
        launch_k(rows_perm_inplace_kernel, dim3((unsigned)ceil_div(a.cols, w)), dim3(256), a.rows * w * 4, b.st, a.d,
                 a.ld, (uint32_t)a.rows, (uint32_t)a.cols, (uint32_t)w, src);
        b.ws.prof.end(b.st, PROF_PERM, 16.0 * a.rows * a.cols);
        FFG_CUDA(cudaGetLastError());
        b.count();
        return;
    }
    uint32_t* tmp = nullptr;
    FFG_CUDA(cudaMallocAsync(&tmp, a.rows * a.cols * 4, b.st));
    dim3 g((unsigned)ceil_div(a.cols, 256), (unsigned)a.rows);
    b.ws.prof.begin(b.st);
    launch_k(rows_gather_kernel, g, dim3(256), 0, b.st, a.d, a.ld, (uint32_t)a.rows, (uint32_t)a.cols, src, tmp);
    launch_k(rows_store_kernel, g, dim3(256), 0, b.st, a.d, a.ld, (uint32_t)a.rows, (uint32_t)a.cols, tmp);
    b.ws.prof.end(b.st, PROF_PERM, 16.0 * a.rows * a.cols);
    FFG_CUDA(cudaGetLastError());
    FFG_CUDA(cudaFreeAsync(tmp, b.st));
    b.count(2);
}
void gather_cols(const Blas& b, DView a, PermSrc src) {
    if (a.empty()) return;
    if ((a.cols * 4 + a.cols * 4) * 4 <= PERM_SMEM) {  // at least 4 rows per CTA
        perm_smem_attr();
        const size_t h = std::min<size_t>(a.rows, std::min<size_t>(64, (PERM_SMEM - a.cols * 4) / (a.cols * 4)));
        b.ws.prof.begin(b.st);
        launch_k(cols_perm_inplace_kernel, dim3((unsigned)ceil_div(a.rows, h)), dim3(256), (h + 1) * a.cols * 4, b.st,
                 a.d, a.ld, (uint32_t)a.rows, (uint32_t)a.cols, (uint32_t)h, src);
        b.ws.prof.end(b.st, PROF_PERM, 16.0 * a.rows * a.cols);
        FFG_CUDA(cudaGetLastError());
        b.count();
        return;
    }
    uint32_t* tmp = nullptr;
    FFG_CUDA(cudaMallocAsync(&tmp, a.rows * a.cols * 4, b.st));
    dim3 g((unsigned)ceil_div(a.cols, 256), (unsigned)a.rows);
    b.ws.prof.begin(b.st);
    launch_k(cols_gather_kernel, g, dim3(256), 0, b.st, a.d, a.ld, (uint32_t)a.rows, (uint32_t)a.cols, src, tmp);
    launch_k(rows_store_kernel, g, dim3(256), 0, b.st, a.d, a.ld, (uint32_t)a.rows, (uint32_t)a.cols, tmp);
    b.ws.prof.end(b.st, PROF_PERM, 16.0 * a.rows * a.cols);
    FFG_CUDA(cudaGetLastError());
    FFG_CUDA(cudaFreeAsync(tmp, b.st));
    b.count(2);
}
}  // namespace

void perm_apply_range(const Blas& b, DView a, int axis, const uint32_t* perm, size_t lo, size_t hi) {
    if (hi <= lo || a.empty()) return;
    PermSrc src{perm, (uint32_t)lo, 0, 0};
    if (axis == 0)
        gather_rows(b, a.sub(lo, 0, hi - lo, a.cols), src);
    else
        gather_cols(b, a.sub(0, lo, a.rows, hi - lo), src);
}

void rotate_block_dev(const Blas& b, DView a, int axis, size_t first, size_t mid, size_t len) {
    if (len == 0 || mid == first || a.empty()) return;  // perm.hpp:198, 210
    const size_t span = mid - first;
    PermSrc src{nullptr, 0, (uint32_t)span, (uint32_t)len};
    if (axis == 0)
        gather_rows(b, a.sub(first, 0, span + len, a.cols), src);
    else
        gather_cols(b, a.sub(0, first, a.rows, span + len), src);
}

static void array_gather(const Blas& b, uint32_t* a, size_t len, PermSrc src) {
    if (len == 0) return;
    const size_t bytes = len * 4;
    if (bytes <= 200 * 1024) {
        static PerDeviceOnce once;
        once([] {
            FFG_CUDA(cudaFuncSetAttribute(array_gather_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        });
        launch_k(array_gather_kernel, dim3(1), dim3(1024), bytes, b.st, a, (uint32_t)len, src);
        b.count();
    } else {
        uint32_t* tmp = nullptr;
        FFG_CUDA(cudaMallocAsync(&tmp, bytes, b.st));
        launch_k(array_gather_global_kernel, dim3((unsigned)ceil_div(len, 256)), dim3(256), 0, b.st, a, (uint32_t)len,
                 src, tmp);
        FFG_CUDA(cudaMemcpyAsync(a, tmp, bytes, cudaMemcpyDeviceToDevice, b.st));
        FFG_CUDA(cudaFreeAsync(tmp, b.st));
        b.count();
    }
    FFG_CUDA(cudaGetLastError());
}

void perm_compose_dev(const Blas& b, uint32_t* dst, size_t off, const uint32_t* child, size_t lo, size_t hi) {
    if (hi <= lo) return;
    // dst[off + t] = dst[off + child[t]] for t in [lo, hi); child is identity outside the range
    PermSrc src{child, (uint32_t)lo, 0, 0};
    array_gather(b, dst + off + lo, hi - lo, src);
}

void perm_rot_dev(const Blas& b, uint32_t* arr, size_t first, size_t mid, size_t len) {
    if (len == 0 || mid == first) return;
    PermSrc src{nullptr, 0, (uint32_t)(mid - first), (uint32_t)len};
    array_gather(b, arr + first, mid - first + len, src);
}

void perm_iota_dev(const Blas& b, uint32_t* arr, size_t len) {
    if (!len) return;
    launch_k(iota_kernel, dim3((unsigned)ceil_div(len, 256)), dim3(256), 0, b.st, arr, (uint32_t)len);
    FFG_CUDA(cudaGetLastError());
    b.count();
}

__global__ void invert_perm_kernel(const uint32_t* p, uint32_t* q, uint32_t n) {
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t < n) q[p[t]] = t;
}

void apply_perm_dev(const Blas& b, DView a, int axis, int inverse, const uint32_t* perm) {
    const size_t dim = axis == 0 ? a.rows : a.cols;
    if (!inverse) {
        perm_apply_range(b, a, axis, perm, 0, dim);
        return;
    }
    // inverse (perm.hpp:190-192): out[perm[t]] = in[t] -> gather by the inverse index array
    uint32_t* invp = nullptr;
    FFG_CUDA(cudaMallocAsync(&invp, dim * 4, b.st));
    invert_perm_kernel<<<(unsigned)ceil_div(dim, 256), 256, 0, b.st>>>(perm, invp, (uint32_t)dim);
    b.count();
    perm_apply_range(b, a, axis, invp, 0, dim);
    FFG_CUDA(cudaFreeAsync(invp, b.st));
}

// dst <- src (same shape): 16-byte accesses when both views allow them.  The host entry's
// speculative path backs its input up in HBM with this (a kernel, not a DMA copy: the copy
// engines are busy with the PCIe transfers).
__global__ void copy_block_kernel(const uint32_t* __restrict__ S, uint64_t lds, uint32_t* __restrict__ D, uint64_t ldd,
                                  uint32_t rows, uint32_t cols, uint32_t vec) {
    const uint32_t per = vec ? cols / 4 : cols;
    const uint64_t total = (uint64_t)rows * per;
    for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < total; t += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t r = t / per, c = t % per;
        if (vec)
            reinterpret_cast<uint4*>(D + r * ldd)[c] = reinterpret_cast<const uint4*>(S + r * lds)[c];
        else
            D[r * ldd + c] = S[r * lds + c];
    }
}

void copy_2d_dev(const uint32_t* src, size_t lds, uint32_t* dst, size_t ldd, size_t rows, size_t cols,
                 cudaStream_t st) {
    if (!rows || !cols) return;
    const bool vec = cols % 4 == 0 && lds % 4 == 0 && ldd % 4 == 0 && (reinterpret_cast<uintptr_t>(src) & 15) == 0 &&
                     (reinterpret_cast<uintptr_t>(dst) & 15) == 0;
    const uint64_t items = (uint64_t)rows * (vec ? cols / 4 : cols);
    const unsigned grid = (unsigned)std::min<uint64_t>(ceil_div(items, 256), (uint64_t)148 * 4);
    copy_block_kernel<<<grid, 256, 0, st>>>(src, lds, dst, ldd, (uint32_t)rows, (uint32_t)cols, vec ? 1u : 0u);
    FFG_CUDA(cudaGetLastError());
}

void copy_block_dev(const Blas& b, DView src, DView dst) {
    if (src.empty()) return;
    const bool vec = src.cols % 4 == 0 && src.ld % 4 == 0 && dst.ld % 4 == 0 &&
                     (reinterpret_cast<uintptr_t>(src.d) & 15) == 0 && (reinterpret_cast<uintptr_t>(dst.d) & 15) == 0;
    const uint64_t items = (uint64_t)src.rows * (vec ? src.cols / 4 : src.cols);
    int sms = 148;
    const unsigned grid = (unsigned)std::min<uint64_t>(ceil_div(items, 256), (uint64_t)sms * 4);
    copy_block_kernel<<<grid, 256, 0, b.st>>>(src.d, src.ld, dst.d, dst.ld, (uint32_t)src.rows, (uint32_t)src.cols,
                                              vec ? 1u : 0u);
    FFG_CUDA(cudaGetLastError());
    b.count();
}

// a.cols <= 64 columns of every row of a gathered by a local index array: a[i][t] <- a[i][q[t]].
// One warp per row; all reads before any write.  The panel schedule applies a base case's column
// pivots to the rows above its block with it (tile_rec applies R's Q to D, rankrev.hpp:158-161).
__global__ void block_cols_perm_kernel(uint32_t* __restrict__ A, uint64_t lda, uint32_t rows, uint32_t s,
                                       const uint32_t* __restrict__ q) {
    ptx::pdl_enter();
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t row = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
    if (row >= rows) return;
    uint32_t* r = A + (uint64_t)row * lda;
    const uint32_t v0 = lane < s ? r[q[lane]] : 0u, v1 = lane + 32 < s ? r[q[lane + 32]] : 0u;
    __syncwarp();
    if (lane < s) r[lane] = v0;
    if (lane + 32 < s) r[lane + 32] = v1;
}

void block_cols_perm_dev(const Blas& b, DView a, const uint32_t* q) {
    if (a.empty()) return;
    if (a.cols > 64) throw Error(FFG_ERR_INTERNAL, "block_cols_perm: more than 64 columns");
    launch_k(block_cols_perm_kernel, dim3((unsigned)ceil_div(a.rows, 8)), dim3(256), 0, b.st, a.d, a.ld,
             (uint32_t)a.rows, (uint32_t)a.cols, q);
    FFG_CUDA(cudaGetLastError());
    b.count();
}

// Byte storage of small-field matrices (p <= 256, BASELINE config 5 "stored as uint8"): the
// host entry moves bytes over PCIe and widens / narrows them to the u32 working layout in HBM.
__global__ void widen_u8_kernel(const uint8_t* __restrict__ S, uint64_t lds, uint32_t* __restrict__ D, uint64_t ldd,
                                uint32_t rows, uint32_t cols, uint32_t p) {
    const uint64_t total = (uint64_t)rows * cols;
    for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < total; t += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t r = t / cols, c = t % cols;
        const uint32_t v = S[r * lds + c];
        D[r * ldd + c] = v < p ? v : v % p;
    }
}
__global__ void narrow_u8_kernel(const uint32_t* __restrict__ S, uint64_t lds, uint8_t* __restrict__ D, uint64_t ldd,
                                 uint32_t rows, uint32_t cols) {
    const uint64_t total = (uint64_t)rows * cols;
    for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < total; t += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t r = t / cols, c = t % cols;
        D[r * ldd + c] = (uint8_t)S[r * lds + c];
    }
}

void widen_u8_dev(const Blas& b, const uint8_t* src, size_t lds, DView dst) {
    if (dst.empty()) return;
    const unsigned grid = (unsigned)std::min<uint64_t>(ceil_div((uint64_t)dst.rows * dst.cols, 256), 148 * 8);
    widen_u8_kernel<<<grid, 256, 0, b.st>>>(src, lds, dst.d, dst.ld, (uint32_t)dst.rows, (uint32_t)dst.cols, b.F.p);
    FFG_CUDA(cudaGetLastError());
    b.count();
}
void narrow_u8_dev(const Blas& b, DView src, uint8_t* dst, size_t ldd) {
    if (src.empty()) return;
    const unsigned grid = (unsigned)std::min<uint64_t>(ceil_div((uint64_t)src.rows * src.cols, 256), 148 * 8);
    narrow_u8_kernel<<<grid, 256, 0, b.st>>>(src.d, src.ld, dst, ldd, (uint32_t)src.rows, (uint32_t)src.cols);
    FFG_CUDA(cudaGetLastError());
    b.count();
}

}  // namespace ffg
