// capi.cu -- the extern "C" boundary (include/ffg.h): context, status codes, host/device entry points.
#include <algorithm>
#include <cstdio>
#include <vector>
#include <cstring>
#include <string>

#include "common.cuh"
#include "gemm.cuh"
#include "pluq.cuh"
#include "profile.cuh"

struct ffg_ctx {
    int device = 0;
    cudaStream_t own_stream = nullptr;
    cudaStream_t stream = nullptr;
    ffg::Workspace ws;
    uint64_t launches = 0;
};

namespace {

thread_local std::string g_err;
thread_local size_t g_err_index = 0;

template <class Fn>
int guarded(ffg_ctx* ctx, Fn&& fn) {
    if (!ctx) {
        g_err = "null context";
        return FFG_ERR_INVALID_ARG;
    }
    try {
        cudaSetDevice(ctx->device);
        fn();
        return FFG_OK;
    } catch (const ffg::Error& e) {
        g_err = e.what();
        g_err_index = e.index;
        return e.code;
    } catch (const std::bad_alloc&) {
        g_err = "host allocation failed";
        return FFG_ERR_NO_MEMORY;
    } catch (const std::exception& e) {
        g_err = e.what();
        return FFG_ERR_INTERNAL;
    }
}

// device copy of a strided host matrix (pinned staging is the caller's choice; cudaMemcpy2D handles pageable)
struct DevMat {
    uint32_t* d = nullptr;
    size_t rows = 0, cols = 0;
    DevMat(size_t r, size_t c, cudaStream_t st) : rows(r), cols(c) {
        if (r && c) FFG_CUDA(cudaMallocAsync(&d, r * c * sizeof(uint32_t), st));
        stream = st;
    }
    ~DevMat() {
        if (d) cudaFreeAsync(d, stream);
    }
    ffg::DView view() { return ffg::DView{d, rows, cols, cols}; }
    void upload(const uint32_t* h, size_t ld) {
        if (d)
            FFG_CUDA(cudaMemcpy2DAsync(d, cols * 4, h, ld * 4, cols * 4, rows, cudaMemcpyHostToDevice, stream));
    }
    void download(uint32_t* h, size_t ld) {
        if (d)
            FFG_CUDA(cudaMemcpy2DAsync(h, ld * 4, d, cols * 4, cols * 4, rows, cudaMemcpyDeviceToHost, stream));
    }
    cudaStream_t stream;
};

// every entry point: a non-empty matrix needs a pointer and ld >= cols (the MatView invariant,
// matrix.hpp:13-43); anything else would be read out of bounds on the device
void check_mat(const char* what, const void* ptr, size_t rows, size_t cols, size_t ld) {
    if (rows == 0 || cols == 0) return;
    if (!ptr) throw ffg::Error(FFG_ERR_INVALID_ARG, std::string(what) + ": null matrix pointer");
    if (ld < cols) throw ffg::Error(FFG_ERR_INVALID_DIM, std::string(what) + ": leading dimension < columns");
}

}  // namespace

extern "C" {

void ffg_knobs_reload(void) { ffg::knobs_reload(); }

const char* ffg_version(void) { return "ffg_b200 0.1 (sm_100a tcgen05 kind::i8 limb GEMM)"; }
const char* ffg_last_error(void) { return g_err.c_str(); }
size_t ffg_last_error_index(void) { return g_err_index; }

int ffg_create(ffg_ctx** out, int device) {
    if (!out) return FFG_ERR_INVALID_ARG;
    *out = nullptr;
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n <= device) {
        (void)cudaGetLastError();
        g_err = "no CUDA device";
        return FFG_ERR_NO_DEVICE;
    }
    cudaDeviceProp prop;
    if (cudaGetDeviceProperties(&prop, device) != cudaSuccess || prop.major != 10) {
        g_err = "device is not sm_100 (compute capability 10.x); this library has no other code path";
        return FFG_ERR_NO_DEVICE;
    }
    ffg_ctx* c = new ffg_ctx;
    c->device = device;
    cudaSetDevice(device);
    if (cudaStreamCreateWithFlags(&c->own_stream, cudaStreamNonBlocking) != cudaSuccess) {
        delete c;
        g_err = "stream creation failed";
        return FFG_ERR_CUDA;
    }
    c->stream = c->own_stream;
    if (const char* s = ffg::knob_str("FFG_SIMT_MACS")) ffg::g_simt_macs = strtoull(s, nullptr, 10);
    if (const char* s = ffg::knob_str("FFG_SIMT_KMAX")) ffg::g_simt_kmax = strtoull(s, nullptr, 10);
    // keep freed stream-ordered allocations cached in the pool
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
        uint64_t thr = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    *out = c;
    return FFG_OK;
}

void ffg_destroy(ffg_ctx* ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    if (ctx->own_stream) cudaStreamDestroy(ctx->own_stream);
    delete ctx;
}

int ffg_set_stream(ffg_ctx* ctx, void* stream) {
    return guarded(ctx, [&] { ctx->stream = stream ? static_cast<cudaStream_t>(stream) : ctx->own_stream; });
}
void* ffg_get_stream(ffg_ctx* ctx) { return ctx ? ctx->stream : nullptr; }
int ffg_synchronize(ffg_ctx* ctx) { return guarded(ctx, [&] { FFG_CUDA(cudaStreamSynchronize(ctx->stream)); }); }
uint64_t ffg_launch_count(ffg_ctx* ctx) { return ctx ? ctx->launches : 0; }

int ffg_spec_stats(ffg_ctx* ctx, uint64_t* out) {
    return guarded(ctx, [&] {
        if (!out) throw ffg::Error(FFG_ERR_INVALID_DIM, "spec_stats: null output");
        out[0] = ctx->ws.st_guess;
        out[1] = ctx->ws.st_guess_failed;
        out[2] = ctx->ws.st_node;
        out[3] = ctx->ws.st_node_failed;
        out[4] = ctx->ws.st_profile_first;
    });
}

int ffg_profile_enable(ffg_ctx* ctx, int on) {
    return guarded(ctx, [&] { ctx->ws.prof.mode = on < 0 || on > 2 ? 1 : on; });
}

int ffg_profile_read(ffg_ctx* ctx, double* out, int nclasses) {
    return guarded(ctx, [&] {
        double ms[ffg::PROF_NKINDS], n[ffg::PROF_NKINDS], w[ffg::PROF_NKINDS], f[ffg::PROF_NKINDS];
        ctx->ws.prof.read(ms, n, w, f);
        ctx->ws.prof.clear();
        for (int c = 0; c < nclasses && c < ffg::PROF_NKINDS; ++c) {
            out[4 * c + 0] = ms[c];
            out[4 * c + 1] = n[c];
            out[4 * c + 2] = w[c];
            out[4 * c + 3] = f[c];
        }
    });
}

int ffg_field_info(uint64_t p, int* limbs, uint64_t* kmax, int* nt) {
    try {
        ffg::Field F = ffg::make_field(p);
        if (limbs) *limbs = F.limbs;
        if (kmax) *kmax = F.kmax;
        if (nt) *nt = ffg::tile_n(F.limbs);
        return FFG_OK;
    } catch (const ffg::Error& e) {
        g_err = e.what();
        return e.code;
    }
}

int ffg_tile_rec_perms(size_t m, size_t n, size_t threshold, size_t rank, const uint32_t* prow, const uint32_t* pcol,
                       uint32_t* P, uint32_t* Q) {
    try {
        if ((rank && (!prow || !pcol)) || (m && !P) || (n && !Q)) throw ffg::Error(FFG_ERR_INVALID_ARG, "null array");
        ffg::tile_rec_perms(m, n, threshold, rank, prow, pcol, P, Q);
        return FFG_OK;
    } catch (const ffg::Error& e) {
        g_err = e.what();
        return e.code;
    } catch (const std::bad_alloc&) {
        g_err = "host allocation failed";
        return FFG_ERR_NO_MEMORY;
    }
}

int ffg_rank_profile_dev(ffg_ctx* ctx, uint64_t p, const uint32_t* A, size_t m, size_t n, size_t lda, uint32_t* prow,
                         uint32_t* pcol, size_t* rank) {
    return guarded(ctx, [&] {
        ffg::Field F = ffg::make_field(p);
        check_mat("rank_profile", A, m, n, lda);
        if (std::min(m, n) && (!prow || !pcol)) throw ffg::Error(FFG_ERR_INVALID_ARG, "rank_profile: null output");
        if (!ffg::profile_first_fits(n)) throw ffg::Error(FFG_ERR_INVALID_DIM, "rank_profile: too many columns");
        ffg::Blas blas{F, ctx->ws, ctx->stream, &ctx->launches};
        DevMat W(m, n, ctx->stream);
        if (m && n) ffg::copy_block_dev(blas, ffg::DView{const_cast<uint32_t*>(A), m, n, lda}, W.view());
        std::vector<uint32_t> pr, pc;
        const size_t r = ffg::rank_profile_dev(blas, W.view(), pr, pc);
        std::copy(pr.begin(), pr.end(), prow);
        std::copy(pc.begin(), pc.end(), pcol);
        if (rank) *rank = r;
    });
}

int ffg_pluq_from_profile_dev(ffg_ctx* ctx, uint64_t p, uint32_t* A, size_t m, size_t n, size_t lda, size_t threshold,
                              size_t rank, const uint32_t* prow, const uint32_t* pcol, uint32_t* P, uint32_t* Q) {
    return guarded(ctx, [&] {
        ffg::Field F = ffg::make_field(p);
        check_mat("pluq_from_profile", A, m, n, lda);
        if ((rank && (!prow || !pcol)) || (m && !P) || (n && !Q)) throw ffg::Error(FFG_ERR_INVALID_ARG, "null array");
        ffg::Blas blas{F, ctx->ws, ctx->stream, &ctx->launches};
        DevMat W(m, n, ctx->stream);
        ffg::pluq_from_profile_dev(blas, ffg::DView{A, m, n, lda}, threshold, rank, prow, pcol, P, Q, W.d);
        FFG_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

int ffg_random_mat_dev(ffg_ctx* ctx, uint64_t p, uint64_t seed, uint32_t* A, size_t m, size_t n, size_t lda) {
    return guarded(ctx, [&] {
        ffg::Field F = ffg::make_field(p);
        check_mat("random_mat", A, m, n, lda);
        ffg::Blas blas{F, ctx->ws, ctx->stream, &ctx->launches};
        ffg::random_mat_dev(blas, ffg::DView{A, m, n, lda}, seed);
    });
}

int ffg_lru_matrix_dev(ffg_ctx* ctx, uint64_t p, uint64_t seed, uint32_t* M, size_t n, size_t ldm, size_t r,
                       uint32_t* rows, uint32_t* cols) {
    return guarded(ctx, [&] {
        ffg::Field F = ffg::make_field(p);
        check_mat("lru_matrix", M, n, n, ldm);
        if (r > n) throw ffg::Error(FFG_ERR_INVALID_RANK, "lru_matrix: r > n");
        ffg::Blas blas{F, ctx->ws, ctx->stream, &ctx->launches};
        ffg::lru_matrix_dev(blas, ffg::DView{M, n, n, ldm}, r, seed, rows, cols);
    });
}

int ffg_fgemm_dev(ffg_ctx* ctx, uint64_t p, uint32_t alpha, const uint32_t* A, size_t lda, const uint32_t* B,
                  size_t ldb, uint32_t beta, uint32_t* C, size_t ldc, size_t m, size_t n, size_t k) {
    return guarded(ctx, [&] {
        ffg::Field F = ffg::make_field(p);
        check_mat("fgemm A", A, m, k, lda);
        check_mat("fgemm B", B, k, n, ldb);
        check_mat("fgemm C", C, m, n, ldc);
        ffg::fgemm_dev(F, alpha, ffg::DView{const_cast<uint32_t*>(A), m, k, lda},
                       ffg::DView{const_cast<uint32_t*>(B), k, n, ldb}, beta, ffg::DView{C, m, n, ldc}, ctx->stream,
                       ctx->ws, &ctx->launches);
    });
}

int ffg_fgemm(ffg_ctx* ctx, uint64_t p, uint32_t alpha, const uint32_t* A, size_t lda, const uint32_t* B,
              size_t ldb, uint32_t beta, uint32_t* C, size_t ldc, size_t m, size_t n, size_t k) {
    return guarded(ctx, [&] {
        ffg::Field F = ffg::make_field(p);
        check_mat("fgemm A", A, m, k, lda);
        check_mat("fgemm B", B, k, n, ldb);
        check_mat("fgemm C", C, m, n, ldc);
        cudaStream_t st = ctx->stream;
        DevMat dA(m, k, st), dB(k, n, st), dC(m, n, st);
        dA.upload(A, lda);
        dB.upload(B, ldb);
        dC.upload(C, ldc);
        ffg::fgemm_dev(F, alpha, dA.view(), dB.view(), beta, dC.view(), st, ctx->ws, &ctx->launches);
        dC.download(C, ldc);
        FFG_CUDA(cudaStreamSynchronize(st));
    });
}

int ffg_ftrsm_dev(ffg_ctx* ctx, uint64_t p, int side, int uplo, int diag, const uint32_t* A, size_t lda, uint32_t* B,
                  size_t ldb, size_t m, size_t n) {
    return guarded(ctx, [&] {
        ffg::Field F = ffg::make_field(p);
        const size_t t = side == 0 ? m : n;
        check_mat("ftrsm A", A, t, t, lda);
        check_mat("ftrsm B", B, m, n, ldb);
        ffg::Blas blas{F, ctx->ws, ctx->stream, &ctx->launches};
        ffg::ftrsm_dev(blas, side, uplo, diag, ffg::DView{const_cast<uint32_t*>(A), t, t, lda}, ffg::DView{B, m, n, ldb},
                       /*check_diag=*/true);
    });
}

int ffg_ftrsm(ffg_ctx* ctx, uint64_t p, int side, int uplo, int diag, const uint32_t* A, size_t lda, uint32_t* B,
              size_t ldb, size_t m, size_t n) {
    return guarded(ctx, [&] {
        ffg::Field F = ffg::make_field(p);
        cudaStream_t st = ctx->stream;
        const size_t t = side == 0 ? m : n;
        check_mat("ftrsm A", A, t, t, lda);
        check_mat("ftrsm B", B, m, n, ldb);
        DevMat dA(t, t, st), dB(m, n, st);
        dA.upload(A, lda);
        dB.upload(B, ldb);
        ffg::Blas blas{F, ctx->ws, st, &ctx->launches};
        ffg::ftrsm_dev(blas, side, uplo, diag, dA.view(), dB.view(), true);
        dB.download(B, ldb);
        FFG_CUDA(cudaStreamSynchronize(st));
    });
}

int ffg_pluq_tile_recursive_dev(ffg_ctx* ctx, uint64_t p, uint32_t* A, size_t m, size_t n, size_t lda,
                                size_t threshold, uint32_t* P, uint32_t* Q, size_t* rank) {
    return guarded(ctx, [&] {
        ffg::Field F = ffg::make_field(p);
        check_mat("pluq", A, m, n, lda);
        ffg::Blas blas{F, ctx->ws, ctx->stream, &ctx->launches};
        size_t r = ffg::pluq_tile_recursive_dev(blas, ffg::DView{A, m, n, lda}, threshold, P, Q);
        if (rank) *rank = r;
    });
}

int ffg_pluq_tile_recursive(ffg_ctx* ctx, uint64_t p, uint32_t* A, size_t m, size_t n, size_t lda, size_t threshold,
                            uint32_t* P, uint32_t* Q, size_t* rank) {
    return guarded(ctx, [&] {
        ffg::Field F = ffg::make_field(p);
        ffg::Blas blas{F, ctx->ws, ctx->stream, &ctx->launches};
        check_mat("pluq", A, m, n, lda);
        size_t r = ffg::pluq_tile_recursive_host(blas, A, m, n, lda, threshold, P, Q);
        if (rank) *rank = r;
    });
}

int ffg_pluq_tile_recursive_u8(ffg_ctx* ctx, uint64_t p, uint8_t* A, size_t m, size_t n, size_t lda,
                               size_t threshold, uint32_t* P, uint32_t* Q, size_t* rank) {
    return guarded(ctx, [&] {
        ffg::Field F = ffg::make_field(p);
        ffg::Blas blas{F, ctx->ws, ctx->stream, &ctx->launches};
        check_mat("pluq", A, m, n, lda);
        size_t r = ffg::pluq_tile_recursive_host_u8(blas, A, m, n, lda, threshold, P, Q);
        if (rank) *rank = r;
    });
}

int ffg_rr_base(ffg_ctx* ctx, uint64_t p, uint32_t* A, size_t m, size_t n, size_t lda, uint32_t* P, uint32_t* Q,
                size_t* rank) {
    return guarded(ctx, [&] {
        ffg::Field F = ffg::make_field(p);
        check_mat("rr_base", A, m, n, lda);
        cudaStream_t st = ctx->stream;
        DevMat dA(m, n, st);
        dA.upload(A, lda);
        ffg::Blas blas{F, ctx->ws, st, &ctx->launches};
        size_t r = ffg::rr_base_dev(blas, dA.view(), P, Q);
        dA.download(A, lda);
        FFG_CUDA(cudaStreamSynchronize(st));
        if (rank) *rank = r;
    });
}

int ffg_apply_perm_dev(ffg_ctx* ctx, uint32_t* A, size_t m, size_t n, size_t lda, int axis, int inverse,
                       const uint32_t* perm) {
    return guarded(ctx, [&] {
        ffg::Field F = ffg::make_field(2);
        check_mat("apply_perm", A, m, n, lda);
        if (axis != 0 && axis != 1) throw ffg::Error(FFG_ERR_INVALID_ARG, "apply_perm: axis must be 0 or 1");
        if (!perm && (axis == 0 ? m : n) > 0) throw ffg::Error(FFG_ERR_INVALID_ARG, "apply_perm: null perm");
        ffg::Blas blas{F, ctx->ws, ctx->stream, &ctx->launches};
        ffg::apply_perm_dev(blas, ffg::DView{A, m, n, lda}, axis, inverse, perm);
    });
}

int ffg_dist_unique_id(unsigned char id[128]) {
    if (!id) return FFG_ERR_INVALID_ARG;
    try {
        ffg::nccl_unique_id(id);
        return FFG_OK;
    } catch (const ffg::Error& e) {
        g_err = e.what();
        return e.code;
    }
}

int ffg_dist_init(ffg_ctx* ctx, int world, int rank, const unsigned char id[128]) {
    return guarded(ctx, [&] {
        if (!id) throw ffg::Error(FFG_ERR_INVALID_ARG, "dist: null unique id");
        FFG_CUDA(cudaStreamSynchronize(ctx->stream));
        ffg::dist_init_nccl(ctx->ws.dist, world, rank, id, ctx->device);
    });
}

int ffg_dist_init_virtual(ffg_ctx* ctx, int world, int loopback) {
    return guarded(ctx, [&] {
        if (world < 1) throw ffg::Error(FFG_ERR_INVALID_ARG, "dist: world must be >= 1");
        FFG_CUDA(cudaStreamSynchronize(ctx->stream));
        ctx->ws.dist.reset();
        ctx->ws.dist.world = world;
        ctx->ws.dist.virt = world > 1;
        ctx->ws.dist.loopback = world > 1 && loopback != 0;
    });
}

int ffg_dist_set_min_work(ffg_ctx* ctx, uint64_t macs) {
    return guarded(ctx, [&] { ctx->ws.dist.min_work = macs; });
}

int ffg_dist_info(ffg_ctx* ctx, int* world, int* rank, int* is_virtual, uint64_t* exchanges, uint64_t* bytes) {
    return guarded(ctx, [&] {
        const ffg::Dist& d = ctx->ws.dist;
        if (world) *world = d.world;
        if (rank) *rank = d.rank;
        if (is_virtual) *is_virtual = d.virt ? 1 : 0;
        if (exchanges) *exchanges = d.exchanges;
        if (bytes) *bytes = d.bytes;
    });
}

int ffg_dist_finalize(ffg_ctx* ctx) {
    return guarded(ctx, [&] {
        FFG_CUDA(cudaStreamSynchronize(ctx->stream));
        ctx->ws.dist.reset();
    });
}

int ffg_dist_partition(size_t total, int world, int rank, size_t align, size_t* lo, size_t* hi) {
    if (world < 1 || rank < 0 || rank >= world || !lo || !hi) {
        g_err = "dist: bad partition arguments";
        return FFG_ERR_INVALID_ARG;
    }
    const ffg::Slice s = ffg::partition(total, world, rank, align);
    *lo = s.lo;
    *hi = s.hi;
    return FFG_OK;
}

}  // extern "C"
