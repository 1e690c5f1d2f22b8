// Per-launch GPU cost of dependent back-to-back kernels: empty body with 384 threads and
// (a) no smem, (b) large dynamic smem, (c) TMEM alloc/dealloc of 512 columns, (d) both,
// (e) alternating with a small-smem kernel (carveout switches), (f) 103 CTAs instead of 1.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/launch_cost launch_cost.cu
#include <cstdint>
#include <cstdio>

__global__ void __launch_bounds__(384, 1) k_plain(int* x) {
    if (threadIdx.x == 0 && x[0] == 12345) x[1] = 1;
}
__global__ void __launch_bounds__(384, 1) k_smem(int* x) {
    extern __shared__ int s[];
    s[threadIdx.x] = threadIdx.x;
    __syncthreads();
    if (threadIdx.x == 0 && s[5] == 12345) x[1] = 1;
}
__global__ void __launch_bounds__(384, 1) k_tmem(int* x) {
    __shared__ uint32_t slot;
    const uint32_t warp = threadIdx.x >> 5;
    if (warp == 2) {
        uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(&slot));
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(a));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t t = slot;
    __syncthreads();
    if (warp == 2) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(t));
    if (threadIdx.x == 0 && x[0] == 12345) x[1] = 1;
}
__global__ void __launch_bounds__(384, 1) k_both(int* x) {
    extern __shared__ int s[];
    __shared__ uint32_t slot;
    const uint32_t warp = threadIdx.x >> 5;
    s[threadIdx.x] = threadIdx.x;
    if (warp == 2) {
        uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(&slot));
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(a));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t t = slot;
    __syncthreads();
    if (warp == 2) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(t));
    if (threadIdx.x == 0 && s[5] == 12345) x[1] = 1;
}
__global__ void k_small(int* x) {
    __shared__ int s[256];
    s[threadIdx.x] = threadIdx.x;
    __syncthreads();
    if (threadIdx.x == 0 && s[5] == 12345) x[1] = 1;
}

int main() {
    int* x;
    cudaMalloc(&x, 1 << 20);
    cudaMemset(x, 0, 1 << 20);
    const int BIG = 160 * 1024;
    cudaFuncSetAttribute(k_smem, cudaFuncAttributeMaxDynamicSharedMemorySize, BIG);
    cudaFuncSetAttribute(k_both, cudaFuncAttributeMaxDynamicSharedMemorySize, BIG);
    cudaStream_t st;
    cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const char* names[] = {"plain 1 CTA",      "smem160K 1 CTA",        "tmem512 1 CTA",
                           "smem+tmem 1 CTA",  "smem+tmem 103 CTAs",    "small 148 CTAs",
                           "alt smem+tmem / small", "alt plain / small", "smem 4K 1 CTA"};
    for (int mode = 0; mode < 9; ++mode) {
        float best = 1e9f;
        for (int rep = 0; rep < 3; ++rep) {
            const int N = 200;
            cudaEventRecord(a, st);
            for (int i = 0; i < N; ++i) {
                switch (mode) {
                    case 0: k_plain<<<1, 384, 0, st>>>(x); break;
                    case 1: k_smem<<<1, 384, BIG, st>>>(x); break;
                    case 2: k_tmem<<<1, 384, 0, st>>>(x); break;
                    case 3: k_both<<<1, 384, BIG, st>>>(x); break;
                    case 4: k_both<<<103, 384, BIG, st>>>(x); break;
                    case 5: k_small<<<148, 256, 0, st>>>(x); break;
                    case 6:
                        k_both<<<1, 384, BIG, st>>>(x);
                        k_small<<<148, 256, 0, st>>>(x);
                        break;
                    case 7:
                        k_plain<<<1, 384, 0, st>>>(x);
                        k_small<<<148, 256, 0, st>>>(x);
                        break;
                    case 8: k_smem<<<1, 384, 4096, st>>>(x); break;
                }
            }
            cudaEventRecord(b, st);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            const float per = ms * 1000 / N / ((mode == 6 || mode == 7) ? 2 : 1);
            if (per < best) best = per;
        }
        printf("%-24s %7.2f us per launch\n", names[mode], best);
    }
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
