// Does alternating large/small shared-memory kernels cost a carveout switch?
#include <cstdio>
__global__ void big(float* x) {
    extern __shared__ float s[];
    s[threadIdx.x] = x[threadIdx.x];
    __syncthreads();
    x[threadIdx.x] = s[(threadIdx.x + 1) % blockDim.x];
}
__global__ void small(float* x) {
    __shared__ float s[256];
    s[threadIdx.x] = x[threadIdx.x];
    __syncthreads();
    x[threadIdx.x] = s[(threadIdx.x + 1) % blockDim.x] + 1;
}
int main() {
    float* x;
    cudaMalloc(&x, 1 << 20);
    const int big_smem = 149 * 1024;
    cudaFuncSetAttribute(big, cudaFuncAttributeMaxDynamicSharedMemorySize, big_smem);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int mode = 0; mode < 4; ++mode) {
        for (int w = 0; w < 2; ++w) {
            cudaEventRecord(a);
            for (int i = 0; i < 100; ++i) {
                if (mode == 0) big<<<1, 256, big_smem>>>(x);
                if (mode == 1) small<<<148, 256>>>(x);
                if (mode == 2) { big<<<1, 256, big_smem>>>(x); small<<<148, 256>>>(x); }
                if (mode == 3) { big<<<1, 256, 1024>>>(x); small<<<148, 256>>>(x); }
            }
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (w) printf("mode %d: %.2f us per iteration\n", mode, ms * 10);
        }
    }
    return 0;
}
