// Cycles per pivot step of the base kernel's loop skeleton (512 threads): barrier + header
// load, optionally the 8-element lazy Shoup update per thread, and the lead warp's publish
// (ballot, 2 stores, shuffle chain).  nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdint>
#include <cstdio>

template <int MODE>  // 0: barrier only, 1: + header/publish chain, 2: + update, 3: update only (no publish)
__global__ void __launch_bounds__(512, 1) skel(uint32_t* out, uint32_t p, uint32_t pvp0, long long* cyc) {
    __shared__ uint4 hdr[2];
    __shared__ uint32_t row[2][64];
    const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    uint32_t v[8];
    for (int u = 0; u < 8; ++u) v[u] = tid * 8 + u + 1;
    if (tid == 0) hdr[0] = make_uint4(0, 1, 12345, pvp0);
    for (int j = tid; j < 128; j += 512) (&row[0][0])[j] = j + 1;
    __syncthreads();
    long long t0 = clock64();
    uint32_t buf = 0, acc = 0;
    for (int step = 0; step < 64; ++step) {
        uint4 h = make_uint4(1, 2, 3, pvp0);
        if (MODE == 1 || MODE == 2 || MODE == 3) h = hdr[buf];
        if (MODE >= 2) {
            const uint32_t numer = h.x * 7 + 3, nump = h.w ^ numer;
            const uint4 b0 = reinterpret_cast<const uint4*>(&row[buf][(tid & 7) * 8])[0];
            const uint4 b1 = reinterpret_cast<const uint4*>(&row[buf][(tid & 7) * 8])[1];
            const uint32_t b[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const uint32_t a = v[u] * h.z - __umulhi(v[u], h.w) * p;
                const uint32_t s = b[u] * numer - __umulhi(b[u], nump) * p;
                v[u] = a + 2 * p - s;
            }
        }
        if ((MODE == 1 || MODE == 2) && warp == (uint32_t)(step / 4)) {
            uint32_t o = 0;
            for (int u = 0; u < 8; ++u) o |= v[u];
            const uint32_t bal = __ballot_sync(0xffffffffu, o != 0);
            const uint32_t lead = __ffs(bal) - 1;
            if ((lane & ~7u) == (lead & ~7u)) {
                reinterpret_cast<uint4*>(&row[buf ^ 1][(lane & 7) * 8])[0] = make_uint4(v[0], v[1], v[2], v[3]);
                reinterpret_cast<uint4*>(&row[buf ^ 1][(lane & 7) * 8])[1] = make_uint4(v[4], v[5], v[6], v[7]);
            }
            __syncwarp();
            const uint32_t x0 = row[buf ^ 1][lane], x1 = row[buf ^ 1][lane + 32];
            const uint32_t b0 = __ballot_sync(0xffffffffu, x0 != 0), b1 = __ballot_sync(0xffffffffu, x1 != 0);
            const uint32_t pj = b0 ? __ffs(b0) - 1 : 31 + __ffs(b1);
            if (lane == 0) hdr[buf ^ 1] = make_uint4(step + 1, pj, row[buf ^ 1][pj], pvp0 + pj);
        }
        buf ^= 1;
        __syncthreads();
    }
    const long long t1 = clock64();
    for (int u = 0; u < 8; ++u) acc += v[u];
    out[tid] = acc;
    if (tid == 0) *cyc = t1 - t0;
}

int main() {
    uint32_t* out;
    long long* cyc;
    cudaMalloc(&out, 4096);
    cudaMallocManaged(&cyc, 8);
    const char* names[] = {"barrier only", "barrier+header+publish", "barrier+header+update+publish",
                           "barrier+header+update"};
    for (int mode = 0; mode < 4; ++mode) {
        long long best = 1LL << 60;
        for (int rep = 0; rep < 5; ++rep) {
            if (mode == 0) skel<0><<<1, 512>>>(out, 131071, 77, cyc);
            if (mode == 1) skel<1><<<1, 512>>>(out, 131071, 77, cyc);
            if (mode == 2) skel<2><<<1, 512>>>(out, 131071, 77, cyc);
            if (mode == 3) skel<3><<<1, 512>>>(out, 131071, 77, cyc);
            cudaDeviceSynchronize();
            if (*cyc < best) best = *cyc;
        }
        printf("%-34s %6.1f cycles/step\n", names[mode], best / 64.0);
    }
    return 0;
}
