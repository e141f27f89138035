// how long does the issuing thread spend in one cp.async.bulk (global -> smem)?
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "/root/repo/paper_2306_07629_b200/csrc/ptx.cuh"
using namespace sqz;
__global__ void k(const uint8_t* g, int bytes, int ncopies, long long* out, int warps_issuing) {
    extern __shared__ __align__(1024) uint8_t sm[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm);
    uint8_t* buf = sm + 1024;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) { for (int i = 0; i < 32; ++i) mbar_init(&bar[i], 1); fence_barrier_init(); }
    __syncthreads();
    if (warp >= warps_issuing) return;
    const uint64_t pol = policy_evict_first();
    long long tot = 0;
    uint32_t ph = 0;
    for (int i = 0; i < ncopies; ++i) {
        if (lane == 0) {
            const uint8_t* src = g + (size_t(blockIdx.x) * 64 + warp * 8 + (i & 7)) * size_t(bytes) % (size_t(1) << 30);
            long long t0 = clock64();
            mbar_arrive_expect_tx(&bar[warp], bytes);
            bulk_g2s(buf + warp * bytes, src, bytes, &bar[warp], pol);
            long long t1 = clock64();
            tot += t1 - t0;
        }
        __syncwarp();
        mbar_wait(&bar[warp], ph);
        ph ^= 1;
    }
    if (lane == 0) out[blockIdx.x * 32 + warp] = tot / ncopies;
}
int main() {
    uint8_t* g; cudaMalloc(&g, size_t(1) << 30); cudaMemset(g, 1, size_t(1) << 30);
    long long* out; cudaMalloc(&out, 148 * 32 * 8);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    for (int w : {1, 8, 16})
        for (int bytes : {1536, 6144, 12288}) {
            if (1024 + w * bytes > 200 * 1024) continue;
            k<<<148, w * 32, 1024 + w * bytes>>>(g, bytes, 200, out, w);
            cudaDeviceSynchronize();
            long long h[148 * 32]; cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost);
            double s = 0; int n = 0;
            for (int b = 0; b < 148; ++b) for (int i = 0; i < w; ++i) { s += h[b * 32 + i]; ++n; }
            printf("issuing warps %2d bytes %6d: %.0f cycles in arrive.expect_tx + cp.async.bulk\n", w, bytes, s / n);
        }
    return 0;
}
