// Consumer-loop microbenchmark (dev tool): the stack kernel's 3-bit decode
// (tile.cuh span3_frags: PRMT byte planes -> fp16 A fragments -> mma.sync)
// run over shared-memory-resident unit records, to compare loop structures at
// the kernel's warp counts.  Reports weights/clk/SM.
//   V0  span pair (2 units / iter, one accumulator each) -- the kernel's loop
//   V1  span pair, software-pipelined (next pair's words + x loaded first)
//   V2  4 units / iter (two span pairs, 4 accumulators)
//   V3  2 tiles x 2 spans / iter (x shared by the two tiles, 4 accumulators)
//   V4  V1 + 2 tiles x 1 span per half-iteration (x shared), pipelined
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o loop_mb loop_mb.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include "../../paper_2306_07629_b200/csrc/tile.cuh"

#define CK(x)                                                                          \
    do {                                                                               \
        cudaError_t e = (x);                                                           \
        if (e != cudaSuccess) {                                                        \
            printf("CUDA %s @%d: %s\n", #x, __LINE__, cudaGetErrorString(e));          \
            return 1;                                                                  \
        }                                                                              \
    } while (0)

using namespace sqz;
constexpr int NU = 32;  // unit records per warp in smem (cycled)

__device__ __forceinline__ uint4 ldx(const uint16_t* xs, uint32_t off) {
    return *reinterpret_cast<const uint4*>(xs + off);
}

template <int VAR>
__global__ void __launch_bounds__(1024, 1) k_loop(int niter, float* out, int consumers, ShiftK K,
                                                  long long* clk) {
    extern __shared__ __align__(16) uint32_t sm[];
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t* words = sm + warp * NU * 96;
    uint16_t* xs = reinterpret_cast<uint16_t*>(sm + consumers * NU * 96);  // NU spans of x
    if (int(warp) < consumers)
        for (uint32_t i = lane; i < NU * 96; i += 32) words[i] = (i * 2654435761u) ^ (warp * 77u);
    for (uint32_t i = threadIdx.x; i < NU * 256; i += blockDim.x) xs[i] = uint16_t(0x3800 + (i & 0x3ff));
    __syncthreads();
    if (int(warp) >= consumers) {  // idle role warps (the kernel's 5..7)
        __nanosleep(100000);
        return;
    }
    const ShiftK k = K;
    const uint32_t xoff = tile_x_offset(lane);
    const Planes8 PA{0x3c3a3836u ^ lane, 0x44424140u, 0x3c3b3a39u, 0x3d3e3f40u ^ lane};
    const Planes8 PB{0x34363839u ^ lane, 0x40414243u, 0x39393a3bu, 0x3a3b3c3du ^ lane};
    float d0[4] = {0, 0, 0, 0}, d1[4] = {0, 0, 0, 0}, d2[4] = {0, 0, 0, 0}, d3[4] = {0, 0, 0, 0};
    long long c0 = clock64();
#pragma unroll 1
    for (int it = 0; it < niter; ++it) {
        if constexpr (VAR == 0) {
#pragma unroll 1
            for (int u = 0; u < NU; u += 2) {
                const uint32_t* sp = words + u * 96;
                const uint16_t* xp = xs + u * 256 + xoff;
                const uint32_t a0 = sp[lane], a1 = sp[32 + lane], a2 = sp[64 + lane];
                const uint32_t b0 = sp[96 + lane], b1 = sp[128 + lane], b2 = sp[160 + lane];
                const uint4 xa0 = ldx(xp, 0), xb0 = ldx(xp, 128), xa1 = ldx(xp, 256),
                            xb1 = ldx(xp, 384);
                span3_mma_one(a0, a1, a2, PA, xa0, xb0, d0, k);
                span3_mma_one(b0, b1, b2, PA, xa1, xb1, d1, k);
            }
        } else if constexpr (VAR == 1) {
            const uint32_t* sp = words;
            const uint16_t* xp = xs + xoff;
            uint32_t a0 = sp[lane], a1 = sp[32 + lane], a2 = sp[64 + lane];
            uint32_t b0 = sp[96 + lane], b1 = sp[128 + lane], b2 = sp[160 + lane];
            uint4 xa0 = ldx(xp, 0), xb0 = ldx(xp, 128), xa1 = ldx(xp, 256), xb1 = ldx(xp, 384);
#pragma unroll 1
            for (int u = 0; u < NU; u += 2) {
                const uint32_t ca0 = a0, ca1 = a1, ca2 = a2, cb0 = b0, cb1 = b1, cb2 = b2;
                const uint4 cxa0 = xa0, cxb0 = xb0, cxa1 = xa1, cxb1 = xb1;
                const int un = (u + 2) & (NU - 1);
                sp = words + un * 96;
                xp = xs + un * 256 + xoff;
                a0 = sp[lane]; a1 = sp[32 + lane]; a2 = sp[64 + lane];
                b0 = sp[96 + lane]; b1 = sp[128 + lane]; b2 = sp[160 + lane];
                xa0 = ldx(xp, 0); xb0 = ldx(xp, 128); xa1 = ldx(xp, 256); xb1 = ldx(xp, 384);
                span3_mma_one(ca0, ca1, ca2, PA, cxa0, cxb0, d0, k);
                span3_mma_one(cb0, cb1, cb2, PA, cxa1, cxb1, d1, k);
            }
        } else if constexpr (VAR == 2) {
#pragma unroll 1
            for (int u = 0; u < NU; u += 4) {
                const uint32_t* sp = words + u * 96;
                const uint16_t* xp = xs + u * 256 + xoff;
                const uint32_t a0 = sp[lane], a1 = sp[32 + lane], a2 = sp[64 + lane];
                const uint32_t b0 = sp[96 + lane], b1 = sp[128 + lane], b2 = sp[160 + lane];
                const uint32_t c0_ = sp[192 + lane], c1 = sp[224 + lane], c2 = sp[256 + lane];
                const uint32_t e0 = sp[288 + lane], e1 = sp[320 + lane], e2 = sp[352 + lane];
                const uint4 xa0 = ldx(xp, 0), xb0 = ldx(xp, 128), xa1 = ldx(xp, 256),
                            xb1 = ldx(xp, 384), xa2 = ldx(xp, 512), xb2 = ldx(xp, 640),
                            xa3 = ldx(xp, 768), xb3 = ldx(xp, 896);
                span3_mma_one(a0, a1, a2, PA, xa0, xb0, d0, k);
                span3_mma_one(b0, b1, b2, PA, xa1, xb1, d1, k);
                span3_mma_one(c0_, c1, c2, PA, xa2, xb2, d2, k);
                span3_mma_one(e0, e1, e2, PA, xa3, xb3, d3, k);
            }
        } else if constexpr (VAR == 7 || VAR == 8) {
            // V0 split into "layers" of 14 units (7 pairs): a loop restart per
            // layer (VAR 8 also: a (warp*U) % NS division and a LUT reload)
            for (int l0 = 0; l0 < NU; l0 += 14) {
                const int U = min(14, NU - l0);
                Planes8 PL = PA;
                uint32_t sdiv = 0;
                if constexpr (VAR == 8) {  // LUT planes reloaded from smem per layer
                    const uint4 q = *reinterpret_cast<const uint4*>(xs + ((l0 + it) & 31) * 8 + 8 * (lane & 3));
                    PL = Planes8{q.x ^ PA.l0, q.y ^ PA.l1, PA.h0, PA.h1};
                }
#pragma unroll 1
                for (int u = 0; u + 1 < U; u += 2) {
                    const uint32_t* sp = words + (l0 + u) * 96;
                    const uint16_t* xp = xs + ((l0 + u + sdiv) & 31) * 256 + xoff;
                    const uint32_t a0 = sp[lane], a1 = sp[32 + lane], a2 = sp[64 + lane];
                    const uint32_t b0 = sp[96 + lane], b1 = sp[128 + lane], b2 = sp[160 + lane];
                    const uint4 xa0 = ldx(xp, 0), xb0 = ldx(xp, 128), xa1 = ldx(xp, 256),
                                xb1 = ldx(xp, 384);
                    span3_mma_one(a0, a1, a2, PL, xa0, xb0, d0, k);
                    span3_mma_one(b0, b1, b2, PL, xa1, xb1, d1, k);
                }

            }
        } else if constexpr (VAR == 5 || VAR == 6) {
#pragma unroll 1
            for (int u = 0; u < NU; u += 2) {
                const uint32_t* sp = words + u * 96;
                const uint16_t* xp = xs + u * 256 + xoff;
                const uint32_t a0 = sp[lane], a1 = sp[32 + lane], a2 = sp[64 + lane];
                const uint32_t b0 = sp[96 + lane], b1 = sp[128 + lane], b2 = sp[160 + lane];
                const uint4 xa0 = ldx(xp, 0), xb0 = ldx(xp, 128), xa1 = ldx(xp, 256),
                            xb1 = ldx(xp, 384);
                if constexpr (VAR == 5) {  // full decode, no HMMA: fold fragments into d
                    auto fold = [&](float (&d)[4]) {
                        return [&](int j, uint32_t f0, uint32_t f1, uint32_t f2, uint32_t f3) {
                            d[j] += __uint_as_float((f0 ^ f1) & 0x3fffffffu) + __uint_as_float((f2 ^ f3) & 0x3fffffffu);
                        };
                    };
                    span3_frags(a0, a1, a2, PA, fold(d0), k);
                    span3_frags(b0, b1, b2, PA, fold(d1), k);
                    d0[0] += __uint_as_float((xa0.x ^ xb0.y) & 0x3fffffffu);
                    d1[0] += __uint_as_float((xa1.x ^ xb1.y) & 0x3fffffffu);
                } else {  // HMMA only: raw words as fragments
                    hmma16816(d0, a0, a1, a2, b0, xa0.x, xa0.y);
                    hmma16816(d0, a1, a2, b0, b1, xa0.z, xa0.w);
                    hmma16816(d0, a2, b0, b1, b2, xb0.x, xb0.y);
                    hmma16816(d0, b0, b1, b2, a0, xb0.z, xb0.w);
                    hmma16816(d1, a0, a1, a2, b0, xa1.x, xa1.y);
                    hmma16816(d1, a1, a2, b0, b1, xa1.z, xa1.w);
                    hmma16816(d1, a2, b0, b1, b2, xb1.x, xb1.y);
                    hmma16816(d1, b0, b1, b2, a0, xb1.z, xb1.w);
                }
            }
        } else if constexpr (VAR == 3) {
            // units u, u+1 = tile A spans s, s+1; u+2, u+3 = tile B spans s, s+1
#pragma unroll 1
            for (int u = 0; u < NU; u += 4) {
                const uint32_t* sp = words + u * 96;
                const uint16_t* xp = xs + (u & ~3) * 128 + xoff;
                const uint32_t a0 = sp[lane], a1 = sp[32 + lane], a2 = sp[64 + lane];
                const uint32_t b0 = sp[96 + lane], b1 = sp[128 + lane], b2 = sp[160 + lane];
                const uint32_t c0_ = sp[192 + lane], c1 = sp[224 + lane], c2 = sp[256 + lane];
                const uint32_t e0 = sp[288 + lane], e1 = sp[320 + lane], e2 = sp[352 + lane];
                const uint4 xa0 = ldx(xp, 0), xb0 = ldx(xp, 128), xa1 = ldx(xp, 256),
                            xb1 = ldx(xp, 384);
                span3_mma_one(a0, a1, a2, PA, xa0, xb0, d0, k);
                span3_mma_one(b0, b1, b2, PA, xa1, xb1, d1, k);
                span3_mma_one(c0_, c1, c2, PB, xa0, xb0, d2, k);
                span3_mma_one(e0, e1, e2, PB, xa1, xb1, d3, k);
            }
        } else {
            // pipelined, 2 tiles x 1 span per half-iteration (x shared)
            const uint32_t* sp = words;
            const uint16_t* xp = xs + xoff;
            uint32_t a0 = sp[lane], a1 = sp[32 + lane], a2 = sp[64 + lane];
            uint32_t b0 = sp[96 + lane], b1 = sp[128 + lane], b2 = sp[160 + lane];
            uint4 xa0 = ldx(xp, 0), xb0 = ldx(xp, 128);
#pragma unroll 1
            for (int u = 0; u < NU; u += 2) {
                const uint32_t ca0 = a0, ca1 = a1, ca2 = a2, cb0 = b0, cb1 = b1, cb2 = b2;
                const uint4 cxa0 = xa0, cxb0 = xb0;
                const int un = (u + 2) & (NU - 1);
                sp = words + un * 96;
                xp = xs + un * 128 + xoff;
                a0 = sp[lane]; a1 = sp[32 + lane]; a2 = sp[64 + lane];
                b0 = sp[96 + lane]; b1 = sp[128 + lane]; b2 = sp[160 + lane];
                xa0 = ldx(xp, 0); xb0 = ldx(xp, 128);
                span3_mma_one(ca0, ca1, ca2, PA, cxa0, cxb0, d0, k);
                span3_mma_one(cb0, cb1, cb2, PB, cxa0, cxb0, d1, k);
            }
        }
    }
    long long c1 = clock64();
    if (threadIdx.x == 0) atomicAdd(reinterpret_cast<unsigned long long*>(clk), c1 - c0);
    float a = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) a += d0[q] + d1[q] + d2[q] + d3[q];
    out[blockIdx.x * blockDim.x + threadIdx.x] = a;
}

// V5: the same pair loop fed from HBM through a private per-warp TMA ring
// (cp.async.bulk + mbarrier, like the stack kernel's consumers): each warp
// streams its own contiguous `per_warp` units of a large buffer in chunks of
// `cu` units through `ws` slots.  Role warps: none.
__global__ void __launch_bounds__(1024, 1) k_stream(const uint32_t* __restrict__ g, int per_warp,
                                                    int cu, int ws, int consumers, float* out,
                                                    ShiftK K, long long* clk) {
    extern __shared__ __align__(1024) uint8_t smb[];
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint64_t* full = reinterpret_cast<uint64_t*>(smb);  // [consumers][ws]
    uint16_t* xs = reinterpret_cast<uint16_t*>(smb + 2048);
    uint8_t* ring = smb + 2048 + 64 * 256 * 2;
    const uint32_t slot_bytes = cu * 384;
    for (uint32_t i = threadIdx.x; i < 64 * 256; i += blockDim.x) xs[i] = uint16_t(0x3800 + (i & 0x3ff));
    if (threadIdx.x == 0) {
        for (int i = 0; i < consumers * ws; ++i) mbar_init(&full[i], 1);
        fence_barrier_init();
    }
    __syncthreads();
    if (int(warp) >= consumers) return;
    const uint64_t pol = policy_evict_first();
    const size_t wbase = (size_t(blockIdx.x) * consumers + warp) * per_warp * 96;  // words
    int issued = 0, slot_i = 0;
    auto issue = [&]() {
        if (issued >= per_warp) return;
        const int n = min(cu, per_warp - issued);
        if (lane == 0) {
            uint64_t* bar = &full[warp * ws + slot_i];
            mbar_arrive_expect_tx(bar, n * 384);
            bulk_g2s(ring + size_t(warp * ws + slot_i) * slot_bytes, g + wbase + size_t(issued) * 96,
                     n * 384, bar, pol);
        }
        issued += n;
        if (++slot_i == ws) slot_i = 0;
    };
    for (int k = 0; k < ws; ++k) issue();
    const ShiftK k = K;
    const uint32_t xoff = tile_x_offset(lane);
    const Planes8 PA{0x3c3a3836u ^ lane, 0x44424140u, 0x3c3b3a39u, 0x3d3e3f40u ^ lane};
    float d0[4] = {0, 0, 0, 0}, d1[4] = {0, 0, 0, 0};
    long long c0 = clock64();
    int cslot = 0;
    uint32_t ph = 0;
    for (int done = 0; done < per_warp;) {
        const int n = min(cu, per_warp - done);
        mbar_wait(&full[warp * ws + cslot], ph);
        const uint32_t* chunk = reinterpret_cast<const uint32_t*>(ring + size_t(warp * ws + cslot) * slot_bytes);
#pragma unroll 1
        for (int u = 0; u + 1 < n; u += 2) {
            const uint32_t* sp = chunk + u * 96;
            const uint16_t* xp = xs + ((done + u) & 63) * 256 + xoff;
            const uint32_t a0 = sp[lane], a1 = sp[32 + lane], a2 = sp[64 + lane];
            const uint32_t b0 = sp[96 + lane], b1 = sp[128 + lane], b2 = sp[160 + lane];
            const uint4 xa0 = ldx(xp, 0), xb0 = ldx(xp, 128), xa1 = ldx(xp, 256), xb1 = ldx(xp, 384);
            span3_mma_one(a0, a1, a2, PA, xa0, xb0, d0, k);
            span3_mma_one(b0, b1, b2, PA, xa1, xb1, d1, k);
        }
        __syncwarp();
        done += n;
        if (++cslot == ws) { cslot = 0; ph ^= 1u; }
        issue();
    }
    long long c1 = clock64();
    if (lane == 0) atomicAdd(reinterpret_cast<unsigned long long*>(clk), c1 - c0);
    float a = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) a += d0[q] + d1[q];
    out[blockIdx.x * blockDim.x + threadIdx.x] = a;
}

// V6: as V5, but one producer warp issues every TMA refill (consumers only
// wait on `full` and arrive on `empty`): warp `consumers` is the producer
__global__ void __launch_bounds__(1024, 1) k_stream_prod(const uint32_t* __restrict__ g, int per_warp,
                                                         int cu, int ws, int consumers, float* out,
                                                         ShiftK K, long long* clk) {
    extern __shared__ __align__(1024) uint8_t smb[];
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint64_t* full = reinterpret_cast<uint64_t*>(smb);        // [consumers][ws]
    uint64_t* empty = full + 128;                              // [consumers][ws]
    uint16_t* xs = reinterpret_cast<uint16_t*>(smb + 2048);
    uint8_t* ring = smb + 2048 + 64 * 256 * 2;
    const uint32_t slot_bytes = cu * 384;
    for (uint32_t i = threadIdx.x; i < 64 * 256; i += blockDim.x) xs[i] = uint16_t(0x3800 + (i & 0x3ff));
    if (threadIdx.x == 0) {
        for (int i = 0; i < consumers * ws; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 1);
        }
        fence_barrier_init();
    }
    __syncthreads();
    const int nch = (per_warp + cu - 1) / cu;
    if (int(warp) == consumers) {  // producer
        if (lane != 0) return;
        const uint64_t pol = policy_evict_first();
        // non-blocking round robin: refill whichever warp's next slot is free
        int next[32];
        for (int w = 0; w < consumers; ++w) next[w] = 0;
        int left = consumers;
        while (left) {
            for (int w = 0; w < consumers; ++w) {
                const int j = next[w];
                if (j >= nch) continue;
                const int slot = j % ws;
                if (j >= ws && !mbar_test_wait(&empty[w * ws + slot], ((j / ws) - 1) & 1u)) continue;
                const int n = min(cu, per_warp - j * cu);
                const size_t wbase = (size_t(blockIdx.x) * consumers + w) * per_warp * 96;
                uint64_t* bar = &full[w * ws + slot];
                mbar_arrive_expect_tx(bar, n * 384);
                bulk_g2s(ring + size_t(w * ws + slot) * slot_bytes, g + wbase + size_t(j) * cu * 96,
                         n * 384, bar, pol);
                if (++next[w] == nch) --left;
            }
        }
        return;
    }
    if (int(warp) > consumers) return;
    const ShiftK k = K;
    const uint32_t xoff = tile_x_offset(lane);
    const Planes8 PA{0x3c3a3836u ^ lane, 0x44424140u, 0x3c3b3a39u, 0x3d3e3f40u ^ lane};
    float d0[4] = {0, 0, 0, 0}, d1[4] = {0, 0, 0, 0};
    long long c0 = clock64();
    for (int j = 0; j < nch; ++j) {
        const int slot = j % ws;
        const int n = min(cu, per_warp - j * cu);
        mbar_wait(&full[warp * ws + slot], (j / ws) & 1u);
        const uint32_t* chunk = reinterpret_cast<const uint32_t*>(ring + size_t(warp * ws + slot) * slot_bytes);
#pragma unroll 1
        for (int u = 0; u + 1 < n; u += 2) {
            const uint32_t* sp = chunk + u * 96;
            const uint16_t* xp = xs + ((j * cu + u) & 63) * 256 + xoff;
            const uint32_t a0 = sp[lane], a1 = sp[32 + lane], a2 = sp[64 + lane];
            const uint32_t b0 = sp[96 + lane], b1 = sp[128 + lane], b2 = sp[160 + lane];
            const uint4 xa0 = ldx(xp, 0), xb0 = ldx(xp, 128), xa1 = ldx(xp, 256), xb1 = ldx(xp, 384);
            span3_mma_one(a0, a1, a2, PA, xa0, xb0, d0, k);
            span3_mma_one(b0, b1, b2, PA, xa1, xb1, d1, k);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[warp * ws + slot]);
    }
    long long c1 = clock64();
    if (lane == 0) atomicAdd(reinterpret_cast<unsigned long long*>(clk), c1 - c0);
    float a = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) a += d0[q] + d1[q];
    out[blockIdx.x * blockDim.x + threadIdx.x] = a;
}

// V7: no smem ring -- each lane loads its own index words straight from HBM
// into registers, D unit pairs ahead of the decode (ld.global.nc, L1 no-
// allocate), so there is no TMA issue, no mbarrier and no ring slot
template <int D>
__global__ void __launch_bounds__(1024, 1) k_ldg(const uint32_t* __restrict__ g, int per_warp,
                                                 int consumers, float* out, ShiftK K,
                                                 long long* clk) {
    extern __shared__ __align__(1024) uint8_t smb[];
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint16_t* xs = reinterpret_cast<uint16_t*>(smb);
    for (uint32_t i = threadIdx.x; i < 64 * 256; i += blockDim.x) xs[i] = uint16_t(0x3800 + (i & 0x3ff));
    __syncthreads();
    if (int(warp) >= consumers) return;
    const uint32_t* base = g + (size_t(blockIdx.x) * consumers + warp) * per_warp * 96 + lane;
    const ShiftK k = K;
    const uint32_t xoff = tile_x_offset(lane);
    const Planes8 PA{0x3c3a3836u ^ lane, 0x44424140u, 0x3c3b3a39u, 0x3d3e3f40u ^ lane};
    float d0[4] = {0, 0, 0, 0}, d1[4] = {0, 0, 0, 0};
    uint32_t q[D][6];
    auto ld = [&](int pair, uint32_t (&r)[6]) {
        const uint32_t* p = base + size_t(pair) * 192;
#pragma unroll
        for (int i = 0; i < 6; ++i) {
            uint32_t v;
            asm volatile("ld.global.nc.L1::no_allocate.b32 %0, [%1];" : "=r"(v) : "l"(p + 32 * i));
            r[i] = v;
        }
    };
#pragma unroll
    for (int i = 0; i < D; ++i) ld(i, q[i]);
    const int npairs = per_warp / 2;
    long long c0 = clock64();
#pragma unroll 1
    for (int pr = 0; pr < npairs; pr += D) {
#pragma unroll
        for (int i = 0; i < D; ++i) {
            uint32_t c[6];
#pragma unroll
            for (int z = 0; z < 6; ++z) c[z] = q[i][z];
            if (pr + i + D < npairs) ld(pr + i + D, q[i]);
            const uint16_t* xp = xs + (((pr + i) * 2) & 63) * 256 + xoff;
            const uint4 xa0 = ldx(xp, 0), xb0 = ldx(xp, 128), xa1 = ldx(xp, 256), xb1 = ldx(xp, 384);
            span3_mma_one(c[0], c[1], c[2], PA, xa0, xb0, d0, k);
            span3_mma_one(c[3], c[4], c[5], PA, xa1, xb1, d1, k);
        }
    }
    long long c1 = clock64();
    if (lane == 0) atomicAdd(reinterpret_cast<unsigned long long*>(clk), c1 - c0);
    float a = 0;
#pragma unroll
    for (int z = 0; z < 4; ++z) a += d0[z] + d1[z];
    out[blockIdx.x * blockDim.x + threadIdx.x] = a;
}

// V8: the kernel's per-layer structure in isolation: each warp streams L
// "layers" of U units each (one TMA chunk per layer, 2 slots), per layer a
// LUT-plane load, span-pair loop over tiles of NS spans (a flush = row reduce
// + smem partial store at every tile change and at the layer end)
__global__ void __launch_bounds__(1024, 1) k_layers(const uint32_t* __restrict__ g, int L, int U,
                                                    int NS, int consumers, float* out, ShiftK K,
                                                    long long* clk, int mode = 0) {
    extern __shared__ __align__(1024) uint8_t smb[];
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint64_t* full = reinterpret_cast<uint64_t*>(smb);
    uint16_t* xs = reinterpret_cast<uint16_t*>(smb + 2048);
    float* part = reinterpret_cast<float*>(smb + 2048 + 64 * 256 * 2);  // [16][256]
    uint32_t* luts = reinterpret_cast<uint32_t*>(smb + 2048 + 64 * 512 + 16 * 1024);  // 256 rows x 4
    uint8_t* ring = smb + 2048 + 64 * 512 + 16 * 1024 + 4096;
    const uint32_t slot_bytes = ((U * 384 + 127) / 128) * 128;
    for (uint32_t i = threadIdx.x; i < 64 * 256; i += blockDim.x) xs[i] = uint16_t(0x3800 + (i & 0x3ff));
    for (uint32_t i = threadIdx.x; i < 1024; i += blockDim.x) luts[i] = 0x3c3a3836u ^ i;
    if (threadIdx.x == 0) {
        for (int i = 0; i < consumers * 2; ++i) mbar_init(&full[i], 1);
        fence_barrier_init();
    }
    __syncthreads();
    if (int(warp) >= consumers) return;
    const uint64_t pol = policy_evict_first();
    const size_t wbase = (size_t(blockIdx.x) * consumers + warp) * size_t(L) * U * 96;
    auto issue = [&](int l) {
        if (l >= L) return;
        if ((mode & 4) && l >= 2) return;  // mode 4: no per-layer TMA (slots reused)
        if (lane == 0) {
            uint64_t* bar = &full[warp * 2 + (l & 1)];
            mbar_arrive_expect_tx(bar, U * 384);
            bulk_g2s(ring + size_t(warp * 2 + (l & 1)) * slot_bytes, g + wbase + size_t(l) * U * 96,
                     U * 384, bar, pol);
        }
    };
    issue(0);
    issue(1);
    const ShiftK k = K;
    const uint32_t xoff = tile_x_offset(lane), trow = (lane >> 2) & 3u;
    if (mode & 64) {  // overwrite the ring with hashed words (data-value experiment)
        mbar_wait(&full[warp * 2], 0);
        mbar_wait(&full[warp * 2 + 1], 0);
        uint32_t* rw = reinterpret_cast<uint32_t*>(ring + size_t(warp * 2) * slot_bytes);
        for (uint32_t i = lane; i < 2 * slot_bytes / 4; i += 32) rw[i] = (i * 2654435761u) ^ (warp * 77u);
        __syncwarp();
    }
    long long c0 = clock64();
    float acc = 0.f;
    for (int l = 0; l < L; ++l) {
        if ((!(mode & 4) || l < 2) && !(mode & 64)) mbar_wait(&full[warp * 2 + (l & 1)], (l >> 1) & 1u);
        const uint32_t* chunk = reinterpret_cast<const uint32_t*>(ring + size_t(warp * 2 + (l & 1)) * slot_bytes);
        const uint16_t* xh = xs + (l & 3) * 4096;
        // the warp's range starts mid-tile like the kernel's (warp-dependent offset)
        uint32_t s = (mode & 8) ? 0u : (warp * U) % NS, tile = (mode & 8) ? warp : (warp * U) / NS;
        float d0[4] = {0, 0, 0, 0}, d1[4] = {0, 0, 0, 0};
        const uint4 q0 = *reinterpret_cast<const uint4*>(luts + ((tile * 4 + trow) & 255) * 4);
        Planes8 P{q0.x, q0.y, q0.z, q0.w};
        auto flush = [&]() {
            const float v = tile_rows_reduce(d0, d1, lane);
            if ((lane & 3) == 0 && lane < 16) part[warp * 256 + ((tile * 4 + trow) & 255)] += v;
#pragma unroll
            for (int z = 0; z < 4; ++z) d0[z] = d1[z] = 0.f;
        };
        int u = 0;
        while (u < U) {
            const int s_end = min(NS, int(s) + (U - u));
            int kk = s;
            const uint32_t* sp = chunk + u * 96;
            const uint16_t* xp = xh + (s & 15) * 256 + xoff;
#pragma unroll 1
            for (; kk + 1 < s_end; kk += 2) {
                const uint32_t a0 = sp[lane], a1 = sp[32 + lane], a2 = sp[64 + lane];
                const uint32_t b0 = sp[96 + lane], b1 = sp[128 + lane], b2 = sp[160 + lane];
                const uint4 xa0 = ldx(xp, 0), xb0 = ldx(xp, 128), xa1 = ldx(xp, 256), xb1 = ldx(xp, 384);
                span3_mma_one(a0, a1, a2, P, xa0, xb0, d0, k);
                span3_mma_one(b0, b1, b2, P, xa1, xb1, d1, k);
                sp += 192;
                xp = xh + (((kk + 2) & 15) * 256) + xoff;
            }
            if (kk < s_end) {
                const uint4 xa0 = ldx(xp, 0), xb0 = ldx(xp, 128);
                span3_mma_one(sp[lane], sp[32 + lane], sp[64 + lane], P, xa0, xb0, d0, k);
                ++kk;
            }
            u += s_end - s;
            s = s_end;
            if (s == uint32_t(NS)) {
                if (!(mode & 1)) flush();  // mode 1: no tile flush
                ++tile;
                s = 0;
                if (!(mode & 16)) {  // mode 16: keep the LUT planes
                    const uint4 q = *reinterpret_cast<const uint4*>(luts + ((tile * 4 + trow) & 255) * 4);
                    P = Planes8{q.x, q.y, q.z, q.w};
                }
            }
        }
        if (!(mode & 2)) flush();  // mode 2: no layer-end flush
        else if (!(mode & 32)) acc += d0[0] + d1[1];  // mode 32: no drain at all
        __syncwarp();
        issue(l + 2);
    }
    long long c1 = clock64();
    if (lane == 0) atomicAdd(reinterpret_cast<unsigned long long*>(clk), c1 - c0);
    out[blockIdx.x * blockDim.x + threadIdx.x] = part[lane] + acc;
}

// V9: V8's per-layer structure with the words streamed by LDG into a
// register queue (2 unit pairs ahead, across layer boundaries): no TMA issue,
// no mbarrier, no ring
__global__ void __launch_bounds__(1024, 1) k_layers_ldg(const uint32_t* __restrict__ g, int L, int U,
                                                        int NS, int consumers, float* out, ShiftK K,
                                                        long long* clk) {
    extern __shared__ __align__(1024) uint8_t smb[];
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint16_t* xs = reinterpret_cast<uint16_t*>(smb + 2048);
    float* part = reinterpret_cast<float*>(smb + 2048 + 64 * 256 * 2);
    uint32_t* luts = reinterpret_cast<uint32_t*>(smb + 2048 + 64 * 512 + 16 * 1024);
    for (uint32_t i = threadIdx.x; i < 64 * 256; i += blockDim.x) xs[i] = uint16_t(0x3800 + (i & 0x3ff));
    for (uint32_t i = threadIdx.x; i < 1024; i += blockDim.x) luts[i] = 0x3c3a3836u ^ i;
    __syncthreads();
    if (int(warp) >= consumers) return;
    const uint32_t* base = g + (size_t(blockIdx.x) * consumers + warp) * size_t(L) * U * 96 + lane;
    const int total = L * U;  // units in this warp's stream
    // queue: words of units n, n+1 (cur) and n+2, n+3 (nxt)
    uint32_t cur[6], nxt[6];
    auto ld = [&](int unit, uint32_t* r) {
        const uint32_t* p = base + size_t(min(unit, total - 1)) * 96;
#pragma unroll
        for (int i = 0; i < 3; ++i)
            asm volatile("ld.global.nc.L1::no_allocate.b32 %0, [%1];" : "=r"(r[i]) : "l"(p + 32 * i));
    };
    ld(0, cur); ld(1, cur + 3); ld(2, nxt); ld(3, nxt + 3);
    int qn = 0;  // stream index of cur[0..2]
    const ShiftK k = K;
    const uint32_t xoff = tile_x_offset(lane), trow = (lane >> 2) & 3u;
    long long c0 = clock64();
    for (int l = 0; l < L; ++l) {
        const uint16_t* xh = xs + (l & 3) * 4096;
        uint32_t s = (warp * U) % NS, tile = (warp * U) / NS;
        float d0[4] = {0, 0, 0, 0}, d1[4] = {0, 0, 0, 0};
        const uint4 q0 = *reinterpret_cast<const uint4*>(luts + ((tile * 4 + trow) & 255) * 4);
        Planes8 P{q0.x, q0.y, q0.z, q0.w};
        auto flush = [&]() {
            const float v = tile_rows_reduce(d0, d1, lane);
            if ((lane & 3) == 0 && lane < 16) part[warp * 256 + ((tile * 4 + trow) & 255)] += v;
#pragma unroll
            for (int z = 0; z < 4; ++z) d0[z] = d1[z] = 0.f;
        };
        // units of this layer are stream indices [l*U, (l+1)*U); pop two at a time
        int u = 0;
        while (u < U) {
            const int s_end = min(NS, int(s) + (U - u));
            int kk = s;
            const uint16_t* xp = xh + (s & 15) * 256 + xoff;
#pragma unroll 1
            for (; kk + 1 < s_end; kk += 2) {
                const uint32_t a0 = cur[0], a1 = cur[1], a2 = cur[2], b0 = cur[3], b1 = cur[4], b2 = cur[5];
#pragma unroll
                for (int z = 0; z < 6; ++z) cur[z] = nxt[z];
                qn += 2;
                ld(qn + 2, nxt); ld(qn + 3, nxt + 3);
                const uint4 xa0 = ldx(xp, 0), xb0 = ldx(xp, 128), xa1 = ldx(xp, 256), xb1 = ldx(xp, 384);
                span3_mma_one(a0, a1, a2, P, xa0, xb0, d0, k);
                span3_mma_one(b0, b1, b2, P, xa1, xb1, d1, k);
                xp = xh + (((kk + 2) & 15) * 256) + xoff;
            }
            if (kk < s_end) {  // single unit: shift the queue by one
                const uint32_t a0 = cur[0], a1 = cur[1], a2 = cur[2];
                cur[0] = cur[3]; cur[1] = cur[4]; cur[2] = cur[5];
                cur[3] = nxt[0]; cur[4] = nxt[1]; cur[5] = nxt[2];
                nxt[0] = nxt[3]; nxt[1] = nxt[4]; nxt[2] = nxt[5];
                qn += 1;
                ld(qn + 3, nxt + 3);
                const uint4 xa0 = ldx(xp, 0), xb0 = ldx(xp, 128);
                span3_mma_one(a0, a1, a2, P, xa0, xb0, d0, k);
                ++kk;
            }
            u += s_end - s;
            s = s_end;
            if (s == uint32_t(NS)) {
                flush();
                ++tile;
                s = 0;
                const uint4 q = *reinterpret_cast<const uint4*>(luts + ((tile * 4 + trow) & 255) * 4);
                P = Planes8{q.x, q.y, q.z, q.w};
            }
        }
        flush();
    }
    long long c1 = clock64();
    if (lane == 0) atomicAdd(reinterpret_cast<unsigned long long*>(clk), c1 - c0);
    out[blockIdx.x * blockDim.x + threadIdx.x] = part[lane] + float(cur[0] & 1);
}

// V10: V8 with one flat pair loop per layer -- the tile change is a rare
// uniform branch inside the loop (no segment restarts), accumulators d0/d1
// alternate by unit parity and are flushed together
__global__ void __launch_bounds__(1024, 1) k_flat(const uint32_t* __restrict__ g, int L, int U,
                                                  int NS, int consumers, float* out, ShiftK K,
                                                  long long* clk, int mode = 0) {
    extern __shared__ __align__(1024) uint8_t smb[];
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint64_t* full = reinterpret_cast<uint64_t*>(smb);
    uint16_t* xs = reinterpret_cast<uint16_t*>(smb + 2048);
    float* part = reinterpret_cast<float*>(smb + 2048 + 64 * 256 * 2);
    uint32_t* luts = reinterpret_cast<uint32_t*>(smb + 2048 + 64 * 512 + 16 * 1024);
    uint8_t* ring = smb + 2048 + 64 * 512 + 16 * 1024 + 4096;
    const uint32_t slot_bytes = ((U * 384 + 127) / 128) * 128;
    for (uint32_t i = threadIdx.x; i < 64 * 256; i += blockDim.x) xs[i] = uint16_t(0x3800 + (i & 0x3ff));
    for (uint32_t i = threadIdx.x; i < 1024; i += blockDim.x) luts[i] = 0x3c3a3836u ^ i;
    if (threadIdx.x == 0) {
        for (int i = 0; i < consumers * 2; ++i) mbar_init(&full[i], 1);
        fence_barrier_init();
    }
    __syncthreads();
    if (int(warp) >= consumers) return;
    const uint64_t pol = policy_evict_first();
    const size_t wbase = (size_t(blockIdx.x) * consumers + warp) * size_t(L) * U * 96;
    auto issue = [&](int l) {
        if (l >= L || ((mode & 4) && l >= 2)) return;
        if (lane == 0) {
            uint64_t* bar = &full[warp * 2 + (l & 1)];
            mbar_arrive_expect_tx(bar, U * 384);
            bulk_g2s(ring + size_t(warp * 2 + (l & 1)) * slot_bytes, g + wbase + size_t(l) * U * 96,
                     U * 384, bar, pol);
        }
    };
    issue(0);
    issue(1);
    const ShiftK k = K;
    const uint32_t xoff = tile_x_offset(lane), trow = (lane >> 2) & 3u;
    const uint32_t s_start = (warp * U) % NS, t_start = (warp * U) / NS;
    long long c0 = clock64();
    float d0[4] = {0, 0, 0, 0}, d1[4] = {0, 0, 0, 0};
    for (int l = 0; l < L; ++l) {
        if (!(mode & 4) || l < 2) mbar_wait(&full[warp * 2 + (l & 1)], (l >> 1) & 1u);
        const uint32_t* sp = reinterpret_cast<const uint32_t*>(ring + size_t(warp * 2 + (l & 1)) * slot_bytes) + lane;
        const uint16_t* xh = xs + (l & 3) * 4096 + xoff;
        uint32_t s = s_start, tile = t_start;
        uint4 q0 = *reinterpret_cast<const uint4*>(luts + ((tile * 4 + trow) & 255) * 4);
        Planes8 P{q0.x, q0.y, q0.z, q0.w};
        auto flush = [&]() {
            const float v = tile_rows_reduce(d0, d1, lane);
            if ((lane & 3) == 0 && lane < 16) part[warp * 256 + ((tile * 4 + trow) & 255)] += v;
#pragma unroll
            for (int z = 0; z < 4; ++z) d0[z] = d1[z] = 0.f;
        };
        auto next_tile = [&]() {
            flush();
            ++tile;
            s = 0;
            const uint4 q = *reinterpret_cast<const uint4*>(luts + ((tile * 4 + trow) & 255) * 4);
            P = Planes8{q.x, q.y, q.z, q.w};
        };
        int u = 0;
#pragma unroll 1
        for (; u + 1 < U; u += 2) {
            const uint32_t a0 = sp[0], a1 = sp[32], a2 = sp[64];
            const uint32_t b0 = sp[96], b1 = sp[128], b2 = sp[160];
            sp += 192;
            if (s == uint32_t(NS)) next_tile();
            const uint16_t* xa = xh + (s & 15) * 256;
            const uint4 xa0 = ldx(xa, 0), xb0 = ldx(xa, 128);
            span3_mma_one(a0, a1, a2, P, xa0, xb0, d0, k);
            ++s;
            if (s == uint32_t(NS)) next_tile();
            const uint16_t* xb = xh + (s & 15) * 256;
            const uint4 xa1 = ldx(xb, 0), xb1 = ldx(xb, 128);
            span3_mma_one(b0, b1, b2, P, xa1, xb1, d1, k);
            ++s;
        }
        if (u < U) {
            if (s == uint32_t(NS)) next_tile();
            const uint16_t* xa = xh + (s & 15) * 256;
            const uint4 xa0 = ldx(xa, 0), xb0 = ldx(xa, 128);
            span3_mma_one(sp[0], sp[32], sp[64], P, xa0, xb0, d0, k);
        }
        if (!(mode & 2)) flush();
        __syncwarp();
        issue(l + 2);
    }
    long long c1 = clock64();
    if (lane == 0) atomicAdd(reinterpret_cast<unsigned long long*>(clk), c1 - c0);
    out[blockIdx.x * blockDim.x + threadIdx.x] = part[lane] + d0[0] + d1[1];
}

// V11: k_flat with cross-layer software pipelining: the next layer's LUT
// planes and the current pair's words/x are always loaded one pair ahead
// (the pair loop carries the loaded operands in registers across the tile
// change and the layer boundary), so a restart never exposes the LDS latency
__global__ void __launch_bounds__(1024, 1) k_pipe(const uint32_t* __restrict__ g, int L, int U,
                                                  int NS, int consumers, float* out, ShiftK K,
                                                  long long* clk, int mode = 0) {
    extern __shared__ __align__(1024) uint8_t smb[];
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint64_t* full = reinterpret_cast<uint64_t*>(smb);
    uint16_t* xs = reinterpret_cast<uint16_t*>(smb + 2048);
    float* part = reinterpret_cast<float*>(smb + 2048 + 64 * 256 * 2);
    uint32_t* luts = reinterpret_cast<uint32_t*>(smb + 2048 + 64 * 512 + 16 * 1024);
    uint8_t* ring = smb + 2048 + 64 * 512 + 16 * 1024 + 4096;
    const uint32_t slot_bytes = ((U * 384 + 127) / 128) * 128;
    for (uint32_t i = threadIdx.x; i < 64 * 256; i += blockDim.x) xs[i] = uint16_t(0x3800 + (i & 0x3ff));
    for (uint32_t i = threadIdx.x; i < 1024; i += blockDim.x) luts[i] = 0x3c3a3836u ^ i;
    if (threadIdx.x == 0) {
        for (int i = 0; i < consumers * 2; ++i) mbar_init(&full[i], 1);
        fence_barrier_init();
    }
    __syncthreads();
    if (int(warp) >= consumers) return;
    const uint64_t pol = policy_evict_first();
    const size_t wbase = (size_t(blockIdx.x) * consumers + warp) * size_t(L) * U * 96;
    auto issue = [&](int l) {
        if (l >= L || ((mode & 4) && l >= 2)) return;
        if (lane == 0) {
            uint64_t* bar = &full[warp * 2 + (l & 1)];
            mbar_arrive_expect_tx(bar, U * 384);
            bulk_g2s(ring + size_t(warp * 2 + (l & 1)) * slot_bytes, g + wbase + size_t(l) * U * 96,
                     U * 384, bar, pol);
        }
    };
    issue(0);
    issue(1);
    const ShiftK k = K;
    const uint32_t xoff = tile_x_offset(lane), trow = (lane >> 2) & 3u;
    const uint32_t s_start = (warp * U) % NS, t_start = (warp * U) / NS;
    long long c0 = clock64();
    float d0[4] = {0, 0, 0, 0}, d1[4] = {0, 0, 0, 0};
    // unit cursor state (units of the warp's whole stream: L layers x U)
    int l = 0, u = 0;
    uint32_t s = s_start, tile = t_start;
    const uint32_t* sp = nullptr;
    const uint16_t* xh = nullptr;
    auto enter_layer = [&](int ll) {
        if (!(mode & 4) || ll < 2) mbar_wait(&full[warp * 2 + (ll & 1)], (ll >> 1) & 1u);
        sp = reinterpret_cast<const uint32_t*>(ring + size_t(warp * 2 + (ll & 1)) * slot_bytes) + lane;
        xh = xs + (ll & 3) * 4096 + xoff;
        s = s_start;
        tile = t_start;
    };
    enter_layer(0);
    uint4 q0 = *reinterpret_cast<const uint4*>(luts + ((tile * 4 + trow) & 255) * 4);
    Planes8 P{q0.x, q0.y, q0.z, q0.w};
    // operands of the next unit, loaded ahead
    uint32_t w0 = sp[0], w1 = sp[32], w2 = sp[64];
    uint4 xa = ldx(xh + (s & 15) * 256, 0), xb = ldx(xh + (s & 15) * 256, 128);
    int parity = 0;
    const int total = L * U;
    for (int n = 0; n < total; ++n) {
        const uint32_t cw0 = w0, cw1 = w1, cw2 = w2;
        const uint4 cxa = xa, cxb = xb;
        const Planes8 CP = P;
        // advance the cursor to the next unit and load its operands now
        ++u;
        ++s;
        sp += 96;
        bool flush_after = false;
        if (u == U) {  // layer end: flush after this unit, next layer
            flush_after = true;
            __syncwarp();
            issue(l + 1 + 1 - 1 + 1);  // refill the slot of layer l with layer l + 2
            ++l;
            u = 0;
            if (l < L) enter_layer(l);
        } else if (s == uint32_t(NS)) {  // tile end
            flush_after = true;
            s = 0;
            ++tile;
        }
        if (n + 1 < total) {
            w0 = sp[0]; w1 = sp[32]; w2 = sp[64];
            xa = ldx(xh + (s & 15) * 256, 0);
            xb = ldx(xh + (s & 15) * 256, 128);
            if (flush_after) {
                const uint4 q = *reinterpret_cast<const uint4*>(luts + ((tile * 4 + trow) & 255) * 4);
                P = Planes8{q.x, q.y, q.z, q.w};
            }
        }
        if (parity == 0) span3_mma_one(cw0, cw1, cw2, CP, cxa, cxb, d0, k);
        else span3_mma_one(cw0, cw1, cw2, CP, cxa, cxb, d1, k);
        parity ^= 1;
        if (flush_after && !(mode & 2)) {
            const float v = tile_rows_reduce(d0, d1, lane);
            if ((lane & 3) == 0 && lane < 16) part[warp * 256 + ((tile * 4 + trow) & 255)] += v;
#pragma unroll
            for (int z = 0; z < 4; ++z) d0[z] = d1[z] = 0.f;
        }
    }
    long long c1 = clock64();
    if (lane == 0) atomicAdd(reinterpret_cast<unsigned long long*>(clk), c1 - c0);
    out[blockIdx.x * blockDim.x + threadIdx.x] = part[lane] + d0[0] + d1[1];
}

int main(int argc, char** argv) {
    cudaDeviceProp pr;
    CK(cudaGetDeviceProperties(&pr, 0));
    const int nsm = pr.multiProcessorCount;
    float* out;
    CK(cudaMalloc(&out, size_t(nsm) * 1024 * 4));
    long long* clk;
    CK(cudaMalloc(&clk, 8));
    const ShiftK K = SQZ_SHIFTK_INIT;
    auto run = [&](auto kern, const char* name, int consumers, int idle) -> int {
        const size_t smem = size_t(consumers) * NU * 96 * 4 + NU * 256 * 2;
        CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        const int threads = (consumers + idle) * 32, niter = 400;
        kern<<<nsm, threads, smem>>>(10, out, consumers, K, clk);
        CK(cudaDeviceSynchronize());
        CK(cudaMemset(clk, 0, 8));
        kern<<<nsm, threads, smem>>>(niter, out, consumers, K, clk);
        CK(cudaDeviceSynchronize());
        long long c;
        CK(cudaMemcpy(&c, clk, 8, cudaMemcpyDeviceToHost));
        const double cyc = double(c) / nsm;  // per SM (thread 0 of each CTA)
        const double w = double(consumers) * niter * NU * 1024.0;
        printf("%-44s consumers %2d idle %d: %6.1f w/clk/SM\n", name, consumers, idle, w / cyc);
        return 0;
    };
    {
        const size_t total_units = size_t(nsm) * 16 * 2048;  // 1.86 GB of words at 16 warps
        uint32_t* g;
        CK(cudaMalloc(&g, total_units * 384));
        CK(cudaMemset(g, 0x5a, total_units * 384));
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        for (int prod = 0; prod < 1; ++prod)
        for (int c : {8})
            for (int ws : {2})
                for (int cu : {16, 14}) {
                    auto kern = prod ? k_stream_prod : k_stream;
                    const size_t smem = 2048 + 64 * 256 * 2 + size_t(c) * ws * cu * 384;
                    if (smem > 227 * 1024) continue;
                    const int per_warp = int(total_units / nsm / c);
                    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
                    kern<<<nsm, (c + prod) * 32, smem>>>(g, per_warp / 8, cu, ws, c, out, K, clk);
                    CK(cudaDeviceSynchronize());
                    CK(cudaMemset(clk, 0, 8));
                    cudaEventRecord(e0);
                    kern<<<nsm, (c + prod) * 32, smem>>>(g, per_warp, cu, ws, c, out, K, clk);
                    cudaEventRecord(e1);
                    CK(cudaDeviceSynchronize());
                    float ms;
                    cudaEventElapsedTime(&ms, e0, e1);
                    const double w = double(nsm) * c * per_warp * 1024.0;
                    printf(prod ? "V6 prod   c%2d ws %d cu %2d: %.3f ms  %6.1f w/clk/SM @1.965  %6.0f GB/s\n" : "V5 stream c%2d ws %d cu %2d: %.3f ms  %6.1f w/clk/SM @1.965  %6.0f GB/s\n", c, ws,
                           cu, ms, w / (ms * 1e-3) / nsm / 1.965e9, w * 0.375 / (ms * 1e-3) / 1e9);
                }
        auto ldg = [&](auto kern, const char* name, int c) -> int {
            const int per_warp = int(total_units / nsm / c);
            CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 512));
            kern<<<nsm, c * 32, 64 * 512>>>(g, per_warp / 8, c, out, K, clk);
            CK(cudaDeviceSynchronize());
            cudaEventRecord(e0);
            kern<<<nsm, c * 32, 64 * 512>>>(g, per_warp, c, out, K, clk);
            cudaEventRecord(e1);
            CK(cudaDeviceSynchronize());
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            const double w = double(nsm) * c * per_warp * 1024.0;
            printf("%-24s c%2d: %.3f ms  %6.1f w/clk/SM @1.965  %6.0f GB/s\n", name, c, ms,
                   w / (ms * 1e-3) / nsm / 1.965e9, w * 0.375 / (ms * 1e-3) / 1e9);
            return 0;
        };
        for (int c : {0}) {
            if (!c) break;
            ldg(k_ldg<2>, "V7 ldg D=2 pairs", c);
            ldg(k_ldg<4>, "V7 ldg D=4 pairs", c);
            ldg(k_ldg<6>, "V7 ldg D=6 pairs", c);
        }
        auto lay = [&](int c, int U, int NS, bool use_ldg = false, int mode = 0, int flat = 0) -> int {
            const int L = int(total_units / nsm / c / U);
            const size_t smem = 2048 + 64 * 512 + 16 * 1024 + 4096 + size_t(c) * 2 * (((U * 384 + 127) / 128) * 128);
            if (smem > 227 * 1024) return 0;
            CK(cudaFuncSetAttribute(k_flat, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
            CK(cudaFuncSetAttribute(k_pipe, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
            if (use_ldg) CK(cudaFuncSetAttribute(k_layers_ldg, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
            else CK(cudaFuncSetAttribute(k_layers, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
            if (flat == 2) k_pipe<<<nsm, c * 32, smem>>>(g, L / 8, U, NS, c, out, K, clk, mode);
            else if (flat) k_flat<<<nsm, c * 32, smem>>>(g, L / 8, U, NS, c, out, K, clk, mode);
            else if (use_ldg) k_layers_ldg<<<nsm, c * 32, smem>>>(g, L / 8, U, NS, c, out, K, clk);
            else k_layers<<<nsm, c * 32, smem>>>(g, L / 8, U, NS, c, out, K, clk, mode);
            CK(cudaDeviceSynchronize());
            CK(cudaMemset(clk, 0, 8));
            cudaEventRecord(e0);
            if (flat == 2) k_pipe<<<nsm, c * 32, smem>>>(g, L, U, NS, c, out, K, clk, mode);
            else if (flat) k_flat<<<nsm, c * 32, smem>>>(g, L, U, NS, c, out, K, clk, mode);
            else if (use_ldg) k_layers_ldg<<<nsm, c * 32, smem>>>(g, L, U, NS, c, out, K, clk);
            else k_layers<<<nsm, c * 32, smem>>>(g, L, U, NS, c, out, K, clk, mode);
            cudaEventRecord(e1);
            CK(cudaDeviceSynchronize());
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            const double w = double(nsm) * c * L * U * 1024.0;
            long long cyc = 0;
            CK(cudaMemcpy(&cyc, clk, 8, cudaMemcpyDeviceToHost));
            printf("[cycle-based %.1f w/clk/SM, SM clock %.0f MHz] ", w / (double(cyc) / (nsm * c)) / nsm,
                   double(cyc) / (nsm * c) / (ms * 1e-3) / 1e6);
            printf("%s mode %d ", flat == 2 ? "PIPE" : flat ? "FLAT" : "seg ", mode);
            printf(use_ldg ? "V9 ldg    c%2d U %3d NS %2d: %.3f ms  %6.1f w/clk/SM @1.965  %6.0f GB/s  %.0f ns/layer\n" : "V8 layers c%2d U %3d NS %2d: %.3f ms  %6.1f w/clk/SM @1.965  %6.0f GB/s  %.0f ns/layer\n", c, U, NS,
                   ms, w / (ms * 1e-3) / nsm / 1.965e9, w * 0.375 / (ms * 1e-3) / 1e9, ms * 1e6 / L);
            return 0;
        };
        if (argc > 1) {  // one configuration: c U NS mode flat
            lay(atoi(argv[1]), atoi(argv[2]), atoi(argv[3]), false, atoi(argv[4]), atoi(argv[5]));
            return 0;
        }
        for (int mode : {15, 15 | 32, 15 | 32 | 64}) lay(8, 14, 16, false, mode, 0);
        lay(8, 14, 1024, false, 7, 0);
        lay(8, 14, 14, false, 7, 0);
        lay(8, 14, 1024, false, 15, 0);
        for (int flat = 0; flat < 0; flat += 2) {
            for (int mode : {0, 4, 6}) lay(8, 14, 16, false, mode, flat);
            for (int mode : {0, 6}) lay(8, 28, 16, false, mode, flat);
            for (int mode : {0, 6}) lay(8, 37, 16, false, mode, flat);
            for (int mode : {0, 6}) lay(16, 7, 16, false, mode, flat);
            for (int mode : {0, 6}) lay(16, 19, 16, false, mode, flat);
        }
        lay(8, 37, 16);   // 7B 11008x4096
        lay(8, 38, 43);   // 7B 4096x11008
        lay(16, 7, 16);
        lay(16, 19, 16);
        lay(16, 16, 16);
        lay(16, 32, 16);
        lay(8, 64, 16);
        CK(cudaFree(g));
    }
    for (int c : {8, 16}) {
        run(k_loop<7>, "V0 restart every 14 units", c, 5);
        run(k_loop<8>, "V0 restart + LUT reload from smem", c, 5);
        run(k_loop<0>, "V0 span pair (kernel loop)", c, 5);
        run(k_loop<1>, "V1 span pair, pipelined loads", c, 5);
        run(k_loop<2>, "V2 4 units / iter", c, 5);
        run(k_loop<3>, "V3 2 tiles x 2 spans, x shared", c, 5);
        run(k_loop<4>, "V4 pipelined, 2 tiles x 1 span, x shared", c, 5);
    }
    return 0;
}
