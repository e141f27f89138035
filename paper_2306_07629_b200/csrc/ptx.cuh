// ptx.cuh -- PTX helpers and the LUT decode micro-kernels shared by the
// sm_100a kernels (kernels.cu: per-layer stream-K path; stack.cu: persistent
// multi-layer path).
#pragma once

#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "layout.hpp"

namespace sqz {

// ---------------------------------------------------------------------------
// PTX helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t s) {
    uint32_t r;
    asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(s));
    return r;
}
// acc + lo16(w) * lo16(x)   (fp16 x fp16 -> fp32, single FHFMA)
__device__ __forceinline__ float fma_lo(uint32_t w, uint32_t x, float acc) {
    float d;
    asm("fma.rn.f32.f16 %0, %1, %2, %3;"
        : "=f"(d)
        : "h"((unsigned short)(w & 0xffffu)), "h"((unsigned short)(x & 0xffffu)), "f"(acc));
    return d;
}
__device__ __forceinline__ float fma_hi(uint32_t w, uint32_t x, float acc) {
    float d;
    asm("fma.rn.f32.f16 %0, %1, %2, %3;"
        : "=f"(d)
        : "h"((unsigned short)(w >> 16)), "h"((unsigned short)(x >> 16)), "f"(acc));
    return d;
}
__device__ __forceinline__ float fma_h(uint16_t w, uint16_t x, float acc) {
    float d;
    asm("fma.rn.f32.f16 %0, %1, %2, %3;" : "=f"(d) : "h"(w), "h"(x), "f"(acc));
    return d;
}
__device__ __forceinline__ uint4 ldg_nc_v4(const void* p) {
    uint4 r;
    asm volatile("ld.global.nc.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}
__device__ __forceinline__ uint16_t ldg_nc_u16(const uint16_t* p) {
    uint16_t r;
    asm volatile("ld.global.nc.u16 %0, [%1];" : "=h"(r) : "l"(p));
    return r;
}
__device__ __forceinline__ float ld_cg_f32(const float* p) {
    float r;
    asm volatile("ld.global.cg.f32 %0, [%1];" : "=f"(r) : "l"(p));
    return r;
}
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_barrier_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
// raise the expected transaction count without arriving
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar, uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
        "[%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
    uint32_t done;
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return done != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    const uint32_t a = smem_u32(bar);
    uint32_t done = 0;
    do {
        // suspend-time hint: the thread sleeps in hardware until the phase
        // completes (or ~1 ms), instead of re-issuing the probe
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n"
            " selp.u32 %0, 1, 0, p;\n}"
            : "=r"(done)
            : "r"(a), "r"(parity), "r"(1000000u)
            : "memory");
    } while (!done);
}
// consumer-side wait: try_wait with the hardware's default time limit (no
// suspend hint), re-probed in a loop -- the decode warps resume as soon as
// the phase completes instead of after a suspend wake-up
__device__ __forceinline__ void mbar_wait_spin(uint64_t* bar, uint32_t parity) {
    const uint32_t a = smem_u32(bar);
    uint32_t done = 0;
    do {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
            " selp.u32 %0, 1, 0, p;\n}"
            : "=r"(done)
            : "r"(a), "r"(parity)
            : "memory");
    } while (!done);
}
// role-warp wait off the critical path: a non-blocking probe, then a plain
// nanosleep (not woken by unrelated mbarrier traffic, unlike the suspend
// hint's NANOSLEEP.SYNCS) so a long wait costs a few issue slots per
// `ns`, not a probe loop the decoding warps pay for
__device__ __forceinline__ bool mbar_test_wait(uint64_t* bar, uint32_t parity) {
    uint32_t done;
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return done != 0;
}
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity, uint32_t ns) {
    while (!mbar_test_wait(bar, parity)) __nanosleep(ns);
}
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

template <typename T>
__device__ __forceinline__ void store_y(T* y, uint32_t i, float v);
template <>
__device__ __forceinline__ void store_y<float>(float* y, uint32_t i, float v) {
    y[i] = v;
}
template <>
__device__ __forceinline__ void store_y<__half>(__half* y, uint32_t i, float v) {
    y[i] = __float2half_rn(v);
}

// ---------------------------------------------------------------------------
// LUT byte planes: entries e[0..7] fp16 -> lo/hi byte planes for PRMT lookup
// ---------------------------------------------------------------------------
struct Planes8 {
    uint32_t l0, l1, h0, h1;  // l0 = lo bytes of e0..e3, l1 = e4..e7, h* = hi bytes
};
__device__ __forceinline__ Planes8 make_planes8(uint4 q) {
    // q.x = e0 | e1<<16, q.y = e2 | e3<<16, q.z = e4|e5<<16, q.w = e6|e7<<16
    Planes8 p;
    p.l0 = prmt(q.x, q.y, 0x6420);
    p.h0 = prmt(q.x, q.y, 0x7531);
    p.l1 = prmt(q.z, q.w, 0x6420);
    p.h1 = prmt(q.z, q.w, 0x7531);
    return p;
}

// 4 weights selected by the low 4 nibbles of `sel` (bit 3 of each nibble 0)
// -> two half2 words (w0,w1), (w2,w3) -> 4 FHFMA with x pair words xa, xb
__device__ __forceinline__ void lookup4_fma(uint32_t sel, const Planes8& P, uint32_t xa,
                                            uint32_t xb, float& a0, float& a1, float& a2,
                                            float& a3) {
    const uint32_t lo = prmt(P.l0, P.l1, sel);
    const uint32_t hi = prmt(P.h0, P.h1, sel);
    const uint32_t h01 = prmt(lo, hi, 0x5140);
    const uint32_t h23 = prmt(lo, hi, 0x7362);
    a0 = fma_lo(h01, xa, a0);
    a1 = fma_hi(h01, xa, a1);
    a2 = fma_lo(h23, xb, a2);
    a3 = fma_hi(h23, xb, a3);
}

// one 3-bit unit of one lane: 32 weights, x as 4 uint4 (32 halves, column order)
__device__ __forceinline__ void unit3(uint32_t w0, uint32_t w1, uint32_t w2, const Planes8& P,
                                      const uint4 (&xv)[4], float& a0, float& a1, float& a2,
                                      float& a3) {
    const uint32_t m0 = w0 & 0x77777777u;
    const uint32_t m1 = w1 & 0x77777777u;
    const uint32_t m2 = w2 & 0x77777777u;
    const uint32_t t = ((w0 >> 3) & 0x11111111u) | ((w1 >> 2) & 0x22222222u) |
                       ((w2 >> 1) & 0x44444444u);
    const uint32_t s[4] = {m0, m1, m2, t};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        lookup4_fma(s[q], P, xv[q].x, xv[q].y, a0, a1, a2, a3);
        lookup4_fma(s[q] >> 16, P, xv[q].z, xv[q].w, a0, a1, a2, a3);
    }
}

struct Planes16 {
    Planes8 a, b;  // entries 0..7 and 8..15
};

// 4-bit: nibble n = idx (4 bits); lookups in both half tables, pick by bit 3
__device__ __forceinline__ void lookup4_fma16(uint32_t sel, uint32_t pick, const Planes16& P,
                                              uint32_t xa, uint32_t xb, float& a0, float& a1,
                                              float& a2, float& a3) {
    const uint32_t loA = prmt(P.a.l0, P.a.l1, sel);
    const uint32_t loB = prmt(P.b.l0, P.b.l1, sel);
    const uint32_t hiA = prmt(P.a.h0, P.a.h1, sel);
    const uint32_t hiB = prmt(P.b.h0, P.b.h1, sel);
    const uint32_t lo = prmt(loA, loB, pick);
    const uint32_t hi = prmt(hiA, hiB, pick);
    const uint32_t h01 = prmt(lo, hi, 0x5140);
    const uint32_t h23 = prmt(lo, hi, 0x7362);
    a0 = fma_lo(h01, xa, a0);
    a1 = fma_hi(h01, xa, a1);
    a2 = fma_lo(h23, xb, a2);
    a3 = fma_hi(h23, xb, a3);
}

__device__ __forceinline__ void unit4(const uint32_t (&w)[4], const Planes16& P,
                                      const uint4 (&xv)[4], float& a0, float& a1, float& a2,
                                      float& a3) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const uint32_t sl = w[q] & 0x77777777u;
        const uint32_t pk = ((w[q] >> 1) & 0x44444444u) | 0x32103210u;
        lookup4_fma16(sl, pk, P, xv[q].x, xv[q].y, a0, a1, a2, a3);
        lookup4_fma16(sl >> 16, pk >> 16, P, xv[q].z, xv[q].w, a0, a1, a2, a3);
    }
}

// generic width (1..8): little-endian 32*bits-bit stream, LUT from global (L1)
template <int BITS>
__device__ __forceinline__ void unit_generic(const uint32_t (&w)[8], const uint16_t* lut_row,
                                             const uint4 (&xv)[4], float& a0, float& a1) {
    const uint16_t* xh = reinterpret_cast<const uint16_t*>(&xv[0]);
#pragma unroll
    for (int j = 0; j < 32; ++j) {
        const int bp = j * BITS;
        const int wi = bp >> 5, off = bp & 31;
        uint32_t v = w[wi] >> off;
        if (off + BITS > 32) v |= w[wi + 1] << (32 - off);
        const uint32_t idx = v & ((1u << BITS) - 1u);
        const uint16_t c = ldg_nc_u16(lut_row + idx);
        if (j & 1)
            a1 = fma_h(c, xh[j], a1);
        else
            a0 = fma_h(c, xh[j], a0);
    }
}

// load x halves [g*32, g*32+32) as 4 uint4; zero beyond cols
__device__ __forceinline__ void load_x(const uint16_t* x, uint32_t g, uint32_t cols,
                                       uint4 (&xv)[4]) {
    const uint32_t c0 = g * kGroupCols;
    if (c0 + kGroupCols <= cols) {
        const uint4* p = reinterpret_cast<const uint4*>(x + c0);
#pragma unroll
        for (int q = 0; q < 4; ++q) xv[q] = ldg_nc_v4(p + q);
    } else {
        uint16_t h[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) h[j] = (c0 + j < cols) ? ldg_nc_u16(x + c0 + j) : 0;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            xv[q].x = h[8 * q + 0] | (uint32_t(h[8 * q + 1]) << 16);
            xv[q].y = h[8 * q + 2] | (uint32_t(h[8 * q + 3]) << 16);
            xv[q].z = h[8 * q + 4] | (uint32_t(h[8 * q + 5]) << 16);
            xv[q].w = h[8 * q + 6] | (uint32_t(h[8 * q + 7]) << 16);
        }
    }
}


// bulk copy without a cache-policy operand
__device__ __forceinline__ void bulk_g2s_plain(void* dst, const void* src, uint32_t bytes,
                                               uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
            "r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
// order this thread's prior generic-proxy global accesses (incl. an acquire)
// before subsequent async-proxy (TMA) accesses
__device__ __forceinline__ void fence_proxy_async_global() {
    asm volatile("fence.proxy.async.global;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_gpu(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void red_release_gpu_add(uint32_t* p, uint32_t v) {
    asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// peer-memory words (64-bit single-copy atomic, not cached in L1)
__device__ __forceinline__ void st_volatile_u64(unsigned long long* p, unsigned long long v) {
    asm volatile("st.volatile.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_volatile_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.volatile.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
// system scope (peers over NVLink): release add / acquire load
__device__ __forceinline__ void red_release_sys_add(uint32_t* p, uint32_t v) {
    asm volatile("red.release.sys.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_gpu(uint32_t* p, uint32_t v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// uncached 16-byte load (host memory rewritten between steps); no compiler
// memory barrier, so a batch of them stays in flight together
__device__ __forceinline__ uint4 ld_volatile_v4(const uint4* p) {
    uint4 r;
    asm volatile("ld.volatile.global.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}
__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint4 ld_cg_v4(const void* p) {
    uint4 r;
    asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}
__device__ __forceinline__ uint16_t ld_cg_u16(const uint16_t* p) {
    uint16_t r;
    asm volatile("ld.global.cg.u16 %0, [%1];" : "=h"(r) : "l"(p));
    return r;
}
// named barrier among a subset of warps; the non-.aligned form, so the
// warps may reach it from different code paths / convergence states
__device__ __forceinline__ void named_bar_sync(uint32_t id, uint32_t threads) {
    asm volatile("barrier.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}

}  // namespace sqz
