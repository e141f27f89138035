// stack.cu -- K7: persistent multi-layer Dense-and-Sparse LUT-GEMV (sm_100a).
//
// One CTA per SM, all co-resident.  For every layer l of the stack each CTA
// owns a contiguous range of 4-row tiles (tiles split evenly over the grid, so
// the balance granularity is one tile and no output row is ever shared
// between CTAs -> no global merge, no floating-point atomics).
//
// Warp roles:
//   consumers 0..NC-1: each owns a contiguous range of the CTA's (tile,
//              256-column span) units of every layer and streams it through a
//              private 2-slot TMA ring (cp.async.bulk, mbarrier completion)
//              that runs ahead across layer boundaries (weights never depend
//              on x).  Per unit a lane decodes 32 indices of one tile row with
//              PRMT byte-plane lookups into fp16 A fragments and 4
//              mma.sync.m16n8k16 accumulate them against x in fp32 (tile.cuh);
//              on a tile change the D fragments collapse to the tile's 4 row
//              partials in the warp's column of a [warp][row] smem table.
//   publisher (NC): copies each layer's descriptor (+ the CTA's tile share
//              and CSR range) into an 8-slot shared-memory cache.
//   loader    (NC+1): stages the CTA's LUT planes, CSR slice (row_ptr,
//              entries, row-start bitmap) and, once the layer producing x is
//              complete on ALL CTAs (grid-wide completion counter,
//              ld.acquire), the activation vector(s) x -- all by TMA into
//              double-buffered shared memory.
//   finisher  (NC+2) and CSR warps (NC+3 ..): the CSR warps scan the CTA's
//              deltas (segmented warp scans, host-built row-start bitmap)
//              while the consumers decode; then all of them finish rows: the
//              dense partials in warp order plus the row's CSR round results
//              in round order (deterministic), the store of y (or the TP
//              exchange), and the layer's completion signal (red.release).
// Reference semantics: per row, LUT dot + CSR delta dot == fused_dns_matvec
// (reference kernels.cpp:108-141); the hybrid split is unnecessary because the
// CSR rounds are balanced regardless of per-row skew.
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdint>

#include "layout.hpp"
#include "ptx.cuh"
#include "stack.hpp"
#include "tile.cuh"

namespace sqz {

// Shared-memory descriptor cache: the producer (the role furthest ahead)
// copies layer l's descriptor + this CTA's CSR entry range into slot l % 8;
// the other roles wait on dfull and release the slot through dempty when they
// are done with the layer.  Descriptors of long stacks live in global memory,
// and re-reading them per field from every warp is slow.
constexpr uint32_t kDescSlots = 8;
// ring slots per consumer warp: p.n_slots / consumers (host plan, 2..kMaxWarpSlots)
// CSR warps: p.csr_warps (1..kCsrWarps) process the CSR deltas -- chosen per
// plan from the largest per-CTA entry count (each extra role warp costs the
// decoding warps issue slots, so light outlier loads get fewer)
constexpr uint32_t kCsrWarps = 4;
struct __align__(16) SDesc {
    StackLayerDesc d;
    uint32_t e0, e1;  // CSR entries of this CTA's rows: [e0, e1)
    uint32_t t0, nt;  // this CTA's tiles [t0, t0 + nt)
};
static_assert(sizeof(SDesc) == 128, "descriptor slot is one 128-byte line");

__device__ __forceinline__ const StackLayerDesc& layer_desc(const StackParams& p, uint32_t l) {
    return l < kInlineLayers && p.n_layers <= kInlineLayers ? p.inl[l] : p.layers[l];
}

// layer l's x in shared memory: p.x_step != 0 -> a region of x_step bytes
// with even layers at its bottom and odd layers at its top (the host sizes it
// for the largest pair of consecutive layers, so layer l's x never overlaps
// layer l-1's; it may overlap l-2's, whose readers the loader waits for
// through bempty, as with two fixed buffers); 0 -> one shared buffer.  Each
// of the NB vectors takes ns * 256 halves.
__device__ __forceinline__ uint32_t x_region(const StackParams& p, uint32_t l, uint32_t ns) {
    return (p.x_step && (l & 1u)) ? p.x_step - ns * kSpanCols * 2u * p.nbatch : 0u;
}

// CTA tile share from the host-precomputed quotient/remainder (no division)
struct Share {
    uint32_t t0, nt;       // first tile, tiles
    uint32_t r0, nrows;    // real rows [r0, r0 + nrows) (tiles clipped to the layer)
};
__device__ __forceinline__ Share cta_share(const StackLayerDesc& d, uint32_t cta) {
    Share s;
    const bool hi = cta < d.tr;
    s.t0 = cta * d.tq + (hi ? cta : d.tr);
    s.nt = d.tq + (hi ? 1u : 0u);
    s.r0 = min(s.t0 * kTileRows, d.rows);
    s.nrows = min((s.t0 + s.nt) * kTileRows, d.rows) - s.r0;
    return s;
}

// dev-only experiment switches (StackParams::dbg bits 1 / 8 skip the decode
// math / the weight loads): compiled in only with -DDSQ_STACK_DEV (the
// variant-lib / profile builds), so the product library can never skip work
#ifdef DSQ_MULTI_SIGNAL  // dev comparison: one release per finishing warp
constexpr bool kOneSignal = false;
#else
constexpr bool kOneSignal = true;
#endif
#if defined(DSQ_STACK_DEV) || defined(DSQ_STACK_PROFILE)
constexpr bool kDevSwitches = true;
#else
constexpr bool kDevSwitches = false;
#endif

__device__ __forceinline__ unsigned long long gtimer_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

#ifdef DSQ_STACK_WATCHDOG
// debug build (make watchdog-lib): every mbarrier wait and dependency poll of
// the stack kernel gives up after ~2 s with the waiting site printed, so a
// protocol deadlock turns into a trap with a location instead of a hung GPU
__device__ __noinline__ void mbar_wait_wd(uint64_t* bar, uint32_t parity, int line) {
    const unsigned long long t0 = gtimer_ns();
    while (!mbar_try_wait(bar, parity)) {
        if (gtimer_ns() - t0 > 2000000000ull) {
            if ((threadIdx.x & 31) == 0)
                printf("stack watchdog: cta %u warp %u line %d parity %u\n", blockIdx.x,
                       threadIdx.x >> 5, line, parity);
            __trap();
        }
    }
}
#define mbar_wait(bar, parity) mbar_wait_wd(bar, parity, __LINE__)
#define mbar_wait_cons(bar, parity) mbar_wait_wd(bar, parity, __LINE__)
#define mbar_wait_edge(bar, parity) mbar_wait_wd(bar, parity, __LINE__)
#define mbar_wait_role(bar, parity, ns) mbar_wait_wd(bar, parity, __LINE__)
#define mbar_wait_fin(bar, parity) mbar_wait_wd(bar, parity, __LINE__)
#define DSQ_WD_POLL(cond, ...)                                \
    do {                                                      \
        const unsigned long long wd0_ = gtimer_ns();          \
        while (cond) {                                        \
            if (gtimer_ns() - wd0_ > 2000000000ull) {         \
                printf(__VA_ARGS__);                          \
                __trap();                                     \
            }                                                 \
            __nanosleep(20);                                  \
        }                                                     \
    } while (0)
#else
// decode warps: the suspend-hint wait (DSQ_CONS_SPIN: plain try_wait spin,
// measured neutral)
#ifdef DSQ_CONS_SPIN
#define mbar_wait_cons(bar, parity) mbar_wait_spin(bar, parity)
#else
#define mbar_wait_cons(bar, parity) mbar_wait(bar, parity)
#endif
// decode warps at a layer start (x staged, partial buffer free): the
// suspend-hint wait, or with DSQ_EDGE_SLEEP=ns a probe + plain nanosleep
#ifndef DSQ_EDGE_SLEEP
#define DSQ_EDGE_SLEEP 0
#endif
#define mbar_wait_edge(bar, parity)                                         \
    do {                                                                    \
        if (DSQ_EDGE_SLEEP) mbar_wait_sleep(bar, parity, DSQ_EDGE_SLEEP);    \
        else mbar_wait(bar, parity);                                        \
    } while (0)
// role-warp waits (publisher / loader: off the critical path; finishing and
// CSR warps: DSQ_FIN_SLEEP ns, 0 = the suspend-hint wait)
#ifndef DSQ_ROLE_SLEEP
#define DSQ_ROLE_SLEEP 1
#endif
#ifndef DSQ_FIN_SLEEP
#define DSQ_FIN_SLEEP 0
#endif
#define mbar_wait_role(bar, parity, ns)                                     \
    do {                                                                    \
        if (DSQ_ROLE_SLEEP) mbar_wait_sleep(bar, parity, (ns));             \
        else mbar_wait(bar, parity);                                        \
    } while (0)
#define mbar_wait_fin(bar, parity)                                          \
    do {                                                                    \
        if (DSQ_FIN_SLEEP) mbar_wait_sleep(bar, parity, DSQ_FIN_SLEEP);      \
        else mbar_wait(bar, parity);                                        \
    } while (0)
#define DSQ_WD_POLL(cond, ...)          \
    do {                                \
        while (cond) __nanosleep(20);   \
    } while (0)
#endif
#define DSQ_TRACE(l, slot)                                                                 \
    do {                                                                                   \
        if (p.trace && !(p.dbg & 4u))                                                      \
            p.trace[(size_t(blockIdx.x) * p.n_layers + (l)) * kTrSlots + (slot)] = gtimer_ns(); \
    } while (0)

// CSR deltas of the CTA's rows.  The entries [e0, e1) are addressed by
// position p = q - ea (ea = e0 rounded down to 4, so every lane's 4-entry
// chunk is one aligned 16-byte load).  A round is 128 positions: lane L takes
// positions 4L..4L+3, forms the products and their running sums restarted at
// row starts (hb: host-built bitmap, bit q set <=> entry q begins a row), and
// one segmented warp scan over the lanes' open tails carries rows across
// lanes.  Result: S[p] = sum of entry p's row's products from max(row start,
// round start) through p -- the finishers read S at each row's last position
// in every round the row touches.  Positions outside [e0, e1) count 0.
__device__ __forceinline__ void csr_stream(uint32_t ea, uint32_t e0, uint32_t e1,
                                           const uint32_t* ent, const uint32_t* hb,
                                           uint32_t hbase, uint32_t hlast, const uint16_t* xh,
                                           float* S, uint32_t first, uint32_t stride,
                                           uint32_t lane) {
    const uint32_t np = e1 - ea;
    const uint32_t rounds = (np + 127) / 128;
    for (uint32_t j = first; j < rounds; j += stride) {
        const uint32_t p0 = j * 128 + 4 * lane;
        const uint32_t g = ea + p0;  // global entry index of position p0
        float v[4] = {0.f, 0.f, 0.f, 0.f};
        uint32_t hbits = 0;
        if (p0 < np) {
            const uint4 e4 = *reinterpret_cast<const uint4*>(ent + p0);
            const uint32_t es[4] = {e4.x, e4.y, e4.z, e4.w};
#pragma unroll
            for (int m = 0; m < 4; ++m)
                if (g + m >= e0 && g + m < e1)
                    v[m] = fma_h(uint16_t(es[m] >> 16), xh[es[m] & 0xffffu], 0.f);
            const uint32_t wi = min((g >> 5) - hbase, hlast);
            hbits = (__funnelshift_r(hb[wi], hb[wi + 1], g & 31u)) & 0xfu;
        }
        // running sums inside the chunk, restarted at row starts
        float c[4];
        c[0] = v[0];
#pragma unroll
        for (int m = 1; m < 4; ++m) c[m] = ((hbits >> m) & 1u) ? v[m] : c[m - 1] + v[m];
        // segmented inclusive scan of the open tails across lanes
        const uint32_t starts = __ballot_sync(0xffffffffu, hbits != 0);
        const uint32_t upto = starts & (0xffffffffu >> (31 - lane));
        const uint32_t seg0 = upto ? (31u - __clz(upto)) : 0u;
        float incl = c[3];
#pragma unroll
        for (uint32_t off = 1; off < 32; off <<= 1) {
            const float t = __shfl_up_sync(0xffffffffu, incl, off);
            if (lane >= seg0 + off) incl += t;
        }
        float excl = __shfl_up_sync(0xffffffffu, incl, 1);
        if (lane == 0) excl = 0.f;
        // positions before this lane's first row start continue the open row
        const uint32_t first_head = hbits ? uint32_t(__ffs(hbits) - 1) : 4u;
        float4 o;
        o.x = c[0] + (0 < first_head ? excl : 0.f);
        o.y = c[1] + (1 < first_head ? excl : 0.f);
        o.z = c[2] + (2 < first_head ? excl : 0.f);
        o.w = c[3] + (3 < first_head ? excl : 0.f);
        if (p0 < np) *reinterpret_cast<float4*>(S + p0) = o;
    }
}

// SERVE: the serving-loop variant (gates / notify, StackParams::serve_*)
template <int BITS, int NC, int NB, bool SERVE = false>
__global__ void __launch_bounds__((NC + 3 + kCsrWarps) * 32, 1)
    stack_gemv(const __grid_constant__ StackParams p) {
    constexpr uint32_t LW = BITS == 3 ? 4u : 8u;   // LUT words per tile row
    constexpr uint32_t UW = BITS * 32u;             // words per (tile, span) unit
    extern __shared__ __align__(1024) uint8_t sm[];
    // mbarriers: per-warp ring slots, then per buffer parity b in {0,1}
    const uint32_t WS = p.n_slots / NC;
    uint64_t* full = reinterpret_cast<uint64_t*>(sm);  // [NC][WS] unit chunk landed
    uint64_t* xfull = full + NC * WS;      // x + LUT planes staged (TMA transaction count)
    uint64_t* cfull = xfull + 2;           // CSR slice staged (TMA transaction count)
    uint64_t* bempty = cfull + 2;          // x / LUT / CSR buffers free (consumers + finisher)
    uint64_t* pfull = bempty + 2;          // dense partials written (consumers)
    uint64_t* pempty = pfull + 2;          // partials consumed (finisher)
    uint64_t* dfull = pempty + 2;          // descriptor slot written (32 producer lanes)
    uint64_t* dempty = dfull + kDescSlots; // descriptor slot released (consumers, loader, finisher)
    SDesc* sdesc = reinterpret_cast<SDesc*>(sm + p.off_desc);
    uint8_t* ring = sm + p.off_ring;
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t cta = blockIdx.x, G = p.grid;
    // completion signals per CTA and layer (the dependency target is G x this)
    const uint32_t sig_per_cta = kOneSignal ? 1u : 1u + p.csr_warps;

    if (threadIdx.x == 0) {
        for (uint32_t s = 0; s < NC * WS; ++s) mbar_init(&full[s], 1);
        for (int b = 0; b < 2; ++b) {
            mbar_init(&xfull[b], 1);
            mbar_init(&cfull[b], 1);
            mbar_init(&bempty[b], NC + 1 + p.csr_warps);
            mbar_init(&pfull[b], NC + p.csr_warps);
            mbar_init(&pempty[b], 1 + p.csr_warps);
        }
        for (uint32_t k = 0; k < kDescSlots; ++k) {
            mbar_init(&dfull[k], 32);
            mbar_init(&dempty[k], NC + 2 + p.csr_warps);
        }
        fence_barrier_init();
    }
    // the partial tables start at zero; the finisher re-zeroes what it reads
    {
        float* part = reinterpret_cast<float*>(sm + p.off_part);
        for (uint32_t i = threadIdx.x; i < p.nbuf * NB * NC * p.part_rows; i += blockDim.x) part[i] = 0.f;
    }
    __syncthreads();

    auto desc_wait = [&](uint32_t l) -> const SDesc& {
        mbar_wait(&dfull[l % kDescSlots], (l / kDescSlots) & 1u);
        return sdesc[l % kDescSlots];
    };
    auto desc_release = [&](uint32_t l) {
        if (lane == 0) mbar_arrive(&dempty[l % kDescSlots]);
    };

    if (warp == NC) {
        // ---------------- publisher: layer descriptors into the smem cache ----
        pdl_trigger();
        for (uint32_t l = 0; l < p.n_layers; ++l) {
            const uint32_t k = l % kDescSlots;
            if (l >= kDescSlots) mbar_wait_role(&dempty[k], ((l / kDescSlots) - 1) & 1u, 2000);
            const StackLayerDesc& gd = layer_desc(p, l);
            uint32_t* dst = reinterpret_cast<uint32_t*>(&sdesc[k]);
            constexpr uint32_t kDW = sizeof(StackLayerDesc) / 4;
            if (lane < kDW) {
                dst[lane] = reinterpret_cast<const uint32_t*>(&gd)[lane];
            } else if (lane < kDW + 2) {
                dst[lane] = gd.csr_rng[2 * cta + (lane - kDW)];
            } else if (lane < kDW + 4) {
                const Share sh = cta_share(gd, cta);
                dst[lane] = lane == kDW + 2 ? sh.t0 : sh.nt;
            }
            mbar_arrive(&dfull[k]);
            __syncwarp();
        }
        return;
    }

    if (warp == NC + 1) {
        // ---------------- loader: LUT planes, CSR slice, x (the dependency) ---
        // layer 0's LUT planes are launch constants and go before the PDL
        // wait; x (possibly the previous kernel's output) goes after it
        pdl_trigger();
        uint32_t fed = 0;  // served stacks: the last step whose x CTA 0 copied in
        for (uint32_t l = 0; l < p.n_layers; ++l) {
            const uint32_t b = l & 1u;
            if (l >= 2) mbar_wait_role(&bempty[b], ((l >> 1) - 1) & 1u, 500);
            mbar_wait_role(&dfull[l % kDescSlots], (l / kDescSlots) & 1u, 200);
            const SDesc& sd = sdesc[l % kDescSlots];
            const StackLayerDesc& d = sd.d;
            const Share sh = cta_share(d, cta);
            const uint32_t r0 = sh.r0, r1 = sh.r0 + sh.nrows;
            uint8_t* xb = sm + p.off_x + x_region(p, l, d.ns);
            const uint32_t xvl = d.ns * kSpanCols;  // halves per vector
            if (lane == 0) {
                DSQ_TRACE(l, kTrLoaderStart);
                // the CTA's LUT planes ride on the x barrier (expected first,
                // so the phase cannot complete before x is staged too)
                const uint32_t lb = sh.nt * kTileRows * LW * 4;
                if (lb) {
                    mbar_expect_tx(&xfull[b], lb);
                    bulk_g2s_plain(sm + p.off_lut + b * p.lut_bytes,
                                   d.lut + size_t(sh.t0) * kTileRows * LW, lb, &xfull[b]);
                }
            }
            // x: one TMA bulk copy of the 16-byte-aligned body (+ scalar tail,
            // zero padding to the span count), completion on xfull[b]
            auto stage_x = [&]() {
                const uint32_t body = (d.cols / 8) * 16;  // bytes
                const uint32_t nv = NB == 1 ? 1u : p.nvec;
                // a chained layer's x vectors are its producer's y vectors
                const uint32_t xstride = d.dep == kNoDep ? p.x_bstride : p.y_bstride;
                // vectors past nvec are not staged: their B columns and
                // accumulators are separate from the real vectors' and their
                // results are never stored, so stale data there is harmless
#pragma unroll
                for (int v = 0; v < NB; ++v) {  // batch vector v at xb + v * xvec halves
                    if (uint32_t(v) >= nv) continue;
                    uint16_t* xv = reinterpret_cast<uint16_t*>(xb) + v * xvl;
                    const uint16_t* gx = d.x + size_t(v) * xstride;
                    for (uint32_t i = body / 2 + lane; i < d.ns * kSpanCols; i += 32)
                        xv[i] = i < d.cols ? ld_cg_u16(gx + i) : uint16_t(0);
                }
                __syncwarp();
                if (lane == 0) {
                    fence_proxy_async_global();
                    mbar_arrive_expect_tx(&xfull[b], nv * body);
                    if (body)
#pragma unroll
                        for (int v = 0; v < NB; ++v)
                            if (uint32_t(v) < nv)
                                bulk_g2s_plain(reinterpret_cast<uint16_t*>(xb) + v * xvl,
                                               d.x + size_t(v) * xstride, body, &xfull[b]);
                }
            };
            // one shared x buffer (large batched stacks, p.x_step == 0): layer
            // l may overwrite x only after every reader of layer l-1's x is done
            if (p.x_step == 0 && l >= 1) mbar_wait(&bempty[(l - 1) & 1u], ((l - 1) >> 1) & 1u);
            if (l == 0) pdl_wait();
            // served stacks: an external input of step k waits for the host's doorbell
            const uint32_t gate = SERVE ? p.serve_gate[l] : 0u;
            if (d.dep == kNoDep && !gate) stage_x();  // external input: no wait at all
            // row_ptr slice + CSR entries + row-start bitmap of the CTA's rows:
            // TMA bulk copies (16-byte granules; the device arrays are padded),
            // sized from the host-precomputed per-CTA entry range
            if (lane == 0) {
                const uint32_t e0 = sd.e0, e1 = sd.e1;
                // (r0 is a multiple of 4 -> 16-byte aligned, except for CTAs
                // past the last tile, which own no rows and copy nothing)
                const uint32_t rp_bytes = r1 > r0 ? (((r1 - r0 + 1) * 4 + 15) & ~15u) : 0u;
                const uint32_t ea = e0 & ~3u;
                const uint32_t c_bytes =
                    (e1 > e0 && e1 - e0 <= p.csr_cap - 4) ? (((e1 - ea) * 4 + 15) & ~15u) : 0u;
                const uint32_t hw0 = (e0 >> 5) & ~3u;
                const uint32_t h_bytes = c_bytes ? ((((e1 >> 5) + 2 - hw0) * 4 + 15) & ~15u) : 0u;
                uint32_t* rp = reinterpret_cast<uint32_t*>(sm + p.off_rp) + b * p.rp_words;
                uint32_t* cb = reinterpret_cast<uint32_t*>(sm + p.off_csr) + b * p.csr_cap;
                uint32_t* hb = reinterpret_cast<uint32_t*>(sm + p.off_hb) + b * p.hb_words;
                mbar_arrive_expect_tx(&cfull[b], rp_bytes + c_bytes + h_bytes);
                if (rp_bytes) bulk_g2s_plain(rp, d.row_ptr + r0, rp_bytes, &cfull[b]);
                if (c_bytes) {
                    bulk_g2s_plain(cb, d.csr + ea, c_bytes, &cfull[b]);
                    bulk_g2s_plain(hb, d.csr_heads + hw0, h_bytes, &cfull[b]);
                }
                DSQ_TRACE(l, kTrCsrStaged);
            }
            if (gate) {
                // CTA 0 feeds step `gate`'s x (host doorbell -> PCIe copy ->
                // device flag); everyone else waits for the flag
                const uint32_t* wait_on = cta == 0 ? p.doorbell : p.serve_flag;
                // no timeout: an idle server may wait any time for its next
                // step, and computing on a stale x is never right -- only the
                // host's doorbell (serve_step) or serve_end's release
                // (0xffffffff: the steps not fed, results discarded) ends it
                if (lane == 0 && !(cta == 0 && fed >= gate)) {
                    while ((cta == 0 ? ld_acquire_sys(wait_on) : ld_acquire_gpu(wait_on)) < gate)
                        if (cta != 0) __nanosleep(32);  // CTA 0's polls cross PCIe anyway
                }
                __syncwarp();
                if (cta == 0 && fed < gate) {
                    // 16 loads in flight per lane: one PCIe round trip per 8 KB
                    const uint32_t n16 = p.serve_x_bytes / 16;
                    for (uint32_t i0 = 0; i0 < n16; i0 += 32 * 16) {
                        uint4 v[16];
#pragma unroll
                        for (int u = 0; u < 16; ++u) {
                            const uint32_t i = i0 + 32 * u + lane;
                            if (i < n16) v[u] = ld_volatile_v4(p.serve_x_src + i);
                        }
#pragma unroll
                        for (int u = 0; u < 16; ++u) {
                            const uint32_t i = i0 + 32 * u + lane;
                            if (i < n16) p.serve_x_dst[i] = v[u];
                        }
                    }
                    __syncwarp();
                    if (lane == 0) {
                        __threadfence();
                        st_release_gpu(p.serve_flag, gate);
                    }
                    fed = gate;
                }
                __syncwarp();
                stage_x();
            }
            if (d.dep != kNoDep) {
                if (lane == 0) {
                    DSQ_WD_POLL(ld_acquire_gpu(p.counters + d.dep) < G * sig_per_cta,
                                "stack watchdog: cta %u layer %u dep %u counter %u\n", cta, l, d.dep,
                                *(volatile const uint32_t*)(p.counters + d.dep));
                    DSQ_TRACE(l, kTrDepMet);
                }
                __syncwarp();
                stage_x();
            }
            if (lane == 0) DSQ_TRACE(l, kTrXIssued);
            __syncwarp();
            desc_release(l);
        }
        return;
    }

    // ---- finishing (finisher warp + the CSR warps, kFin warps): rows
    // i = 32*f + lane (mod 32*kFin) of the layer get their dense partials in
    // warp order (warps that did not touch a row left 0) plus their CSR
    // rounds in round order, y is stored, and each finishing warp bumps the
    // layer's completion counter (target grid * kFin)
    const uint32_t kFin = 1 + p.csr_warps;
    auto finish_rows = [&](uint32_t l, uint32_t f) {
        const uint32_t b = l & 1u, ph = (l >> 1) & 1u;
        const SDesc& sd = sdesc[l % kDescSlots];
        const StackLayerDesc& d = sd.d;
        const Share sh = cta_share(d, cta);
        const uint32_t r0 = sh.r0, nrows = sh.nrows;
        const uint32_t* rp = reinterpret_cast<const uint32_t*>(sm + p.off_rp) + b * p.rp_words;
        mbar_wait_fin(&pfull[b], ph);
        if (f == 0 && lane == 0) DSQ_TRACE(l, kTrAllDense);
        // the CSR scan results (position-indexed, see csr_stream)
        const uint32_t ea = sd.e0 & ~3u;
        const bool staged_csr = sd.e1 - sd.e0 <= p.csr_cap - 4;
        const float* S = staged_csr
                             ? reinterpret_cast<const float*>(sm + p.off_seg) + size_t(b) * NB * p.seg_cap
                             : p.gseg + (size_t(cta) * 2 + b) * NB * p.gseg_cap;
        const uint32_t s_vec = staged_csr ? p.seg_cap : p.gseg_cap;  // between batch vectors
        float* part = reinterpret_cast<float*>(sm + p.off_part) + size_t(b) * NB * p.part_rows * NC;
        const bool tp = d.reduce_ord != kNoDep;
        const uint32_t par = tp ? (p.tp_base + d.reduce_ord) & 1u : 0u;
        for (uint32_t i = 32 * f + lane; i < sh.nt * kTileRows; i += 32 * kFin) {
            float s = 0.f;
#pragma unroll
            for (uint32_t w = 0; w < NC; ++w) {
                s += part[w * p.part_rows + i];
                part[w * p.part_rows + i] = 0.f;
            }
            float sv[NB > 1 ? NB - 1 : 1];  // batch vectors 1.. (NB > 1)
#pragma unroll
            for (int v = 1; v < NB; ++v) {
                float* pv = part + v * NC * p.part_rows;
                float t = 0.f;
#pragma unroll
                for (uint32_t w = 0; w < NC; ++w) {
                    t += pv[w * p.part_rows + i];
                    pv[w * p.part_rows + i] = 0.f;
                }
                sv[v - 1] = t;
            }
            const bool valid = i < nrows;  // else a padding row of the last tile
            const uint32_t a = valid ? rp[i] - ea : 0u, e = valid ? rp[i + 1] - ea : 0u;
            for (uint32_t j = a / 128; e > a && j <= (e - 1) / 128; ++j) {
                const uint32_t q = j * 128 + min(e - 1 - j * 128, 127u);
                s += S[q];
#pragma unroll
                for (int v = 1; v < NB; ++v) sv[v - 1] += S[v * s_vec + q];
            }
            if (SERVE && p.serve_y_words && p.serve_notify[l]) {
                // served output: rows 2j / 2j+1 sit in lanes 2m / 2m+1 (r0 is a
                // multiple of 4, the row stride 32 * kFin even), both live or
                // both past the loop end
                const unsigned long long tag = static_cast<unsigned long long>(p.serve_notify[l]) << 32;
                if (d.y_f16) {
                    const uint32_t h = valid ? uint32_t(__half_as_ushort(__float2half_rn(s))) : 0u;
                    const uint32_t h1 = __shfl_down_sync(__activemask(), h, 1);
                    const uint32_t w = (r0 + i) >> 1;
                    if (valid && !(lane & 1u) && w < p.serve_y_words)
                        st_volatile_u64(p.serve_y_ll + w, tag | (h1 << 16) | h);
                } else if (valid && r0 + i < p.serve_y_words) {  // fp32: one row per word
                    st_volatile_u64(p.serve_y_ll + r0 + i, tag | __float_as_uint(s));
                }
            }
            if (!valid) continue;
#pragma unroll
            for (int v = 1; v < NB; ++v) {
                if (uint32_t(v) >= p.nvec) continue;
                if (d.y_f16)
                    static_cast<__half*>(d.y)[v * p.y_bstride + r0 + i] = __float2half_rn(sv[v - 1]);
                else
                    static_cast<float*>(d.y)[v * p.y_bstride + r0 + i] = sv[v - 1];
            }
            if (tp) {
                // a partial sum: hand it to every rank (own included) at slot
                // [parity][this rank][row] as one 64-bit word {value, tag} --
                // single-copy atomic, so no fence or separate flag is needed
                // (the receiver polls the tag, NCCL's LL protocol idea)
                const unsigned long long word =
                    (static_cast<unsigned long long>(p.tp_base + d.reduce_ord + 1) << 32) |
                    __float_as_uint(s);
                for (uint32_t k = 0; k < p.tp_world; ++k)
                    st_volatile_u64(p.tp_peer_recv[k] +
                                        (size_t(par) * p.tp_world + p.tp_rank) * p.tp_max_rows + r0 + i,
                                    word);
            } else if (d.y_f16) {
                static_cast<__half*>(d.y)[r0 + i] = __float2half_rn(s);
            } else {
                static_cast<float*>(d.y)[r0 + i] = s;
            }
        }
        if (tp) {
            // wait for every rank's tagged partial of these rows and sum them
            // in rank order (identical on every rank).  Watchdog: a peer that
            // never arrives (ranks that ran different launch sequences, a dead
            // peer) must not hang the GPU -- give up after ~4 s and raise the
            // context's error flag.
            const uint32_t tag = p.tp_base + d.reduce_ord + 1;
            const unsigned long long* recv =
                p.tp_recv + size_t(par) * p.tp_world * p.tp_max_rows;
            const unsigned long long t_start = gtimer_ns();
            for (uint32_t i = 32 * f + lane; i < nrows; i += 32 * kFin) {
                float s = 0.f;
                for (uint32_t k = 0; k < p.tp_world; ++k) {
                    const unsigned long long* src = recv + k * p.tp_max_rows + r0 + i;
                    unsigned long long v = ld_volatile_u64(src);
                    while (uint32_t(v >> 32) != tag) {
                        if (gtimer_ns() - t_start > 4000000000ull) {
                            atomicExch(p.tp_flags, 1u);
                            break;
                        }
                        __nanosleep(20);
                        v = ld_volatile_u64(src);
                    }
                    s += __uint_as_float(uint32_t(v));
                }
                if (d.y_f16)
                    static_cast<__half*>(d.y)[r0 + i] = __float2half_rn(s);
                else
                    static_cast<float*>(d.y)[r0 + i] = s;
            }
        }
        __syncwarp();
        const uint32_t notify = SERVE ? p.serve_notify[l] : 0u;
        if (lane == 0) {
            if (f == 0) DSQ_TRACE(l, kTrFinalDone);
            mbar_arrive(&pempty[b]);
            mbar_arrive(&bempty[b]);
            if (!kOneSignal) red_release_gpu_add(p.counters + l, 1u);
        }
        if (kOneSignal) {
            // the CTA's finishing warps meet (CTA-scope ordering of all their
            // y stores), then ONE release per CTA: 148 same-address atomics
            // per layer instead of 148 x (1 + csr_warps)
            named_bar_sync(2, 32 * kFin);
            if (f == 0 && lane == 0) red_release_gpu_add(p.counters + l, 1u);
        }
        if (f == 0 && lane == 0) DSQ_TRACE(l, kTrSignaled);
        if (notify && f == 0 && cta == 0 && !p.serve_y_words) {
            // no output buffer: announce the step once every finishing warp
            // of every CTA is done
            if (lane == 0) {
                while (ld_acquire_gpu(p.counters + l) < G * sig_per_cta) __nanosleep(32);
                __threadfence_system();
                st_release_sys(p.host_done, notify);
            }
        }
        __syncwarp();
    };
    // the last finishing warp of the last CTA resets the counters for the
    // next launch (all finishing warps of a CTA meet at named barrier 1)
    auto finish_kernel = [&]() {
        __syncwarp();  // bar.sync is .aligned: the warp must arrive converged
                       // (desc_release's lane-0 arrive diverged it; synccheck)
        named_bar_sync(1, 32 * kFin);
        if (warp == NC + 2 && lane == 0) {
            const uint32_t old = atomicAdd(p.counters + p.n_layers, 1u);
            if (old == G - 1) {
                for (uint32_t l = 0; l <= p.n_layers; ++l) p.counters[l] = 0;
            }
        }
    };

    if (warp == NC + 2) {
        // ---------------- finisher ----------------------------------------------
        pdl_wait();
        pdl_trigger();
        for (uint32_t l = 0; l < p.n_layers; ++l) {
            desc_wait(l);
            finish_rows(l, 0);
            desc_release(l);
        }
        finish_kernel();
        return;
    }

    if (warp >= NC + 3) {
        // ---------------- CSR warps: the deltas of the CTA's rows, then finishing
        pdl_wait();
        pdl_trigger();
        const uint32_t cw = warp - (NC + 3);
        for (uint32_t l = 0; l < p.n_layers; ++l) {
            const uint32_t b = l & 1u, ph = (l >> 1) & 1u;
            const SDesc& sd = desc_wait(l);
            const Share sh = cta_share(sd.d, cta);
            mbar_wait_fin(&xfull[b], ph);
            mbar_wait_fin(&cfull[b], ph);
            if (l >= 2) mbar_wait_fin(&pempty[b], ((l >> 1) - 1) & 1u);  // segs consumed
            if (cw == 0 && lane == 0) DSQ_TRACE(l, kTrCsrStaged);
            const uint16_t* xh = reinterpret_cast<const uint16_t*>(sm + p.off_x + x_region(p, l, sd.d.ns));
            const uint32_t xvl = sd.d.ns * kSpanCols;
            const uint32_t* rp = reinterpret_cast<const uint32_t*>(sm + p.off_rp) + b * p.rp_words;
            (void)rp;
            const uint32_t e0 = sd.e0, e1 = sd.e1, ea = e0 & ~3u;
            const bool staged = e1 - e0 <= p.csr_cap - 4;
            const uint32_t* ent = staged ? reinterpret_cast<const uint32_t*>(sm + p.off_csr) + b * p.csr_cap
                                         : sd.d.csr + ea;
            const uint32_t* hb = staged ? reinterpret_cast<const uint32_t*>(sm + p.off_hb) + b * p.hb_words
                                        : sd.d.csr_heads;
            const uint32_t hbase = staged ? ((e0 >> 5) & ~3u) : 0u;
            const uint32_t hlast = staged ? p.hb_words - 2 : ((e1 + 31) >> 5) + 1;
            float* S = staged ? reinterpret_cast<float*>(sm + p.off_seg) + size_t(b) * NB * p.seg_cap
                              : p.gseg + (size_t(cta) * 2 + b) * NB * p.gseg_cap;
            if (e1 > e0) {
#pragma unroll
                for (int v = 0; v < NB; ++v)
                    if (v == 0 || uint32_t(v) < p.nvec)
                        csr_stream(ea, e0, e1, ent, hb, hbase, hlast, xh + v * xvl,
                                   S + v * (staged ? p.seg_cap : p.gseg_cap), cw, p.csr_warps, lane);
            }
            __syncwarp();
            if (cw == 0 && lane == 0) DSQ_TRACE(l, kTrCsrDone);
            if (lane == 0) mbar_arrive(&pfull[b]);
            finish_rows(l, 1 + cw);
            desc_release(l);
        }
        finish_kernel();
        return;
    }

    // ---------------- consumers: dense LUT products ----------------------------
    // (the first ring chunks are requested before the PDL wait: the weights
    // are launch constants, so their HBM latency overlaps the previous
    // kernel's tail; everything that reads x or writes shared state waits)
    const uint32_t cw = warp;
    // this lane's B-column x halves (NB == 2: B columns 4..7, lanes 16..31,
    // read batch vector 1)
    const uint32_t xoff0 = tile_x_offset(lane);  // + the lane's vector (per layer)
    const uint32_t trow = (lane >> 2) & 3u;         // tile row of this lane
    const ShiftK K{p.k29, p.k30, p.k31, p.kneg};
    const uint64_t policy = policy_evict_first();
    // this warp's weight stream: its unit range of every layer, in chunks of
    // cu units, through WS private ring slots.  The prefetch cursor (pl, pc)
    // runs WS chunks ahead of consumption, across layer boundaries (weights
    // never depend on x), so HBM keeps streaming while the warp waits for a
    // layer's input.
    uint32_t cslot = 0, cphase = 0;       // consumption
    // prefetch cursor: layer pl, next unit pa of this warp's range [pa, pe)
    // of that layer, whose first unit's words are at psrc; slot pslot
    uint32_t pl = 0, pa = 0, pe = 0, pslot = 0, pcu = 0;
    const uint32_t* psrc = nullptr;
    bool pvalid = false;
    auto issue_next = [&]() {
        while (true) {
            if (!pvalid) {
                if (pl >= p.n_layers) return;
                const SDesc& sn = desc_wait(pl);
                const uint32_t Un = sn.nt * sn.d.ns;
                // warps past the layer's active count own no units of it
                const bool act = cw < sn.d.nca;
                pa = act ? (cw * Un) >> sn.d.nca_shift : 0u;
                pe = act ? ((cw + 1) * Un) >> sn.d.nca_shift : 0u;
                pcu = sn.d.cu;
                psrc = sn.d.idx + (size_t(sn.t0) * sn.d.ns + pa) * UW;
                pvalid = true;
            }
            if (pa < pe) {
                const uint32_t n = min(pcu, pe - pa);
                if (lane == 0 && !(kDevSwitches && (p.dbg & 8u))) {
                    uint64_t* bar = &full[cw * WS + pslot];
                    mbar_arrive_expect_tx(bar, n * UW * 4);
                    bulk_g2s(ring + size_t(cw * WS + pslot) * p.slot_bytes, psrc, n * UW * 4, bar,
                             policy);
                }
                pa += n;
                psrc += size_t(n) * UW;
                if (++pslot == WS) pslot = 0;
                return;
            }
            pvalid = false;
            ++pl;
        }
    };
    for (uint32_t k = 0; k < WS; ++k) issue_next();
    pdl_wait();
    pdl_trigger();
    // dev profile (build with -DDSQ_STACK_PROFILE, run with DSQ_STACK_DBG bit
    // 2): cycles per consumer warp spent waiting for x / partial buffers,
    // waiting for ring data, in chunk / segment bookkeeping ("dense"), in the
    // unit loops (slot 3), and at layer boundaries
#ifdef DSQ_STACK_PROFILE
    const bool prof = (p.dbg & 4u) && p.trace;
    long long c_xw = 0, c_fw = 0, c_dense = 0, c_csr = 0, c_top = 0, t_mark = clock64();
    auto lap = [&](long long& acc) {
        if (prof) {
            const long long t = clock64();
            acc += t - t_mark;
            t_mark = t;
        }
    };
#define DSQ_LAP(acc) lap(acc)
#else
#define DSQ_LAP(acc) \
    do {             \
    } while (0)
#endif
    for (uint32_t l = 0; l < p.n_layers; ++l) {
        const uint32_t b = l & 1u;
        const SDesc& sd = desc_wait(l);
        const StackLayerDesc& d = sd.d;
        const uint32_t NS = d.ns, cu = d.cu;
        if (cw == 0 && lane == 0) DSQ_TRACE(l, kTrConsStart);
        DSQ_LAP(c_top);
        mbar_wait_edge(&xfull[b], (l >> 1) & 1u);
        if (l >= 2) mbar_wait_edge(&pempty[b], ((l >> 1) - 1) & 1u);
        DSQ_LAP(c_xw);
        if (cw == 0 && lane == 0) DSQ_TRACE(l, kTrXReady);
        const uint16_t* xh = reinterpret_cast<const uint16_t*>(sm + p.off_x + x_region(p, l, d.ns));
        const uint32_t xvl = d.ns * kSpanCols;  // halves per vector in this layer's x
        const uint32_t xoff = xoff0 + (NB >= 2 ? (lane >> 4) * xvl : 0u);
        const uint32_t* luts = reinterpret_cast<const uint32_t*>(sm + p.off_lut + b * p.lut_bytes);
        float* part = reinterpret_cast<float*>(sm + p.off_part) + size_t(b) * NB * p.part_rows * NC;

        // dense units: warp cw owns the contiguous unit range [u0, u1) of the
        // CTA share (tile-major: unit u = (tile u / NS, span u % NS)), which
        // its own TMA ring brings in, cu units per chunk.  The accumulators
        // follow the warp across chunks and are flushed into part[cw][row]
        // on a tile change.
        const uint32_t U = sd.nt * NS;
        const bool act = cw < d.nca;
        const uint32_t u0 = act ? (cw * U) >> d.nca_shift : 0u;
        const uint32_t u1 = act ? ((cw + 1) * U) >> d.nca_shift : 0u;
        uint32_t cur_tile = 0xffffffffu;
        Planes16 P;
        float d0[4] = {0.f, 0.f, 0.f, 0.f}, d1[4] = {0.f, 0.f, 0.f, 0.f};
        // vector pairs 2/3, 4/5, 6/7 (NB >= 4): one accumulator pair each
        constexpr int NX = NB >= 4 ? NB / 2 - 1 : 1;
        float ex[NX][2][4];
#pragma unroll
        for (int q = 0; q < NX; ++q)
#pragma unroll
            for (int k = 0; k < 4; ++k) ex[q][0][k] = ex[q][1][k] = 0.f;
        auto flush = [&]() {
            if (cur_tile != 0xffffffffu) {
                if constexpr (NB == 1) {
                    const float v = tile_rows_reduce(d0, d1, lane);
                    if ((lane & 3) == 0 && lane < 16) part[cw * p.part_rows + cur_tile * kTileRows + trow] += v;
                } else {  // vector 0 in lanes 4i, vector 1 in lanes 4i + 2
                    const float v = tile_rows_reduce2(d0, d1, lane);
                    if ((lane & 1) == 0 && lane < 16)
                        part[((lane >> 1) & 1u) * NC * p.part_rows + cw * p.part_rows +
                             cur_tile * kTileRows + trow] += v;
                    if constexpr (NB >= 4) {  // the other vector pairs
#pragma unroll
                        for (int q = 0; q < NX; ++q) {
                            const float v2 = tile_rows_reduce2(ex[q][0], ex[q][1], lane);
                            if ((lane & 1) == 0 && lane < 16)
                                part[(2u * (q + 1) + ((lane >> 1) & 1u)) * NC * p.part_rows +
                                     cw * p.part_rows + cur_tile * kTileRows + trow] += v2;
#pragma unroll
                            for (int k = 0; k < 4; ++k) ex[q][0][k] = ex[q][1][k] = 0.f;
                        }
                    }
                }
#pragma unroll
                for (int k = 0; k < 4; ++k) d0[k] = d1[k] = 0.f;
            }
        };
        // (tile, span) of the next unit, carried across chunks (chunks are
        // consecutive ranges): one division per layer, not per chunk
        uint32_t tile_c = u0 / NS, s_c = u0 - tile_c * NS;
        for (uint32_t cb = u0; cb < u1; cb += cu) {
            DSQ_LAP(c_dense);
            if (!(kDevSwitches && (p.dbg & 8u)))  // dev bit 8: compute only
                mbar_wait_cons(&full[cw * WS + cslot], cphase);
            DSQ_LAP(c_fw);
            const uint32_t* chunk = reinterpret_cast<const uint32_t*>(ring + size_t(cw * WS + cslot) * p.slot_bytes);
            uint32_t u = cb;
            const uint32_t ue = min(u1, cb + cu);
            if (!(kDevSwitches && (p.dbg & 1u))) {  // dev bit 1: streaming only
                uint32_t tile = tile_c, s = s_c;
                const uint32_t* sp = chunk;
                while (u < ue) {
                    if (tile != cur_tile) {
                        flush();
                        cur_tile = tile;
                        const uint32_t* lp = luts + (tile * kTileRows + trow) * LW;
                        const uint4 q0 = *reinterpret_cast<const uint4*>(lp);
                        P.a = Planes8{q0.x, q0.y, q0.z, q0.w};
                        if constexpr (BITS == 4) {
                            const uint4 q1 = *reinterpret_cast<const uint4*>(lp + 4);
                            P.b = Planes8{q1.x, q1.y, q1.z, q1.w};
                        }
                    }
                    // spans [s, s_end) of this tile; software-pipelined: the
                    // next span's words and x are loaded before the current
                    // span is decoded
                    DSQ_LAP(c_dense);  // (profile: segment set-up counts as dense)
                    const uint32_t s_end = min(NS, s + (ue - u));
                    const uint16_t* xs = xh + s * kSpanCols + xoff;
                    uint32_t w[BITS];
                    uint4 xa, xb2;
                    auto load = [&](const uint32_t* spp, const uint16_t* xsp) {
                        if constexpr (BITS == 3) {
                            w[0] = spp[lane];
                            w[1] = spp[32 + lane];
                            w[2] = spp[64 + lane];
                        } else {
                            const uint4 q = reinterpret_cast<const uint4*>(spp)[lane];
                            w[0] = q.x;
                            w[1] = q.y;
                            w[2] = q.z;
                            w[3] = q.w;
                        }
                        xa = *reinterpret_cast<const uint4*>(xsp);
                        xb2 = *reinterpret_cast<const uint4*>(xsp + 128);
                    };
                    uint32_t k = s;
                    if constexpr (NB >= 4) {
                        // 4 / 8 vectors: every decoded fragment feeds NB/2
                        // HMMAs (vector pair q's x at +2q vector strides)
                        for (; k < s_end; ++k) {
                            const uint4 xa0 = *reinterpret_cast<const uint4*>(xs);
                            const uint4 xb0 = *reinterpret_cast<const uint4*>(xs + 128);
                            uint4 ya[NX], yb[NX];
#pragma unroll
                            for (int q = 0; q < NX; ++q) {
                                ya[q] = *reinterpret_cast<const uint4*>(xs + 2 * (q + 1) * xvl);
                                yb[q] = *reinterpret_cast<const uint4*>(xs + 2 * (q + 1) * xvl + 128);
                            }
                            if constexpr (BITS == 3) {
                                span3_mma_xn<NX>(sp[lane], sp[32 + lane], sp[64 + lane], P.a, xa0,
                                                 xb0, ya, yb, d0, d1, ex, K);
                            } else {
                                span4_mma_xn<NX>(reinterpret_cast<const uint4*>(sp)[lane], P, xa0,
                                                 xb0, ya, yb, d0, d1, ex);
                            }
                            sp += UW;
                            xs += kSpanCols;
                        }
                    }
                    if constexpr (BITS == 3 && NB < 4) {
                        // 8-consumer kernels: four units per iteration (two
                        // pairs interleaved: twice the independent work per
                        // warp with only two decode warps per SMSP; +2.6% on
                        // the 7B chain; the 16-consumer kernels, capped at 88
                        // registers, measured slower with it)
                        for (; NC == 8 && k + 3 < s_end; k += 4) {
                            const uint32_t a0 = sp[lane], a1 = sp[32 + lane], a2 = sp[64 + lane];
                            const uint32_t b0 = sp[96 + lane], b1 = sp[128 + lane],
                                           b2 = sp[160 + lane];
                            const uint32_t c0 = sp[192 + lane], c1 = sp[224 + lane],
                                           c2 = sp[256 + lane];
                            const uint32_t e0 = sp[288 + lane], e1 = sp[320 + lane],
                                           e2 = sp[352 + lane];
                            const uint4 xa0 = *reinterpret_cast<const uint4*>(xs);
                            const uint4 xb0 = *reinterpret_cast<const uint4*>(xs + 128);
                            const uint4 xa1 = *reinterpret_cast<const uint4*>(xs + kSpanCols);
                            const uint4 xb1 = *reinterpret_cast<const uint4*>(xs + kSpanCols + 128);
                            const uint4 xa2 = *reinterpret_cast<const uint4*>(xs + 2 * kSpanCols);
                            const uint4 xb2 = *reinterpret_cast<const uint4*>(xs + 2 * kSpanCols + 128);
                            const uint4 xa3 = *reinterpret_cast<const uint4*>(xs + 3 * kSpanCols);
                            const uint4 xb3 = *reinterpret_cast<const uint4*>(xs + 3 * kSpanCols + 128);
                            span3_mma_one(a0, a1, a2, P.a, xa0, xb0, d0, K);
                            span3_mma_one(b0, b1, b2, P.a, xa1, xb1, d1, K);
                            span3_mma_one(c0, c1, c2, P.a, xa2, xb2, d0, K);
                            span3_mma_one(e0, e1, e2, P.a, xa3, xb3, d1, K);
                            sp += 4 * UW;
                            xs += 4 * kSpanCols;
                        }
                        // span pairs: two independent units per iteration
                        for (; k + 1 < s_end; k += 2) {
                            const uint32_t a0 = sp[lane], a1 = sp[32 + lane], a2 = sp[64 + lane];
                            const uint32_t b0 = sp[96 + lane], b1 = sp[128 + lane],
                                           b2 = sp[160 + lane];
                            const uint4 xa0 = *reinterpret_cast<const uint4*>(xs);
                            const uint4 xb0 = *reinterpret_cast<const uint4*>(xs + 128);
                            const uint4 xa1 = *reinterpret_cast<const uint4*>(xs + kSpanCols);
                            const uint4 xb1 = *reinterpret_cast<const uint4*>(xs + kSpanCols + 128);
                            span3_mma_one(a0, a1, a2, P.a, xa0, xb0, d0, K);
                            span3_mma_one(b0, b1, b2, P.a, xa1, xb1, d1, K);
                            sp += 2 * UW;
                            xs += 2 * kSpanCols;
                        }
                    }
                    if (k < s_end) load(sp, xs);
                    for (; k < s_end; ++k) {
                        uint32_t wc[BITS];
#pragma unroll
                        for (int q = 0; q < BITS; ++q) wc[q] = w[q];
                        const uint4 xac = xa, xbc = xb2;
                        sp += UW;
                        xs += kSpanCols;
                        if (k + 1 < s_end) load(sp, xs);
                        if constexpr (BITS == 3) {
                            span3_mma(wc[0], wc[1], wc[2], P.a, xac, xbc, d0, d1, K);
                        } else {
                            span4_mma(make_uint4(wc[0], wc[1], wc[2], wc[3]), P, xac, xbc, d0, d1);
                        }
                    }
                    DSQ_LAP(c_csr);  // (profile slot 3: the unit loops themselves)
                    u += s_end - s;
                    s = s_end;
                    if (s == NS) {
                        ++tile;
                        s = 0;
                    }
                }
                tile_c = tile;
                s_c = s;
            }
            // the slot's words are consumed (their values were used): refill
            // it with the next chunk of this warp's stream
            __syncwarp();
            if (++cslot == WS) {
                cslot = 0;
                cphase ^= 1u;
            }
            DSQ_LAP(c_dense);
            issue_next();
            DSQ_LAP(c_fw);  // (profile: the refill issue counts with the ring wait)
        }
        flush();
        if (cw == 0 && lane == 0) DSQ_TRACE(l, kTrDenseDone);
        DSQ_LAP(c_dense);
        __syncwarp();
        desc_release(l);
        if (lane == 0) {
            mbar_arrive(&pfull[b]);
            mbar_arrive(&bempty[b]);
        }
    }
#ifdef DSQ_STACK_PROFILE
    if (prof && lane == 0) {
        long long* o = reinterpret_cast<long long*>(p.trace) + (size_t(cta) * NC + cw) * 5;
        o[0] = c_xw;
        o[1] = c_fw;
        o[2] = c_dense;
        o[3] = c_csr;
        o[4] = c_top;
    }
#endif
}

cudaError_t launch_stack(const StackParams& p, cudaStream_t st, bool pdl) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(p.grid);
    cfg.blockDim = dim3((p.consumers + 3 + p.csr_warps) * 32);
    cfg.dynamicSmemBytes = p.smem_bytes;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    static bool attr_done[18][64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    const int ci = p.consumers == 8 ? 0 : 1;
    // nbatch 8 has only 8-consumer kernels (the accumulators of four vector
    // pairs need the registers)
    if (p.serve_gate && p.nbatch != 1) return cudaErrorInvalidValue;  // served: batch 1
    const int bi = p.serve_gate       ? 14 + (p.bits == 3 ? 0 : 1) * 2 + ci
                   : p.nbatch == 8 ? 12 + (p.bits == 3 ? 0 : 1)
                                 : (p.nbatch == 4 ? 8 : p.nbatch == 2 ? 4 : 0) +
                                       (p.bits == 3 ? 0 : 1) * 2 + ci;
    using K = void (*)(StackParams);
    static const K kerns[18] = {
        stack_gemv<3, 8, 1>, stack_gemv<3, 16, 1>, stack_gemv<4, 8, 1>, stack_gemv<4, 16, 1>,
        stack_gemv<3, 8, 2>, stack_gemv<3, 16, 2>, stack_gemv<4, 8, 2>, stack_gemv<4, 16, 2>,
        stack_gemv<3, 8, 4>, stack_gemv<3, 16, 4>, stack_gemv<4, 8, 4>, stack_gemv<4, 16, 4>,
        stack_gemv<3, 8, 8>, stack_gemv<4, 8, 8>,
        stack_gemv<3, 8, 1, true>, stack_gemv<3, 16, 1, true>, stack_gemv<4, 8, 1, true>,
        stack_gemv<4, 16, 1, true>};
    const K kern = kerns[bi];
    if (dev < 0 || dev >= 64 || !attr_done[bi][dev]) {
        int max_optin = 0;
        cudaDeviceGetAttribute(&max_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             max_optin);
        if (e != cudaSuccess) return e;
        if (dev >= 0 && dev < 64) attr_done[bi][dev] = true;
    }
    // every grid-wide wait in the kernel (layer completion counters, the TP
    // exchange, the serving flags) assumes all CTAs are co-resident: check
    // that one CTA of this size fits per SM and that the grid does not
    // exceed the SM count (cooperative-launch guarantee, without the
    // cooperative attribute, which programmatic dependent launch excludes)
    {
        int per_sm = 0, sms = 0;
        cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(
            &per_sm, kern, int(cfg.blockDim.x), cfg.dynamicSmemBytes);
        if (e != cudaSuccess) return e;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (per_sm < 1 || uint64_t(p.grid) > uint64_t(per_sm) * uint64_t(sms))
            return cudaErrorCooperativeLaunchTooLarge;
    }
    return cudaLaunchKernelEx(&cfg, kern, p);
}

// ---------------------------------------------------------------------------
// K5/K6 for the tile layout: decode indices / values of every (row, col)
// ---------------------------------------------------------------------------
template <int BITS, int MODE>  // MODE 0: u16 indices, 1: fp16 values, 2: fp32 values
__global__ void decode_tiles(const uint32_t* __restrict__ idx, const uint32_t* __restrict__ lutp,
                             uint32_t rows, uint32_t cols, uint32_t ns, void* out) {
    const uint32_t ng = ns * (kSpanCols / 32);
    const size_t t = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= size_t(rows) * ng) return;
    const uint32_t row = uint32_t(t / ng), g = uint32_t(t % ng);
    constexpr uint32_t LW = BITS == 3 ? 4 : 8;
    const uint32_t tile = row / kTileRows, i = row % kTileRows, s = g / 8, gs = g % 8;
    const uint32_t h = gs >> 2, tt = gs & 3, lane = 16 * h + 4 * i + tt;
    const uint32_t* sp = idx + (size_t(tile) * ns + s) * BITS * 32;
    uint32_t w[4];
#pragma unroll
    for (int k = 0; k < 4; ++k)
        w[k] = k < BITS ? (BITS == 3 ? sp[k * 32 + lane] : sp[lane * 4 + k]) : 0u;
    // fp16 entries back from the byte planes
    const uint32_t* r = lutp + (size_t(tile) * kTileRows + i) * LW;
    uint16_t lut[16];
#pragma unroll
    for (int e = 0; e < (1 << BITS); ++e) {
        const uint32_t base = (e >> 3) * 4;  // plane set
        const uint32_t ee = e & 7;
        const uint32_t lo = (r[base + (ee >> 2)] >> (8 * (ee & 3))) & 0xffu;
        const uint32_t hi = (r[base + 2 + (ee >> 2)] >> (8 * (ee & 3))) & 0xffu;
        lut[e] = uint16_t(lo | (hi << 8));
    }
    for (int j = 0; j < 32; ++j) {
        const uint32_t c = s * kSpanCols + tile_col(h, tt, j);
        if (c >= cols) continue;
        uint32_t ix;
        if constexpr (BITS == 3) {
            if (j < 24) {
                ix = (w[j >> 3] >> (4 * (j & 7))) & 7u;
            } else {
                const int nn = j - 24;
                ix = ((w[0] >> (4 * nn + 3)) & 1u) | (((w[1] >> (4 * nn + 3)) & 1u) << 1) |
                     (((w[2] >> (4 * nn + 3)) & 1u) << 2);
            }
        } else {
            ix = (w[j >> 3] >> (4 * (j & 7))) & 15u;
        }
        const size_t o = size_t(row) * cols + c;
        if (MODE == 0) static_cast<uint16_t*>(out)[o] = uint16_t(ix);
        else if (MODE == 1) static_cast<uint16_t*>(out)[o] = lut[ix];
        else static_cast<float*>(out)[o] = __half2float(__ushort_as_half(lut[ix]));
    }
}

// Fragment dump (parity tests): the fp16 A fragments exactly as the product
// kernels build them -- the same span3_frags / span4_frags decode (PRMT byte
// planes, selector preparation) the timed stack kernel runs -- scattered back
// to (row, col) of a dense rows x cols fp16 matrix.  One warp per unit.
template <int BITS>
__global__ void dump_frags(const uint32_t* __restrict__ idx, const uint32_t* __restrict__ lutp,
                           uint32_t rows, uint32_t cols, uint32_t tiles, uint32_t ns,
                           uint16_t* __restrict__ out, ShiftK K) {
    constexpr uint32_t LW = BITS == 3 ? 4u : 8u, UW = BITS * 32u;
    const size_t unit = (size_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const uint32_t lane = threadIdx.x & 31;
    if (unit >= size_t(tiles) * ns) return;
    const uint32_t tile = uint32_t(unit / ns), s = uint32_t(unit % ns);
    const uint32_t h = lane >> 4, i = (lane >> 2) & 3u, t = lane & 3u;
    const uint32_t* lp = lutp + (size_t(tile) * kTileRows + i) * LW;
    Planes16 P;
    P.a = Planes8{lp[0], lp[1], lp[2], lp[3]};
    if constexpr (BITS == 4) P.b = Planes8{lp[4], lp[5], lp[6], lp[7]};
    const uint32_t* sp = idx + unit * UW;
    const uint32_t row = tile * kTileRows + i;
    auto sink = [&](int j, uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3) {
        const uint32_t a[4] = {a0, a1, a2, a3};
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) {
                const uint32_t c = s * kSpanCols + tile_col(h, t, frag_pos(j, r, hh));
                if (row < rows && c < cols)
                    out[size_t(row) * cols + c] = uint16_t(a[r] >> (16 * hh));
            }
    };
    if constexpr (BITS == 3)
        span3_frags(sp[lane], sp[32 + lane], sp[64 + lane], P.a, sink, K);
    else
        span4_frags(reinterpret_cast<const uint4*>(sp)[lane], P, sink);
}

cudaError_t launch_dump_frags(uint32_t bits, const uint32_t* idx, const uint32_t* lut,
                              uint32_t rows, uint32_t cols, uint32_t tiles, uint32_t ns,
                              uint16_t* out, cudaStream_t st) {
    const ShiftK K = SQZ_SHIFTK_INIT;
    const size_t threads = size_t(tiles) * ns * 32;
    const uint32_t blocks = uint32_t((threads + 255) / 256);
    if (bits == 3)
        dump_frags<3><<<blocks, 256, 0, st>>>(idx, lut, rows, cols, tiles, ns, out, K);
    else
        dump_frags<4><<<blocks, 256, 0, st>>>(idx, lut, rows, cols, tiles, ns, out, K);
    return cudaGetLastError();
}

cudaError_t launch_decode_tiles(int mode, uint32_t bits, const uint32_t* idx, const uint32_t* lut,
                                uint32_t rows, uint32_t cols, uint32_t ns, void* out,
                                cudaStream_t st) {
    const size_t n = size_t(rows) * ns * (kSpanCols / 32);
    const uint32_t blocks = uint32_t((n + 255) / 256);
#define DSQ_DEC(B, M) decode_tiles<B, M><<<blocks, 256, 0, st>>>(idx, lut, rows, cols, ns, out)
    if (bits == 3) {
        if (mode == 0) DSQ_DEC(3, 0);
        else if (mode == 1) DSQ_DEC(3, 1);
        else DSQ_DEC(3, 2);
    } else {
        if (mode == 0) DSQ_DEC(4, 0);
        else if (mode == 1) DSQ_DEC(4, 1);
        else DSQ_DEC(4, 2);
    }
#undef DSQ_DEC
    return cudaGetLastError();
}

}  // namespace sqz
