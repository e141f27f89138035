// stack.cu -- K7: persistent multi-layer Dense-and-Sparse LUT-GEMV (sm_100a).
//
// One CTA per SM, all co-resident.  For every layer l of the stack each CTA
// owns a contiguous range of 4-row tiles (tiles split evenly over the grid, so
// the balance granularity is one tile and no output row is ever shared
// between CTAs -> no global merge, no floating-point atomics).
//
// Warp roles (consumers take the low warp ids, control warps the top ones,
// which the issue arbiter favours):
//   consumers 0..NC-1: every ring chunk (a fixed number of (tile, 256-column
//              span) units of the CTA's share) is split in equal contiguous
//              unit ranges over the NC warps; per unit a lane decodes 32
//              indices of one tile row with PRMT byte-plane lookups into fp16
//              A fragments and 4 mma.sync m16n8k16 accumulate them against x
//              in fp32 (tile.cuh).  When a warp moves to another tile its D
//              fragments collapse to the tile's 4 row partials, added into the
//              warp's column of a shared-memory [warp][row] partial table.
//              The CSR deltas of the CTA's rows are shared by the warps in
//              32-entry rounds (segmented warp scan, host-built row-start
//              bitmap); half of the warps do them before their dense units,
//              half after, so the rounds' latency overlaps dense work.
//   producer  (NC):   publishes each layer's descriptor to a shared-memory
//              cache and streams the CTA's index units of layer 0, 1, 2, ...
//              HBM -> shared-memory ring with cp.async.bulk (TMA bulk
//              engine), completion on mbarriers.  Weights never depend on x,
//              so it runs ahead across layer boundaries, bounded only by the
//              ring -- the HBM pipe stays busy while other warps wait on a
//              layer dependency.
//   loader    (NC+1): stages the CTA's LUT planes, CSR slice (row_ptr,
//              entries, row-start bitmap) and, once the layer producing x is
//              complete on ALL CTAs (grid-wide completion counter,
//              ld.acquire), the activation vector x -- all by TMA into
//              double-buffered shared memory.
//   finisher  (NC+2): per row, the dense partials in warp order plus the
//              row's CSR round results in round order (deterministic), the
//              store of y, and the layer's completion signal (red.release).
// Reference semantics: per row, LUT dot + CSR delta dot == fused_dns_matvec
// (reference kernels.cpp:108-141); the hybrid split is unnecessary because the
// CSR rounds are balanced regardless of per-row skew.
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
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
constexpr uint32_t kWarpSlots = 2;  // ring slots per consumer warp
struct __align__(16) SDesc {
    StackLayerDesc d;
    uint32_t e0, e1;  // CSR entries of this CTA's rows: [e0, e1)
    uint32_t pad[(128 - sizeof(StackLayerDesc) - 8) / 4];
};
static_assert(sizeof(SDesc) == 128, "descriptor slot is one 128-byte line");

__device__ __forceinline__ const StackLayerDesc& layer_desc(const StackParams& p, uint32_t l) {
    return l < kInlineLayers && p.n_layers <= kInlineLayers ? p.inl[l] : p.layers[l];
}

// CTA tile share from the host-precomputed quotient/remainder (no division)
struct Share {
    uint32_t t0, nt, nch;  // first tile, tiles, ring chunks
    uint32_t r0, nrows;    // real rows [r0, r0 + nrows) (tiles clipped to the layer)
};
__device__ __forceinline__ Share cta_share(const StackLayerDesc& d, uint32_t cta) {
    Share s;
    const bool hi = cta < d.tr;
    s.t0 = cta * d.tq + (hi ? cta : d.tr);
    s.nt = d.tq + (hi ? 1u : 0u);
    s.nch = hi ? d.nch_hi : d.nch_lo;
    s.r0 = min(s.t0 * kTileRows, d.rows);
    s.nrows = min((s.t0 + s.nt) * kTileRows, d.rows) - s.r0;
    return s;
}

__device__ __forceinline__ unsigned long long gtimer_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#define DSQ_TRACE(l, slot)                                                                 \
    do {                                                                                   \
        if (p.trace && !(p.dbg & 4u))                                                      \
            p.trace[(size_t(blockIdx.x) * p.n_layers + (l)) * kTrSlots + (slot)] = gtimer_ns(); \
    } while (0)

// CSR deltas of the CTA's rows: 32-entry rounds j = first, first+stride, ...
// of the CTA's contiguous entry slice.  hb is the host-built bitmap of row
// starts (bit q = entry q begins a row), so a lane knows where its segment
// begins without scanning row pointers; a segmented inclusive warp scan
// (5 shuffles) then leaves each row's partial of the round at its last entry.
// Two rounds are processed together for instruction-level parallelism.
__device__ __forceinline__ void csr_round_pair(uint32_t e0, uint32_t nz, const uint32_t* ent,
                                               const uint32_t* hb, uint32_t hbase,
                                               const uint16_t* xh, float* segs, float* gseg,
                                               uint32_t seg_rounds, uint32_t j0, uint32_t j1,
                                               bool two, uint32_t lane) {
    float v[2];
    uint32_t seg0[2];
#pragma unroll
    for (int k = 0; k < 2; ++k) {
        const uint32_t j = k ? j1 : j0;
        const uint32_t pi = j * 32 + lane;
        v[k] = 0.f;
        if ((k == 0 || two) && pi < nz) {
            const uint32_t e = ent[pi];
            v[k] = fma_h(uint16_t(e >> 16), xh[e & 0xffffu], 0.f);
        }
        const uint32_t g = e0 + j * 32, w = (g >> 5) - hbase;
        const uint32_t heads = __funnelshift_r(hb[w], hb[w + 1], g & 31u);
        const uint32_t upto = heads & (0xffffffffu >> (31 - lane));
        seg0[k] = upto ? (31u - __clz(upto)) : 0u;
    }
#pragma unroll
    for (uint32_t off = 1; off < 32; off <<= 1) {
        const float t0 = __shfl_up_sync(0xffffffffu, v[0], off);
        const float t1 = __shfl_up_sync(0xffffffffu, v[1], off);
        if (lane >= seg0[0] + off) v[0] += t0;
        if (lane >= seg0[1] + off) v[1] += t1;
    }
#pragma unroll
    for (int k = 0; k < 2; ++k) {
        if (k == 1 && !two) break;
        const uint32_t j = k ? j1 : j0;
        float* dst = j < seg_rounds ? segs + j * 32 : gseg + (j - seg_rounds) * 32;
        dst[lane] = v[k];
    }
}

__device__ __forceinline__ void csr_rounds(uint32_t e0, uint32_t nz, const uint32_t* ent,
                                           const uint32_t* hb, uint32_t hbase, const uint16_t* xh,
                                           float* segs, float* gseg, uint32_t seg_rounds,
                                           uint32_t first, uint32_t stride, uint32_t lane) {
    const uint32_t rounds = (nz + 31) / 32;
    for (uint32_t j = first; j < rounds; j += 2 * stride)
        csr_round_pair(e0, nz, ent, hb, hbase, xh, segs, gseg, seg_rounds, j, j + stride,
                       j + stride < rounds, lane);
}

template <int BITS, int NC>
__global__ void __launch_bounds__((NC + 3) * 32, 1) stack_gemv(const __grid_constant__ StackParams p) {
    constexpr uint32_t LW = BITS == 3 ? 4u : 8u;   // LUT words per tile row
    constexpr uint32_t UW = BITS * 32u;             // words per (tile, span) unit
    extern __shared__ __align__(1024) uint8_t sm[];
    // mbarriers: per-warp ring slots, then per buffer parity b in {0,1}
    constexpr uint32_t WS = kWarpSlots;
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

    if (threadIdx.x == 0) {
        for (uint32_t s = 0; s < NC * WS; ++s) mbar_init(&full[s], 1);
        for (int b = 0; b < 2; ++b) {
            mbar_init(&xfull[b], 1);
            mbar_init(&cfull[b], 1);
            mbar_init(&bempty[b], NC + 1);
            mbar_init(&pfull[b], NC);
            mbar_init(&pempty[b], 1);
        }
        for (uint32_t k = 0; k < kDescSlots; ++k) {
            mbar_init(&dfull[k], 32);
            mbar_init(&dempty[k], NC + 2);
        }
        fence_barrier_init();
    }
    // the partial tables start at zero; the finisher re-zeroes what it reads
    {
        float* part = reinterpret_cast<float*>(sm + p.off_part);
        for (uint32_t i = threadIdx.x; i < 2 * NC * p.part_rows; i += blockDim.x) part[i] = 0.f;
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
            if (l >= kDescSlots) mbar_wait(&dempty[k], ((l / kDescSlots) - 1) & 1u);
            const StackLayerDesc& gd = layer_desc(p, l);
            uint32_t* dst = reinterpret_cast<uint32_t*>(&sdesc[k]);
            constexpr uint32_t kDW = sizeof(StackLayerDesc) / 4;
            if (lane < kDW) dst[lane] = reinterpret_cast<const uint32_t*>(&gd)[lane];
            else if (lane < kDW + 2) dst[lane] = gd.csr_rng[2 * cta + (lane - kDW)];
            mbar_arrive(&dfull[k]);
            __syncwarp();
        }
        return;
    }

    if (warp == NC + 1) {
        // ---------------- loader: LUT planes, CSR slice, x (the dependency) ---
        pdl_wait();
        pdl_trigger();
        for (uint32_t l = 0; l < p.n_layers; ++l) {
            const uint32_t b = l & 1u;
            if (l >= 2) mbar_wait(&bempty[b], ((l >> 1) - 1) & 1u);
            const SDesc& sd = desc_wait(l);
            const StackLayerDesc& d = sd.d;
            const Share sh = cta_share(d, cta);
            const uint32_t r0 = sh.r0, r1 = sh.r0 + sh.nrows;
            uint8_t* xb = sm + p.off_x + b * p.x_bytes;
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
                for (uint32_t i = body / 2 + lane; i < d.ns * kSpanCols; i += 32)
                    reinterpret_cast<uint16_t*>(xb)[i] = i < d.cols ? ld_cg_u16(d.x + i) : uint16_t(0);
                __syncwarp();
                if (lane == 0) {
                    fence_proxy_async_global();
                    mbar_arrive_expect_tx(&xfull[b], body);
                    if (body) bulk_g2s_plain(xb, d.x, body, &xfull[b]);
                }
            };
            if (d.dep == kNoDep) stage_x();  // external input: no wait at all
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
            if (d.dep != kNoDep) {
                if (lane == 0) {
                    while (ld_acquire_gpu(p.counters + d.dep) < G) __nanosleep(20);
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

    if (warp == NC + 2) {
        // ---------------- finisher: row totals, y, grid signal ----------------
        pdl_wait();
        pdl_trigger();
        for (uint32_t l = 0; l < p.n_layers; ++l) {
            const uint32_t b = l & 1u, ph = (l >> 1) & 1u;
            float* segs = reinterpret_cast<float*>(sm + p.off_seg) + size_t(b) * p.seg_rounds * 32;
            float* gseg = p.gseg + (size_t(cta) * 2 + b) * p.gseg_rounds * 32;
            const StackLayerDesc& d = desc_wait(l).d;
            const Share sh = cta_share(d, cta);
            const uint32_t r0 = sh.r0, nrows = sh.nrows;
            const uint32_t* rp = reinterpret_cast<const uint32_t*>(sm + p.off_rp) + b * p.rp_words;
            mbar_wait(&pfull[b], ph);
            if (lane == 0) DSQ_TRACE(l, kTrAllDense);
            const uint32_t e0 = rp[0];
            float* part = reinterpret_cast<float*>(sm + p.off_part) + size_t(b) * p.part_rows * NC;
            // row totals: dense partials in warp order (warps that did not
            // touch a row left 0), then the row's CSR rounds in round order
            for (uint32_t i = lane; i < sh.nt * kTileRows; i += 32) {
                float s = 0.f;
#pragma unroll
                for (uint32_t w = 0; w < NC; ++w) {
                    s += part[w * p.part_rows + i];
                    part[w * p.part_rows + i] = 0.f;
                }
                if (i >= nrows) continue;  // padding rows of the last tile
                const uint32_t a = rp[i] - e0, e = rp[i + 1] - e0;
                for (uint32_t j = a / 32; e > a && j <= (e - 1) / 32; ++j) {
                    const uint32_t end = min(e - 1 - j * 32, 31u);
                    const float* src = j < p.seg_rounds ? segs + j * 32 : gseg + (j - p.seg_rounds) * 32;
                    s += src[end];
                }
                if (d.y_f16)
                    static_cast<__half*>(d.y)[r0 + i] = __float2half_rn(s);
                else
                    static_cast<float*>(d.y)[r0 + i] = s;
            }
            __syncwarp();
            if (lane == 0) {
                DSQ_TRACE(l, kTrFinalDone);
                mbar_arrive(&pempty[b]);
                mbar_arrive(&bempty[b]);
                red_release_gpu_add(p.counters + l, 1u);
                DSQ_TRACE(l, kTrSignaled);
            }
            __syncwarp();
            desc_release(l);
        }
        // the last CTA to finish resets the counters for the next launch
        if (lane == 0) {
            const uint32_t old = atomicAdd(p.counters + p.n_layers, 1u);
            if (old == G - 1) {
                for (uint32_t l = 0; l <= p.n_layers; ++l) p.counters[l] = 0;
            }
        }
        return;
    }

    // ---------------- consumers: dense LUT products + CSR rounds --------------
    pdl_wait();
    pdl_trigger();
    const uint32_t cw = warp;
    const uint32_t xoff = tile_x_offset(lane);     // this lane's B-column x halves
    const uint32_t trow = (lane >> 2) & 3u;         // tile row of this lane
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
                const StackLayerDesc& dn = desc_wait(pl).d;
                const Share shn = cta_share(dn, cta);
                const uint32_t Un = shn.nt * dn.ns;
                pa = (cw * Un) / NC;
                pe = ((cw + 1) * Un) / NC;
                pcu = dn.cu;
                psrc = dn.idx + (size_t(shn.t0) * dn.ns + pa) * UW;
                pvalid = true;
            }
            if (pa < pe) {
                const uint32_t n = min(pcu, pe - pa);
                if (lane == 0) {
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
    // dev profile (DSQ_STACK_DBG bit 2): cycles per consumer warp spent
    // waiting for x / partial buffers, waiting for ring data, decoding, in
    // the CSR rounds, and at layer boundaries (descriptor + CSR staging waits)
    const bool prof = (p.dbg & 4u) && p.trace;
    long long c_xw = 0, c_fw = 0, c_dense = 0, c_csr = 0, c_top = 0, t_mark = clock64();
    auto lap = [&](long long& acc) {
        if (prof) {
            const long long t = clock64();
            acc += t - t_mark;
            t_mark = t;
        }
    };
    for (uint32_t l = 0; l < p.n_layers; ++l) {
        const uint32_t b = l & 1u;
        const StackLayerDesc& d = desc_wait(l).d;
        const Share sh = cta_share(d, cta);
        const uint32_t nrows = sh.nrows, NS = d.ns, cu = d.cu;
        (void)cu;
        if (cw == 0 && lane == 0) DSQ_TRACE(l, kTrConsStart);
        lap(c_top);
        mbar_wait(&xfull[b], (l >> 1) & 1u);
        if (l >= 2) mbar_wait(&pempty[b], ((l >> 1) - 1) & 1u);
        lap(c_xw);
        if (cw == 0 && lane == 0) DSQ_TRACE(l, kTrXReady);
        const uint16_t* xh = reinterpret_cast<const uint16_t*>(sm + p.off_x + b * p.x_bytes);
        const uint32_t* luts = reinterpret_cast<const uint32_t*>(sm + p.off_lut + b * p.lut_bytes);
        float* part = reinterpret_cast<float*>(sm + p.off_part) + size_t(b) * p.part_rows * NC;

        // CSR deltas: rounds distributed over the consumer warps; half of the
        // warps (alternating per layer) do theirs before the dense units
        auto csr_phase = [&]() {
            mbar_wait(&cfull[b], (l >> 1) & 1u);
            lap(c_top);
            const uint32_t* rp = reinterpret_cast<const uint32_t*>(sm + p.off_rp) + b * p.rp_words;
            const uint32_t e0 = rp[0], nz = rp[nrows] - e0;
            const bool staged = nz <= p.csr_cap - 4;
            const uint32_t* ent = staged ? reinterpret_cast<const uint32_t*>(sm + p.off_csr) +
                                               b * p.csr_cap + (e0 & 3u)
                                         : d.csr + e0;
            const uint32_t* hb = staged ? reinterpret_cast<const uint32_t*>(sm + p.off_hb) + b * p.hb_words
                                        : d.csr_heads;
            csr_rounds(e0, nz, ent, hb, staged ? ((e0 >> 5) & ~3u) : 0u, xh,
                       reinterpret_cast<float*>(sm + p.off_seg) + size_t(b) * p.seg_rounds * 32,
                       p.gseg + (size_t(cta) * 2 + b) * p.gseg_rounds * 32, p.seg_rounds, cw, NC,
                       lane);
            __syncwarp();
            lap(c_csr);
        };
        const bool csr_first = !(p.dbg & 8u) && ((cw + l) & 1u) != 0;
        if (csr_first) csr_phase();

        // dense units: warp cw owns the contiguous unit range [u0, u1) of the
        // CTA share (tile-major: unit u = (tile u / NS, span u % NS)), which
        // its own TMA ring brings in, cu units per chunk.  The accumulators
        // follow the warp across chunks and are flushed into part[cw][row]
        // on a tile change.
        const uint32_t U = sh.nt * NS;
        const uint32_t u0 = (cw * U) / NC, u1 = ((cw + 1) * U) / NC;
        uint32_t cur_tile = 0xffffffffu;
        Planes16 P;
        float d0[4] = {0.f, 0.f, 0.f, 0.f}, d1[4] = {0.f, 0.f, 0.f, 0.f};
        auto flush = [&]() {
            if (cur_tile != 0xffffffffu) {
                const float v = tile_rows_reduce(d0, d1, lane);
                if ((lane & 3) == 0 && lane < 16) part[cw * p.part_rows + cur_tile * kTileRows + trow] += v;
#pragma unroll
                for (int k = 0; k < 4; ++k) d0[k] = d1[k] = 0.f;
            }
        };
        for (uint32_t cb = u0; cb < u1; cb += cu) {
            lap(c_dense);
            mbar_wait(&full[cw * WS + cslot], cphase);
            lap(c_fw);
            const uint32_t* chunk = reinterpret_cast<const uint32_t*>(ring + size_t(cw * WS + cslot) * p.slot_bytes);
            uint32_t u = cb;
            const uint32_t ue = min(u1, cb + cu);
            if (!(p.dbg & 1u)) {
                uint32_t tile = u / NS, s = u - tile * NS;
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
                    load(sp, xs);
                    for (uint32_t k = s; k < s_end; ++k) {
                        uint32_t wc[BITS];
#pragma unroll
                        for (int q = 0; q < BITS; ++q) wc[q] = w[q];
                        const uint4 xac = xa, xbc = xb2;
                        sp += UW;
                        xs += kSpanCols;
                        if (k + 1 < s_end) load(sp, xs);
                        if constexpr (BITS == 3) {
                            span3_mma(wc[0], wc[1], wc[2], P.a, xac, xbc, d0, d1);
                        } else {
                            span4_mma(make_uint4(wc[0], wc[1], wc[2], wc[3]), P, xac, xbc, d0, d1);
                        }
                    }
                    u += s_end - s;
                    s = s_end;
                    if (s == NS) {
                        ++tile;
                        s = 0;
                    }
                }
            }
            // the slot's words are consumed (their values were used): refill
            // it with the next chunk of this warp's stream
            __syncwarp();
            if (++cslot == WS) {
                cslot = 0;
                cphase ^= 1u;
            }
            issue_next();
        }
        flush();
        if (cw == 0 && lane == 0) DSQ_TRACE(l, kTrDenseDone);
        lap(c_dense);
        if (!csr_first) csr_phase();
        __syncwarp();
        desc_release(l);
        if (lane == 0) {
            mbar_arrive(&pfull[b]);
            mbar_arrive(&bempty[b]);
        }
    }
    if (prof && lane == 0) {
        long long* o = reinterpret_cast<long long*>(p.trace) + (size_t(cta) * NC + cw) * 5;
        o[0] = c_xw;
        o[1] = c_fw;
        o[2] = c_dense;
        o[3] = c_csr;
        o[4] = c_top;
    }
}

cudaError_t launch_stack(const StackParams& p, cudaStream_t st, bool pdl) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(p.grid);
    cfg.blockDim = dim3((p.consumers + 3) * 32);
    cfg.dynamicSmemBytes = p.smem_bytes;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    static bool attr_done[6][64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    const int ci = p.consumers == 8 ? 0 : p.consumers == 16 ? 1 : 2;
    const int bi = (p.bits == 3 ? 0 : 1) * 3 + ci;
    using K = void (*)(StackParams);
    static const K kerns[6] = {stack_gemv<3, 8>, stack_gemv<3, 16>, stack_gemv<3, 24>,
                               stack_gemv<4, 8>, stack_gemv<4, 16>, stack_gemv<4, 24>};
    const K kern = kerns[bi];
    if (dev < 0 || dev >= 64 || !attr_done[bi][dev]) {
        int max_optin = 0;
        cudaDeviceGetAttribute(&max_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             max_optin);
        if (e != cudaSuccess) return e;
        if (dev >= 0 && dev < 64) attr_done[bi][dev] = true;
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
