// stack.cu -- K7: persistent multi-layer Dense-and-Sparse LUT-GEMV (sm_100a).
//
// One CTA per SM, all co-resident.  For every layer l of the stack each CTA
// owns a contiguous row range [r0, r1) (rows split evenly over the grid, so
// the balance granularity is one row and no output row is ever shared
// between CTAs -> no global merge, no floating-point atomics).
//
// Warp roles:
//   warp 0     producer: streams the CTA's row records of layer 0, 1, 2, ...
//              HBM -> shared-memory ring with cp.async.bulk (TMA bulk
//              engine), completion on mbarriers.  Weights never depend on x,
//              so it runs ahead across layer boundaries, bounded only by the
//              ring -- the HBM pipe stays busy while other warps wait on a
//              layer dependency.
//   warp 1     x-loader: stages the CTA's CSR slice (row_ptr + entries) and,
//              once the layer producing x is complete on ALL CTAs (grid-wide
//              completion counter, ld.acquire), the activation vector x into
//              a double-buffered shared-memory x buffer.
//   warps 2-17 consumers: (row, 32-group slice) pairs of each ring chunk are
//              split over the 16 warps (slice-major runs, rotating start for
//              balance); lane = group of 32 columns; per row the LUT byte
//              planes come from the record (one broadcast LDS.128), indices
//              are decoded with PRMT lookups and multiplied with fp16 x by
//              FHFMA into fp32.  Up to 4 rows are reduced at once with a
//              4-value butterfly; per-(row, slice) partials land in shared
//              memory and are summed in slice order (deterministic).  The
//              CSR deltas of the CTA's rows are processed in 32-entry rounds
//              with a segmented warp scan (skew-robust), then each row's
//              total is stored and the layer's completion counter bumped
//              (red.release.gpu).
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

namespace sqz {

__device__ __forceinline__ const StackLayerDesc& layer_desc(const StackParams& p, uint32_t l) {
    return l < kInlineLayers && p.n_layers <= kInlineLayers ? p.inl[l] : p.layers[l];
}

// 4-value butterfly: lane holds v[0..3] (partials of 4 rows over its group);
// afterwards lane 8*i holds the warp total of row i.  Fixed order.
__device__ __forceinline__ float reduce4(float v0, float v1, float v2, float v3, uint32_t lane) {
    const bool hi = lane & 16;
    float k0 = hi ? v2 : v0, k1 = hi ? v3 : v1;
    const float s0 = hi ? v0 : v2, s1 = hi ? v1 : v3;
    k0 += __shfl_xor_sync(0xffffffffu, s0, 16);
    k1 += __shfl_xor_sync(0xffffffffu, s1, 16);
    const bool b3 = lane & 8;
    float k = b3 ? k1 : k0;
    const float s = b3 ? k0 : k1;
    k += __shfl_xor_sync(0xffffffffu, s, 8);
    k += __shfl_xor_sync(0xffffffffu, k, 4);
    k += __shfl_xor_sync(0xffffffffu, k, 2);
    k += __shfl_xor_sync(0xffffffffu, k, 1);
    return k;
}

// Operands of one (row, 32-group slice) for one lane: LUT planes + words.
template <int BITS>
struct RowOps {
    uint4 pl[BITS == 3 ? 1 : 2];
    uint32_t w[BITS];
};

template <int BITS>
__device__ __forceinline__ void load_row(const uint32_t* rec, uint32_t g, bool on, RowOps<BITS>& o) {
    if constexpr (BITS == 3) {
        o.pl[0] = on ? *reinterpret_cast<const uint4*>(rec) : make_uint4(0, 0, 0, 0);
        const uint32_t* w = rec + 4 + 3 * g;
        o.w[0] = on ? w[0] : 0u;
        o.w[1] = on ? w[1] : 0u;
        o.w[2] = on ? w[2] : 0u;
    } else {
        o.pl[0] = on ? *reinterpret_cast<const uint4*>(rec) : make_uint4(0, 0, 0, 0);
        o.pl[1] = on ? *reinterpret_cast<const uint4*>(rec + 4) : make_uint4(0, 0, 0, 0);
        const uint4 w4 = on ? *reinterpret_cast<const uint4*>(rec + 8 + 4 * g) : make_uint4(0, 0, 0, 0);
        o.w[0] = w4.x;
        o.w[1] = w4.y;
        o.w[2] = w4.z;
        o.w[3] = w4.w;
    }
}

// zero operands decode to LUT entries 0.0 -> contribute exactly 0
template <int BITS>
__device__ __forceinline__ float row_dot(const RowOps<BITS>& o, const uint4 (&xv)[4]) {
    float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
    if constexpr (BITS == 3) {
        const Planes8 P{o.pl[0].x, o.pl[0].y, o.pl[0].z, o.pl[0].w};
        unit3(o.w[0], o.w[1], o.w[2], P, xv, a0, a1, a2, a3);
    } else {
        Planes16 P;
        P.a = Planes8{o.pl[0].x, o.pl[0].y, o.pl[0].z, o.pl[0].w};
        P.b = Planes8{o.pl[1].x, o.pl[1].y, o.pl[1].z, o.pl[1].w};
        const uint32_t ww[4] = {o.w[0], o.w[1], o.w[2], o.w[3]};
        unit4(ww, P, xv, a0, a1, a2, a3);
    }
    return (a0 + a1) + (a2 + a3);
}

// CTA row share from the host-precomputed quotient/remainder (no division)
struct Share {
    uint32_t r0, n, nch;
};
__device__ __forceinline__ Share cta_share(const StackLayerDesc& d, uint32_t cta) {
    Share s;
    const bool hi = cta < d.rr;
    s.r0 = cta * d.rq + (hi ? cta : d.rr);
    s.n = d.rq + (hi ? 1u : 0u);
    s.nch = hi ? d.nch_hi : d.nch_lo;
    return s;
}

// 2-value butterfly: lane 0 -> row 0 total, lane 16 -> row 1 total
__device__ __forceinline__ float reduce2(float v0, float v1, uint32_t lane) {
    const bool hi = lane & 16;
    float k = hi ? v1 : v0;
    const float s = hi ? v0 : v1;
    k += __shfl_xor_sync(0xffffffffu, s, 16);
    k += __shfl_xor_sync(0xffffffffu, k, 8);
    k += __shfl_xor_sync(0xffffffffu, k, 4);
    k += __shfl_xor_sync(0xffffffffu, k, 2);
    k += __shfl_xor_sync(0xffffffffu, k, 1);
    return k;
}
__device__ __forceinline__ float reduce1(float v) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    return v;
}

// warp-cooperative global -> shared copy with 8 loads in flight per lane
__device__ __forceinline__ void warp_stage(uint32_t* dst, const uint32_t* src, uint32_t n,
                                           uint32_t lane) {
    for (uint32_t base = 0; base < n; base += 256) {
        uint32_t v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const uint32_t i = base + u * 32 + lane;
            v[u] = i < n ? __ldg(src + i) : 0u;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const uint32_t i = base + u * 32 + lane;
            if (i < n) dst[i] = v[u];
        }
    }
}

__device__ __forceinline__ unsigned long long gtimer_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#define DSQ_TRACE(l, slot)                                                                 \
    do {                                                                                   \
        if (p.trace) p.trace[(size_t(blockIdx.x) * p.n_layers + (l)) * kTrSlots + (slot)] = \
            gtimer_ns();                                                                   \
    } while (0)

// CSR deltas of the CTA's rows: 32-entry rounds j = first, first+stride, ...
// of the CTA's contiguous entry slice; a lane starts a segment where a row
// starts (row starts found in parallel: each lane tests <= ceil(nrows/32) row
// pointers), then a segmented inclusive warp scan; round results go to segs.
__device__ __forceinline__ void csr_rounds(const uint32_t* rp, uint32_t nrows, const uint32_t* ent,
                                           const uint16_t* xh, float* segs, float* gseg,
                                           uint32_t seg_rounds, uint32_t first, uint32_t stride,
                                           uint32_t lane) {
    const uint32_t e0 = rp[0], nz = rp[nrows] - e0;
    const uint32_t rounds = (nz + 31) / 32;
    for (uint32_t j = first; j < rounds; j += stride) {
        const uint32_t base = e0 + j * 32;
        const uint32_t pi = j * 32 + lane;
        float prod = 0.f;
        if (pi < nz) {
            const uint32_t e = ent[pi];
            prod = fma_h(uint16_t(e >> 16), xh[e & 0xffffu], 0.f);
        }
        uint32_t mybits = 0;
        for (uint32_t r = lane; r < nrows; r += 32) {
            const uint32_t a = rp[r];
            if (a >= base && a < base + 32 && a < rp[r + 1]) mybits |= 1u << (a - base);
        }
        const uint32_t heads = __reduce_or_sync(0xffffffffu, mybits);
        const uint32_t upto = heads & (0xffffffffu >> (31 - lane));
        const uint32_t seg0 = upto ? (31u - __clz(upto)) : 0u;
        float v = prod;
#pragma unroll
        for (uint32_t off = 1; off < 32; off <<= 1) {
            const float t = __shfl_up_sync(0xffffffffu, v, off);
            if (lane >= seg0 + off) v += t;
        }
        float* dst = j < seg_rounds ? segs + j * 32 : gseg + (j - seg_rounds) * 32;
        dst[lane] = v;
    }
}

template <int BITS, int NC>
__global__ void __launch_bounds__((NC + 3) * 32, 1) stack_gemv(const __grid_constant__ StackParams p) {
    constexpr int kStackConsumers = NC;
    extern __shared__ __align__(1024) uint8_t sm[];
    // mbarriers: ring full/empty, then per buffer parity b in {0,1}
    uint64_t* full = reinterpret_cast<uint64_t*>(sm);
    uint64_t* empty = full + p.n_slots;
    uint64_t* xfull = empty + p.n_slots;   // x staged (TMA transaction count)
    uint64_t* cfull = xfull + 2;           // CSR slice staged (32 loader lanes)
    uint64_t* bempty = cfull + 2;          // x + CSR buffers free (consumers + finisher)
    uint64_t* pfull = bempty + 2;          // dense partials written (consumers)
    uint64_t* pempty = pfull + 2;          // partials consumed (finisher)
    uint8_t* ring = sm + p.off_ring;
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t cta = blockIdx.x, G = p.grid;

    if (threadIdx.x == 0) {
        for (uint32_t s = 0; s < p.n_slots; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kStackConsumers);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&xfull[b], 1);
            mbar_init(&cfull[b], 32);
            mbar_init(&bempty[b], kStackConsumers + 1);
            mbar_init(&pfull[b], kStackConsumers);
            mbar_init(&pempty[b], 1);
        }
        fence_barrier_init();
    }
    __syncthreads();

    // Warp roles.  The issue arbiter favours the highest warp id, so the
    // latency-critical control warps take the top ids: consumers 0..NC-1,
    // producer NC, loader NC+1, finisher NC+2.
    if (warp == NC) {
        // ---------------- producer: weights only, never waits on x ----------
        pdl_trigger();
        if (lane == 0) {
            const uint64_t policy = policy_evict_first();
            uint32_t slot = 0, phase = 0;
            for (uint32_t l = 0; l < p.n_layers; ++l) {
                const StackLayerDesc& d = layer_desc(p, l);
                const uint32_t rw = d.rw, cr = d.chunk_rows;
                const uint32_t* rec = d.rec;
                const Share sh = cta_share(d, cta);
                for (uint32_t c = 0; c < sh.nch; ++c) {
                    const uint32_t r = sh.r0 + c * cr;
                    const uint32_t n = min(cr, sh.n - c * cr);
                    const uint32_t bytes = n * rw * 4;
                    mbar_wait(&empty[slot], phase ^ 1u);
                    if (c == 0) DSQ_TRACE(l, kTrProdFirst);
                    mbar_arrive_expect_tx(&full[slot], bytes);
                    bulk_g2s(ring + size_t(slot) * p.slot_bytes, rec + size_t(r) * rw, bytes,
                             &full[slot], policy);
                    if (++slot == p.n_slots) {
                        slot = 0;
                        phase ^= 1u;
                    }
                }
            }
        }
        return;
    }

    if (warp == NC + 1) {
        // ---------------- loader: CSR slice + x, handles the dependency -------
        pdl_wait();
        pdl_trigger();
        for (uint32_t l = 0; l < p.n_layers; ++l) {
            const uint32_t b = l & 1u;
            if (l >= 2) mbar_wait(&bempty[b], ((l >> 1) - 1) & 1u);
            const StackLayerDesc& d = layer_desc(p, l);
            const Share sh = cta_share(d, cta);
            const uint32_t r0 = sh.r0, r1 = sh.r0 + sh.n;
            uint8_t* xb = sm + p.off_x + b * p.x_bytes;
            if (lane == 0) DSQ_TRACE(l, kTrLoaderStart);
            // x: one TMA bulk copy of the 16-byte-aligned body (+ scalar tail,
            // zero padding to the group count), completion on xfull[b]
            auto stage_x = [&]() {
                const uint32_t body = (d.cols / 8) * 16;  // bytes
                for (uint32_t i = body / 2 + lane; i < d.ng * 32; i += 32)
                    reinterpret_cast<uint16_t*>(xb)[i] = i < d.cols ? ld_cg_u16(d.x + i) : uint16_t(0);
                __syncwarp();
                if (lane == 0) {
                    fence_proxy_async_global();
                    mbar_arrive_expect_tx(&xfull[b], body);
                    if (body) bulk_g2s_plain(xb, d.x, body, &xfull[b]);
                }
            };
            if (d.dep == kNoDep) stage_x();  // external input: no wait at all
            uint32_t* rp = reinterpret_cast<uint32_t*>(sm + p.off_rp) + b * p.rp_words;
            warp_stage(rp, d.row_ptr + r0, r1 - r0 + 1, lane);
            __syncwarp();
            const uint32_t e0 = rp[0], e1 = rp[r1 - r0];
            if (e1 - e0 <= p.csr_cap) {
                uint32_t* cb = reinterpret_cast<uint32_t*>(sm + p.off_csr) + b * p.csr_cap;
                warp_stage(cb, d.csr + e0, e1 - e0, lane);
            }
            mbar_arrive(&cfull[b]);
            if (lane == 0) DSQ_TRACE(l, kTrCsrStaged);
            if (d.dep != kNoDep) {
                if (lane == 0) {
                    while (ld_acquire_gpu(p.counters + d.dep) < G) __nanosleep(20);
                    DSQ_TRACE(l, kTrDepMet);
                }
                __syncwarp();
                stage_x();
            }
            if (lane == 0) DSQ_TRACE(l, kTrXIssued);
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
            const StackLayerDesc& d = layer_desc(p, l);
            const Share sh = cta_share(d, cta);
            const uint32_t r0 = sh.r0, nrows = sh.n, S = d.nslices;
            const uint32_t* rp = reinterpret_cast<const uint32_t*>(sm + p.off_rp) + b * p.rp_words;
            // row totals: dense slices in order, then the row's CSR rounds
            mbar_wait(&pfull[b], ph);
            if (lane == 0) DSQ_TRACE(l, kTrAllDense);
            const uint32_t e0 = rp[0];
            const float* part = reinterpret_cast<const float*>(sm + p.off_part) +
                                size_t(b) * p.part_rows * p.part_stride;
            for (uint32_t i = lane; i < nrows; i += 32) {
                float s = 0.f;
                for (uint32_t cs = 0; cs < S; ++cs) s += part[i * p.part_stride + cs];
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

    // ---------------- consumers: dense LUT products only ----------------------
    pdl_wait();
    pdl_trigger();
    const uint32_t cw = warp;
    uint32_t slot = 0, phase = 0;
    for (uint32_t l = 0; l < p.n_layers; ++l) {
        const uint32_t b = l & 1u;
        const StackLayerDesc& d = layer_desc(p, l);
        const Share sh = cta_share(d, cta);
        const uint32_t nrows = sh.n, S = d.nslices, rw = d.rw, cr = d.chunk_rows;
        const uint32_t ng = d.ng;
        if (cw == 0 && lane == 0) DSQ_TRACE(l, kTrConsStart);
        mbar_wait(&xfull[b], (l >> 1) & 1u);
        if (l >= 2) mbar_wait(&pempty[b], ((l >> 1) - 1) & 1u);
        if (cw == 0 && lane == 0) DSQ_TRACE(l, kTrXReady);
        const uint4* xb = reinterpret_cast<const uint4*>(sm + p.off_x + b * p.x_bytes);
        float* part = reinterpret_cast<float*>(sm + p.off_part) + size_t(b) * p.part_rows * p.part_stride;

        for (uint32_t ci = 0; ci < sh.nch; ++ci) {
            const uint32_t rbase = ci * cr;  // local row of chunk start
            const uint32_t n = min(cr, nrows - rbase);
            mbar_wait(&full[slot], phase);
            const uint32_t* chunk = reinterpret_cast<const uint32_t*>(ring + size_t(slot) * p.slot_bytes);
            // (row, slice) pairs in slice-major order, an equal share per warp,
            // rotating which warps get the remainder
            const uint32_t P = n * S;
            const uint32_t wr = (cw + ci + l) % kStackConsumers;
            uint32_t q = (wr * P) / kStackConsumers;
            const uint32_t q1 = ((wr + 1) * P) / kStackConsumers;
            // cs = q / n without an integer division
            uint32_t cs = uint32_t(__fmul_rz(float(q), __frcp_rn(float(n))));
            if (cs * n > q) --cs;
            if ((cs + 1) * n <= q) ++cs;
            uint32_t ra = q - cs * n;
            while (q < q1) {
                const uint32_t rb_ = min(n, ra + (q1 - q));
                const uint32_t g = cs * 32 + lane;
                const bool gv = g < ng;
                uint4 xv[4];
#pragma unroll
                for (int j = 0; j < 4; ++j) xv[j] = gv ? xb[g * 4 + j] : make_uint4(0, 0, 0, 0);
                float* pcol = part + cs;
                uint32_t rr = ra;
                const uint32_t* rowp = chunk + size_t(ra) * rw;
                for (; rr + 4 <= rb_; rr += 4, rowp += 4 * rw) {
                    RowOps<BITS> ops[4];
#pragma unroll
                    for (int i = 0; i < 4; ++i) load_row<BITS>(rowp + i * rw, g, gv, ops[i]);
                    float v[4];
#pragma unroll
                    for (int i = 0; i < 4; ++i) v[i] = row_dot<BITS>(ops[i], xv);
                    const float t = reduce4(v[0], v[1], v[2], v[3], lane);
                    if ((lane & 7) == 0) pcol[(rbase + rr + (lane >> 3)) * p.part_stride] = t;
                }
                if (rr + 2 <= rb_) {
                    RowOps<BITS> o0, o1;
                    load_row<BITS>(rowp, g, gv, o0);
                    load_row<BITS>(rowp + rw, g, gv, o1);
                    const float t = reduce2(row_dot<BITS>(o0, xv), row_dot<BITS>(o1, xv), lane);
                    if ((lane & 15) == 0) pcol[(rbase + rr + (lane >> 4)) * p.part_stride] = t;
                    rr += 2;
                    rowp += 2 * rw;
                }
                if (rr < rb_) {
                    RowOps<BITS> o0;
                    load_row<BITS>(rowp, g, gv, o0);
                    const float t = reduce1(row_dot<BITS>(o0, xv));
                    if (lane == 0) pcol[(rbase + rr) * p.part_stride] = t;
                }
                q += rb_ - ra;
                ++cs;
                ra = 0;
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[slot]);
            if (++slot == p.n_slots) {
                slot = 0;
                phase ^= 1u;
            }
        }
        if (cw == 0 && lane == 0) DSQ_TRACE(l, kTrDenseDone);

        // CSR deltas: rounds distributed over the consumer warps
        mbar_wait(&cfull[b], (l >> 1) & 1u);
        {
            const uint32_t* rp = reinterpret_cast<const uint32_t*>(sm + p.off_rp) + b * p.rp_words;
            const uint32_t e0 = rp[0], nz = rp[nrows] - e0;
            const uint32_t* ent = nz <= p.csr_cap
                                      ? reinterpret_cast<const uint32_t*>(sm + p.off_csr) + b * p.csr_cap
                                      : d.csr + e0;
            csr_rounds(rp, nrows, ent, reinterpret_cast<const uint16_t*>(xb),
                       reinterpret_cast<float*>(sm + p.off_seg) + size_t(b) * p.seg_rounds * 32,
                       p.gseg + (size_t(cta) * 2 + b) * p.gseg_rounds * 32, p.seg_rounds, cw,
                       kStackConsumers, lane);
        }
        __syncwarp();
        if (lane == 0) {
            mbar_arrive(&pfull[b]);
            mbar_arrive(&bempty[b]);
        }
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
// K5/K6 for the row-record layout: decode indices / values of every (row, col)
// ---------------------------------------------------------------------------
template <int BITS, int MODE>  // MODE 0: u16 indices, 1: fp16 values, 2: fp32 values
__global__ void decode_records(const uint32_t* __restrict__ rec, uint32_t rows, uint32_t cols,
                               uint32_t ng, uint32_t ngp, uint32_t rw, void* out) {
    const size_t t = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= size_t(rows) * ng) return;
    const uint32_t row = uint32_t(t / ng), g = uint32_t(t % ng);
    const uint32_t* r = rec + size_t(row) * rw;
    constexpr uint32_t LW = BITS == 3 ? 4 : 8;
    uint32_t w[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) w[i] = (i < BITS) ? r[LW + g * BITS + i] : 0u;
    // fp16 entries back from the byte planes
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
        const uint32_t c = g * kGroupCols + j;
        if (c >= cols) break;
        uint32_t idx;
        if constexpr (BITS == 3) {
            if (j < 24) {
                idx = (w[j >> 3] >> (4 * (j & 7))) & 7u;
            } else {
                const int nn = j - 24;
                idx = ((w[0] >> (4 * nn + 3)) & 1u) | (((w[1] >> (4 * nn + 3)) & 1u) << 1) |
                      (((w[2] >> (4 * nn + 3)) & 1u) << 2);
            }
        } else {
            idx = (w[j >> 3] >> (4 * (j & 7))) & 15u;
        }
        const size_t o = size_t(row) * cols + c;
        if (MODE == 0) static_cast<uint16_t*>(out)[o] = uint16_t(idx);
        else if (MODE == 1) static_cast<uint16_t*>(out)[o] = lut[idx];
        else static_cast<float*>(out)[o] = __half2float(__ushort_as_half(lut[idx]));
    }
}

cudaError_t launch_decode_records(int mode, uint32_t bits, const uint32_t* rec, uint32_t rows,
                                  uint32_t cols, uint32_t ng, uint32_t ngp, uint32_t rw,
                                  void* out, cudaStream_t st) {
    const size_t n = size_t(rows) * ng;
    const uint32_t blocks = uint32_t((n + 255) / 256);
#define DSQ_DEC(B, M) decode_records<B, M><<<blocks, 256, 0, st>>>(rec, rows, cols, ng, ngp, rw, out)
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
