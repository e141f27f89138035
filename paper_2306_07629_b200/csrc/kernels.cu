// kernels.cu -- sm_100a kernels of the Dense-and-Sparse LUT-GEMV hot path.
//
//   K1/K3  fused_gemv<BITS, DENSE, SPARSE>   LUT-GEMV (+ CSR outlier SpMV) in
//          one launch.  Replaces dsq::lut_matvec / fused_dns_matvec
//          (reference kernels.cpp:18-33, 51-67, 108-141); with DENSE=false it
//          is K2, the CSR SpMV (kernels.cpp:35-41, 69-85).
//   K4     dense_gemv_f16                    fp16 dense GEMV (dense_matvec,
//          kernels.cpp:43-47, 87-106; the bench "reference" kernel).
//   K5/K6  unpack_tiled / dequant_tiled      bit-exact debug decoders
//          (unpack packfmt.cpp:57-80, ref::dequant_dense kernels.cpp:149-159).
//
// Fused kernel design (B200):
//   * Work = units of (32 rows x 32 cols).  The host scheduler (api.cpp)
//     splits the unit sequence (row-block major) into one contiguous,
//     cost-balanced range per warp ("stream-K"), so every SM gets the same
//     bytes regardless of layer shape, and CSR work (weighted by nnz) rides
//     along with the dense work of its row block -> outlier-skew robust.
//   * Each warp streams its contiguous byte range HBM -> shared memory with
//     cp.async.bulk (TMA bulk engine) into a kStages-deep ring completed on
//     mbarriers; the copies for the first stages are issued BEFORE
//     griddepcontrol.wait, so under programmatic dependent launch the weight
//     stream of layer i+1 starts while layer i drains.
//   * lane = row: each lane keeps its row's 8/16 fp16 centroids as byte
//     planes in registers and decodes 4 weights with 4 PRMT (2 lookups + 2
//     interleaves); the 3-bit packer layout makes the selectors nearly free.
//   * products fp16 x fp16 are exact in fp32 and accumulated in fp32 with the
//     sm_100 mixed-precision FMA (fma.rn.f32.f16 -> SASS FHFMA).
//   * A row block split across warps is merged without floating-point
//     atomics: partials go to a scratch slot, an integer arrival counter
//     picks the last warp, which sums the partials in segment order
//     (deterministic) and writes y.  Counters self-reset.
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "layout.hpp"
#include "ptx.cuh"

namespace sqz {

// Cooperative CSR window of one row block: entries [c0, c1) of the rows
// rb*32 .. rb*32+31 (lane = row).  Returns lane's row contribution.
// Segmented warp scan, fixed order -> deterministic; skew-robust because the
// 32 lanes always process 32 consecutive entries, whatever their rows.
// `e_first` is the (prefetched) entry c0 + lane of the first round.
__device__ __forceinline__ float csr_window(const uint32_t* __restrict__ csr, const uint16_t* x,
                                            uint32_t c0, uint32_t c1, uint32_t rp_l,
                                            uint32_t rp_n, uint32_t lane, uint32_t e_first) {
    float rowsum = 0.f;
    const bool nonempty = rp_l < rp_n;
    for (uint32_t base = c0; base < c1; base += 32) {
        const uint32_t p = base + lane;
        float prod = 0.f;
        if (p < c1) {
            const uint32_t e = (base == c0) ? e_first : __ldg(csr + p);
            const uint16_t xv = ldg_nc_u16(x + (e & 0xffffu));
            prod = fma_h(uint16_t(e >> 16), xv, 0.f);
        }
        const uint32_t mybit =
            (nonempty && rp_l >= base && rp_l < base + 32) ? (1u << (rp_l - base)) : 0u;
        const uint32_t heads = __reduce_or_sync(0xffffffffu, mybit);
        const uint32_t upto = heads & (0xffffffffu >> (31 - lane));
        const uint32_t seg0 = upto ? (31u - __clz(upto)) : 0u;
        float v = prod;
#pragma unroll
        for (uint32_t off = 1; off < 32; off <<= 1) {
            const float t = __shfl_up_sync(0xffffffffu, v, off);
            if (lane >= seg0 + off) v += t;
        }
        // my row's entries in this round: [max(rp_l, base, c0), min(rp_n, base+32, c1))
        const uint32_t lo = max(max(rp_l, base), c0);
        const uint32_t hi = min(min(rp_n, base + 32), c1);
        const uint32_t src = (hi > lo) ? (hi - 1 - base) : 0u;
        const float got = __shfl_sync(0xffffffffu, v, src);
        if (hi > lo) rowsum += got;
    }
    return rowsum;
}

// release-only arrival: orders this warp's partial stores (made visible to
// lane 0 by __syncwarp) before the count; the last arriver reads the other
// partials with ld.global.cg (L2, never a stale L1 line), so no acquire-side
// L1 invalidation is needed.
__device__ __forceinline__ uint32_t atom_add_release_gpu(uint32_t* p, uint32_t v) {
    uint32_t old;
    asm volatile("atom.release.gpu.global.add.u32 %0, [%1], %2;"
                 : "=r"(old)
                 : "l"(p), "r"(v)
                 : "memory");
    return old;
}

// largest w with W.u0[w] <= u
__device__ __forceinline__ uint32_t find_worker(const WorkTable& W, uint32_t u) {
    uint32_t lo = 0, hi = W.n;
    while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        if (W.u0[mid] <= u) lo = mid;
        else hi = mid;
    }
    return lo;
}

// Per-segment metadata (row LUT, merge bookkeeping, CSR bounds).  Loaded one
// segment ahead -- the first one before griddepcontrol.wait -- so no warp
// waits on a metadata round trip at a segment start.
struct SegMeta {
    uint4 lut0, lut1;
    uint32_t a, b, rp_l, rp_n;
};

template <int BITS, bool DENSE, bool SPARSE>
__device__ __forceinline__ void load_meta(const LayerParams& P, uint32_t rb, uint32_t lane,
                                          SegMeta& m) {
    const uint32_t row = rb * kRowBlock + lane;
    if constexpr (DENSE && (BITS == 3 || BITS == 4)) {
        const uint16_t* lr = P.lut + size_t(row) * (1u << BITS);
        m.lut0 = ldg_nc_v4(lr);
        if constexpr (BITS == 4) m.lut1 = ldg_nc_v4(lr + 8);
    }
    if constexpr (SPARSE) {
        const uint32_t r0 = min(rb * kRowBlock, P.rows);
        const uint32_t r1 = min(r0 + kRowBlock, P.rows);
        m.a = __ldg(P.row_ptr + r0);
        m.b = __ldg(P.row_ptr + r1);
        m.rp_l = __ldg(P.row_ptr + min(row, P.rows));
        m.rp_n = __ldg(P.row_ptr + min(row + 1, P.rows));
    }
}

// ---------------------------------------------------------------------------
// K1/K2/K3: fused LUT-GEMV + CSR
// ---------------------------------------------------------------------------
template <int BITS, bool DENSE, bool SPARSE, typename YT>
__global__ void __launch_bounds__(kWarpsPerCta * 32, 2)
    fused_gemv(const LayerParams P, const __grid_constant__ WorkTable W,
               const uint16_t* __restrict__ x, YT* __restrict__ y) {
    constexpr uint32_t WPU = BITS;                       // words per lane per unit
    constexpr uint32_t UNIT_WORDS = WPU * 32;            // words per unit
    constexpr uint32_t STAGE_WORDS = kChunkUnits * UNIT_WORDS;
    extern __shared__ __align__(128) uint8_t smem_raw[];
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t warp = threadIdx.x >> 5;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw) + warp * kStages;
    uint32_t* stage_base = reinterpret_cast<uint32_t*>(smem_raw + kWarpsPerCta * kStages * 8) +
                           warp * (kStages * STAGE_WORDS);
    const uint32_t worker = blockIdx.x * kWarpsPerCta + warp;
    const bool active = worker < W.n;
    uint32_t u0 = 0, u1 = 0;
    if (active) {
        u0 = W.u0[worker];
        u1 = W.u0[worker + 1];
    }
    const uint32_t K = u1 - u0;
    const uint32_t nchunks = (K + kChunkUnits - 1) / kChunkUnits;
    // everything below until pdl_wait() reads only layer-constant data
    // (weights, LUTs, CSR structure, schedule) -> overlaps the previous grid
    SegMeta cur{};
    if (active) load_meta<BITS, DENSE, SPARSE>(P, u0 / P.ng, lane, cur);
    uint64_t policy = 0;
    if (DENSE) {
        policy = policy_evict_first();
        if (lane == 0) {
            for (int s = 0; s < kStages; ++s) mbar_init(&bars[s], 1);
            fence_barrier_init();
        }
        __syncwarp();
        if (lane == 0) {
            for (uint32_t c = 0; c < nchunks && c < uint32_t(kStages); ++c) {
                const uint32_t n = min(uint32_t(kChunkUnits), K - c * kChunkUnits);
                const uint32_t bytes = n * UNIT_WORDS * 4;
                mbar_arrive_expect_tx(&bars[c], bytes);
                bulk_g2s(stage_base + c * STAGE_WORDS,
                         P.words + size_t(u0 + c * kChunkUnits) * UNIT_WORDS, bytes, &bars[c],
                         policy);
            }
        }
    }
    pdl_wait();
    pdl_trigger();
    if (!active) return;

    uint32_t k = 0;  // unit counter within this worker's range
    uint32_t u = u0;
    const uint32_t rb_first = u0 / P.ng;
    const uint32_t* my_stage = stage_base + lane;
    while (u < u1) {
        const uint32_t rb = u / P.ng;
        const uint32_t seg_end = min(u1, (rb + 1) * P.ng);
        const uint32_t g0 = u - rb * P.ng;
        const uint32_t g1 = seg_end - rb * P.ng;
        const uint32_t row = rb * kRowBlock + lane;
        SegMeta nxt{};
        if (seg_end < u1) load_meta<BITS, DENSE, SPARSE>(P, rb + 1, lane, nxt);
        uint32_t c0 = 0, c1 = 0, e_first = 0;
        if constexpr (SPARSE) {
            c0 = cur.a + uint32_t((uint64_t(cur.b - cur.a) * g0) / P.ng);
            c1 = cur.a + uint32_t((uint64_t(cur.b - cur.a) * g1) / P.ng);
            if (c0 + lane < c1) e_first = __ldg(P.csr + c0 + lane);
        }

        float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
        if constexpr (DENSE) {
            const uint16_t* lut_row = P.lut + size_t(row) * (1u << BITS);
            Planes8 P8;
            Planes16 P16;
            if constexpr (BITS == 3) {
                P8 = make_planes8(cur.lut0);
            } else if constexpr (BITS == 4) {
                P16.a = make_planes8(cur.lut0);
                P16.b = make_planes8(cur.lut1);
            }
            for (uint32_t g = g0; g < g1; ++g, ++k) {
                const uint32_t c = k / kChunkUnits;
                const uint32_t slot = c % kStages;
                const uint32_t within = k - c * kChunkUnits;
                uint4 xv[4];
                load_x(x, g, P.cols, xv);
                if (within == 0) mbar_wait(&bars[slot], (c / kStages) & 1u);
                const uint32_t* sw = my_stage + slot * STAGE_WORDS + within * UNIT_WORDS;
                if constexpr (BITS == 3) {
                    unit3(sw[0], sw[32], sw[64], P8, xv, a0, a1, a2, a3);
                } else if constexpr (BITS == 4) {
                    const uint32_t w[4] = {sw[0], sw[32], sw[64], sw[96]};
                    unit4(w, P16, xv, a0, a1, a2, a3);
                } else {
                    uint32_t w[8];
#pragma unroll
                    for (int i = 0; i < 8; ++i) w[i] = (i < BITS) ? sw[i * 32] : 0u;
                    unit_generic<BITS>(w, lut_row, xv, a0, a1);
                }
                // recycle the stage after its last unit
                if (within == kChunkUnits - 1 || k + 1 == K) {
                    __syncwarp();
                    const uint32_t cn = c + kStages;
                    if (lane == 0 && cn < nchunks) {
                        fence_proxy_async();
                        const uint32_t n = min(uint32_t(kChunkUnits), K - cn * kChunkUnits);
                        const uint32_t bytes = n * UNIT_WORDS * 4;
                        mbar_arrive_expect_tx(&bars[slot], bytes);
                        bulk_g2s(stage_base + slot * STAGE_WORDS,
                                 P.words + size_t(u0 + cn * kChunkUnits) * UNIT_WORDS, bytes,
                                 &bars[slot], policy);
                    }
                }
            }
        } else {
            k += g1 - g0;
        }
        float part = (a0 + a1) + (a2 + a3);
        if constexpr (SPARSE) {
            if (c1 > c0) part += csr_window(P.csr, x, c0, c1, cur.rp_l, cur.rp_n, lane, e_first);
        }
        // merge (atomic-free in floating point)
        if (g0 == 0 && g1 == P.ng) {  // this warp owns the whole row block
            if (row < P.rows) store_y<YT>(y, row, part);
        } else {
            float* scr = P.scratch + size_t(2 * worker + (rb == rb_first ? 0 : 1)) * kRowBlock;
            scr[lane] = part;
            __syncwarp();
            const uint32_t fw = find_worker(W, rb * P.ng);
            const uint32_t lw = find_worker(W, (rb + 1) * P.ng - 1);
            uint32_t old = 0;
            if (lane == 0) old = atom_add_release_gpu(P.counters + rb, 1u);
            old = __shfl_sync(0xffffffffu, old, 0);
            if (old == lw - fw) {  // last of the nseg = lw - fw + 1 arrivals
                float sum = 0.f;
                for (uint32_t t = fw; t <= lw; ++t) {
                    const uint32_t which = (W.u0[t] / P.ng == rb) ? 0u : 1u;
                    const float v = (t == worker)
                                        ? part
                                        : ld_cg_f32(P.scratch +
                                                    size_t(2 * t + which) * kRowBlock + lane);
                    sum += v;
                }
                if (row < P.rows) store_y<YT>(y, row, sum);
                if (lane == 0) P.counters[rb] = 0;
            }
        }
        cur = nxt;
        u = seg_end;
    }
}

// ---------------------------------------------------------------------------
// K4: dense fp16 GEMV  y[r] = sum_c W[r][c] x[c]   (warp per row, fp32 acc)
// ---------------------------------------------------------------------------
template <typename YT>
__global__ void __launch_bounds__(256)
    dense_gemv_f16(const uint16_t* __restrict__ w, uint32_t rows, uint32_t cols,
                   const uint16_t* __restrict__ x, YT* __restrict__ y) {
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
    pdl_wait();
    pdl_trigger();
    const bool vec = (cols % 8 == 0);
    for (uint32_t r = gw; r < rows; r += nw) {
        const uint16_t* wr = w + size_t(r) * cols;
        float a0 = 0.f, a1 = 0.f;
        if (vec) {
            const uint32_t nv = cols / 8;
            for (uint32_t v = lane; v < nv; v += 32) {
                const uint4 wv = ldg_nc_v4(wr + v * 8);
                const uint4 xv = ldg_nc_v4(x + v * 8);
                a0 = fma_lo(wv.x, xv.x, a0);
                a1 = fma_hi(wv.x, xv.x, a1);
                a0 = fma_lo(wv.y, xv.y, a0);
                a1 = fma_hi(wv.y, xv.y, a1);
                a0 = fma_lo(wv.z, xv.z, a0);
                a1 = fma_hi(wv.z, xv.z, a1);
                a0 = fma_lo(wv.w, xv.w, a0);
                a1 = fma_hi(wv.w, xv.w, a1);
            }
        } else {
            for (uint32_t c = lane; c < cols; c += 32) a0 = fma_h(wr[c], x[c], a0);
        }
        float s = a0 + a1;
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
        if (lane == 0) store_y<YT>(y, r, s);
    }
}

// ---------------------------------------------------------------------------
// K5 / K6: decode the tiled layout (one thread = one (row, group))
// ---------------------------------------------------------------------------
template <int BITS>
__device__ __forceinline__ uint32_t tiled_index(const uint32_t (&w)[8], int j) {
    if constexpr (BITS == 3) {
        if (j < 24) return (w[j >> 3] >> (4 * (j & 7))) & 7u;
        const int n = j - 24;
        return ((w[0] >> (4 * n + 3)) & 1u) | (((w[1] >> (4 * n + 3)) & 1u) << 1) |
               (((w[2] >> (4 * n + 3)) & 1u) << 2);
    } else if constexpr (BITS == 4) {
        return (w[j >> 3] >> (4 * (j & 7))) & 15u;
    } else {
        const int bp = j * BITS;
        const int wi = bp >> 5, off = bp & 31;
        uint32_t v = w[wi] >> off;
        if (off + BITS > 32) v |= w[wi + 1] << (32 - off);
        return v & ((1u << BITS) - 1u);
    }
}

template <int BITS, int MODE>  // MODE 0: u16 indices, 1: fp16 values, 2: fp32 values
__global__ void decode_tiled(const LayerParams P, void* out) {
    const size_t t = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const size_t n_units = size_t(P.n_rb) * P.ng;
    if (t >= n_units * 32) return;
    const uint32_t lane = t & 31;
    const size_t u = t >> 5;
    const uint32_t rb = uint32_t(u / P.ng), g = uint32_t(u % P.ng);
    const uint32_t row = rb * kRowBlock + lane;
    if (row >= P.rows) return;
    uint32_t w[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) w[i] = (i < BITS) ? P.words[u * BITS * 32 + i * 32 + lane] : 0u;
    const uint16_t* lut_row = P.lut + size_t(row) * (1u << BITS);
    for (int j = 0; j < 32; ++j) {
        const uint32_t c = g * kGroupCols + j;
        if (c >= P.cols) break;
        const uint32_t idx = tiled_index<BITS>(w, j);
        const size_t o = size_t(row) * P.cols + c;
        if (MODE == 0) {
            static_cast<uint16_t*>(out)[o] = uint16_t(idx);
        } else if (MODE == 1) {
            static_cast<uint16_t*>(out)[o] = lut_row[idx];
        } else {
            static_cast<float*>(out)[o] = __half2float(__ushort_as_half(lut_row[idx]));
        }
    }
}

__global__ void f32_to_f16(const float* __restrict__ in, uint16_t* __restrict__ out, uint32_t n) {
    pdl_wait();
    pdl_trigger();
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        out[i] = __half_as_ushort(__float2half_rn(in[i]));
}

// ---------------------------------------------------------------------------
// host-side launchers (called from api.cpp)
// ---------------------------------------------------------------------------
size_t fused_smem_bytes(uint32_t bits) {
    return size_t(kWarpsPerCta) * kStages * 8 +
           size_t(kWarpsPerCta) * kStages * kChunkUnits * bits * 32 * 4;
}

template <int BITS, bool D, bool S, typename YT>
static cudaError_t launch_fused_t(const LayerParams& P, const WorkTable& Wt, const uint16_t* x,
                                  void* y, uint32_t ctas, cudaStream_t st, bool pdl) {
    auto kern = fused_gemv<BITS, D, S, YT>;
    const size_t smem = fused_smem_bytes(BITS);
    // the opt-in smem attribute is per function and device: set it once
    static bool attr_done[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64 || !attr_done[dev]) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             int(smem));
        if (e != cudaSuccess) return e;
        if (dev >= 0 && dev < 64) attr_done[dev] = true;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(ctas);
    cfg.blockDim = dim3(kWarpsPerCta * 32);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, P, Wt, x, static_cast<YT*>(y));
}

template <int BITS, typename YT>
static cudaError_t launch_bits(int mode, const LayerParams& P, const WorkTable& Wt,
                               const uint16_t* x, void* y, uint32_t ctas, cudaStream_t st,
                               bool pdl) {
    switch (mode) {
        case 0: return launch_fused_t<BITS, true, false, YT>(P, Wt, x, y, ctas, st, pdl);
        case 1: return launch_fused_t<BITS, false, true, YT>(P, Wt, x, y, ctas, st, pdl);
        default: return launch_fused_t<BITS, true, true, YT>(P, Wt, x, y, ctas, st, pdl);
    }
}

template <typename YT>
static cudaError_t launch_y(int mode, const LayerParams& P, const WorkTable& Wt,
                            const uint16_t* x, void* y, uint32_t ctas, cudaStream_t st,
                            bool pdl) {
    switch (P.bits) {
        case 1: return launch_bits<1, YT>(mode, P, Wt, x, y, ctas, st, pdl);
        case 2: return launch_bits<2, YT>(mode, P, Wt, x, y, ctas, st, pdl);
        case 3: return launch_bits<3, YT>(mode, P, Wt, x, y, ctas, st, pdl);
        case 4: return launch_bits<4, YT>(mode, P, Wt, x, y, ctas, st, pdl);
        case 5: return launch_bits<5, YT>(mode, P, Wt, x, y, ctas, st, pdl);
        case 6: return launch_bits<6, YT>(mode, P, Wt, x, y, ctas, st, pdl);
        case 7: return launch_bits<7, YT>(mode, P, Wt, x, y, ctas, st, pdl);
        default: return launch_bits<8, YT>(mode, P, Wt, x, y, ctas, st, pdl);
    }
}

// mode: 0 = LUT only (K1), 1 = CSR only (K2), 2 = fused (K3); y_f16 selects fp16 output
cudaError_t launch_fused(int mode, const LayerParams& P, const WorkTable& Wt, const uint16_t* x,
                         void* y, bool y_f16, uint32_t ctas, cudaStream_t st, bool pdl) {
    return y_f16 ? launch_y<__half>(mode, P, Wt, x, y, ctas, st, pdl)
                 : launch_y<float>(mode, P, Wt, x, y, ctas, st, pdl);
}

cudaError_t launch_dense(const uint16_t* w, uint32_t rows, uint32_t cols, const uint16_t* x,
                         void* y, bool y_f16, int num_sms, cudaStream_t st, bool pdl) {
    cudaLaunchConfig_t cfg = {};
    const uint32_t want = (rows + 7) / 8;
    cfg.gridDim = dim3(std::min<uint32_t>(want, uint32_t(num_sms) * 8));
    cfg.blockDim = dim3(256);
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (y_f16)
        return cudaLaunchKernelEx(&cfg, dense_gemv_f16<__half>, w, rows, cols, x,
                                  static_cast<__half*>(y));
    return cudaLaunchKernelEx(&cfg, dense_gemv_f16<float>, w, rows, cols, x,
                              static_cast<float*>(y));
}

// ---------------------------------------------------------------------------
// Grouped LUTs (groups_per_row > 1, the reference's grouping ablation,
// packfmt.hpp:28-31): the reference packed layout read directly (LSB-first
// bitstream rows, packfmt.cpp:40-53) and lut_at(r, c) = luts[(r * groups +
// c / gcols) * K], as in lut_row_dot (kernels.cpp:18-33).  One warp per row,
// exact fp16 x fp16 products accumulated in fp32.  MODE 0 LUT, 1 CSR, 2 fused.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t grouped_index(const uint8_t* row, uint32_t stride, uint32_t c,
                                                  uint32_t bits) {
    const uint32_t bp = c * bits, b = bp >> 3;
    const uint32_t w = uint32_t(row[b]) | (b + 1 < stride ? uint32_t(row[b + 1]) << 8 : 0u);
    return (w >> (bp & 7u)) & ((1u << bits) - 1u);
}

template <typename YT, int MODE>
__global__ void grouped_gemv(const GroupedParams p, const uint16_t* __restrict__ x,
                             YT* __restrict__ y) {
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    pdl_wait();
    pdl_trigger();
    if (r >= p.rows) return;
    const uint32_t K = 1u << p.bits;
    float acc = 0.f;
    if (MODE != 1) {
        const uint8_t* row = p.payload + size_t(r) * p.stride;
        const uint16_t* lr = p.lut + size_t(r) * p.groups * K;
        for (uint32_t c = lane; c < p.cols; c += 32) {
            const uint32_t idx = grouped_index(row, p.stride, c, p.bits);
            acc = fma_h(lr[(c / p.gcols) * K + idx], x[c], acc);
        }
    }
    if (MODE != 0) {
        for (uint32_t q = p.row_ptr[r] + lane; q < p.row_ptr[r + 1]; q += 32) {
            const uint32_t e = p.csr[q];
            acc = fma_h(uint16_t(e >> 16), x[e & 0xffffu], acc);
        }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
    if (lane == 0) store_y<YT>(y, r, acc);
}

// K5 / K6 for grouped layers: MODE 0 u16 indices, 1 fp16 values, 2 fp32 values
template <int MODE>
__global__ void grouped_decode(const GroupedParams p, void* out) {
    const size_t t = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= size_t(p.rows) * p.cols) return;
    const uint32_t r = uint32_t(t / p.cols), c = uint32_t(t % p.cols);
    const uint32_t idx = grouped_index(p.payload + size_t(r) * p.stride, p.stride, c, p.bits);
    const uint16_t h = p.lut[(size_t(r) * p.groups + c / p.gcols) * (1u << p.bits) + idx];
    if (MODE == 0) static_cast<uint16_t*>(out)[t] = uint16_t(idx);
    else if (MODE == 1) static_cast<uint16_t*>(out)[t] = h;
    else static_cast<float*>(out)[t] = __half2float(__ushort_as_half(h));
}

cudaError_t launch_grouped(int mode, const GroupedParams& p, const uint16_t* x, void* y, bool y_f16,
                           cudaStream_t st, bool pdl) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((p.rows + 7) / 8);
    cfg.blockDim = dim3(256);
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
#define DSQ_G(T, M) cudaLaunchKernelEx(&cfg, grouped_gemv<T, M>, p, x, static_cast<T*>(y))
    if (y_f16) return mode == 0 ? DSQ_G(__half, 0) : mode == 1 ? DSQ_G(__half, 1) : DSQ_G(__half, 2);
    return mode == 0 ? DSQ_G(float, 0) : mode == 1 ? DSQ_G(float, 1) : DSQ_G(float, 2);
#undef DSQ_G
}

cudaError_t launch_grouped_decode(int mode, const GroupedParams& p, void* out, cudaStream_t st) {
    const size_t n = size_t(p.rows) * p.cols;
    const uint32_t blocks = uint32_t((n + 255) / 256);
    if (mode == 0) grouped_decode<0><<<blocks, 256, 0, st>>>(p, out);
    else if (mode == 1) grouped_decode<1><<<blocks, 256, 0, st>>>(p, out);
    else grouped_decode<2><<<blocks, 256, 0, st>>>(p, out);
    return cudaGetLastError();
}

// dequantize_layer (pipeline.cpp:49-75), second half: after the LUT dequant
// (K6, fp32) every extracted position becomes lut_row[0] + delta, one fp32
// addition like the reference's float arithmetic (the widened fp16 operands
// are exact).  One warp per row, entries in CSR order.
__global__ void apply_deltas(const uint32_t* __restrict__ row_ptr, const uint32_t* __restrict__ csr,
                             const uint16_t* __restrict__ lut, uint32_t K, uint32_t groups,
                             uint32_t gcols, uint32_t rows, uint32_t cols, float* __restrict__ w) {
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (r >= rows) return;
    for (uint32_t q = row_ptr[r] + lane; q < row_ptr[r + 1]; q += 32) {
        const uint32_t e = csr[q], c = e & 0xffffu;
        // lut_at(r, c)[0]: the codebook of c's group (packfmt.hpp:28-31)
        const float l0 = __half2float(__ushort_as_half(lut[(size_t(r) * groups + c / gcols) * K]));
        const float d = __half2float(__ushort_as_half(uint16_t(e >> 16)));
        w[size_t(r) * cols + c] = __fadd_rn(l0, d);
    }
}

cudaError_t launch_apply_deltas(const uint32_t* row_ptr, const uint32_t* csr, const uint16_t* lut,
                                uint32_t K, uint32_t groups, uint32_t gcols, uint32_t rows,
                                uint32_t cols, float* w, cudaStream_t st) {
    apply_deltas<<<(rows + 7) / 8, 256, 0, st>>>(row_ptr, csr, lut, K, groups, gcols, rows, cols,
                                                 w);
    return cudaGetLastError();
}

// dense_matvec with fp32 weights (kernels.cpp:43-47, 87-106): the products
// double(m) * double(x) are exact, accumulated in fp64.  One warp per row.
__global__ void dense_gemv_f32(const float* __restrict__ w, uint32_t rows, uint32_t cols,
                               const float* __restrict__ x, double* __restrict__ y) {
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t r = gw; r < rows; r += nw) {
        const float* wr = w + size_t(r) * cols;
        double a = 0.0;
        for (uint32_t c = lane; c < cols; c += 32) a = fma(double(wr[c]), double(x[c]), a);
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) a += __shfl_xor_sync(0xffffffffu, a, off);
        if (lane == 0) y[r] = a;
    }
}

cudaError_t launch_dense_f32(const float* w, uint32_t rows, uint32_t cols, const float* x,
                             double* y, int num_sms, cudaStream_t st) {
    const uint32_t blocks = std::min<uint32_t>((rows + 7) / 8, uint32_t(num_sms) * 8);
    dense_gemv_f32<<<blocks, 256, 0, st>>>(w, rows, cols, x, y);
    return cudaGetLastError();
}

template <int BITS>
static cudaError_t launch_decode_bits(int mode, const LayerParams& P, void* out, cudaStream_t st) {
    const size_t n = size_t(P.n_rb) * P.ng * 32;
    const uint32_t blocks = uint32_t((n + 255) / 256);
    if (mode == 0) decode_tiled<BITS, 0><<<blocks, 256, 0, st>>>(P, out);
    else if (mode == 1) decode_tiled<BITS, 1><<<blocks, 256, 0, st>>>(P, out);
    else decode_tiled<BITS, 2><<<blocks, 256, 0, st>>>(P, out);
    return cudaGetLastError();
}

// mode 0: indices (u16), 1: fp16 values, 2: fp32 values
cudaError_t launch_decode(int mode, const LayerParams& P, void* out, cudaStream_t st) {
    switch (P.bits) {
        case 1: return launch_decode_bits<1>(mode, P, out, st);
        case 2: return launch_decode_bits<2>(mode, P, out, st);
        case 3: return launch_decode_bits<3>(mode, P, out, st);
        case 4: return launch_decode_bits<4>(mode, P, out, st);
        case 5: return launch_decode_bits<5>(mode, P, out, st);
        case 6: return launch_decode_bits<6>(mode, P, out, st);
        case 7: return launch_decode_bits<7>(mode, P, out, st);
        default: return launch_decode_bits<8>(mode, P, out, st);
    }
}

// host -> device copy of a step's input by the GPU itself (reads mapped pinned
// host memory over PCIe).  It triggers its dependents at once, so the stack
// kernel launched after it (PDL) runs its weight prologue -- ring loads, LUT
// planes -- while the bytes cross the bus, and waits for them at its
// griddepcontrol.wait; a copy-engine memcpy would serialise the two instead.
__global__ void __launch_bounds__(256) upload_x(const uint4* __restrict__ src, uint4* dst,
                                                uint32_t n16) {
    pdl_trigger();
    pdl_wait();  // dst may still be read by the previous launch on the stream
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += gridDim.x * blockDim.x)
        dst[i] = src[i];
}

cudaError_t launch_upload_x(const void* host, void* dev, size_t bytes, cudaStream_t st) {
    const uint32_t n16 = uint32_t(bytes / 16);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(std::max<uint32_t>(1, std::min<uint32_t>((n16 + 255) / 256, 16)));
    cfg.blockDim = dim3(256);
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, upload_x, static_cast<const uint4*>(host),
                              static_cast<uint4*>(dev), n16);
}

cudaError_t launch_f32_to_f16(const float* in, uint16_t* out, uint32_t n, cudaStream_t st,
                              bool pdl) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(std::min<uint32_t>((n + 255) / 256, 1024));
    cfg.blockDim = dim3(256);
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, f32_to_f16, in, out, n);
}

}  // namespace sqz
