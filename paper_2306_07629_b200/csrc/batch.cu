// batch.cu -- K8: batched Dense-and-Sparse LUT-GEMM, Y[b] = W X[b] for
// B = 2..16 activation vectors (BASELINE configs[4], the roofline crossover).
//
// Same HBM layout as the batch-1 stack kernel (stack.hpp tile layout: 4-row
// tiles, 256-column spans), read with a DENSE fragment map: a warp owns a
// 16-row tile (4 consecutive 4-row tiles) and every mma.sync.m16n8k16 uses all
// 16 A rows and all 8 B columns -- 8 batch vectors per HMMA.  The index decode
// (PRMT byte-plane lookups, tile.cuh) is paid once per weight and amortised
// over the batch; B > 8 adds a second HMMA per decoded fragment.
//
//   thread (g, t): A rows g and g+8 = tile rows (16Q + g) and (16Q + g + 8);
//   it reads the two lanes (h = 0/1, i = g%4, t) of each row's 4-row tile, 64
//   indices per row per span = 16 quads; HMMA m takes quad m of both rows as
//   its k-slots (2t, 2t+1, 2t+8, 2t+9) and x[batch g] at the quad's 4 columns
//   as its B fragment.  D[g][n] / D[g+8][n] are rows x batch n.
//
// Grid: CTA = (group of 8 16-row tiles, column slice); the slice's x for all
// batches is staged in shared memory once and shared by the 8 warps.  Each
// warp writes its tile's partial products for the slice; a second kernel sums
// the slices in order and adds the CSR deltas (deterministic, no atomics).
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "ptx.cuh"
#include "stack.hpp"
#include "tile.cuh"

namespace sqz {

constexpr int kBatchWarps = 8;

struct BatchParams {
    const uint32_t* idx;      // [tiles4][ns][32 x 3 or 4]
    const uint32_t* lut;      // [tiles4][4][LW]
    const uint16_t* x;        // [B][cols] fp16, rows 16-byte aligned (x_stride halves)
    float* part;              // [kslices][rows16][B] fp32 partials
    uint16_t* xT;             // [cols][8 * NB] x transposed (column-major batch), for the CSR pass
    uint32_t rows, cols, ns, tiles4, tiles16, B, x_stride;
    uint32_t kslices, spans_per_slice;
    uint32_t xs_stride;       // halves per batch row in smem (slice cols + 8 pad)
};

// one 4-row-tile lane's 32 indices -> 8 quads (selector words, low 16 bits)
template <int BITS>
__device__ __forceinline__ void lane_quads(const uint32_t* w, uint32_t (&q)[8], uint32_t (&pk)[8]) {
    if constexpr (BITS == 3) {
        const uint32_t m0 = w[0] & 0x77777777u, m1 = w[1] & 0x77777777u, m2 = w[2] & 0x77777777u;
        const uint32_t t = ((w[0] >> 3) & 0x11111111u) | ((w[1] >> 2) & 0x22222222u) |
                           ((w[2] >> 1) & 0x44444444u);
        q[0] = m0; q[1] = hi16(m0); q[2] = m1; q[3] = hi16(m1);
        q[4] = m2; q[5] = hi16(m2); q[6] = t; q[7] = hi16(t);
    } else {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const uint32_t sl = w[k] & 0x77777777u;
            const uint32_t p = ((w[k] >> 1) & 0x44444444u) | 0x32103210u;
            q[2 * k] = sl;
            q[2 * k + 1] = hi16(sl);
            pk[2 * k] = p;
            pk[2 * k + 1] = hi16(p);
        }
    }
}

// quad m of a lane -> span columns (4 consecutive)
__device__ __forceinline__ uint32_t quad_col(uint32_t h, uint32_t t, uint32_t qi) {
    // qi 0..3: positions 4qi.. of piece 4h+t; qi 4..7: positions 4(qi-4).. of piece 8+4h+t
    return tile_col(h, t, qi < 4 ? 4 * qi : 16 + 4 * (qi - 4));
}

template <int BITS, int NB>  // NB = HMMA column groups (1: B <= 8, 2: B <= 16)
__global__ void __launch_bounds__(kBatchWarps * 32) batch_gemv(const __grid_constant__ BatchParams p) {
    extern __shared__ __align__(16) uint16_t xs[];  // [B][xs_stride]
    constexpr uint32_t LW = BITS == 3 ? 4u : 8u;
    constexpr uint32_t UW = BITS * 32u;
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t g = lane >> 2, t = lane & 3, i = g & 3;
    const uint32_t groups = (p.tiles16 + kBatchWarps - 1) / kBatchWarps;
    const uint32_t grp = blockIdx.x % groups, ks = blockIdx.x / groups;
    const uint32_t s0 = ks * p.spans_per_slice;
    const uint32_t s1 = min(p.ns, s0 + p.spans_per_slice);
    const uint32_t c0 = s0 * kSpanCols;
    const uint32_t ccount = min(p.cols, s1 * kSpanCols) - min(p.cols, c0);
    // the weights are immutable: the LUT planes and the first span's index
    // words are requested before the PDL wait and the x staging, so their
    // DRAM latency overlaps both
    const uint32_t Q = grp * kBatchWarps + warp;  // 16-row tile
    // the thread's two rows: A row g -> 4-row tile 4Q + g/4, A row g+8 -> 4Q + 2 + g/4
    const uint32_t T0 = 4 * Q + (g >> 2), T1 = T0 + 2;
    const bool v0 = T0 < p.tiles4, v1 = T1 < p.tiles4;
    Planes16 P0, P1;
    {
        const uint32_t* l0 = p.lut + (size_t(min(T0, p.tiles4 - 1)) * kTileRows + i) * LW;
        const uint32_t* l1 = p.lut + (size_t(min(T1, p.tiles4 - 1)) * kTileRows + i) * LW;
        P0.a = Planes8{v0 ? l0[0] : 0u, v0 ? l0[1] : 0u, v0 ? l0[2] : 0u, v0 ? l0[3] : 0u};
        P1.a = Planes8{v1 ? l1[0] : 0u, v1 ? l1[1] : 0u, v1 ? l1[2] : 0u, v1 ? l1[3] : 0u};
        if constexpr (BITS == 4) {
            P0.b = Planes8{v0 ? l0[4] : 0u, v0 ? l0[5] : 0u, v0 ? l0[6] : 0u, v0 ? l0[7] : 0u};
            P1.b = Planes8{v1 ? l1[4] : 0u, v1 ? l1[5] : 0u, v1 ? l1[6] : 0u, v1 ? l1[7] : 0u};
        }
    }
    float d[2][NB][4];  // two accumulator chains (h = 0 / 1)
#pragma unroll
    for (int c = 0; c < 2; ++c)
#pragma unroll
        for (int n = 0; n < NB; ++n) d[c][n][0] = d[c][n][1] = d[c][n][2] = d[c][n][3] = 0.f;
    const uint16_t* xg0 = xs + g * p.xs_stride;            // batch g
    const uint16_t* xg1 = xs + (8 + g) * p.xs_stride;      // batch 8 + g (NB == 2)
    // index words of one span: [h][row g / g+8][k], prefetched one span ahead
    uint32_t wn[2][2][BITS];
    auto fetch = [&](uint32_t s) {
        const uint32_t* u0 = p.idx + (size_t(min(T0, p.tiles4 - 1)) * p.ns + s) * UW;
        const uint32_t* u1 = p.idx + (size_t(min(T1, p.tiles4 - 1)) * p.ns + s) * UW;
#pragma unroll
        for (uint32_t h = 0; h < 2; ++h) {
            const uint32_t L = 16 * h + 4 * i + t;
#pragma unroll
            for (int k = 0; k < BITS; ++k) {
                const uint32_t o = BITS == 3 ? k * 32 + L : L * 4 + k;
                wn[h][0][k] = v0 ? __ldg(u0 + o) : 0u;
                wn[h][1][k] = v1 ? __ldg(u1 + o) : 0u;
            }
        }
    };
    if (s0 < s1) fetch(s0);
    // x and the partial buffer may belong to the previous launch on this
    // stream (programmatic dependent launch): wait for it first
    pdl_trigger();
    pdl_wait();
    // stage the slice's x for all 8*NB B-columns (zero beyond B and cols),
    // 16 bytes per load (x rows are 16-byte aligned, cols % 8 == 0)
    {
        const uint32_t per_row = (s1 - s0) * kSpanCols / 8;  // uint4 per batch row
        for (uint32_t k = threadIdx.x; k < 8 * NB * per_row; k += blockDim.x) {
            const uint32_t b = k / per_row, c = (k - b * per_row) * 8;
            uint4 v = make_uint4(0, 0, 0, 0);
            if (b < p.B && c < ccount)
                v = __ldg(reinterpret_cast<const uint4*>(p.x + size_t(b) * p.x_stride + c0 + c));
            *reinterpret_cast<uint4*>(xs + b * p.xs_stride + c) = v;
        }
    }
    __syncthreads();
    if (grp == 0 && p.xT) {
        // the slice's x transposed: all batch values of a column in one 16- or
        // 32-byte run, so the CSR pass gathers one sector per column, not per vector
        const uint32_t nbv = 8 * NB;
        for (uint32_t k = threadIdx.x; k < ccount * nbv; k += blockDim.x) {
            const uint32_t c = k / nbv, b = k - c * nbv;
            p.xT[size_t(c0 + c) * nbv + b] = xs[b * p.xs_stride + c];
        }
    }
    if (Q >= p.tiles16) return;
    for (uint32_t s = s0; s < s1; ++s) {
        const uint32_t sl = (s - s0) * kSpanCols;
        uint32_t wc[2][2][BITS];
#pragma unroll
        for (uint32_t h = 0; h < 2; ++h)
#pragma unroll
            for (int r = 0; r < 2; ++r)
#pragma unroll
                for (int k = 0; k < BITS; ++k) wc[h][r][k] = wn[h][r][k];
        if (s + 1 < s1) fetch(s + 1);
#pragma unroll
        for (uint32_t h = 0; h < 2; ++h) {
            const uint32_t* w0 = wc[h][0];
            const uint32_t* w1 = wc[h][1];
            uint32_t q0[8], q1[8], k0[8], k1[8];
            lane_quads<BITS>(w0, q0, k0);
            lane_quads<BITS>(w1, q1, k1);
#pragma unroll
            for (uint32_t qi = 0; qi < 8; ++qi) {
                uint32_t a0, a1, a2, a3;
                if constexpr (BITS == 3) {
                    quad8(q0[qi], P0.a, a0, a2);
                    quad8(q1[qi], P1.a, a1, a3);
                } else {
                    quad16(q0[qi], k0[qi], P0, a0, a2);
                    quad16(q1[qi], k1[qi], P1, a1, a3);
                }
                const uint32_t col = sl + quad_col(h, t, qi);
                const uint2 xb = *reinterpret_cast<const uint2*>(xg0 + col);
                hmma16816(d[h][0], a0, a1, a2, a3, xb.x, xb.y);
                if constexpr (NB == 2) {
                    const uint2 xc = *reinterpret_cast<const uint2*>(xg1 + col);
                    hmma16816(d[h][NB - 1], a0, a1, a2, a3, xc.x, xc.y);
                }
            }
        }
    }
    // partials: D[g][n], D[g+8][n] -> part[ks][row][batch]
    float* out = p.part + size_t(ks) * p.tiles16 * 16 * p.B;
    const uint32_t r0 = Q * 16 + g, r1 = r0 + 8;
#pragma unroll
    for (int n = 0; n < NB; ++n) {
        const uint32_t b0 = 8 * n + 2 * t, b1 = b0 + 1;
        if (b0 < p.B) {
            out[size_t(r0) * p.B + b0] = d[0][n][0] + d[1][n][0];
            out[size_t(r1) * p.B + b0] = d[0][n][2] + d[1][n][2];
        }
        if (b1 < p.B) {
            out[size_t(r0) * p.B + b1] = d[0][n][1] + d[1][n][1];
            out[size_t(r1) * p.B + b1] = d[0][n][3] + d[1][n][3];
        }
    }
}

// y[b][r] = sum over slices (in order) + sum over the row's CSR deltas.  One
// warp per row: lane = part * XB + b (XB = 8 or 16 batch slots, P = 32 / XB
// parts); part k takes the row's entries in groups of 8, group j when
// j % P == k, and the parts are added in a fixed shuffle order (deterministic).
// Loads are issued 8 at a time so the latency of the dependent entry -> x
// loads is paid once per 8 entries; with the transposed x (xT) the XB lanes of
// one part read one column's batch values from one 16- / 32-byte run.
template <int XB>
__global__ void batch_finish(const float* __restrict__ part, uint32_t kslices, uint32_t rows16,
                             uint32_t rows, uint32_t B, const uint32_t* __restrict__ row_ptr,
                             const uint32_t* __restrict__ csr, const uint16_t* __restrict__ x,
                             uint32_t x_stride, const uint16_t* __restrict__ xT, void* y,
                             uint32_t y_stride, int y_f16, int with_dense, int with_csr) {
    constexpr uint32_t P = 32 / XB;
    pdl_trigger();
    pdl_wait();  // the partials of the preceding batch_gemv
    const uint32_t r = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
    const uint32_t lane = threadIdx.x & 31, b = lane % XB, k = lane / XB;
    if (r >= rows) return;  // whole warps
    const bool live = b < B;
    float s = 0.f;
    if (with_csr && live) {
        // x[b][col] = xb[col * xs] (transposed copy from batch_gemv when present)
        const uint16_t* xb = xT ? xT + b : x + size_t(b) * x_stride;
        const uint32_t xs = xT ? uint32_t(XB) : 1u;
        const uint32_t q0 = row_ptr[r], q1 = row_ptr[r + 1];
        for (uint32_t q = q0 + 8 * k; q < q1; q += 8 * P) {
            uint32_t e[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) e[u] = q + u < q1 ? __ldg(csr + q + u) : 0u;
            uint16_t xv[8];
#pragma unroll
            for (int u = 0; u < 8; ++u)
                xv[u] = q + u < q1 ? __ldg(xb + size_t(e[u] & 0xffffu) * xs) : uint16_t(0);
#pragma unroll
            for (int u = 0; u < 8; ++u)
                if (q + u < q1) s = fma_h(uint16_t(e[u] >> 16), xv[u], s);
        }
    }
#pragma unroll
    for (uint32_t o = XB; o < 32; o <<= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (k != 0 || !live) return;
    if (with_dense) {
        float d = 0.f;
        uint32_t j = 0;
        for (; j + 4 <= kslices; j += 4) {
            float v[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) v[u] = part[(size_t(j + u) * rows16 * 16 + r) * B + b];
#pragma unroll
            for (int u = 0; u < 4; ++u) d += v[u];
        }
        for (; j < kslices; ++j) d += part[(size_t(j) * rows16 * 16 + r) * B + b];
        s = d + s;
    }
    if (y_f16)
        static_cast<__half*>(y)[size_t(b) * y_stride + r] = __float2half_rn(s);
    else
        static_cast<float*>(y)[size_t(b) * y_stride + r] = s;
}

// launch with programmatic stream serialization (the kernel calls pdl_wait
// before touching data of the previous launch), so back-to-back products
// overlap one kernel's tail with the next one's launch
template <class K, class... A>
cudaError_t launch_pdl(K kern, dim3 grid, dim3 block, size_t smem, cudaStream_t st, A... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, args...);
}

size_t batch_smem_bytes(uint32_t B, uint32_t spans_per_slice) {
    return size_t(B > 8 ? 16 : 8) * (spans_per_slice * kSpanCols + 8) * 2;
}

cudaError_t launch_batch(uint32_t bits, const uint32_t* idx, const uint32_t* lut,
                         const uint32_t* row_ptr, const uint32_t* csr, uint32_t rows,
                         uint32_t cols, uint32_t ns, uint32_t tiles4, const uint16_t* x,
                         uint32_t x_stride, uint32_t B, void* y, uint32_t y_stride, bool y_f16,
                         float* part, uint32_t kslices, uint32_t spans_per_slice, int mode,
                         cudaStream_t st) {
    BatchParams p{};
    p.idx = idx;
    p.lut = lut;
    p.x = x;
    p.part = part;
    p.rows = rows;
    p.cols = cols;
    p.ns = ns;
    p.tiles4 = tiles4;
    p.tiles16 = (tiles4 + 3) / 4;
    p.B = B;
    p.x_stride = x_stride;
    p.kslices = kslices;
    p.spans_per_slice = spans_per_slice;
    p.xs_stride = spans_per_slice * kSpanCols + 8;
    const int with_dense = mode != 1, with_csr = mode != 0;
    // the transposed x lives after the partials (api.cpp sizes the buffer)
    p.xT = with_dense && with_csr
               ? reinterpret_cast<uint16_t*>(part + size_t(kslices) * p.tiles16 * 16 * 16)
               : nullptr;
    const uint32_t xT_stride = B > 8 ? 16u : 8u;
    if (with_dense) {
        const uint32_t groups = (p.tiles16 + kBatchWarps - 1) / kBatchWarps;
        const size_t smem = batch_smem_bytes(B, spans_per_slice);
        using K = void (*)(BatchParams);
        K k = bits == 3 ? (B > 8 ? batch_gemv<3, 2> : batch_gemv<3, 1>)
                        : (B > 8 ? batch_gemv<4, 2> : batch_gemv<4, 1>);
        cudaError_t e = cudaSuccess;
        if (smem > 48 * 1024)
            e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        if (e != cudaSuccess) return e;
        if ((e = launch_pdl(k, dim3(groups * kslices), dim3(kBatchWarps * 32), smem, st, p)) !=
            cudaSuccess)
            return e;
    }
    const dim3 fg((rows + 7) / 8), fb(256);  // one warp per row
    const uint16_t* xT = p.xT;
    return xT_stride == 16
               ? launch_pdl(batch_finish<16>, fg, fb, 0, st, part, kslices, p.tiles16, rows, B,
                            row_ptr, csr, x, x_stride, xT, y, y_stride, y_f16 ? 1 : 0, with_dense,
                            with_csr)
               : launch_pdl(batch_finish<8>, fg, fb, 0, st, part, kslices, p.tiles16, rows, B,
                            row_ptr, csr, x, x_stride, xT, y, y_stride, y_f16 ? 1 : 0, with_dense,
                            with_csr);
}

}  // namespace sqz
