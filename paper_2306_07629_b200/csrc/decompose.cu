// K10: GPU Dense-and-Sparse decomposition -- the
// reference's dsq::decompose (src/dns.cpp:56-145): mark the
// ceil(sensitive_fraction*N) weights of highest sensitivity, then the
// ceil(outlier_fraction*N) of largest magnitude among the rest (ties: lower
// row-major index first, mark_top_m :56-71), and gather the marked positions
// into a CSR matrix of their original values (row-major, columns ascending,
// csr_from_triplets :31-51).
//
// The selection order is a strict total order on (key descending, index
// ascending), so the top-m set is unique and a radix select finds it
// exactly: the 64-bit composite (~orderable(key) << 32 | index) is unique
// per position and the m smallest composites are the marked ones.  Eight
// 8-bit digit passes (histogram kernel + host digit choice), then one marking
// pass.  The CSR is built one warp per row with ballot compaction (column
// order preserved).
#include <cuda_runtime.h>

#include <cstdint>

namespace sqz {
namespace {

__device__ __forceinline__ uint32_t okey(float f) {  // ascending order, -0 == +0
    uint32_t u = __float_as_uint(f);
    if ((u & 0x7fffffffu) == 0) u = 0;
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

// composite selection key: smaller = selected first
__device__ __forceinline__ unsigned long long ckey(const float* keys, int use_abs, uint32_t i) {
    float k = keys[i];
    if (use_abs) k = fabsf(k);
    return ((unsigned long long)(~okey(k)) << 32) | i;
}

__global__ void select_hist(const float* keys, int use_abs, const uint8_t* excluded, uint32_t n,
                            unsigned long long prefix, uint32_t shift, unsigned int* hist) {
    __shared__ unsigned int h[256];
    for (uint32_t b = threadIdx.x; b < 256; b += blockDim.x) h[b] = 0;
    __syncthreads();
    const unsigned long long hi_mask = shift >= 56 ? 0ull : (~0ull << (shift + 8));
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        if (excluded && excluded[i]) continue;
        const unsigned long long k = ckey(keys, use_abs, i);
        if ((k & hi_mask) != prefix) continue;
        atomicAdd(&h[uint32_t(k >> shift) & 255u], 1u);
    }
    __syncthreads();
    for (uint32_t b = threadIdx.x; b < 256; b += blockDim.x)
        if (h[b]) atomicAdd(&hist[b], h[b]);
}

__global__ void select_mark(const float* keys, int use_abs, uint8_t* mark, uint32_t n,
                            unsigned long long threshold, uint8_t value) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        if (mark[i]) continue;  // already extracted (the sensitive set)
        if (ckey(keys, use_abs, i) <= threshold) mark[i] = value;
    }
}

// one warp per row: number of marked positions
__global__ void row_counts(const uint8_t* mark, uint32_t rows, uint32_t cols, uint32_t* counts) {
    const uint32_t r = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
    if (r >= rows) return;
    uint32_t c = 0;
    for (uint32_t col = lane; col < cols; col += 32) c += mark[size_t(r) * cols + col] ? 1u : 0u;
    for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if (lane == 0) counts[r] = c;
}

// one warp per row: CSR columns / values in column order
__global__ void row_fill(const uint8_t* mark, const float* w, uint32_t rows, uint32_t cols,
                         const uint32_t* row_ptr, uint16_t* col_idx, float* values) {
    const uint32_t r = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
    if (r >= rows) return;
    uint32_t base = row_ptr[r];
    for (uint32_t c0 = 0; c0 < cols; c0 += 32) {
        const uint32_t col = c0 + lane;
        const bool on = col < cols && mark[size_t(r) * cols + col];
        const uint32_t bal = __ballot_sync(0xffffffffu, on);
        if (on) {
            const uint32_t at = base + __popc(bal & ((1u << lane) - 1u));
            col_idx[at] = uint16_t(col);
            values[at] = w[size_t(r) * cols + col];
        }
        base += __popc(bal);
    }
}

}  // namespace

// radix select of the m smallest composite keys among non-excluded positions;
// marks them with `value` in `mark` (positions already marked are skipped,
// which is how the outlier pass excludes the sensitive set)
cudaError_t select_top_m(const float* keys, int use_abs, uint8_t* mark, uint32_t n, uint64_t m,
                         uint8_t value, unsigned int* hist_dev, cudaStream_t st) {
    if (m == 0) return cudaSuccess;
    unsigned long long prefix = 0;
    uint64_t rank = m;  // 1-based rank of the threshold among the candidates
    unsigned int h[256];
    const int grid = 1184, block = 256;
    for (int shift = 56; shift >= 0; shift -= 8) {
        cudaError_t e = cudaMemsetAsync(hist_dev, 0, 256 * sizeof(unsigned int), st);
        if (e != cudaSuccess) return e;
        select_hist<<<grid, block, 0, st>>>(keys, use_abs, mark, n, prefix, uint32_t(shift),
                                            hist_dev);
        if ((e = cudaMemcpyAsync(h, hist_dev, sizeof h, cudaMemcpyDeviceToHost, st)) != cudaSuccess ||
            (e = cudaStreamSynchronize(st)) != cudaSuccess)
            return e;
        uint32_t d = 0;
        for (; d < 256; ++d) {
            if (rank <= h[d]) break;
            rank -= h[d];
        }
        if (d == 256) return cudaErrorInvalidValue;  // fewer candidates than m
        prefix |= (unsigned long long)d << shift;
    }
    select_mark<<<grid, block, 0, st>>>(keys, use_abs, mark, n, prefix, value);
    return cudaGetLastError();
}

cudaError_t csr_counts(const uint8_t* mark, uint32_t rows, uint32_t cols, uint32_t* counts,
                       cudaStream_t st) {
    row_counts<<<(rows + 7) / 8, 256, 0, st>>>(mark, rows, cols, counts);
    return cudaGetLastError();
}

cudaError_t csr_fill(const uint8_t* mark, const float* w, uint32_t rows, uint32_t cols,
                     const uint32_t* row_ptr, uint16_t* col_idx, float* values, cudaStream_t st) {
    row_fill<<<(rows + 7) / 8, 256, 0, st>>>(mark, w, rows, cols, row_ptr, col_idx, values);
    return cudaGetLastError();
}

}  // namespace sqz
