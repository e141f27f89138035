// C ABI of the GPU channel-wise quantizer (K9, quantize.cu): the reference's
// dsq::quantize_channelwise (src/nuq.cpp:673-779) with the same validation
// order and error codes (WeightMatrix::validate tensor.cpp:12-20,
// QuantConfig::validate nuq.cpp:24-34, group_size / empty_channel checks).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "../../include/dsq_cuda.h"
#include "quantize.hpp"

extern "C" int dsq_internal_fail(int code, const char* fmt, ...);

namespace sqz {
cudaError_t select_top_m(const float* keys, int use_abs, uint8_t* mark, uint32_t n, uint64_t m,
                         uint8_t value, unsigned int* hist_dev, cudaStream_t st);
cudaError_t csr_counts(const uint8_t* mark, uint32_t rows, uint32_t cols, uint32_t* counts,
                       cudaStream_t st);
cudaError_t csr_fill(const uint8_t* mark, const float* w, uint32_t rows, uint32_t cols,
                     const uint32_t* row_ptr, uint16_t* col_idx, float* values, cudaStream_t st);
}  // namespace sqz

namespace {
struct DevBuf {
    void* p = nullptr;
    ~DevBuf() {
        if (p) cudaFree(p);
    }
    cudaError_t alloc(size_t bytes) { return cudaMalloc(&p, bytes ? bytes : 1); }
};
}  // namespace

extern "C" int dsq_cuda_quantize_channelwise(const float* w, const float* sens,
                                             const uint8_t* mask, uint32_t rows, uint32_t cols,
                                             const dsq_quant_config* cfg, int method, int device,
                                             float* centroids, uint16_t* assign,
                                             double* weighted_objective,
                                             double* unweighted_mse_sum) {
    if (!cfg || !centroids || !assign)
        return dsq_internal_fail(DSQ_E_INVALID_ARGUMENT, "quantize_channelwise: null argument");
    // matrix.validate()
    if (rows < 1 || cols < 1)
        return dsq_internal_fail(DSQ_E_EMPTY_DIMENSION, "matrix: dimensions must be >= 1");
    if (!w) return dsq_internal_fail(DSQ_E_SHAPE_MISMATCH, "matrix: value count does not match rows*cols");
    const size_t total = size_t(rows) * cols;
    for (size_t i = 0; i < total; ++i)
        if (!std::isfinite(w[i])) return dsq_internal_fail(DSQ_E_NON_FINITE_VALUE, "matrix: non-finite value");
    // cfg.validate()
    if (cfg->bits < 2 || cfg->bits > 8)
        return dsq_internal_fail(DSQ_E_INVALID_ARGUMENT, "bits must be in 2..8");
    if (!(cfg->sensitive_fraction >= 0.0 && cfg->sensitive_fraction <= 0.05))
        return dsq_internal_fail(DSQ_E_INVALID_ARGUMENT, "sensitive_fraction must be in [0, 0.05]");
    if (!(cfg->outlier_fraction >= 0.0 && cfg->outlier_fraction <= 0.05))
        return dsq_internal_fail(DSQ_E_INVALID_ARGUMENT, "outlier_fraction must be in [0, 0.05]");
    if (!(cfg->sensitive_fraction + cfg->outlier_fraction < 1.0))
        return dsq_internal_fail(DSQ_E_INVALID_ARGUMENT, "fraction sum must be < 1");
    if (cfg->kmeans_max_iters < 1)
        return dsq_internal_fail(DSQ_E_INVALID_ARGUMENT, "kmeans_max_iters must be >= 1");
    if (!(cfg->kmeans_tol >= 0.0))
        return dsq_internal_fail(DSQ_E_INVALID_ARGUMENT, "kmeans_tol must be >= 0");
    if (!sens) return dsq_internal_fail(DSQ_E_SHAPE_MISMATCH, "matrix: sensitivity shape mismatch");
    uint32_t gcols = cols;
    if (cfg->group_size > 0) {
        if (cols % cfg->group_size != 0)
            return dsq_internal_fail(DSQ_E_INVALID_ARGUMENT, "matrix: group_size does not divide cols");
        gcols = cfg->group_size;
    }
    if (method < DSQ_CODEBOOK_WEIGHTED_KMEANS || method > DSQ_CODEBOOK_RTN)
        return dsq_internal_fail(DSQ_E_INVALID_ARGUMENT, "quantize_channelwise: unknown method");
    const uint32_t gpr = cols / gcols, k = 1u << cfg->bits;
    const size_t groups = size_t(rows) * gpr;
    size_t np = 1;
    while (np < gcols) np <<= 1;

    cudaError_t e = cudaSetDevice(device);
    if (e != cudaSuccess) return dsq_internal_fail(DSQ_E_CUDA, "cudaSetDevice: %s", cudaGetErrorString(e));
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    // prefix tables in shared memory when they fit; CTAs per SM from the
    // shared-memory footprint (static ~11 KB + the tables)
    int smax = 0;
    cudaDeviceGetAttribute(&smax, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
    const size_t pre = sqz::kmeans_smem_bytes(gcols);
    const bool in_smem = pre + 16 * 1024 <= size_t(smax);
    const size_t per_cta = (in_smem ? pre : 0) + 12 * 1024;
    const size_t per_sm = std::max<size_t>(1, std::min<size_t>(8, (size_t(smax) + 1024) / per_cta));
    const uint32_t grid = uint32_t(std::min<size_t>(groups, size_t(sms > 0 ? sms : 1) * per_sm));
    const size_t stride = sqz::kmeans_scratch_stride(gcols, np);
    DevBuf dw, ds, dm, dc, da, dobj, dmse, dfail, dscr;
    if ((e = dw.alloc(total * 4)) || (e = ds.alloc(total * 4)) ||
        (e = dm.alloc(mask ? total : 1)) || (e = dc.alloc(groups * k * 4)) ||
        (e = da.alloc(total * 2)) || (e = dobj.alloc(groups * 8)) || (e = dmse.alloc(groups * 8)) ||
        (e = dfail.alloc(groups)) || (e = dscr.alloc(stride * grid)))
        return dsq_internal_fail(DSQ_E_CUDA, "quantize_channelwise: cudaMalloc: %s", cudaGetErrorString(e));
    if ((e = cudaMemcpy(dw.p, w, total * 4, cudaMemcpyHostToDevice)) ||
        (e = cudaMemcpy(ds.p, sens, total * 4, cudaMemcpyHostToDevice)) ||
        (mask && (e = cudaMemcpy(dm.p, mask, total, cudaMemcpyHostToDevice))) ||
        (e = cudaMemset(dfail.p, 0, groups)))
        return dsq_internal_fail(DSQ_E_CUDA, "quantize_channelwise: upload: %s", cudaGetErrorString(e));
    sqz::QuantParams P{};
    P.w = static_cast<const float*>(dw.p);
    P.sens = static_cast<const float*>(ds.p);
    P.mask = mask ? static_cast<const uint8_t*>(dm.p) : nullptr;
    P.rows = rows;
    P.cols = cols;
    P.groups_per_row = gpr;
    P.bits = cfg->bits;
    P.max_iters = cfg->kmeans_max_iters;
    P.tol = cfg->kmeans_tol;
    P.method = method;
    P.centroids = static_cast<float*>(dc.p);
    P.assign = static_cast<uint16_t*>(da.p);
    P.group_obj = static_cast<double*>(dobj.p);
    P.group_mse = static_cast<double*>(dmse.p);
    P.group_failed = static_cast<uint8_t*>(dfail.p);
    P.scratch = static_cast<uint8_t*>(dscr.p);
    P.scratch_stride = stride;
    P.npow2 = np;
    P.smem_prefix = in_smem ? 1 : 0;
    DevBuf dprof;
    const bool prof = std::getenv("DSQ_KMEANS_PROFILE") != nullptr;  // dev
    if (prof && dprof.alloc(groups * 6 * 8) == cudaSuccess) {
        cudaMemset(dprof.p, 0, groups * 6 * 8);
        P.prof = static_cast<unsigned long long*>(dprof.p);
    }
    if ((e = sqz::launch_kmeans(P, grid, 0)) || (e = cudaDeviceSynchronize()))
        return dsq_internal_fail(DSQ_E_CUDA, "kmeans_groups: %s", cudaGetErrorString(e));
    if (P.prof) {
        std::vector<unsigned long long> h(groups * 6);
        cudaMemcpy(h.data(), P.prof, h.size() * 8, cudaMemcpyDeviceToHost);
        double a[5] = {0, 0, 0, 0, 0};
        for (size_t g = 0; g < groups; ++g)
            for (int q = 0; q < 5; ++q) a[q] += double(h[g * 6 + q]);
        std::fprintf(stderr, "kmeans profile (mean per group): lloyd %.0f refine %.0f merge %.0f "
                     "cycles, rounds %.2f, iterations %.2f (grid %u)\n", a[0] / groups,
                     a[1] / groups, a[2] / groups, a[3] / groups, a[4] / groups, grid);
    }
    std::vector<uint8_t> failed(groups);
    std::vector<double> obj(groups), mse(groups);
    if ((e = cudaMemcpy(failed.data(), dfail.p, groups, cudaMemcpyDeviceToHost)) ||
        (e = cudaMemcpy(obj.data(), dobj.p, groups * 8, cudaMemcpyDeviceToHost)) ||
        (e = cudaMemcpy(mse.data(), dmse.p, groups * 8, cudaMemcpyDeviceToHost)) ||
        (e = cudaMemcpy(centroids, dc.p, groups * k * 4, cudaMemcpyDeviceToHost)) ||
        (e = cudaMemcpy(assign, da.p, total * 2, cudaMemcpyDeviceToHost)))
        return dsq_internal_fail(DSQ_E_CUDA, "quantize_channelwise: download: %s", cudaGetErrorString(e));
    for (size_t g = 0; g < groups; ++g)
        if (failed[g] == 2) return dsq_internal_fail(DSQ_E_INVALID_ARGUMENT, "kmeans: negative weight");
    for (size_t g = 0; g < groups; ++g)
        if (failed[g] == 1)
            return dsq_internal_fail(DSQ_E_EMPTY_CHANNEL, "matrix: mask covers an entire channel/group");
    double so = 0.0, sm = 0.0;  // summed in group order (nuq.cpp:774-777)
    for (size_t g = 0; g < groups; ++g) {
        so += obj[g];
        sm += mse[g];
    }
    if (weighted_objective) *weighted_objective = so;
    if (unweighted_mse_sum) *unweighted_mse_sum = sm;
    return DSQ_OK;
}

// dsq::decompose (src/dns.cpp:73-145) on the GPU (K10, decompose.cu)
extern "C" int dsq_cuda_decompose(const float* w, const float* sens, uint32_t rows, uint32_t cols,
                                  const dsq_quant_config* cfg, int device, uint8_t* mask,
                                  uint32_t* row_ptr, uint16_t* col_idx, float* values,
                                  uint64_t nnz_cap, uint64_t* nnz, uint32_t* sensitive_count,
                                  uint32_t* outlier_count, float* t_min, float* t_max) {
    if (!cfg || !mask || !row_ptr || !nnz)
        return dsq_internal_fail(DSQ_E_INVALID_ARGUMENT, "decompose: null argument");
    if (rows < 1 || cols < 1)
        return dsq_internal_fail(DSQ_E_EMPTY_DIMENSION, "matrix: dimensions must be >= 1");
    if (!w) return dsq_internal_fail(DSQ_E_SHAPE_MISMATCH, "matrix: value count does not match rows*cols");
    const size_t n = size_t(rows) * cols;
    for (size_t i = 0; i < n; ++i)
        if (!std::isfinite(w[i])) return dsq_internal_fail(DSQ_E_NON_FINITE_VALUE, "matrix: non-finite value");
    if (cfg->bits < 2 || cfg->bits > 8)
        return dsq_internal_fail(DSQ_E_INVALID_ARGUMENT, "bits must be in 2..8");
    if (!(cfg->sensitive_fraction >= 0.0 && cfg->sensitive_fraction <= 0.05))
        return dsq_internal_fail(DSQ_E_INVALID_ARGUMENT, "sensitive_fraction must be in [0, 0.05]");
    if (!(cfg->outlier_fraction >= 0.0 && cfg->outlier_fraction <= 0.05))
        return dsq_internal_fail(DSQ_E_INVALID_ARGUMENT, "outlier_fraction must be in [0, 0.05]");
    if (!(cfg->sensitive_fraction + cfg->outlier_fraction < 1.0))
        return dsq_internal_fail(DSQ_E_INVALID_ARGUMENT, "fraction sum must be < 1");
    if (cfg->kmeans_max_iters < 1)
        return dsq_internal_fail(DSQ_E_INVALID_ARGUMENT, "kmeans_max_iters must be >= 1");
    if (!(cfg->kmeans_tol >= 0.0))
        return dsq_internal_fail(DSQ_E_INVALID_ARGUMENT, "kmeans_tol must be >= 0");
    if (!sens) return dsq_internal_fail(DSQ_E_SHAPE_MISMATCH, "matrix: sensitivity shape mismatch");
    if (cols >= 65536)
        return dsq_internal_fail(DSQ_E_DIMENSION_OVERFLOW, "matrix: cols must be < 65536 for 16-bit CSR columns");
    if (n > 0xffffffffull)
        return dsq_internal_fail(DSQ_E_DIMENSION_OVERFLOW, "decompose: more than 2^32 weights");
    const size_t m_sens = static_cast<size_t>(std::ceil(cfg->sensitive_fraction * double(n)));
    const size_t m_out = static_cast<size_t>(std::ceil(cfg->outlier_fraction * double(n)));
    if (!(m_sens + m_out < n))
        return dsq_internal_fail(DSQ_E_FRACTION_OVERFLOW, "matrix: fractions would mark the entire matrix");
    *nnz = m_sens + m_out;
    if (m_sens + m_out > nnz_cap || ((m_sens + m_out) && (!col_idx || !values)))
        return dsq_internal_fail(DSQ_E_INVALID_ARGUMENT, "decompose: CSR capacity %llu < nnz %llu",
                                 (unsigned long long)nnz_cap, (unsigned long long)(m_sens + m_out));
    cudaError_t e = cudaSetDevice(device);
    if (e != cudaSuccess) return dsq_internal_fail(DSQ_E_CUDA, "cudaSetDevice: %s", cudaGetErrorString(e));
    DevBuf dw, ds, dm, dh, dc, dr, dci, dv;
    const size_t nz = m_sens + m_out;
    if ((e = dw.alloc(n * 4)) || (e = ds.alloc(n * 4)) || (e = dm.alloc(n)) ||
        (e = dh.alloc(256 * 4)) || (e = dc.alloc(size_t(rows) * 4)) ||
        (e = dr.alloc((size_t(rows) + 1) * 4)) || (e = dci.alloc(nz * 2)) || (e = dv.alloc(nz * 4)))
        return dsq_internal_fail(DSQ_E_CUDA, "decompose: cudaMalloc: %s", cudaGetErrorString(e));
    if ((e = cudaMemcpy(dw.p, w, n * 4, cudaMemcpyHostToDevice)) ||
        (e = cudaMemcpy(ds.p, sens, n * 4, cudaMemcpyHostToDevice)) || (e = cudaMemset(dm.p, 0, n)))
        return dsq_internal_fail(DSQ_E_CUDA, "decompose: upload: %s", cudaGetErrorString(e));
    uint8_t* md = static_cast<uint8_t*>(dm.p);
    unsigned int* hist = static_cast<unsigned int*>(dh.p);
    // sensitive values first, then magnitude outliers among the rest
    if ((e = sqz::select_top_m(static_cast<const float*>(ds.p), 0, md, uint32_t(n), m_sens, 1, hist, 0)) ||
        (e = sqz::select_top_m(static_cast<const float*>(dw.p), 1, md, uint32_t(n), m_out, 1, hist, 0)) ||
        (e = sqz::csr_counts(md, rows, cols, static_cast<uint32_t*>(dc.p), 0)))
        return dsq_internal_fail(DSQ_E_CUDA, "decompose: select: %s", cudaGetErrorString(e));
    std::vector<uint32_t> cnt(rows);
    if ((e = cudaMemcpy(cnt.data(), dc.p, size_t(rows) * 4, cudaMemcpyDeviceToHost)))
        return dsq_internal_fail(DSQ_E_CUDA, "decompose: counts: %s", cudaGetErrorString(e));
    row_ptr[0] = 0;
    for (uint32_t r = 0; r < rows; ++r) row_ptr[r + 1] = row_ptr[r] + cnt[r];
    if (row_ptr[rows] != nz) return dsq_internal_fail(DSQ_E_INTERNAL, "decompose: marked %u != %zu", row_ptr[rows], nz);
    if ((e = cudaMemcpy(dr.p, row_ptr, (size_t(rows) + 1) * 4, cudaMemcpyHostToDevice)) ||
        (e = sqz::csr_fill(md, static_cast<const float*>(dw.p), rows, cols,
                           static_cast<const uint32_t*>(dr.p), static_cast<uint16_t*>(dci.p),
                           static_cast<float*>(dv.p), 0)) ||
        (e = cudaMemcpy(mask, md, n, cudaMemcpyDeviceToHost)) ||
        (nz && (e = cudaMemcpy(col_idx, dci.p, nz * 2, cudaMemcpyDeviceToHost))) ||
        (nz && (e = cudaMemcpy(values, dv.p, nz * 4, cudaMemcpyDeviceToHost))))
        return dsq_internal_fail(DSQ_E_CUDA, "decompose: csr: %s", cudaGetErrorString(e));
    // thresholds over the unmarked weights in index order (dns.cpp:118-133)
    float lo = INFINITY, hi = -INFINITY;
    for (size_t i = 0; i < n; ++i)
        if (!mask[i]) {
            lo = std::min(lo, w[i]);
            hi = std::max(hi, w[i]);
        }
    if (t_min) *t_min = lo;
    if (t_max) *t_max = hi;
    if (sensitive_count) *sensitive_count = uint32_t(m_sens);
    if (outlier_count) *outlier_count = uint32_t(m_out);
    return DSQ_OK;
}
