// dsq_cuda.hpp -- header-only C++ layer over the C ABI (dsq_cuda.h) with the
// reference's hot-path signatures (include/dsq/kernels.hpp:17-79).
//
// It is templated on the caller's layer types instead of including the
// reference headers, so a reference user passes their own dsq::PackedDense /
// dsq::CsrMatrix / dsq::QuantizedLayer unchanged (fields used: bits, rows,
// cols, groups_per_row, luts, payload; rows, cols, row_ptr, col_idx, values;
// name, packed, sparse, hybrid_top_k -- packfmt.hpp:16-61, dns.hpp:14-24).
//
//   #include <dsq/kernels.hpp>
//   #include "dsq_cuda.hpp"
//   sqz::DeviceLayer dev(layer);                  // validate + re-tile + upload once
//   std::vector<double> y = dev.fused(x);          // == dsq::fused_dns_matvec(layer, x)
//   std::vector<double> y2 = sqz::fused_dns_matvec(layer, x);   // one-shot form
//   (also sqz::lut_matvec / csr_matvec / dense_matvec / bench_matvec /
//    bytes_touched_estimate / dequantize_layer with the dsq:: signatures)
//
// Errors: a non-OK status is rethrown as sqz::Error whose errc() is the
// reference's dsq::errc value (status - 1), so `static_cast<dsq::errc>(e.errc())`
// reproduces dsq::Error and the CLI exit-code mapping (tools/dsq.cpp:399-411).
#pragma once

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "dsq_cuda.h"

namespace sqz {

class Error : public std::runtime_error {
public:
    Error(int status, const std::string& msg) : std::runtime_error(msg), status_(status) {}
    int status() const { return status_; }
    // dsq::errc ordinal (valid for status 1..15), -1 for device-only failures
    int errc() const { return status_ >= 1 && status_ <= 15 ? status_ - 1 : -1; }

private:
    int status_;
};

inline void check(int rc) {
    if (rc != DSQ_OK) throw Error(rc, dsq_cuda_last_error());
}

template <class Packed>
dsq_packed_view packed_view(const Packed& p) {
    dsq_packed_view v{};
    v.bits = p.bits;
    v.rows = p.rows;
    v.cols = p.cols;
    v.groups_per_row = p.groups_per_row;
    v.luts_f32 = p.luts.data();
    v.payload = p.payload.data();
    v.payload_len = p.payload.size();
    return v;
}

template <class Csr>
dsq_csr_view csr_view(const Csr& s) {
    dsq_csr_view v{};
    v.rows = s.rows;
    v.cols = s.cols;
    v.nnz = s.row_ptr.empty() ? 0u : s.row_ptr.back();
    v.row_ptr = s.row_ptr.data();
    v.col_idx = s.col_idx.empty() ? nullptr : s.col_idx.data();
    v.values_f32 = s.values.empty() ? nullptr : s.values.data();
    return v;
}

template <class Layer>
dsq_layer_view layer_view(const Layer& l) {
    dsq_layer_view v{};
    v.name = l.name.c_str();
    v.rows = l.rows;
    v.cols = l.cols;
    v.packed = packed_view(l.packed);
    v.sparse = csr_view(l.sparse);
    v.hybrid_top_k = l.hybrid_top_k;
    return v;
}

// Owning handle of one uploaded layer.
class DeviceLayer {
public:
    template <class Layer>
    explicit DeviceLayer(const Layer& l, int device = 0) {
        const dsq_layer_view v = layer_view(l);
        dsq_cuda_layer* h = nullptr;
        check(dsq_cuda_layer_create(&v, device, &h));
        h_.reset(h);
        cols_ = l.cols;
        rows_ = l.rows;
    }
    dsq_cuda_layer* get() const { return h_.get(); }

    // host-vector products with the reference's signatures (fp32 x -> fp64 y)
    std::vector<double> lut(const std::vector<float>& x) const { return run(DSQ_KERNEL_LUT, x); }
    std::vector<double> csr(const std::vector<float>& x) const { return run(DSQ_KERNEL_CSR, x); }
    std::vector<double> fused(const std::vector<float>& x) const { return run(DSQ_KERNEL_FUSED, x); }
    std::vector<double> reference(const std::vector<float>& x) const {
        return run(DSQ_KERNEL_REFERENCE, x);
    }

    // device-buffer product on a caller stream (cudaStream_t as void*)
    void gemv(int kernel, const void* x, int x_dtype, void* y, int y_dtype, void* stream) const {
        check(dsq_cuda_gemv(h_.get(), kernel, x, x_dtype, y, y_dtype, 1, stream));
    }

private:
    struct Del {
        void operator()(dsq_cuda_layer* h) const { dsq_cuda_layer_destroy(h); }
    };
    std::vector<double> run(int kernel, const std::vector<float>& x) const {
        if (x.size() != cols_) throw Error(DSQ_E_SHAPE_MISMATCH, "dimension mismatch");
        std::vector<double> y(rows_);
        check(dsq_cuda_matvec_host(h_.get(), kernel, x.data(), y.data()));
        return y;
    }
    std::unique_ptr<dsq_cuda_layer, Del> h_;
    size_t cols_ = 0, rows_ = 0;
};

// ---- the reference's free functions (kernels.hpp:20-79, pipeline.hpp) ------
//
// Same names, argument order and meaning as dsq::, so a reference caller
// switches namespaces: `sqz::fused_dns_matvec(layer, x)`.  The Exec argument
// is accepted as dsq::Exec or sqz::Exec; every value runs on the GPU (the
// device products are deterministic whatever the launch configuration, the
// guarantee dsq::Exec::parallel gives on the host, kernels.hpp:13-16).  The
// one-shot forms upload the layer per call; keep a DeviceLayer for repeated
// products.  Errors are rethrown as sqz::Error with the reference errc.
enum class Exec { serial, parallel, cuda };

// dsq::lut_matvec(const PackedDense&, const ActivationVector&, Exec)
template <class Packed, class E = Exec>
std::vector<double> lut_matvec(const Packed& p, const std::vector<float>& x, E = E{}) {
    if (x.size() != p.cols) throw Error(DSQ_E_SHAPE_MISMATCH, "lut_matvec: dimension mismatch");
    const dsq_packed_view v = packed_view(p);
    std::vector<double> y(p.rows);
    check(dsq_cuda_packed_matvec_host(&v, x.data(), y.data(), 0));
    return y;
}

// dsq::csr_matvec(const CsrMatrix&, const ActivationVector&, Exec)
template <class Csr, class E = Exec>
std::vector<double> csr_matvec(const Csr& s, const std::vector<float>& x, E = E{}) {
    if (x.size() != s.cols) throw Error(DSQ_E_SHAPE_MISMATCH, "csr_matvec: dimension mismatch");
    const dsq_csr_view v = csr_view(s);
    std::vector<double> y(s.rows);
    check(dsq_cuda_csr_matvec_host(&v, x.data(), y.data(), 0));
    return y;
}

// dsq::fused_dns_matvec(const QuantizedLayer&, const ActivationVector&, Exec)
template <class Layer, class E = Exec>
std::vector<double> fused_dns_matvec(const Layer& l, const std::vector<float>& x, E = E{}) {
    return DeviceLayer(l).fused(x);
}

// dsq::dense_matvec(const std::vector<float>& m, rows, cols, x, Exec)
template <class E = Exec>
std::vector<double> dense_matvec(const std::vector<float>& m, uint32_t rows, uint32_t cols,
                                 const std::vector<float>& x, E = E{}) {
    if (m.size() != size_t(rows) * cols || x.size() != cols)
        throw Error(DSQ_E_SHAPE_MISMATCH, "dense_matvec: dimension mismatch");
    std::vector<double> y(rows);
    check(dsq_cuda_dense_matvec_host(m.data(), rows, cols, x.data(), y.data(), 0));
    return y;
}

// dsq::bytes_touched_estimate(const QuantizedLayer&) (kernels.cpp:205-212)
template <class Layer>
uint64_t bytes_touched_estimate(const Layer& l) {
    const uint32_t gpr = l.packed.groups_per_row;
    return dsq_bytes_touched_estimate(l.rows, l.cols, l.packed.bits, gpr == 1 ? 0 : l.cols / gpr,
                                      l.sparse.row_ptr.empty() ? 0 : l.sparse.row_ptr.back());
}
inline uint64_t bytes_touched_estimate(uint32_t rows, uint32_t cols, uint32_t bits,
                                       uint32_t group_size, uint64_t nnz) {
    return dsq_bytes_touched_estimate(rows, cols, bits, group_size, nnz);
}

// dsq::BenchRecord / BenchKernel / bench_matvec (kernels.hpp:63-75,
// kernels.cpp:214-282): median wall time of `repeats` (>= 3) products after
// one warm-up, each timed around the reference-signature host call (fp32
// host x -> fp64 host y on the uploaded layer), and the reference's per-kernel
// byte charge.  The kernel argument may be dsq::BenchKernel or sqz::BenchKernel
// (same order: lut, csr, fused, reference).
struct BenchRecord {
    std::string kernel;
    uint32_t repeats = 0;
    double median_seconds = 0.0;
    std::vector<double> all_seconds;
    uint64_t bytes_touched = 0;
};
enum class BenchKernel { lut, csr, fused, reference };

template <class Layer, class K, class E = Exec>
BenchRecord bench_matvec(const Layer& l, const std::vector<float>& x, uint32_t repeats, K kernel,
                         E = E{}) {
    if (repeats < 3) throw Error(DSQ_E_INVALID_ARGUMENT, "bench: repeats must be >= 3");
    const int k = static_cast<int>(kernel);  // DSQ_KERNEL_LUT..REFERENCE
    static const char* names[] = {"lut", "csr", "fused", "reference"};
    if (k < 0 || k > 3) throw Error(DSQ_E_INVALID_ARGUMENT, "bench: unknown kernel");
    DeviceLayer dev(l);
    auto run = [&]() {
        switch (k) {
            case 0: return dev.lut(x);
            case 1: return dev.csr(x);
            case 2: return dev.fused(x);
            default: return dev.reference(x);
        }
    };
    (void)run();  // warm-up
    BenchRecord rec;
    rec.kernel = names[k];
    rec.repeats = repeats;
    for (uint32_t i = 0; i < repeats; ++i) {
        const auto t0 = std::chrono::steady_clock::now();
        (void)run();
        const auto t1 = std::chrono::steady_clock::now();
        rec.all_seconds.push_back(std::chrono::duration<double>(t1 - t0).count());
    }
    std::vector<double> s = rec.all_seconds;
    std::sort(s.begin(), s.end());
    rec.median_seconds = repeats % 2 ? s[repeats / 2] : 0.5 * (s[repeats / 2 - 1] + s[repeats / 2]);
    const uint32_t gpr = l.packed.groups_per_row;
    const uint32_t gs = gpr == 1 ? 0 : l.cols / gpr;
    const uint64_t io = uint64_t(l.cols) * 2 + uint64_t(l.rows) * 2;
    const uint64_t nnz = l.sparse.row_ptr.empty() ? 0 : l.sparse.row_ptr.back();
    switch (k) {
        case 0: rec.bytes_touched = dsq_bytes_touched_estimate(l.rows, l.cols, l.packed.bits, gs, 0); break;
        case 1: rec.bytes_touched = nnz * 4 + (uint64_t(l.rows) + 1) * 4 + io; break;
        case 2: rec.bytes_touched = bytes_touched_estimate(l); break;
        default: rec.bytes_touched = uint64_t(l.rows) * l.cols * 2 + io; break;
    }
    return rec;
}

// dsq::dequantize_layer(const QuantizedLayer&) -> WeightMatrix (pipeline.cpp:49-75);
// Matrix = dsq::WeightMatrix (name, rows, cols, values)
template <class Matrix, class Layer>
Matrix dequantize_layer(const Layer& l, int device = 0) {
    DeviceLayer dev(l, device);
    Matrix m;
    m.name = l.name;
    m.rows = l.rows;
    m.cols = l.cols;
    m.values.resize(size_t(l.rows) * l.cols);
    check(dsq_cuda_dequantize_layer_host(dev.get(), m.values.data()));
    return m;
}

// ---- the producer side on the GPU, with the caller's reference types ------

template <class Cfg>
dsq_quant_config quant_config(const Cfg& c) {  // dsq::QuantConfig (nuq.hpp:26-37)
    dsq_quant_config q{};
    q.bits = c.bits;
    q.sensitive_fraction = c.sensitive_fraction;
    q.outlier_fraction = c.outlier_fraction;
    q.group_size = c.group_size;
    q.kmeans_max_iters = c.kmeans_max_iters;
    q.kmeans_tol = c.kmeans_tol;
    q.seed = c.seed;
    return q;
}

// == dsq::quantize_channelwise(matrix, sens, cfg, mask, method) (nuq.hpp:106-110);
// Result = dsq::ChannelwiseResult, method = int(dsq::CodebookMethod)
template <class Result, class Matrix, class Cfg>
Result quantize_channelwise(const Matrix& m, const std::vector<float>& sens, const Cfg& cfg,
                            const std::vector<uint8_t>& mask = {}, int method = 0,
                            int device = 0) {
    const dsq_quant_config q = quant_config(cfg);
    const uint32_t k = 1u << cfg.bits;
    const uint32_t gpr = cfg.group_size ? m.cols / cfg.group_size : 1;
    std::vector<float> cent(size_t(m.rows) * gpr * k);
    Result r;
    r.assignment.resize(size_t(m.rows) * m.cols);
    double obj = 0, mse = 0;
    if (sens.size() != m.values.size()) throw Error(DSQ_E_SHAPE_MISMATCH, "sensitivity shape mismatch");
    if (!mask.empty() && mask.size() != m.values.size())
        throw Error(DSQ_E_SHAPE_MISMATCH, "mask shape mismatch");
    check(dsq_cuda_quantize_channelwise(m.values.data(), sens.data(),
                                        mask.empty() ? nullptr : mask.data(), m.rows, m.cols, &q,
                                        method, device, cent.data(), r.assignment.data(), &obj,
                                        &mse));
    r.groups_per_row = gpr;
    r.codebooks.resize(size_t(m.rows) * gpr);
    for (size_t g = 0; g < r.codebooks.size(); ++g)
        r.codebooks[g].centroids.assign(cent.begin() + g * k, cent.begin() + (g + 1) * k);
    r.weighted_objective = obj;
    r.unweighted_mse_sum = mse;
    return r;
}

// == dsq::decompose(matrix, sens, cfg) (dns.hpp:44-49); Decomp = dsq::Decomposition
template <class Decomp, class Matrix, class Cfg>
Decomp decompose(const Matrix& m, const std::vector<float>& sens, const Cfg& cfg, int device = 0) {
    const dsq_quant_config q = quant_config(cfg);
    const size_t n = m.values.size();
    if (sens.size() != n) throw Error(DSQ_E_SHAPE_MISMATCH, "sensitivity shape mismatch");
    Decomp d;
    d.mask.assign(n, 0);
    d.sparse.rows = m.rows;
    d.sparse.cols = m.cols;
    d.sparse.row_ptr.assign(size_t(m.rows) + 1, 0);
    uint64_t nnz = 0;
    // first call sizes the CSR (capacity 0 -> DSQ_E_INVALID_ARGUMENT with nnz set)
    const size_t cap = size_t(std::ceil(cfg.sensitive_fraction * double(n))) +
                       size_t(std::ceil(cfg.outlier_fraction * double(n)));
    d.sparse.col_idx.resize(cap);
    d.sparse.values.resize(cap);
    uint32_t sc = 0, oc = 0;
    float lo = 0, hi = 0;
    check(dsq_cuda_decompose(m.values.data(), sens.data(), m.rows, m.cols, &q, device,
                             d.mask.data(), d.sparse.row_ptr.data(),
                             cap ? d.sparse.col_idx.data() : nullptr,
                             cap ? d.sparse.values.data() : nullptr, cap, &nnz, &sc, &oc, &lo,
                             &hi));
    d.sparse.col_idx.resize(nnz);
    d.sparse.values.resize(nnz);
    d.dense = m;
    for (size_t i = 0; i < n; ++i)
        if (d.mask[i]) d.dense.values[i] = 0.0f;
    d.t_min = lo;
    d.t_max = hi;
    d.sensitive_count = sc;
    d.outlier_count = oc;
    return d;
}

}  // namespace sqz
