// ref_shim.cpp -- C entry points over the UNMODIFIED reference library
// (TEST INFRASTRUCTURE).  Compiled by oracle/Makefile together with the
// reference sources where they lie under /root/reference/proj/src into
// oracle/_ref/libdsqref.so.  No reference source is copied into this repo.
//
// Used by tests/ to pin the C restatement (oracle/dsq_oracle.c) and to make
// golden fixtures, and by bench.py --impl reference / cpu_baseline to time the
// reference's own CPU implementation (dsq::fused_dns_matvec via
// dsq::bench_matvec, kernels.cpp:214-282).
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "dsq/container.hpp"
#include "dsq/kernels.hpp"
#include "dsq/nuq.hpp"
#include "dsq/packfmt.hpp"
#include "dsq/pipeline.hpp"
#include "dsq/sensitivity.hpp"

#ifdef _OPENMP
#include <omp.h>
#endif

using namespace dsq;

namespace {
thread_local std::string g_err;

int code_of(const Error& e) { return int(e.code()) + 1; }  // errc 0.. -> 1..

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const Error& e) {
        g_err = e.what();
        return code_of(e);
    } catch (const std::exception& e) {
        g_err = e.what();
        return 100;
    }
}

Exec exec_of(int parallel) { return parallel ? Exec::parallel : Exec::serial; }
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_max_threads() {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

void ref_set_threads(int n) {
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}

// pack(): codebooks given as a flat f32 array [rows*groups][2^bits]
int ref_pack(const uint16_t* assign, const float* luts, uint32_t bits, uint32_t rows,
             uint32_t cols, uint32_t groups, uint8_t* payload_out) {
    return guarded([&] {
        AssignmentVector a(assign, assign + size_t(rows) * cols);
        std::vector<Codebook> cbs(size_t(rows) * groups);
        const uint32_t k = 1u << bits;
        for (size_t i = 0; i < cbs.size(); ++i) cbs[i].centroids.assign(luts + i * k, luts + (i + 1) * k);
        PackedDense p = pack(a, cbs, bits, rows, cols, groups);
        std::memcpy(payload_out, p.payload.data(), p.payload.size());
    });
}

int ref_unpack(const uint8_t* payload, uint32_t bits, uint32_t rows, uint32_t cols,
               int strict, uint16_t* out) {
    return guarded([&] {
        PackedDense p;
        p.bits = bits;
        p.rows = rows;
        p.cols = cols;
        p.groups_per_row = 1;
        p.luts.assign(size_t(rows) << bits, 0.0f);
        p.payload.assign(payload, payload + size_t(rows) * p.row_stride());
        AssignmentVector a = unpack(p, strict != 0);
        std::memcpy(out, a.data(), a.size() * sizeof(uint16_t));
    });
}

// ---------------------------------------------------------------------------
// layer handle: QuantizedLayer assembled from flat arrays (or quantize_layer)
// ---------------------------------------------------------------------------
struct RefLayer {
    QuantizedLayer l;
};

int ref_layer_new(const char* name, uint32_t bits, uint32_t rows, uint32_t cols,
                  uint32_t groups, const float* luts, const uint8_t* payload,
                  const uint32_t* row_ptr, uint32_t nnz, const uint16_t* col_idx,
                  const float* values, uint32_t hybrid_top_k, RefLayer** out) {
    return guarded([&] {
        auto* h = new RefLayer;
        QuantizedLayer& l = h->l;
        l.name = name;
        l.rows = rows;
        l.cols = cols;
        l.packed.bits = bits;
        l.packed.rows = rows;
        l.packed.cols = cols;
        l.packed.groups_per_row = groups;
        l.packed.luts.assign(luts, luts + size_t(rows) * groups * (1u << bits));
        l.packed.payload.assign(payload, payload + size_t(rows) * l.packed.row_stride());
        l.sparse.rows = rows;
        l.sparse.cols = cols;
        l.sparse.row_ptr.assign(row_ptr, row_ptr + rows + 1);
        l.sparse.col_idx.assign(col_idx, col_idx + nnz);
        l.sparse.values.assign(values, values + nnz);
        l.hybrid_top_k = std::min(hybrid_top_k, rows);
        try {
            l.hybrid = hybrid_split(l.sparse, l.hybrid_top_k);
            l.avg_bits = average_bits(l);
            l.validate();
        } catch (...) {
            delete h;
            throw;
        }
        *out = h;
    });
}

// Full reference quantization flow (pipeline.cpp:7-47) on a given matrix and
// sensitivity map -- used only to make realistic golden fixtures.
int ref_layer_quantize(const char* name, const float* w, const float* sens, uint32_t rows,
                       uint32_t cols, uint32_t bits, double sens_frac, double out_frac,
                       uint32_t hybrid_top_k, uint64_t seed, RefLayer** out) {
    return guarded([&] {
        WeightMatrix m;
        m.name = name;
        m.rows = rows;
        m.cols = cols;
        m.values.assign(w, w + size_t(rows) * cols);
        SensitivityMap s = uniform_sensitivity(m.name, rows, cols);
        s.values.assign(sens, sens + size_t(rows) * cols);
        QuantizeOptions opt;
        opt.cfg.bits = bits;
        opt.cfg.sensitive_fraction = sens_frac;
        opt.cfg.outlier_fraction = out_frac;
        opt.cfg.seed = seed;
        opt.hybrid_top_k = hybrid_top_k;
        auto* h = new RefLayer;
        try {
            h->l = quantize_layer(m, s, opt);
        } catch (...) {
            delete h;
            throw;
        }
        *out = h;
    });
}

void ref_layer_free(RefLayer* h) { delete h; }

void ref_layer_dims(const RefLayer* h, uint32_t* bits, uint32_t* rows, uint32_t* cols,
                    uint32_t* groups, uint32_t* nnz, uint32_t* n_promoted) {
    *bits = h->l.packed.bits;
    *rows = h->l.rows;
    *cols = h->l.cols;
    *groups = h->l.packed.groups_per_row;
    *nnz = h->l.sparse.nnz();
    *n_promoted = uint32_t(h->l.hybrid.dense_row_ids.size());
}

// copies out the layer arrays (any pointer may be null)
void ref_layer_arrays(const RefLayer* h, float* luts, uint8_t* payload, uint32_t* row_ptr,
                      uint16_t* col_idx, float* values, uint32_t* dense_row_ids,
                      float* promoted, uint32_t* res_row_ptr, uint16_t* res_col_idx,
                      float* res_values) {
    const QuantizedLayer& l = h->l;
    auto cp = [](auto* dst, const auto& v) {
        if (dst && !v.empty()) std::memcpy(dst, v.data(), v.size() * sizeof(v[0]));
    };
    cp(luts, l.packed.luts);
    cp(payload, l.packed.payload);
    cp(row_ptr, l.sparse.row_ptr);
    cp(col_idx, l.sparse.col_idx);
    cp(values, l.sparse.values);
    cp(dense_row_ids, l.hybrid.dense_row_ids);
    cp(promoted, l.hybrid.promoted_rows);
    cp(res_row_ptr, l.hybrid.residual.row_ptr);
    cp(res_col_idx, l.hybrid.residual.col_idx);
    cp(res_values, l.hybrid.residual.values);
}

// kernel: 0 lut, 1 csr, 2 fused, 3 reference(ref::fused_dns_matvec), 4 dequant-dense-reference
int ref_matvec(const RefLayer* h, int kernel, const float* x, int parallel, double* out) {
    return guarded([&] {
        ActivationVector xv(x, x + h->l.cols);
        std::vector<double> y;
        switch (kernel) {
            case 0: y = lut_matvec(h->l.packed, xv, exec_of(parallel)); break;
            case 1: y = csr_matvec(h->l.sparse, xv, exec_of(parallel)); break;
            case 2: y = fused_dns_matvec(h->l, xv, exec_of(parallel)); break;
            case 3: y = ref::fused_dns_matvec(h->l, xv); break;
            default: {
                const std::vector<float> m = ref::dequant_dense(h->l.packed);
                y = dense_matvec(m, h->l.rows, h->l.cols, xv, exec_of(parallel));
            }
        }
        std::memcpy(out, y.data(), y.size() * sizeof(double));
    });
}

int ref_dequant_dense(const RefLayer* h, float* out) {
    return guarded([&] {
        const std::vector<float> m = ref::dequant_dense(h->l.packed);
        std::memcpy(out, m.data(), m.size() * sizeof(float));
    });
}

int ref_dequantize_layer(const RefLayer* h, float* out) {
    return guarded([&] {
        const WeightMatrix m = dequantize_layer(h->l);
        std::memcpy(out, m.values.data(), m.values.size() * sizeof(float));
    });
}

// dsq::bench_matvec (kernels.cpp:214-282): median seconds of `repeats` runs
int ref_bench(const RefLayer* h, int kernel, const float* x, uint32_t repeats, int parallel,
              double* median_seconds, uint64_t* bytes_touched) {
    return guarded([&] {
        ActivationVector xv(x, x + h->l.cols);
        BenchKernel k = kernel == 0   ? BenchKernel::lut
                        : kernel == 1 ? BenchKernel::csr
                        : kernel == 2 ? BenchKernel::fused
                                      : BenchKernel::reference;
        BenchRecord r = bench_matvec(h->l, xv, repeats, k, exec_of(parallel));
        *median_seconds = r.median_seconds;
        *bytes_touched = r.bytes_touched;
    });
}

uint64_t ref_bytes_touched(const RefLayer* h) { return bytes_touched_estimate(h->l); }

double ref_avg_bits(const RefLayer* h) { return h->l.avg_bits; }

// container round trip (container.cpp:146-223)
int ref_save_container(RefLayer* const* layers, uint32_t n, uint32_t bits, const char* path) {
    return guarded([&] {
        QuantContainer c;
        c.meta.cfg.bits = bits;
        for (uint32_t i = 0; i < n; ++i) c.layers.push_back(layers[i]->l);
        save_container(c, path);
    });
}

int ref_load_container_layer(const char* path, uint32_t index, RefLayer** out) {
    return guarded([&] {
        QuantContainer c = load_container(path);
        check(index < c.layers.size(), errc::invalid_argument, "layer index out of range");
        auto* h = new RefLayer;
        h->l = c.layers[index];
        *out = h;
    });
}


// dsq::quantize_channelwise (nuq.cpp:673-779) on flat arrays: the GPU
// quantizer's (csrc/quantize.cu) parity reference.  mask may be null.
int ref_quantize_channelwise(const float* w, const float* sens, const uint8_t* mask,
                             uint32_t rows, uint32_t cols, uint32_t bits, uint32_t group_size,
                             uint32_t max_iters, double tol, int method, float* centroids,
                             uint16_t* assign, double* obj, double* mse) {
    return guarded([&] {
        const size_t n = size_t(rows) * cols;
        WeightMatrix m = make_matrix("matrix", rows, cols, std::vector<float>(w, w + n));
        QuantConfig cfg;
        cfg.bits = bits;
        cfg.group_size = group_size;
        cfg.kmeans_max_iters = max_iters;
        cfg.kmeans_tol = tol;
        std::vector<uint8_t> mk;
        if (mask) mk.assign(mask, mask + n);
        const ChannelwiseResult r = quantize_channelwise(
            m, std::vector<float>(sens, sens + n), cfg, mk, static_cast<CodebookMethod>(method));
        const uint32_t k = 1u << bits;
        for (size_t g = 0; g < r.codebooks.size(); ++g)
            std::memcpy(centroids + g * k, r.codebooks[g].centroids.data(), k * sizeof(float));
        std::memcpy(assign, r.assignment.data(), n * sizeof(uint16_t));
        *obj = r.weighted_objective;
        *mse = r.unweighted_mse_sum;
    });
}

}  // extern "C"
