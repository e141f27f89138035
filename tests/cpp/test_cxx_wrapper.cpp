// C++ integration test: the reference's own types (dsq::QuantizedLayer built
// by the reference's quantize_layer, pipeline.cpp:7-47) passed unchanged to
// the B200 library through include/dsq_cuda.hpp, compared with the
// reference's dsq::fused_dns_matvec / lut_matvec / csr_matvec.
//
// Built here against /root/reference/proj/include + oracle/_ref/libdsqref.so
// (make cxx-test); the binary travels to the GPU box and is run by
// tests/test_cxx_wrapper.py (GPU).  Exit code 0 = pass.
#include <omp.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <vector>

#include "dsq/dns.hpp"
#include "dsq/kernels.hpp"
#include "dsq/nuq.hpp"
#include "dsq/pipeline.hpp"
#include "dsq/sensitivity.hpp"
#include "dsq_cuda.hpp"

namespace {

float round_f16(float f) {
    // round to the nearest fp16 value (the device stores fp16): via the
    // library's own behaviour is not allowed here, so use a portable routine
    if (f == 0.0f || !std::isfinite(f)) return f;
    int e;
    const float m = std::frexp(f, &e);              // f = m * 2^e, 0.5 <= |m| < 1
    const int shift = e < -13 ? 24 + e : 11;  // mantissa bits kept (subnormals fewer)
    const float q = std::ldexp(std::nearbyint(std::ldexp(m, shift)), -shift);
    return std::ldexp(q, e);
}

int fail(const char* what, double v) {
    std::printf("FAIL %s (%g)\n", what, v);
    return 1;
}

double normwise(const std::vector<double>& a, const std::vector<double>& b) {
    double d = 0, m = 0;
    for (size_t i = 0; i < a.size(); ++i) {
        d = std::max(d, std::fabs(a[i] - b[i]));
        m = std::max(m, std::fabs(b[i]));
    }
    return m > 0 ? d / m : d;
}

}  // namespace

int main() {
    using namespace dsq;
    const uint32_t rows = 96, cols = 256;
    Rng rng(7);
    WeightMatrix w;
    w.name = "wrapped";
    w.rows = rows;
    w.cols = cols;
    w.values.resize(size_t(rows) * cols);
    for (auto& v : w.values) v = float(rng.student_t(4.0));
    SensitivityMap s = uniform_sensitivity(w.name, rows, cols);
    for (auto& v : s.values) v = float(rng.uniform());
    QuantizeOptions opt;
    opt.cfg.bits = 3;
    opt.cfg.sensitive_fraction = 0.0005;
    opt.cfg.outlier_fraction = 0.004;
    QuantizedLayer layer = quantize_layer(w, s, opt);
    // fp16-exact centroids / deltas / x so the comparison is tolerance-tight
    for (auto& v : layer.packed.luts) v = round_f16(v);
    for (auto& v : layer.sparse.values) v = round_f16(v);
    layer.hybrid = hybrid_split(layer.sparse, layer.hybrid_top_k);
    std::vector<float> x(cols);
    for (auto& v : x) v = round_f16(float(rng.normal()));

    try {
        sqz::DeviceLayer dev(layer);
        const double e_fused = normwise(dev.fused(x), fused_dns_matvec(layer, x));
        const double e_lut = normwise(dev.lut(x), lut_matvec(layer.packed, x));
        const double e_csr = normwise(dev.csr(x), csr_matvec(layer.sparse, x));
        const double e_once = normwise(sqz::fused_dns_matvec(layer, x), fused_dns_matvec(layer, x));
        std::printf("normwise err fused %.3e lut %.3e csr %.3e one-shot %.3e\n", e_fused, e_lut,
                    e_csr, e_once);
        if (e_fused > 1e-5) return fail("fused", e_fused);
        if (e_lut > 1e-5) return fail("lut", e_lut);
        if (e_csr > 1e-5) return fail("csr", e_csr);
        if (e_once > 1e-5) return fail("one-shot", e_once);
        if (sqz::bytes_touched_estimate(rows, cols, 3, 0, layer.sparse.nnz()) !=
            bytes_touched_estimate(layer))
            return fail("bytes_touched_estimate", 0);
        // the reference's free functions, namespace switched (kernels.hpp:20-79)
        const double f_lut = normwise(sqz::lut_matvec(layer.packed, x), lut_matvec(layer.packed, x));
        const double f_csr =
            normwise(sqz::csr_matvec(layer.sparse, x, Exec::serial), csr_matvec(layer.sparse, x));
        const double f_fused = normwise(sqz::fused_dns_matvec(layer, x, Exec::parallel),
                                        fused_dns_matvec(layer, x));
        const std::vector<float> dq = ref::dequant_dense(layer.packed);
        const double f_dense =
            normwise(sqz::dense_matvec(dq, rows, cols, x), dense_matvec(dq, rows, cols, x));
        std::printf("free functions: lut %.3e csr %.3e fused %.3e dense %.3e\n", f_lut, f_csr,
                    f_fused, f_dense);
        if (f_lut > 1e-5) return fail("sqz::lut_matvec", f_lut);
        if (f_csr > 1e-5) return fail("sqz::csr_matvec", f_csr);
        if (f_fused > 1e-5) return fail("sqz::fused_dns_matvec", f_fused);
        if (f_dense > 1e-12) return fail("sqz::dense_matvec", f_dense);
        if (sqz::bytes_touched_estimate(layer) != bytes_touched_estimate(layer))
            return fail("sqz::bytes_touched_estimate(layer)", 0);
        for (BenchKernel k : {BenchKernel::lut, BenchKernel::csr, BenchKernel::fused,
                              BenchKernel::reference}) {
            const BenchRecord r = bench_matvec(layer, x, 3, k, Exec::parallel);
            const sqz::BenchRecord g = sqz::bench_matvec(layer, x, 3, k, Exec::parallel);
            if (g.kernel != r.kernel || g.repeats != 3 || g.all_seconds.size() != 3 ||
                g.bytes_touched != r.bytes_touched || !(g.median_seconds > 0))
                return fail("sqz::bench_matvec", double(int(k)));
            std::printf("bench_matvec %-9s median %.1f us (reference %.1f us), %llu bytes\n",
                        g.kernel.c_str(), g.median_seconds * 1e6, r.median_seconds * 1e6,
                        (unsigned long long)g.bytes_touched);
        }
        try {
            sqz::bench_matvec(layer, x, 2, BenchKernel::fused);
            return fail("bench repeats < 3 accepted", 0);
        } catch (const sqz::Error& e) {
            if (e.errc() != int(errc::invalid_argument)) return fail("bench errc", e.errc());
        }
        // dequantize_layer (pipeline.cpp:49-75): bit-identical for fp16-exact layers
        const WeightMatrix wr = dequantize_layer(layer);
        const WeightMatrix wg = sqz::dequantize_layer<WeightMatrix>(layer);
        if (wg.name != wr.name || wg.rows != wr.rows || wg.cols != wr.cols ||
            wg.values != wr.values)
            return fail("sqz::dequantize_layer", 0);
        // error mapping: a dimension mismatch is dsq::errc::shape_mismatch
        try {
            dev.fused(std::vector<float>(cols + 1));
            return fail("no error on bad x", 0);
        } catch (const sqz::Error& e) {
            if (e.errc() != int(errc::shape_mismatch)) return fail("errc mapping", e.errc());
        }
        // the producer side: decompose + quantize_channelwise on the GPU with
        // the reference's types, bit-identical to the reference's
        const Decomposition dr = decompose(w, s.values, opt.cfg);
        const Decomposition dg = sqz::decompose<Decomposition>(w, s.values, opt.cfg);
        if (dg.mask != dr.mask || dg.sparse.row_ptr != dr.sparse.row_ptr ||
            dg.sparse.col_idx != dr.sparse.col_idx || dg.sparse.values != dr.sparse.values ||
            dg.dense.values != dr.dense.values || dg.t_min != dr.t_min || dg.t_max != dr.t_max ||
            dg.sensitive_count != dr.sensitive_count || dg.outlier_count != dr.outlier_count)
            return fail("decompose", 0);
        const ChannelwiseResult cr = quantize_channelwise(w, s.values, opt.cfg, dr.mask);
        const ChannelwiseResult cg =
            sqz::quantize_channelwise<ChannelwiseResult>(w, s.values, opt.cfg, dr.mask);
        if (cg.assignment != cr.assignment || cg.codebooks.size() != cr.codebooks.size() ||
            cg.weighted_objective != cr.weighted_objective ||
            cg.unweighted_mse_sum != cr.unweighted_mse_sum)
            return fail("quantize_channelwise", 0);
        for (size_t g = 0; g < cr.codebooks.size(); ++g)
            if (cg.codebooks[g].centroids != cr.codebooks[g].centroids)
                return fail("codebook", double(g));
        std::printf("decompose + quantize_channelwise: bit-identical (%u extracted)\n",
                    dr.sparse.row_ptr.back());
    } catch (const sqz::Error& e) {
        std::printf("sqz::Error status %d: %s\n", e.status(), e.what());
        return 2;
    }
    // the reference-signature call at LLaMA-7B shapes (the cmd_matvec path):
    // wall time per product, our host call vs the reference on the host cores
    try {
        for (uint32_t rc2 : {4096u, 11008u}) {
            const uint32_t R = rc2, Cc = 4096;
            Rng r2(11);
            AssignmentVector as(size_t(R) * Cc);
            for (auto& a : as) a = uint16_t(r2.below(8));
            std::vector<Codebook> cbs(R);
            for (auto& cb : cbs) {
                cb.centroids.resize(8);
                for (auto& c : cb.centroids) c = round_f16(float(r2.normal()) * 0.02f);
                std::sort(cb.centroids.begin(), cb.centroids.end());
            }
            QuantizedLayer big;
            big.name = "big";
            big.rows = R;
            big.cols = Cc;
            big.packed = pack(as, cbs, 3, R, Cc);
            std::vector<uint32_t> tr, tc;
            std::vector<float> tv;
            for (uint32_t r = 0; r < R; ++r)
                for (uint32_t c = r % 223; c < Cc; c += 223) {  // ~0.45%
                    tr.push_back(r);
                    tc.push_back(c);
                    tv.push_back(round_f16(float(r2.normal()) * 0.2f));
                }
            big.sparse = csr_from_triplets(R, Cc, tr, tc, tv);
            big.hybrid_top_k = 10;
            big.hybrid = hybrid_split(big.sparse, 10);
            std::vector<float> xb(Cc);
            for (auto& v : xb) v = round_f16(float(r2.normal()));
            const sqz::BenchRecord g = sqz::bench_matvec(big, xb, 51, BenchKernel::fused);
            const BenchRecord rr = bench_matvec(big, xb, 5, BenchKernel::fused, Exec::parallel);
            const double e = normwise(sqz::DeviceLayer(big).fused(xb), fused_dns_matvec(big, xb));
            std::printf("host call %ux%u fused: %.1f us per product (reference %.0f us, %d threads),"
                        " normwise err %.2e\n", R, Cc, g.median_seconds * 1e6,
                        rr.median_seconds * 1e6, omp_get_max_threads(), e);
            if (e > 1e-5) return fail("host call at 7B shape", e);
        }
    } catch (const sqz::Error& e) {
        std::printf("sqz::Error status %d: %s\n", e.status(), e.what());
        return 2;
    }
    std::printf("PASS\n");
    return 0;
}
