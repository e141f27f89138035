// ref_roofline_shim.cpp -- C entry points over the UNMODIFIED reference
// roofline module (TEST INFRASTRUCTURE).  oracle/Makefile compiles it with
// /root/reference/proj/src/roofline.cpp (which needs nlohmann/json.hpp: the
// copy vendored in the cudnn_frontend headers of this image) into
// oracle/_ref/libdsqref_roofline.so.  tests/test_roofline.py pins the
// product's roofline model (paper_2306_07629_b200/csrc/roofline.cpp) to it.
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "dsq/roofline.hpp"

using namespace dsq;

namespace {
thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const Error& e) {
        g_err = e.what();
        return int(e.code()) + 1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 100;
    }
}

ModelShape shape_of(const uint32_t* s) {
    ModelShape m;
    m.name = "shape";
    m.num_layers = s[0];
    m.hidden_dim = s[1];
    m.ffn_dim = s[2];
    m.num_heads = s[3];
    m.vocab_size = s[4];
    m.seq_len = s[5];
    m.weight_bits = s[6];
    return m;
}

HardwareProfile hw_of(double peak, double bw) {
    HardwareProfile h;
    h.name = "hw";
    h.peak_flops = peak;
    h.mem_bandwidth = bw;
    return h;
}

// flops, weight_elems, activation_elems, weight_bytes, activation_bytes,
// predicted_time, memory_bound, kind
void put(const LayerCost& c, const HardwareProfile& hw, double* o) {
    o[0] = c.flops;
    o[1] = c.weight_elems;
    o[2] = c.activation_elems;
    o[3] = c.weight_bytes;
    o[4] = c.activation_bytes;
    o[5] = c.predicted_time(hw);
    o[6] = c.memory_bound(hw) ? 1.0 : 0.0;
    o[7] = double(int(c.kind));
}
}  // namespace

extern "C" {

const char* dsqref_roofline_last_error() { return g_err.c_str(); }

// shape = {layers, hidden, ffn, heads, vocab, seq_len, weight_bits};
// out = (n_layers + 1) x 8 doubles (the total last); returns the layer count
int dsqref_decode_step_costs(const uint32_t* shape, double peak, double bw, double* out,
                             uint32_t cap, uint32_t* n, double* share) {
    return guarded([&] {
        const HardwareProfile hw = hw_of(peak, bw);
        const DecodeCosts dc = decode_step_costs(shape_of(shape), hw);
        if (dc.layers.size() + 1 > cap) fail(errc::invalid_argument, "shim: cap");
        for (size_t i = 0; i < dc.layers.size(); ++i) put(dc.layers[i], hw, out + 8 * i);
        put(dc.total, hw, out + 8 * dc.layers.size());
        *n = uint32_t(dc.layers.size());
        *share = dc.weight_traffic_share;
    });
}

int dsqref_runtime_curve(const uint32_t* shape, double peak, double bw, const uint32_t* bits,
                         uint32_t n, double* seconds, double* normalized) {
    return guarded([&] {
        const auto pts = predicted_runtime_curve(shape_of(shape), hw_of(peak, bw),
                                                 std::vector<uint32_t>(bits, bits + n));
        for (uint32_t i = 0; i < n; ++i) {
            seconds[i] = pts[i].seconds;
            normalized[i] = pts[i].normalized;
        }
    });
}

int dsqref_affine_fit_r2(const uint32_t* bits, const double* normalized, uint32_t n, double* r2) {
    return guarded([&] {
        std::vector<RuntimePoint> pts(n);
        for (uint32_t i = 0; i < n; ++i) {
            pts[i].bits = bits[i];
            pts[i].normalized = normalized[i];
        }
        *r2 = affine_fit_r2(pts);
    });
}

int dsqref_arithmetic_intensity(double flops, double welems, double aelems, double* out) {
    return guarded([&] {
        LayerCost c;
        c.flops = flops;
        c.weight_elems = welems;
        c.activation_elems = aelems;
        *out = arithmetic_intensity(c);
    });
}

int dsqref_load_hardware_profile(const char* path, double* peak, double* bw) {
    return guarded([&] {
        const HardwareProfile h = load_hardware_profile(path);
        *peak = h.peak_flops;
        *bw = h.mem_bandwidth;
    });
}

// out = {layers, hidden, ffn, heads, vocab, seq_len, weight_bits}
int dsqref_load_model_shape(const char* path, uint32_t* out) {
    return guarded([&] {
        const ModelShape s = load_model_shape(path);
        const uint32_t v[7] = {s.num_layers, s.hidden_dim, s.ffn_dim, s.num_heads,
                               s.vocab_size, s.seq_len, s.weight_bits};
        std::memcpy(out, v, sizeof v);
    });
}

}  // extern "C"
