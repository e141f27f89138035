// Roofline performance model: the reference's
// analytical decode-step cost model (include/dsq/roofline.hpp:10-88,
// src/roofline.cpp:10-209, `dsq profile` tools/dsq.cpp:220-271) behind the C
// ABI, plus a B200 HardwareProfile and the per-GEMV prediction of the
// SqueezeLLM path (reference-charged bytes / HBM bandwidth) that bench.py and
// tools/dsq_profile.py print beside measured numbers.
//
// Host arithmetic only (no device code).  Every formula keeps the reference's
// evaluation order so the doubles agree bit for bit with the compiled
// reference (tests/test_roofline.py).
#include <cerrno>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include "../../include/dsq_cuda.h"

extern "C" int dsq_internal_fail(int code, const char* fmt, ...);

namespace {

void set_name(char* dst, size_t cap, const char* src) {
    std::snprintf(dst, cap, "%s", src ? src : "");
}

int check_hw(const dsq_hw_profile* hw) {
    if (!hw) return dsq_internal_fail(DSQ_E_INVALID_ARGUMENT, "hardware profile: null");
    if (!(hw->peak_flops > 0.0 && hw->mem_bandwidth > 0.0))  // roofline.cpp:10-13
        return dsq_internal_fail(DSQ_E_INVALID_ARGUMENT,
                                 "hardware profile: throughput and bandwidth must be positive");
    return DSQ_OK;
}

int check_shape(const dsq_model_shape* s) {  // roofline.cpp:15-23
    if (!s) return dsq_internal_fail(DSQ_E_INVALID_ARGUMENT, "model shape: null");
    if (!(s->num_layers >= 1 && s->hidden_dim >= 1 && s->ffn_dim >= 1 && s->num_heads >= 1 &&
          s->vocab_size >= 1 && s->seq_len >= 1))
        return dsq_internal_fail(DSQ_E_INVALID_ARGUMENT, "model shape: dims must be positive");
    if (s->hidden_dim % s->num_heads != 0)
        return dsq_internal_fail(DSQ_E_INVALID_ARGUMENT,
                                 "model shape: hidden_dim must divide by num_heads");
    if (s->weight_bits < 2 || s->weight_bits > 16)
        return dsq_internal_fail(DSQ_E_INVALID_ARGUMENT, "model shape: weight_bits must be in 2..16");
    return DSQ_OK;
}

void finish_cost(dsq_layer_cost& c, const dsq_hw_profile& hw) {
    const double bytes = c.weight_bytes + c.activation_bytes;
    const double t_mem = bytes / hw.mem_bandwidth, t_cmp = c.flops / hw.peak_flops;
    c.predicted_s = t_cmp > t_mem ? t_cmp : t_mem;  // max(flops/peak, bytes/bw)
    c.memory_bound = t_mem >= t_cmp ? 1 : 0;
    const double elems = c.weight_elems + c.activation_elems;
    c.intensity = (c.flops > 0.0 && elems > 0.0) ? c.flops / elems : 0.0;
}

// a matvec of out x in weights repeated `count` times (roofline.cpp:47-60)
dsq_layer_cost matvec(const char* name, double out_dim, double in_dim, double count,
                      double wbits, double abits) {
    dsq_layer_cost c{};
    set_name(c.name, sizeof c.name, name);
    c.kind = DSQ_LAYER_FC;
    const double w = out_dim * in_dim * count;
    c.flops = 2.0 * w;
    c.weight_elems = w;
    c.activation_elems = (in_dim + out_dim) * count;
    c.weight_bytes = w * wbits / 8.0;
    c.activation_bytes = c.activation_elems * abits / 8.0;
    return c;
}

// per-decode-step costs; n == 8 entries (6 projections, attention, other)
void step_costs(const dsq_model_shape& s, const dsq_hw_profile& hw, dsq_layer_cost* out,
                dsq_layer_cost* total, double* share) {
    const double L = s.num_layers, h = s.hidden_dim, f = s.ffn_dim;
    const double ab = s.activation_bits ? s.activation_bits : 16.0, wb = s.weight_bits;
    const double kv = (double(s.seq_len) - 1.0) / 2.0;  // mean cache length
    out[0] = matvec("qkv_proj", 3.0 * h, h, L, wb, ab);
    out[1] = matvec("out_proj", h, h, L, wb, ab);
    out[2] = matvec("ffn_gate", f, h, L, wb, ab);
    out[3] = matvec("ffn_up", f, h, L, wb, ab);
    out[4] = matvec("ffn_down", h, f, L, wb, ab);
    out[5] = matvec("lm_head", s.vocab_size, h, 1.0, wb, ab);
    {  // score + context products over the cached keys / values
        dsq_layer_cost& c = out[6];
        c = dsq_layer_cost{};
        set_name(c.name, sizeof c.name, "attn_kv");
        c.kind = DSQ_LAYER_ATTENTION;
        c.flops = 4.0 * h * kv * L;
        c.activation_elems = (2.0 * h * kv + 2.0 * h + 2.0 * double(s.num_heads) * kv) * L;
        c.activation_bytes = c.activation_elems * ab / 8.0;
    }
    {  // norms, residuals, nonlinearities, embedding row, logits
        dsq_layer_cost& c = out[7];
        c = dsq_layer_cost{};
        set_name(c.name, sizeof c.name, "other");
        c.kind = DSQ_LAYER_OTHER;
        c.flops = (10.0 * h + 2.0 * f) * L + double(s.vocab_size);
        c.activation_elems = (10.0 * h + 2.0 * f) * L + h + double(s.vocab_size);
        c.activation_bytes = c.activation_elems * ab / 8.0;
    }
    dsq_layer_cost t{};
    set_name(t.name, sizeof t.name, "total");
    t.kind = DSQ_LAYER_OTHER;
    for (int i = 0; i < DSQ_DECODE_COSTS; ++i) {
        finish_cost(out[i], hw);
        t.flops += out[i].flops;
        t.weight_elems += out[i].weight_elems;
        t.activation_elems += out[i].activation_elems;
        t.weight_bytes += out[i].weight_bytes;
        t.activation_bytes += out[i].activation_bytes;
    }
    finish_cost(t, hw);
    if (total) *total = t;
    if (share) *share = t.weight_elems / (t.weight_elems + t.activation_elems);
}

double step_time(const dsq_model_shape& s, const dsq_hw_profile& hw) {
    dsq_layer_cost c[DSQ_DECODE_COSTS];
    step_costs(s, hw, c, nullptr, nullptr);
    double t = 0.0;
    for (const auto& x : c) t += x.predicted_s;  // sum of per-layer times
    return t;
}

// --- minimal reader for the flat JSON profile files (name + numbers) -------
struct Json {
    std::string text;
    // value text of "key": ... (string without quotes, or a number token)
    bool get(const char* key, std::string& v) const {
        const std::string k = std::string("\"") + key + "\"";
        size_t p = text.find(k);
        if (p == std::string::npos) return false;
        p = text.find(':', p + k.size());
        if (p == std::string::npos) return false;
        ++p;
        while (p < text.size() && std::isspace(static_cast<unsigned char>(text[p]))) ++p;
        if (p >= text.size()) return false;
        if (text[p] == '"') {
            const size_t e = text.find('"', p + 1);
            if (e == std::string::npos) return false;
            v = text.substr(p + 1, e - p - 1);
            return true;
        }
        size_t e = p;
        while (e < text.size() && text[e] != ',' && text[e] != '}' && !std::isspace(
                   static_cast<unsigned char>(text[e])))
            ++e;
        v = text.substr(p, e - p);
        return !v.empty();
    }
};

int read_json(const char* path, Json& j) {
    FILE* f = path ? std::fopen(path, "rb") : nullptr;
    if (!f) return dsq_internal_fail(DSQ_E_MISSING_FILE, "cannot open profile: %s", path ? path : "");
    char buf[4096];
    size_t n;
    while ((n = std::fread(buf, 1, sizeof buf, f)) > 0) j.text.append(buf, n);
    std::fclose(f);
    const size_t a = j.text.find_first_not_of(" \t\r\n");
    if (a == std::string::npos || j.text[a] != '{' || j.text.find('}') == std::string::npos)
        return dsq_internal_fail(DSQ_E_MALFORMED_HEADER, "%s: not a JSON object", path);
    return DSQ_OK;
}

int num(const Json& j, const char* path, const char* key, double& out, bool required) {
    std::string v;
    // a missing key / a non-number: the reference's json::at / get<> throw a
    // non-dsq exception, which its CLI reports as an internal error (exit 4)
    if (!j.get(key, v)) {
        if (!required) return DSQ_OK;
        return dsq_internal_fail(DSQ_E_INTERNAL, "%s: missing key \"%s\"", path, key);
    }
    char* end = nullptr;
    errno = 0;
    const double d = std::strtod(v.c_str(), &end);
    if (errno || !end || *end)
        return dsq_internal_fail(DSQ_E_INTERNAL, "%s: \"%s\" is not a number", path, key);
    out = d;
    return DSQ_OK;
}

}  // namespace

extern "C" {

int dsq_decode_step_costs(const dsq_model_shape* shape, const dsq_hw_profile* hw,
                          dsq_layer_cost* costs, dsq_layer_cost* total,
                          double* weight_traffic_share) {
    int rc = check_shape(shape);
    if (rc) return rc;
    if ((rc = check_hw(hw))) return rc;
    if (!costs) return dsq_internal_fail(DSQ_E_INVALID_ARGUMENT, "decode_step_costs: null output");
    step_costs(*shape, *hw, costs, total, weight_traffic_share);
    return DSQ_OK;
}

int dsq_arithmetic_intensity(const dsq_layer_cost* c, double* out) {  // roofline.cpp:34-40
    if (!c || !out) return dsq_internal_fail(DSQ_E_INVALID_ARGUMENT, "arithmetic_intensity: null");
    const double elems = c->weight_elems + c->activation_elems;
    if (!(c->flops > 0.0))
        return dsq_internal_fail(DSQ_E_INVALID_ARGUMENT, "arithmetic_intensity: zero-flop layer");
    if (!(elems > 0.0))
        return dsq_internal_fail(DSQ_E_INVALID_ARGUMENT, "arithmetic_intensity: zero memory ops");
    *out = c->flops / elems;
    return DSQ_OK;
}

int dsq_predicted_runtime_curve(const dsq_model_shape* shape, const dsq_hw_profile* hw,
                                const uint32_t* bits, uint32_t n, double* seconds,
                                double* normalized) {
    int rc = check_shape(shape);
    if (rc) return rc;
    if ((rc = check_hw(hw))) return rc;
    if (n && (!bits || !seconds || !normalized))
        return dsq_internal_fail(DSQ_E_INVALID_ARGUMENT, "runtime curve: null arrays");
    dsq_model_shape s = *shape;
    s.weight_bits = 16;
    const double base = step_time(s, *hw);
    for (uint32_t i = 0; i < n; ++i) {
        if (bits[i] < 2 || bits[i] > 16)
            return dsq_internal_fail(DSQ_E_INVALID_ARGUMENT, "runtime curve: bits must be in 2..16");
        s.weight_bits = bits[i];
        seconds[i] = step_time(s, *hw);
        normalized[i] = seconds[i] / base;
    }
    return DSQ_OK;
}

int dsq_affine_fit_r2(const uint32_t* bits, const double* normalized, uint32_t n, double* r2) {
    if (n < 3 || !bits || !normalized || !r2)
        return dsq_internal_fail(DSQ_E_INVALID_ARGUMENT, "affine fit: need >= 3 points");
    double sx = 0, sy = 0, sxx = 0, sxy = 0;  // least squares of y = a + b x
    for (uint32_t i = 0; i < n; ++i) {
        sx += bits[i];
        sy += normalized[i];
        sxx += double(bits[i]) * bits[i];
        sxy += double(bits[i]) * normalized[i];
    }
    const double cnt = double(n);
    const double b = (cnt * sxy - sx * sy) / (cnt * sxx - sx * sx);
    const double a = (sy - b * sx) / cnt;
    const double mean = sy / cnt;
    double res = 0, tot = 0;
    for (uint32_t i = 0; i < n; ++i) {
        const double e = normalized[i] - (a + b * bits[i]);
        res += e * e;
        tot += (normalized[i] - mean) * (normalized[i] - mean);
    }
    *r2 = tot == 0.0 ? 1.0 : 1.0 - res / tot;
    return DSQ_OK;
}

int dsq_load_hardware_profile(const char* path, dsq_hw_profile* out) {
    if (!out) return dsq_internal_fail(DSQ_E_INVALID_ARGUMENT, "null profile");
    Json j;
    int rc = read_json(path, j);
    if (rc) return rc;
    dsq_hw_profile hw{};
    std::string name;
    if (!j.get("name", name))
        return dsq_internal_fail(DSQ_E_INTERNAL, "%s: missing key \"name\"", path);
    set_name(hw.name, sizeof hw.name, name.c_str());
    if ((rc = num(j, path, "peak_flops", hw.peak_flops, true)) ||
        (rc = num(j, path, "mem_bandwidth_bytes_per_s", hw.mem_bandwidth, true)))
        return rc;
    if ((rc = check_hw(&hw))) return rc;
    *out = hw;
    return DSQ_OK;
}

int dsq_load_model_shape(const char* path, dsq_model_shape* out) {
    if (!out) return dsq_internal_fail(DSQ_E_INVALID_ARGUMENT, "null shape");
    Json j;
    int rc = read_json(path, j);
    if (rc) return rc;
    dsq_model_shape s{};
    std::string name;
    if (!j.get("name", name))
        return dsq_internal_fail(DSQ_E_INTERNAL, "%s: missing key \"name\"", path);
    set_name(s.name, sizeof s.name, name.c_str());
    double v[8] = {0, 0, 0, 0, 0, 128, 16, 16};  // seq_len / weight_bits defaults
    const char* keys[7] = {"num_layers", "hidden_dim", "ffn_dim", "num_heads",
                           "vocab_size", "seq_len", "weight_bits"};
    for (int i = 0; i < 7; ++i)
        if ((rc = num(j, path, keys[i], v[i], i < 5))) return rc;
    for (int i = 0; i < 7; ++i)
        if (v[i] < 0 || v[i] > 4294967295.0 || v[i] != std::floor(v[i]))
            return dsq_internal_fail(DSQ_E_INTERNAL, "%s: \"%s\" is not a u32", path, keys[i]);
    s.num_layers = uint32_t(v[0]);
    s.hidden_dim = uint32_t(v[1]);
    s.ffn_dim = uint32_t(v[2]);
    s.num_heads = uint32_t(v[3]);
    s.vocab_size = uint32_t(v[4]);
    s.seq_len = uint32_t(v[5]);
    s.weight_bits = uint32_t(v[6]);
    s.activation_bits = 16;
    if ((rc = check_shape(&s))) return rc;
    *out = s;
    return DSQ_OK;
}

// B200: the measured copy bandwidth and dense bf16 tensor throughput of this
// pool (MEASURED_PEAKS.json, driver-written: "hbm_gbs", "bf16_tflops"), else
// the profiling recipe's fallback 6.65 TB/s and 1.59 PFLOP/s
int dsq_hw_profile_b200(const char* measured_peaks_json, dsq_hw_profile* out) {
    if (!out) return dsq_internal_fail(DSQ_E_INVALID_ARGUMENT, "null profile");
    dsq_hw_profile hw{};
    double gbs = 6650.0, tflops = 1590.0;
    bool measured = false;
    if (measured_peaks_json) {
        Json j;
        if (read_json(measured_peaks_json, j) == DSQ_OK) {
            double g = 0, t = 0;
            if (num(j, measured_peaks_json, "hbm_gbs", g, false) == DSQ_OK && g > 0) {
                gbs = g;
                measured = true;
            }
            if (num(j, measured_peaks_json, "bf16_tflops", t, false) == DSQ_OK && t > 0) tflops = t;
        }
    }
    set_name(hw.name, sizeof hw.name, measured ? "B200 (measured)" : "B200 (fallback)");
    hw.mem_bandwidth = gbs * 1e9;
    hw.peak_flops = tflops * 1e12;
    *out = hw;
    return DSQ_OK;
}

// one fused Dense-and-Sparse LUT-GEMV of the path: reference-charged bytes
// (kernels.cpp:205-212) and 2*B*(rows*cols+nnz) flops against the profile
int dsq_gemv_cost(uint32_t rows, uint32_t cols, uint32_t bits, uint64_t nnz, uint32_t batch,
                  const dsq_hw_profile* hw, dsq_layer_cost* out) {
    int rc = check_hw(hw);
    if (rc) return rc;
    if (!out || rows == 0 || cols == 0 || bits < 2 || bits > 8 || batch == 0)
        return dsq_internal_fail(DSQ_E_INVALID_ARGUMENT, "gemv_cost: bad arguments");
    dsq_layer_cost c{};
    set_name(c.name, sizeof c.name, "dns_lut_gemv");
    c.kind = DSQ_LAYER_FC;
    const double w = double(rows) * cols;
    c.flops = 2.0 * batch * (w + double(nnz));
    c.weight_elems = w + double(nnz);
    c.activation_elems = double(batch) * (double(cols) + rows);
    const uint64_t once = dsq_bytes_touched_estimate(rows, cols, bits, 0, nnz);  // incl. 1 x + 1 y
    c.activation_bytes = double(batch) * (double(cols) * 2.0 + double(rows) * 2.0);
    c.weight_bytes = double(once) - (double(cols) * 2.0 + double(rows) * 2.0);
    finish_cost(c, *hw);
    *out = c;
    return DSQ_OK;
}

}  // extern "C"
