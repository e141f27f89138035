// container.cpp -- the on-disk input of the hot path: "DSQCONT1" quantized
// model containers (reference src/container.cpp:146-223) parsed on the host
// and uploaded as device layers.
//
// Format (little-endian, container.cpp:82-100,146-179):
//   magic "DSQCONT1" | u32 version (1) | payload | u32 CRC-32(payload)
//   payload: u32 bits | f64 sens_frac | f64 out_frac | u32 group_size |
//            u32 iters | f64 tol | u64 seed | u32 hybrid_top_k | u32 method |
//            u32 n_layers | layer*
//   layer:   str name (u32 len + bytes) | u32 rows | u32 cols | u32 bits |
//            u32 groups | f32 luts[rows*groups*2^bits] | u64 payload_len |
//            payload | u32 nnz | u32 row_ptr[rows+1] | u16 col[nnz] |
//            f32 val[nnz] | u32 hybrid_top_k | f64 avg_bits
// Checks and error codes follow load_container / read_layer
// (container.cpp:102-142,181-223): missing file, short file / bad magic /
// bad bits or groups -> malformed_header, version -> unsupported_version,
// CRC -> checksum_mismatch, truncation / payload length / trailing bytes ->
// truncated_payload, then QuantizedLayer::validate (via the layer view
// validation of dsq_cuda_layer_create).  The hybrid split is not read (the
// reference recomputes it on load, container.cpp:138-139; the device does
// not need it).  CRC-32 is the zlib polynomial, computed here.
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/dsq_cuda.h"

extern "C" int dsq_internal_fail(int code, const char* fmt, ...);
extern "C" int dsq_internal_validate_view(const dsq_layer_view* v);

namespace {

uint32_t crc32_zlib(const uint8_t* p, size_t n) {
    static uint32_t table[256];
    static bool init = false;
    if (!init) {
        for (uint32_t i = 0; i < 256; ++i) {
            uint32_t c = i;
            for (int k = 0; k < 8; ++k) c = (c & 1u) ? 0xEDB88320u ^ (c >> 1) : c >> 1;
            table[i] = c;
        }
        init = true;
    }
    uint32_t c = 0xFFFFFFFFu;
    for (size_t i = 0; i < n; ++i) c = table[(c ^ p[i]) & 0xFFu] ^ (c >> 8);
    return c ^ 0xFFFFFFFFu;
}

struct HostLayer {
    std::string name;
    uint32_t rows = 0, cols = 0, bits = 0, groups = 1, hybrid_top_k = 0;
    double avg_bits = 0;
    std::vector<float> luts;
    std::vector<uint8_t> payload;
    std::vector<uint32_t> row_ptr;
    std::vector<uint16_t> col_idx;
    std::vector<float> values;

    dsq_layer_view view() const {
        dsq_layer_view v{};
        v.name = name.c_str();
        v.rows = rows;
        v.cols = cols;
        v.packed.bits = bits;
        v.packed.rows = rows;
        v.packed.cols = cols;
        v.packed.groups_per_row = groups;
        v.packed.luts_f32 = luts.data();
        v.packed.payload = payload.data();
        v.packed.payload_len = payload.size();
        v.sparse.rows = rows;
        v.sparse.cols = cols;
        v.sparse.nnz = uint32_t(col_idx.size());
        v.sparse.row_ptr = row_ptr.data();
        v.sparse.col_idx = col_idx.empty() ? nullptr : col_idx.data();
        v.sparse.values_f32 = values.empty() ? nullptr : values.data();
        v.hybrid_top_k = hybrid_top_k;
        return v;
    }
};

struct Reader {
    const uint8_t* p;
    const uint8_t* end;
    bool ok = true;
    const uint8_t* take(size_t n) {
        if (!ok || size_t(end - p) < n) {
            ok = false;
            return nullptr;
        }
        const uint8_t* r = p;
        p += n;
        return r;
    }
    uint64_t le(int nb) {
        const uint8_t* q = take(size_t(nb));
        uint64_t v = 0;
        if (q)
            for (int i = nb - 1; i >= 0; --i) v = (v << 8) | q[i];
        return v;
    }
    uint32_t u32() { return uint32_t(le(4)); }
    uint16_t u16() { return uint16_t(le(2)); }
    uint64_t u64() { return le(8); }
    float f32() {
        const uint32_t b = u32();
        float f;
        std::memcpy(&f, &b, 4);
        return f;
    }
    double f64() {
        const uint64_t b = u64();
        double d;
        std::memcpy(&d, &b, 8);
        return d;
    }
};

#define TRUNC() dsq_internal_fail(DSQ_E_TRUNCATED_PAYLOAD, "container: truncated payload")

int parse(const char* path, dsq_container_meta* meta, std::vector<HostLayer>* out) {
    FILE* f = std::fopen(path, "rb");
    if (!f) return dsq_internal_fail(DSQ_E_MISSING_FILE, "cannot open container: %s", path);
    std::fseek(f, 0, SEEK_END);
    const long size = std::ftell(f);
    std::fseek(f, 0, SEEK_SET);
    if (size < 16) {
        std::fclose(f);
        return dsq_internal_fail(DSQ_E_MALFORMED_HEADER, "%s: file too small", path);
    }
    std::vector<uint8_t> raw(static_cast<size_t>(size), 0);
    const size_t got = std::fread(raw.data(), 1, raw.size(), f);
    std::fclose(f);
    if (got != raw.size()) return dsq_internal_fail(DSQ_E_IO_FAILURE, "%s: short read", path);
    if (std::memcmp(raw.data(), "DSQCONT1", 8) != 0)
        return dsq_internal_fail(DSQ_E_MALFORMED_HEADER, "%s: bad magic", path);
    uint32_t version = 0;
    for (int i = 3; i >= 0; --i) version = (version << 8) | raw[8 + i];
    if (version != 1)
        return dsq_internal_fail(DSQ_E_UNSUPPORTED_VERSION,
                                 "%s: unsupported container version %u", path, version);
    const uint8_t* payload = raw.data() + 12;
    const size_t payload_len = raw.size() - 16;
    uint32_t stored = 0;
    for (int i = 3; i >= 0; --i) stored = (stored << 8) | raw[raw.size() - 4 + i];
    if (crc32_zlib(payload, payload_len) != stored)
        return dsq_internal_fail(DSQ_E_CHECKSUM_MISMATCH, "%s: checksum mismatch", path);

    Reader r{payload, payload + payload_len};
    dsq_container_meta m{};
    m.bits = r.u32();
    m.sensitive_fraction = r.f64();
    m.outlier_fraction = r.f64();
    m.group_size = r.u32();
    m.kmeans_max_iters = r.u32();
    m.kmeans_tol = r.f64();
    m.seed = r.u64();
    m.hybrid_top_k = r.u32();
    m.method_code = r.u32();
    m.n_layers = r.u32();
    if (!r.ok) return TRUNC();
    std::vector<HostLayer> layers;
    for (uint32_t li = 0; li < m.n_layers; ++li) {
        HostLayer L;
        const uint32_t nlen = r.u32();
        const uint8_t* nm = r.take(nlen);
        if (!r.ok) return TRUNC();
        L.name.assign(reinterpret_cast<const char*>(nm), nlen);
        L.rows = r.u32();
        L.cols = r.u32();
        L.bits = r.u32();
        L.groups = r.u32();
        if (!r.ok) return TRUNC();
        if (L.bits < 1 || L.bits > 8)
            return dsq_internal_fail(DSQ_E_MALFORMED_HEADER, "container: bad packed bits");
        if (L.groups < 1 || L.cols % L.groups != 0)
            return dsq_internal_fail(DSQ_E_MALFORMED_HEADER, "container: bad group count");
        const uint64_t lut_n = uint64_t(L.rows) * L.groups * (1u << L.bits);
        if (lut_n * 4 > uint64_t(r.end - r.p)) return TRUNC();
        L.luts.resize(size_t(lut_n));
        for (auto& v : L.luts) v = r.f32();
        const uint64_t pn = r.u64();
        if (!r.ok) return TRUNC();
        const uint64_t stride = (uint64_t(L.cols) * L.bits + 7) / 8;
        if (pn != uint64_t(L.rows) * stride)
            return dsq_internal_fail(DSQ_E_TRUNCATED_PAYLOAD, "container: payload length mismatch");
        const uint8_t* pb = r.take(size_t(pn));
        if (!r.ok) return TRUNC();
        L.payload.assign(pb, pb + pn);
        const uint32_t nnz = r.u32();
        if (!r.ok || (uint64_t(L.rows) + 1) * 4 + uint64_t(nnz) * 6 > uint64_t(r.end - r.p))
            return TRUNC();
        L.row_ptr.resize(size_t(L.rows) + 1);
        for (auto& v : L.row_ptr) v = r.u32();
        L.col_idx.resize(nnz);
        for (auto& v : L.col_idx) v = r.u16();
        L.values.resize(nnz);
        for (auto& v : L.values) v = r.f32();
        L.hybrid_top_k = r.u32();
        L.avg_bits = r.f64();
        if (!r.ok) return TRUNC();
        // QuantizedLayer::validate (the reference validates in read_layer)
        const dsq_layer_view v = L.view();
        const int rc = dsq_internal_validate_view(&v);
        if (rc) return rc;
        layers.push_back(std::move(L));
    }
    if (r.p != r.end)
        return dsq_internal_fail(DSQ_E_TRUNCATED_PAYLOAD, "%s: trailing bytes in payload", path);
    if (meta) *meta = m;
    if (out) *out = std::move(layers);
    return DSQ_OK;
}

}  // namespace

struct dsq_cuda_container {
    dsq_container_meta meta{};
    std::vector<std::string> names;
    std::vector<dsq_cuda_layer*> layers;
};

extern "C" {

int dsq_container_check(const char* path, dsq_container_meta* meta) {
    if (!path) return dsq_internal_fail(DSQ_E_INVALID_ARGUMENT, "null path");
    return parse(path, meta, nullptr);
}

int dsq_cuda_container_open(const char* path, int device, dsq_cuda_container** out) {
    if (!path || !out) return dsq_internal_fail(DSQ_E_INVALID_ARGUMENT, "null argument");
    *out = nullptr;
    dsq_container_meta m{};
    std::vector<HostLayer> hl;
    int rc = parse(path, &m, &hl);
    if (rc) return rc;
    auto* c = new dsq_cuda_container;
    c->meta = m;
    for (const HostLayer& L : hl) {
        const dsq_layer_view v = L.view();
        dsq_cuda_layer* h = nullptr;
        rc = dsq_cuda_layer_create(&v, device, &h);
        if (rc) {
            dsq_cuda_container_close(c);
            return rc;
        }
        c->layers.push_back(h);
        c->names.push_back(L.name);
    }
    *out = c;
    return DSQ_OK;
}

int dsq_cuda_container_meta(const dsq_cuda_container* c, dsq_container_meta* meta) {
    if (!c || !meta) return dsq_internal_fail(DSQ_E_INVALID_ARGUMENT, "null argument");
    *meta = c->meta;
    return DSQ_OK;
}

dsq_cuda_layer* dsq_cuda_container_layer(const dsq_cuda_container* c, uint32_t index) {
    if (!c || index >= c->layers.size()) return nullptr;
    return c->layers[index];
}

const char* dsq_cuda_container_layer_name(const dsq_cuda_container* c, uint32_t index) {
    if (!c || index >= c->names.size()) return nullptr;
    return c->names[index].c_str();
}

int dsq_cuda_container_close(dsq_cuda_container* c) {
    if (!c) return DSQ_OK;
    for (dsq_cuda_layer* h : c->layers) dsq_cuda_layer_destroy(h);
    delete c;
    return DSQ_OK;
}

}  // extern "C"
