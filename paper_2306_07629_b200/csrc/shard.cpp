// shard.cpp -- tensor-parallel sharding of a quantized layer (host, C ABI).
//
// The product y = D.x + S.x of one layer shards two ways:
//   * column-parallel (q/k/v/gate/up): rank r owns output rows [r0, r1); the
//     rows' packed indices, LUTs and CSR rows move with them, no exchange;
//   * row-parallel (o/down): rank r owns input columns [c0, c1) (aligned
//     splits keep whole index groups); indices are re-packed for the column
//     slice in the reference's LSB-first layout (packfmt.cpp:40-53), LUTs are
//     replicated (channel-wise codebooks do not depend on the column), CSR
//     entries are filtered by column and rebased; the partial sums are
//     reduced over the ranks (fused into the stack kernel, stack.cu).
// Extracted positions keep packed index 0 and their delta (pipeline.cpp:
// 25-32) in whichever shard owns their column, so every shard's fused product
// is exact for its slice.  The decoder split (tp.py DECODER order v, q, o, k,
// up, gate, down; o and down row-parallel) makes a producer's row split equal
// its consumer's column split, so the only exchanges are the two reduces.
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/dsq_cuda.h"

extern "C" int dsq_internal_fail(int code, const char* fmt, ...);

struct dsq_shard {
    std::string name;
    uint32_t lo = 0, hi = 0;  // rows (column-parallel) or columns (row-parallel)
    dsq_layer_view view{};
    std::vector<float> luts32;
    std::vector<uint16_t> luts16;
    std::vector<uint8_t> payload;
    std::vector<uint32_t> row_ptr;
    std::vector<uint16_t> col_idx;
    std::vector<float> val32;
    std::vector<uint16_t> val16;
};

namespace {

size_t stride_of(uint32_t cols, uint32_t bits) { return (size_t(cols) * bits + 7) / 8; }

int check_view(const dsq_layer_view* v) {
    if (!v || !v->name) return dsq_internal_fail(DSQ_E_INVALID_ARGUMENT, "shard: null layer view");
    const dsq_packed_view& p = v->packed;
    if (p.bits < 1 || p.bits > 8)
        return dsq_internal_fail(DSQ_E_INVALID_ARGUMENT, "shard: bits must be in 1..8");
    if (p.rows != v->rows || p.cols != v->cols || v->sparse.rows != v->rows ||
        v->sparse.cols != v->cols)
        return dsq_internal_fail(DSQ_E_SHAPE_MISMATCH, "shard: %s dims mismatch", v->name);
    if (!p.payload || p.payload_len != size_t(p.rows) * stride_of(p.cols, p.bits))
        return dsq_internal_fail(DSQ_E_SHAPE_MISMATCH, "shard: payload size mismatch");
    if (p.groups_per_row < 1 || p.cols % p.groups_per_row)
        return dsq_internal_fail(DSQ_E_SHAPE_MISMATCH, "shard: groups_per_row must divide cols");
    if (!p.luts_f32 == !p.luts_f16)
        return dsq_internal_fail(DSQ_E_SHAPE_MISMATCH, "shard: exactly one LUT array required");
    const dsq_csr_view& s = v->sparse;
    if (!s.row_ptr || s.row_ptr[0] != 0 || s.row_ptr[s.rows] != s.nnz)
        return dsq_internal_fail(DSQ_E_SHAPE_MISMATCH, "shard: bad CSR row_ptr");
    if (s.nnz && (!s.col_idx || !s.values_f32 == !s.values_f16))
        return dsq_internal_fail(DSQ_E_SHAPE_MISMATCH, "shard: exactly one CSR value array required");
    return DSQ_OK;
}

// the views of an owned shard point into its vectors
void publish(dsq_shard* S, const dsq_layer_view* in, uint32_t rows, uint32_t cols,
             uint32_t groups, uint32_t top_k) {
    dsq_layer_view& v = S->view;
    v.name = S->name.c_str();
    v.rows = rows;
    v.cols = cols;
    v.hybrid_top_k = top_k;
    v.packed.bits = in->packed.bits;
    v.packed.rows = rows;
    v.packed.cols = cols;
    v.packed.groups_per_row = groups;
    v.packed.luts_f32 = in->packed.luts_f32 ? S->luts32.data() : nullptr;
    v.packed.luts_f16 = in->packed.luts_f16 ? S->luts16.data() : nullptr;
    v.packed.payload = S->payload.data();
    v.packed.payload_len = S->payload.size();
    v.sparse.rows = rows;
    v.sparse.cols = cols;
    v.sparse.nnz = S->row_ptr.back();
    v.sparse.row_ptr = S->row_ptr.data();
    v.sparse.col_idx = S->col_idx.empty() ? nullptr : S->col_idx.data();
    const bool f32 = in->sparse.values_f32 != nullptr || in->sparse.values_f16 == nullptr;
    v.sparse.values_f32 = f32 && !S->val32.empty() ? S->val32.data() : nullptr;
    v.sparse.values_f16 = !f32 && !S->val16.empty() ? S->val16.data() : nullptr;
}

}  // namespace

extern "C" {

int dsq_split_range(uint32_t n, uint32_t world, uint32_t rank, uint32_t align, uint32_t* lo,
                    uint32_t* hi) {
    if (!lo || !hi || world == 0 || rank >= world || align == 0)
        return dsq_internal_fail(DSQ_E_INVALID_ARGUMENT, "split_range: bad arguments");
    const uint64_t units = (uint64_t(n) + align - 1) / align;
    *lo = uint32_t(units * rank / world * align);
    *hi = uint32_t(std::min<uint64_t>(n, units * (rank + 1) / world * align));
    if (*lo > *hi) *lo = *hi;
    return DSQ_OK;
}

int dsq_shard_rows(const dsq_layer_view* in, uint32_t rank, uint32_t world, uint32_t align,
                   dsq_shard** out) {
    if (!out) return dsq_internal_fail(DSQ_E_INVALID_ARGUMENT, "shard: null output");
    *out = nullptr;
    int rc = check_view(in);
    if (rc) return rc;
    uint32_t r0, r1;
    if ((rc = dsq_split_range(in->rows, world, rank, align ? align : 1, &r0, &r1))) return rc;
    if (r1 == r0) return dsq_internal_fail(DSQ_E_EMPTY_DIMENSION, "shard_rows: empty shard");
    auto* S = new dsq_shard;
    S->name = std::string(in->name) + ".r" + std::to_string(rank);
    S->lo = r0;
    S->hi = r1;
    const dsq_packed_view& p = in->packed;
    const size_t k = size_t(1u << p.bits) * p.groups_per_row, stride = stride_of(p.cols, p.bits);
    if (p.luts_f32) S->luts32.assign(p.luts_f32 + r0 * k, p.luts_f32 + r1 * k);
    else S->luts16.assign(p.luts_f16 + r0 * k, p.luts_f16 + r1 * k);
    S->payload.assign(p.payload + r0 * stride, p.payload + r1 * stride);
    const dsq_csr_view& s = in->sparse;
    const uint32_t a = s.row_ptr[r0], b = s.row_ptr[r1];
    S->row_ptr.resize(size_t(r1 - r0) + 1);
    for (uint32_t r = r0; r <= r1; ++r) S->row_ptr[r - r0] = s.row_ptr[r] - a;
    if (b > a) {
        S->col_idx.assign(s.col_idx + a, s.col_idx + b);
        if (s.values_f32) S->val32.assign(s.values_f32 + a, s.values_f32 + b);
        else S->val16.assign(s.values_f16 + a, s.values_f16 + b);
    }
    publish(S, in, r1 - r0, in->cols, p.groups_per_row, std::min(in->hybrid_top_k, r1 - r0));
    *out = S;
    return DSQ_OK;
}

int dsq_shard_cols(const dsq_layer_view* in, uint32_t rank, uint32_t world, uint32_t align,
                   dsq_shard** out) {
    if (!out) return dsq_internal_fail(DSQ_E_INVALID_ARGUMENT, "shard: null output");
    *out = nullptr;
    int rc = check_view(in);
    if (rc) return rc;
    const dsq_packed_view& p = in->packed;
    if (p.groups_per_row != 1)
        return dsq_internal_fail(DSQ_E_UNSUPPORTED,
                                 "shard_cols: row-parallel sharding needs channel-wise LUTs");
    uint32_t c0, c1;
    if ((rc = dsq_split_range(in->cols, world, rank, align ? align : 1, &c0, &c1))) return rc;
    if (c1 == c0) return dsq_internal_fail(DSQ_E_EMPTY_DIMENSION, "shard_cols: empty shard");
    auto* S = new dsq_shard;
    S->name = std::string(in->name) + ".c" + std::to_string(rank);
    S->lo = c0;
    S->hi = c1;
    const size_t k = size_t(1u) << p.bits;
    if (p.luts_f32) S->luts32.assign(p.luts_f32, p.luts_f32 + size_t(p.rows) * k);
    else S->luts16.assign(p.luts_f16, p.luts_f16 + size_t(p.rows) * k);
    // re-pack each row's index slice [c0, c1) in the LSB-first bitstream
    // layout (packfmt.cpp:40-53), pad bits zero
    const uint32_t bits = p.bits, nc = c1 - c0;
    const size_t in_stride = stride_of(p.cols, bits), out_stride = stride_of(nc, bits);
    S->payload.assign(size_t(p.rows) * out_stride, 0);
    const uint32_t mask = (1u << bits) - 1u;
    for (uint32_t r = 0; r < p.rows; ++r) {
        const uint8_t* src = p.payload + size_t(r) * in_stride;
        uint8_t* dst = S->payload.data() + size_t(r) * out_stride;
        for (uint32_t c = 0; c < nc; ++c) {
            const size_t sb = size_t(c0 + c) * bits, db = size_t(c) * bits;
            uint32_t w = 0;  // up to 8 bits straddle at most two bytes
            w = src[sb >> 3] | (((sb >> 3) + 1 < in_stride ? uint32_t(src[(sb >> 3) + 1]) : 0u) << 8);
            const uint32_t idx = (w >> (sb & 7)) & mask;
            const uint32_t sh = uint32_t(db & 7);
            dst[db >> 3] |= uint8_t(idx << sh);
            if (sh + bits > 8) dst[(db >> 3) + 1] |= uint8_t(idx >> (8 - sh));
        }
    }
    const dsq_csr_view& s = in->sparse;
    S->row_ptr.assign(size_t(p.rows) + 1, 0);
    for (uint32_t r = 0; r < s.rows; ++r) {
        for (uint32_t q = s.row_ptr[r]; q < s.row_ptr[r + 1]; ++q) {
            const uint32_t c = s.col_idx[q];
            if (c < c0 || c >= c1) continue;
            S->col_idx.push_back(uint16_t(c - c0));
            if (s.values_f32) S->val32.push_back(s.values_f32[q]);
            else S->val16.push_back(s.values_f16[q]);
        }
        S->row_ptr[r + 1] = uint32_t(S->col_idx.size());
    }
    publish(S, in, in->rows, nc, 1, in->hybrid_top_k);
    *out = S;
    return DSQ_OK;
}

int dsq_shard_decoder(const dsq_layer_view* layers, uint32_t rank, uint32_t world,
                      uint32_t align, dsq_shard** out) {
    if (!layers || !out) return dsq_internal_fail(DSQ_E_INVALID_ARGUMENT, "shard_decoder: null");
    // DECODER order v, q, o, k, up, gate, down: o (2) and down (6) row-parallel
    for (int i = 0; i < 7; ++i) out[i] = nullptr;
    for (int i = 0; i < 7; ++i) {
        const int rc = (i == 2 || i == 6) ? dsq_shard_cols(&layers[i], rank, world, align, &out[i])
                                          : dsq_shard_rows(&layers[i], rank, world, align, &out[i]);
        if (rc) {
            for (int j = 0; j < i; ++j) {
                delete out[j];
                out[j] = nullptr;
            }
            return rc;
        }
    }
    return DSQ_OK;
}

int dsq_shard_get(const dsq_shard* s, dsq_layer_view* view, uint32_t* lo, uint32_t* hi) {
    if (!s || !view) return dsq_internal_fail(DSQ_E_INVALID_ARGUMENT, "shard_get: null");
    *view = s->view;
    if (lo) *lo = s->lo;
    if (hi) *hi = s->hi;
    return DSQ_OK;
}

int dsq_shard_destroy(dsq_shard* s) {
    delete s;
    return DSQ_OK;
}

}  // extern "C"
