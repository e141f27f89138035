/*
 * dsq_oracle.c -- CPU restatement of the reference hot path (TEST INFRASTRUCTURE,
 * the parity checker; never linked into the product).  See dsq_oracle.h.
 *
 * Reference: /root/reference/proj (C++20, CPU-only).  Every routine below
 * follows the cited reference routine step for step, including the term
 * order of every double-precision accumulation, so results are bit-identical
 * to the compiled reference (pinned in tests/test_oracle.py against oracle/_ref).
 */
#include "dsq_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

size_t orc_row_stride(uint32_t cols, uint32_t bits) {
    /* packfmt.hpp:26  (cols*bits + 7) / 8 */
    return ((size_t)cols * bits + 7) / 8;
}

int orc_pack(const uint16_t* assign, uint32_t bits, uint32_t rows, uint32_t cols,
             uint8_t* payload) {
    /* packfmt.cpp:18-55 */
    if (bits < 1 || bits > 8) return ORC_E_INVALID_ARGUMENT;
    const uint32_t k = 1u << bits;
    const size_t stride = orc_row_stride(cols, bits);
    memset(payload, 0, (size_t)rows * stride);
    for (uint32_t r = 0; r < rows; ++r) {
        uint8_t* out = payload + (size_t)r * stride;
        size_t bitpos = 0;
        for (uint32_t c = 0; c < cols; ++c) {
            uint16_t idx = assign[(size_t)r * cols + c];
            if (idx == 0xFFFFu) idx = 0; /* kMaskedIndex -> 0 (packfmt.cpp:47) */
            if (idx >= k) return ORC_E_INVALID_ARGUMENT;
            for (uint32_t b = 0; b < bits; ++b, ++bitpos) {
                if ((idx >> b) & 1u) out[bitpos >> 3] |= (uint8_t)(1u << (bitpos & 7));
            }
        }
    }
    return ORC_OK;
}

int orc_unpack(const uint8_t* payload, uint32_t bits, uint32_t rows, uint32_t cols,
               int strict, uint16_t* assign) {
    /* packfmt.cpp:57-80 (validate() preconditions at packfmt.cpp:7-16) */
    if (bits < 1 || bits > 8) return ORC_E_INVALID_ARGUMENT;
    if (rows < 1 || cols < 1) return ORC_E_EMPTY_DIMENSION;
    const size_t stride = orc_row_stride(cols, bits);
    for (uint32_t r = 0; r < rows; ++r) {
        const uint8_t* in = payload + (size_t)r * stride;
        size_t bitpos = 0;
        for (uint32_t c = 0; c < cols; ++c) {
            uint16_t idx = 0;
            for (uint32_t b = 0; b < bits; ++b, ++bitpos) {
                idx |= (uint16_t)(((in[bitpos >> 3] >> (bitpos & 7)) & 1u) << b);
            }
            assign[(size_t)r * cols + c] = idx;
        }
        if (strict) {
            for (; bitpos < stride * 8; ++bitpos) {
                if ((in[bitpos >> 3] >> (bitpos & 7)) & 1u) return ORC_E_TRUNCATED_PAYLOAD;
            }
        }
    }
    return ORC_OK;
}

int orc_csr_validate(uint32_t rows, uint32_t cols, const uint32_t* row_ptr,
                     const uint16_t* col_idx, const float* values, size_t n_col_idx) {
    /* dns.cpp:10-29, same check order */
    if (cols >= 65536u) return ORC_E_DIMENSION_OVERFLOW;
    if (row_ptr[0] != 0) return ORC_E_INTERNAL;
    for (uint32_t r = 0; r < rows; ++r) {
        if (row_ptr[r] > row_ptr[r + 1]) return ORC_E_INTERNAL;
        for (uint32_t p = row_ptr[r]; p < row_ptr[r + 1]; ++p) {
            if (p >= n_col_idx) return ORC_E_SHAPE_MISMATCH;
            if (col_idx[p] >= cols) return ORC_E_INTERNAL;
            if (p > row_ptr[r] && !(col_idx[p - 1] < col_idx[p])) return ORC_E_INTERNAL;
        }
    }
    if (row_ptr[rows] != n_col_idx) return ORC_E_SHAPE_MISMATCH;
    for (size_t i = 0; i < n_col_idx; ++i) {
        if (!isfinite(values[i])) return ORC_E_NON_FINITE_VALUE;
    }
    return ORC_OK;
}

/* kernels.cpp:18-33 lut_row_dot: bit-serial index assembly, double FMA-free
 * multiply-add (acc += double(lut) * double(x)), ascending c */
static double lut_row_dot(uint32_t bits, uint32_t cols, uint32_t groups_per_row,
                          const float* luts, const uint8_t* payload, uint32_t r,
                          const float* x) {
    const size_t stride = orc_row_stride(cols, bits);
    const uint8_t* in = payload + (size_t)r * stride;
    const uint32_t gcols = cols / groups_per_row;
    const uint32_t k = 1u << bits;
    const float* lut = luts + (size_t)r * groups_per_row * k;
    double acc = 0.0;
    size_t bitpos = 0;
    for (uint32_t c = 0; c < cols; ++c) {
        uint32_t idx = 0;
        for (uint32_t b = 0; b < bits; ++b, ++bitpos) {
            idx |= (uint32_t)(((in[bitpos >> 3] >> (bitpos & 7)) & 1u) << b);
        }
        const double prod = (double)lut[(c / gcols) * k + idx] * (double)x[c];
        acc = acc + prod;
    }
    return acc;
}

/* kernels.cpp:35-41 */
static double csr_row_dot(const uint32_t* row_ptr, const uint16_t* col_idx,
                          const float* values, uint32_t r, const float* x) {
    double acc = 0.0;
    for (uint32_t p = row_ptr[r]; p < row_ptr[r + 1]; ++p) {
        const double prod = (double)values[p] * (double)x[col_idx[p]];
        acc = acc + prod;
    }
    return acc;
}

/* kernels.cpp:43-47 */
static double dense_row_dot(const float* row, uint32_t cols, const float* x) {
    double acc = 0.0;
    for (uint32_t c = 0; c < cols; ++c) {
        const double prod = (double)row[c] * (double)x[c];
        acc = acc + prod;
    }
    return acc;
}

void orc_lut_matvec(uint32_t bits, uint32_t rows, uint32_t cols, uint32_t groups_per_row,
                    const float* luts, const uint8_t* payload, const float* x,
                    double* out, int nthreads) {
    /* kernels.cpp:51-67: OpenMP static over rows, one owner per output */
    (void)nthreads;
#ifdef _OPENMP
#pragma omp parallel for schedule(static) num_threads(nthreads > 0 ? nthreads : 1)
#endif
    for (int64_t r = 0; r < (int64_t)rows; ++r) {
        out[r] = lut_row_dot(bits, cols, groups_per_row, luts, payload, (uint32_t)r, x);
    }
}

void orc_csr_matvec(uint32_t rows, const uint32_t* row_ptr, const uint16_t* col_idx,
                    const float* values, const float* x, double* out, int nthreads) {
    /* kernels.cpp:69-85 */
    (void)nthreads;
#ifdef _OPENMP
#pragma omp parallel for schedule(static) num_threads(nthreads > 0 ? nthreads : 1)
#endif
    for (int64_t r = 0; r < (int64_t)rows; ++r) {
        out[r] = csr_row_dot(row_ptr, col_idx, values, (uint32_t)r, x);
    }
}

void orc_dense_matvec(const float* m, uint32_t rows, uint32_t cols, const float* x,
                      double* out, int nthreads) {
    /* kernels.cpp:87-106 */
    (void)nthreads;
#ifdef _OPENMP
#pragma omp parallel for schedule(static) num_threads(nthreads > 0 ? nthreads : 1)
#endif
    for (int64_t r = 0; r < (int64_t)rows; ++r) {
        out[r] = dense_row_dot(m + (size_t)r * cols, cols, x);
    }
}

typedef struct { uint32_t row, nnz; } row_key;

static int cmp_row_key(const void* a, const void* b) {
    /* dns.cpp:155-160: more nnz first; ties -> lower row (stable by row id) */
    const row_key* x = (const row_key*)a;
    const row_key* y = (const row_key*)b;
    if (x->nnz != y->nnz) return x->nnz > y->nnz ? -1 : 1;
    return x->row < y->row ? -1 : (x->row > y->row ? 1 : 0);
}

static int cmp_u32(const void* a, const void* b) {
    const uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
    return x < y ? -1 : (x > y ? 1 : 0);
}

int orc_hybrid_split(uint32_t rows, uint32_t cols, const uint32_t* row_ptr,
                     const uint16_t* col_idx, const float* values, uint32_t top_k,
                     uint32_t* dense_row_ids, float* promoted, uint32_t* res_row_ptr,
                     uint16_t* res_col_idx, float* res_values) {
    /* dns.cpp:151-197 */
    if (top_k > rows) return ORC_E_INVALID_ARGUMENT;
    row_key* order = (row_key*)malloc(sizeof(row_key) * (rows ? rows : 1));
    if (!order) return ORC_E_INTERNAL;
    for (uint32_t r = 0; r < rows; ++r) {
        order[r].row = r;
        order[r].nnz = row_ptr[r + 1] - row_ptr[r];
    }
    qsort(order, rows, sizeof(row_key), cmp_row_key);
    for (uint32_t i = 0; i < top_k; ++i) dense_row_ids[i] = order[i].row;
    free(order);
    qsort(dense_row_ids, top_k, sizeof(uint32_t), cmp_u32);

    uint8_t* is_promoted = (uint8_t*)calloc(rows ? rows : 1, 1);
    if (!is_promoted) return ORC_E_INTERNAL;
    for (uint32_t i = 0; i < top_k; ++i) is_promoted[dense_row_ids[i]] = 1;

    memset(promoted, 0, sizeof(float) * (size_t)top_k * cols);
    for (uint32_t i = 0; i < top_k; ++i) {
        const uint32_t r = dense_row_ids[i];
        for (uint32_t p = row_ptr[r]; p < row_ptr[r + 1]; ++p) {
            promoted[(size_t)i * cols + col_idx[p]] = values[p];
        }
    }
    res_row_ptr[0] = 0;
    uint32_t q = 0;
    for (uint32_t r = 0; r < rows; ++r) {
        if (!is_promoted[r]) {
            for (uint32_t p = row_ptr[r]; p < row_ptr[r + 1]; ++p, ++q) {
                res_col_idx[q] = col_idx[p];
                res_values[q] = values[p];
            }
        }
        res_row_ptr[r + 1] = q;
    }
    free(is_promoted);
    return ORC_OK;
}

void orc_fused_dns_matvec(uint32_t bits, uint32_t rows, uint32_t cols,
                          uint32_t groups_per_row, const float* luts,
                          const uint8_t* payload, uint32_t n_promoted,
                          const uint32_t* dense_row_ids, const float* promoted,
                          const uint32_t* res_row_ptr, const uint16_t* res_col_idx,
                          const float* res_values, const float* x, double* out,
                          int nthreads) {
    /* kernels.cpp:108-141 */
    (void)nthreads;
    int32_t* slot = (int32_t*)malloc(sizeof(int32_t) * (rows ? rows : 1));
    for (uint32_t r = 0; r < rows; ++r) slot[r] = -1;
    for (uint32_t i = 0; i < n_promoted; ++i) slot[dense_row_ids[i]] = (int32_t)i;
#ifdef _OPENMP
#pragma omp parallel for schedule(static) num_threads(nthreads > 0 ? nthreads : 1)
#endif
    for (int64_t r = 0; r < (int64_t)rows; ++r) {
        double acc = lut_row_dot(bits, cols, groups_per_row, luts, payload, (uint32_t)r, x);
        const int32_t s = slot[r];
        if (s >= 0) {
            acc += dense_row_dot(promoted + (size_t)s * cols, cols, x);
        } else {
            acc += csr_row_dot(res_row_ptr, res_col_idx, res_values, (uint32_t)r, x);
        }
        out[r] = acc;
    }
    free(slot);
}

void orc_dequant_dense(uint32_t bits, uint32_t rows, uint32_t cols, uint32_t groups_per_row,
                       const float* luts, const uint8_t* payload, float* out) {
    /* kernels.cpp:149-159: unpack, then lut_at(r,c)[assign] */
    const uint32_t k = 1u << bits;
    const uint32_t gcols = cols / groups_per_row;
    uint16_t* assign = (uint16_t*)malloc(sizeof(uint16_t) * (size_t)rows * cols);
    orc_unpack(payload, bits, rows, cols, 0, assign);
    for (uint32_t r = 0; r < rows; ++r) {
        for (uint32_t c = 0; c < cols; ++c) {
            const size_t i = (size_t)r * cols + c;
            const float* lut = luts + ((size_t)r * groups_per_row + c / gcols) * k;
            out[i] = lut[assign[i]];
        }
    }
    free(assign);
}

uint64_t orc_layer_total_bits(uint32_t rows, uint32_t cols, uint32_t bits,
                              uint32_t group_size, uint64_t nnz) {
    /* packfmt.cpp:98-121 */
    const uint64_t weight_count = (uint64_t)rows * cols;
    if (bits == 16) return weight_count * 16;
    const uint64_t groups_per_row = group_size == 0 ? 1 : cols / group_size;
    const uint64_t row_stride = ((uint64_t)cols * bits + 7) / 8;
    uint64_t total = (uint64_t)rows * row_stride * 8;
    total += (uint64_t)rows * groups_per_row * (1u << bits) * 16;
    if (nnz > 0) {
        total += nnz * (16 + 16);
        total += ((uint64_t)rows + 1) * 32;
    }
    return total;
}

uint64_t orc_bytes_touched(uint32_t rows, uint32_t cols, uint32_t bits,
                           uint32_t group_size, uint64_t nnz) {
    /* kernels.cpp:205-212: stored weights + 16-bit x read + 16-bit y write */
    return orc_layer_total_bits(rows, cols, bits, group_size, nnz) / 8 +
           (uint64_t)cols * 2 + (uint64_t)rows * 2;
}
