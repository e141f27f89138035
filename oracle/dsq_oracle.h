/*
 * dsq_oracle.h -- CPU restatement of the reference hot path (TEST INFRASTRUCTURE).
 *
 * This is the parity CHECKER for the B200 path, not part of the product.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load it.  The product (libdsq_cuda.so) never
 * links or calls it.
 *
 * Each function restates the reference algorithm in plain C and cites the
 * reference file:line it follows (paths relative to /root/reference/proj).
 * Parity of this restatement is PINNED against (a) the SPEC.md known-answer
 * vectors and (b) the reference
 * itself compiled from its own sources into oracle/_ref (see oracle/Makefile
 * and tests/test_oracle.py), bit-exact on every output.
 */
#ifndef DSQ_ORACLE_H
#define DSQ_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* error codes: same numbering as dsq::errc (include/dsq/common.hpp:13-29) */
enum {
    ORC_OK = 0,
    ORC_E_MISSING_FILE = 1,
    ORC_E_MALFORMED_HEADER,
    ORC_E_NON_FINITE_VALUE,
    ORC_E_EMPTY_DIMENSION,
    ORC_E_DIMENSION_OVERFLOW,
    ORC_E_TRUNCATED_PAYLOAD,
    ORC_E_CHECKSUM_MISMATCH,
    ORC_E_UNSUPPORTED_VERSION,
    ORC_E_SHAPE_MISMATCH,
    ORC_E_EMPTY_INPUT,
    ORC_E_INVALID_ARGUMENT,
    ORC_E_FRACTION_OVERFLOW,
    ORC_E_EMPTY_CHANNEL,
    ORC_E_IO_FAILURE,
    ORC_E_INTERNAL
};

/* PackedDense::row_stride (packfmt.hpp:26) */
size_t orc_row_stride(uint32_t cols, uint32_t bits);

/* pack() index stream, LSB-first, masked 0xFFFF -> 0 (packfmt.cpp:18-55).
 * payload must hold rows*row_stride bytes; it is zeroed here. */
int orc_pack(const uint16_t* assign, uint32_t bits, uint32_t rows, uint32_t cols,
             uint8_t* payload);

/* unpack() exact inverse, strict rejects nonzero pad bits (packfmt.cpp:57-80) */
int orc_unpack(const uint8_t* payload, uint32_t bits, uint32_t rows, uint32_t cols,
               int strict, uint16_t* assign);

/* CsrMatrix::validate (dns.cpp:10-29) */
int orc_csr_validate(uint32_t rows, uint32_t cols, const uint32_t* row_ptr,
                     const uint16_t* col_idx, const float* values, size_t n_col_idx);

/* lut_matvec (kernels.cpp:18-33 lut_row_dot, :51-67); double accumulation,
 * ascending c; nthreads<=1 -> serial (results are identical either way) */
void orc_lut_matvec(uint32_t bits, uint32_t rows, uint32_t cols, uint32_t groups_per_row,
                    const float* luts, const uint8_t* payload, const float* x,
                    double* out, int nthreads);

/* csr_matvec (kernels.cpp:35-41 csr_row_dot, :69-85) */
void orc_csr_matvec(uint32_t rows, const uint32_t* row_ptr, const uint16_t* col_idx,
                    const float* values, const float* x, double* out, int nthreads);

/* dense_matvec (kernels.cpp:43-47 dense_row_dot, :87-106) */
void orc_dense_matvec(const float* m, uint32_t rows, uint32_t cols, const float* x,
                      double* out, int nthreads);

/* hybrid_split (dns.cpp:151-197): top_k rows by nnz (ties -> lower row) are
 * promoted to dense rows; the residual CSR excludes them.
 * Outputs: dense_row_ids[top_k] (ascending), promoted[top_k*cols],
 * res_row_ptr[rows+1], res_col_idx/res_values (capacity nnz); returns code. */
int orc_hybrid_split(uint32_t rows, uint32_t cols, const uint32_t* row_ptr,
                     const uint16_t* col_idx, const float* values, uint32_t top_k,
                     uint32_t* dense_row_ids, float* promoted, uint32_t* res_row_ptr,
                     uint16_t* res_col_idx, float* res_values);

/* fused_dns_matvec (kernels.cpp:108-141): per row, LUT dot + (promoted dense
 * row dot | residual CSR row dot). */
void orc_fused_dns_matvec(uint32_t bits, uint32_t rows, uint32_t cols,
                          uint32_t groups_per_row, const float* luts,
                          const uint8_t* payload, uint32_t n_promoted,
                          const uint32_t* dense_row_ids, const float* promoted,
                          const uint32_t* res_row_ptr, const uint16_t* res_col_idx,
                          const float* res_values, const float* x, double* out,
                          int nthreads);

/* ref::dequant_dense (kernels.cpp:149-159) */
void orc_dequant_dense(uint32_t bits, uint32_t rows, uint32_t cols, uint32_t groups_per_row,
                       const float* luts, const uint8_t* payload, float* out);

/* layer_bit_stats().total_bits (packfmt.cpp:98-121); group_size 0 = channel-wise */
uint64_t orc_layer_total_bits(uint32_t rows, uint32_t cols, uint32_t bits,
                              uint32_t group_size, uint64_t nnz);

/* bytes_touched_estimate (kernels.cpp:205-212) */
uint64_t orc_bytes_touched(uint32_t rows, uint32_t cols, uint32_t bits,
                           uint32_t group_size, uint64_t nnz);

#ifdef __cplusplus
}
#endif
#endif
