// quantize.hpp -- parameters of K9 kmeans_groups (quantize.cu), the GPU
// channel-wise quantizer (reference dsq::quantize_channelwise, nuq.cpp:673-779).
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

namespace sqz {

struct QuantParams {
    const float* w;          // [rows * cols] weights (row-major)
    const float* sens;       // [rows * cols] sensitivities (k-means weights)
    const uint8_t* mask;     // [rows * cols] or null: positions already extracted
    uint32_t rows, cols, groups_per_row, bits;
    uint32_t max_iters;
    double tol;
    int method;              // 0 weighted k-means, 1 unweighted, 2 round-to-nearest
    float* centroids;        // [rows * groups_per_row * 2^bits]
    uint16_t* assign;        // [rows * cols] (0xFFFF at masked positions)
    double* group_obj;       // [groups] weighted SSE, sens-weighted
    double* group_mse;       // [groups] plain SSE
    uint8_t* group_failed;   // [groups] 1: empty group, 2: invalid weight
    uint8_t* scratch;        // per-CTA workspace
    size_t scratch_stride;
    size_t npow2;            // sort length (power of two >= group length)
    int smem_prefix;
    unsigned long long* prof;  // dev: [groups][6] cycles lloyd/refine/merge, rounds, iterations         // interval-cost prefix tables in dynamic shared memory
};

cudaError_t launch_kmeans(const QuantParams& p, uint32_t grid, cudaStream_t st);
size_t kmeans_scratch_stride(uint32_t gcols, size_t npow2);
size_t kmeans_smem_bytes(uint32_t gcols);  // dynamic smem with smem_prefix

}  // namespace sqz
