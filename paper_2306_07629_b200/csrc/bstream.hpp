// bstream.hpp -- host side of K11 (bstream.cu): the batched products' work
// plan, shared by the kernel's launcher and api.cpp.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

namespace sqz {

struct BStreamPlanHost {
    uint32_t phases = 0, nseg = 0, max_span = 0, cs = 0, grid = 0;
    std::vector<uint32_t> phase_span, seg_base;
    std::vector<uint32_t> wdesc;  // 4 words per warp: cell begin, end, first segment, phase
};
struct BStreamDevPlan {
    uint32_t phases, nseg, max_span, cs, grid, tiles16;
    uint4* wdesc;
    uint32_t* seg_base;
    uint32_t* phase_span;
    float* part;
    uint16_t* xT;
};
BStreamPlanHost bstream_plan(uint32_t tiles4, uint32_t ns, uint32_t bits, uint32_t nb,
                             uint32_t grid);
size_t bstream_smem_bytes(uint32_t bits, uint32_t nb, uint32_t max_span, uint32_t cs);
cudaError_t launch_bstream(uint32_t bits, uint32_t nb, const BStreamDevPlan& pl, const uint32_t* idx,
                           const uint32_t* lut, const uint32_t* row_ptr, const uint32_t* csr,
                           uint32_t rows, uint32_t cols, uint32_t ns, uint32_t tiles4,
                           const uint16_t* x, uint32_t x_stride, uint32_t B, void* y,
                           uint32_t y_stride, bool y_f16, int mode, cudaStream_t st);

}  // namespace sqz
