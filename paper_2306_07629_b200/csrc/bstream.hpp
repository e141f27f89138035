// bstream.hpp -- host side of K11 (bstream.cu): the batched products' work
// plan, shared by the kernel's launcher and api.cpp.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#ifdef __CUDACC__
#define SQZ_BS_HD __host__ __device__
#else
#define SQZ_BS_HD
#endif

namespace sqz {

// phases carried in the launch parameters: 32 covers every layer the tile
// layout holds (cols < 65536 = 256 spans, 8 spans per phase at B > 8)
constexpr uint32_t kBsMaxPhases = 32;

// the cell range [*wb, *we) of warp w of CTA `cta` (phase tables as in
// BStreamPlanHost): the kernel derives its range from the launch parameters
// with exactly the host plan's arithmetic
SQZ_BS_HD inline void bs_warp_range(const uint32_t* phase_span, const uint32_t* cta_pre,
                                    uint32_t phases, uint32_t tiles16, uint32_t cta, uint32_t w,
                                    uint32_t nw,
                                    uint32_t* phase, uint32_t* a, uint32_t* gp, uint32_t* wb,
                                    uint32_t* we) {
    uint32_t k = 0;
    while (k + 1 < phases && cta >= cta_pre[k + 1]) ++k;
    const uint32_t S = phase_span[k + 1] - phase_span[k];
    const uint64_t C = uint64_t(tiles16) * S;
    const uint32_t g = cta_pre[k + 1] - cta_pre[k], ai = cta - cta_pre[k];
    const uint64_t cb = C * ai / g, ce = C * (ai + 1) / g;
    *phase = k;
    *a = ai;
    *gp = g;
    *wb = uint32_t(cb + (ce - cb) * w / nw);
    *we = uint32_t(cb + (ce - cb) * (w + 1) / nw);
}

struct BStreamPlanHost {
    uint32_t phases = 0, nseg = 0, max_span = 0, cs = 0, grid = 0, warps = 8;
    std::vector<uint32_t> phase_span, seg_base;
    std::vector<uint32_t> cta_pre;  // [phases + 1]: CTAs of phase k are cta_pre[k] .. cta_pre[k+1]
    std::vector<uint32_t> wdesc;  // 4 words per warp: cell begin, end, first segment, packed phase
};
struct BStreamDevPlan {
    uint32_t phases, nseg, max_span, cs, grid, tiles16, warps;
    uint32_t phase_span_h[kBsMaxPhases + 1], cta_pre_h[kBsMaxPhases + 1];  // -> launch params
    uint4* wdesc;
    uint32_t* seg_base;
    float* part;
    uint16_t* xT;
};
// warps: decode warps per CTA, 8 (3 ring slots of 4 / 3 spans) or 16 (2 slots of 2 spans)
BStreamPlanHost bstream_plan(uint32_t tiles4, uint32_t ns, uint32_t bits, uint32_t nb,
                             uint32_t grid, uint32_t warps = 8);
size_t bstream_smem_bytes(uint32_t bits, uint32_t nb, uint32_t max_span, uint32_t cs,
                          uint32_t warps = 8);
cudaError_t launch_bstream(uint32_t bits, uint32_t nb, const BStreamDevPlan& pl, const uint32_t* idx,
                           const uint32_t* lut, const uint32_t* row_ptr, const uint32_t* csr,
                           uint32_t rows, uint32_t cols, uint32_t ns, uint32_t tiles4,
                           const uint16_t* x, uint32_t x_stride, uint32_t B, void* y,
                           uint32_t y_stride, bool y_f16, int mode, cudaStream_t st);

}  // namespace sqz
