// Host-only check of K11's work plan (csrc/bstream.cu, bstream_plan): walks
// every warp's cell range the way bstream_gemv does (chunks of <= cs spans,
// a segment flushed whenever the range leaves a 16-row tile) and checks that
//   * every (16-row tile, span) cell is decoded exactly once,
//   * every segment id is written exactly once, inside its tile's
//     seg_base[p*T + q] .. seg_base[p*T + q + 1] range (what bstream_finish sums),
//   * each phase's x fits the 64 KB staging budget, and the phase's CTAs carry
//     shares a = 0..gp-1 of its transposed x (gp = the phase's CTA count).
// No GPU needed.  Prints PASS.
#include <cstdio>
#include <vector>

#include "bstream.hpp"

using namespace sqz;

static int check(uint32_t tiles4, uint32_t ns, uint32_t bits, uint32_t nb, uint32_t grid,
                 uint32_t warps) {
    const BStreamPlanHost pl = bstream_plan(tiles4, ns, bits, nb, grid, warps);
    const uint32_t W = pl.warps;
    const uint32_t T = (tiles4 + 3) / 4;
    std::vector<int> cover(size_t(T) * ns, 0), seguse(pl.nseg, 0), xt(pl.phases, 0);
    std::vector<uint32_t> xt_gp(pl.phases, 0);
    if (pl.max_span * 256u * 8u * nb * 2u > 65536u) {
        std::printf("FAIL x budget: max_span %u nb %u\n", pl.max_span, nb);
        return 1;
    }
    for (uint32_t c = 0; c < pl.grid; ++c) {
        for (uint32_t w = 0; w < W; ++w) {
            const uint32_t* d = &pl.wdesc[(size_t(c) * W + w) * 4];
            const uint32_t ph = d[3] & 0xffu, a = (d[3] >> 8) & 0xfffu, gp = d[3] >> 20;
            if (ph >= pl.phases) return std::printf("FAIL phase %u\n", ph), 1;
            if (w == 0) {
                // CTAs of a phase are consecutive: share a is the running count
                if (a != uint32_t(xt[ph]) || (xt_gp[ph] && xt_gp[ph] != gp))
                    return std::printf("FAIL xT share %u/%u in phase %u\n", a, gp, ph), 1;
                xt_gp[ph] = gp;
                ++xt[ph];
            }
            const uint32_t sa = pl.phase_span[ph], S = pl.phase_span[ph + 1] - sa;
            uint32_t seg = d[2];
            for (uint32_t cc = d[0]; cc < d[1];) {
                const uint32_t q = cc / S, sl = cc - q * S;
                const uint32_t n = std::min(std::min(pl.cs, S - sl), d[1] - cc);
                for (uint32_t u = 0; u < n; ++u) ++cover[size_t(q) * ns + sa + sl + u];
                cc += n;
                if (cc == d[1] || cc - q * S == S) {
                    if (seg >= pl.nseg || seg < pl.seg_base[size_t(ph) * T + q] ||
                        seg >= pl.seg_base[size_t(ph) * T + q + 1])
                        return std::printf("FAIL segment %u of tile %u phase %u\n", seg, q, ph), 1;
                    ++seguse[seg];
                    if (cc < d[1]) seg = pl.seg_base[size_t(ph) * T + q + 1];
                }
            }
        }
    }
    for (int v : cover)
        if (v != 1) return std::printf("FAIL cell covered %d times\n", v), 1;
    for (int v : seguse)
        if (v != 1) return std::printf("FAIL segment written %d times\n", v), 1;
    for (uint32_t k = 0; k < pl.phases; ++k)
        if (uint32_t(xt[k]) != xt_gp[k]) return std::printf("FAIL %d xT shares of %u\n", xt[k], xt_gp[k]), 1;
    return 0;
}

int main() {
    // (tiles4, spans): 7B / 13B / 65B shapes, ragged and tiny layers
    const uint32_t shapes[][2] = {{1024, 16}, {2752, 16}, {1024, 43}, {1280, 20}, {3456, 20},
                                  {1280, 54}, {2048, 32}, {5504, 32}, {2048, 86}, {1, 1},
                                  {9, 2},     {3, 40},    {17, 3},    {7, 300}};
    int bad = 0, n = 0;
    for (const auto& s : shapes)
        for (uint32_t nb = 1; nb <= 2; ++nb)
            for (uint32_t bits = 3; bits <= 4; ++bits)
                for (uint32_t grid : {148u, 132u, 1u})
                    for (uint32_t warps : {8u, 16u}) bad |= check(s[0], s[1], bits, nb, grid, warps), ++n;
    std::printf("%s (%d plans)\n", bad ? "FAIL" : "PASS", n);
    return bad;
}
