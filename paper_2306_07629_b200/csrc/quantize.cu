// K9 kmeans_groups: GPU channel-wise non-uniform quantization (SURVEY.md §8f
// rank 4) -- the step upstream of the hot path.  Reference:
// dsq::quantize_channelwise (src/nuq.cpp:673-779) with weighted_kmeans_1d
// (:411-502) and its helpers (weighted_quantile_init :65-89,
// make_sorted_problem :120-143, assign_and_repair :154-183, lloyd_converge
// :187-225, boundary_refine :246-327, merge_split_escape :331-408) and
// rtn_uniform (:609-640).
//
// Bit-exact by construction: every floating-point reduction whose order the
// reference fixes (prefix sums, cluster sums, objectives) runs in the same
// order (one thread, or one thread per cluster scanning its members in
// position order); order-free work runs in parallel -- nearest-centroid
// assignment, interval costs, and the reference's sequential "accept a cut
// if it beats the running best by a margin" scans, which warp 0 reproduces
// exactly with ballots (the first lane that beats the record wins, the
// record moves, the scan resumes after it).  Compiled with -fmad=false so no
// a*b+c is contracted (the reference's x86-64 build has no FMA).
//
// One CTA (256 threads) per group, persistent over groups; per-CTA scratch
// in global memory (L1/L2 resident) sized for the group length.
#include <cuda_runtime.h>

#include <cstdint>

#include "quantize.hpp"

namespace sqz {
namespace {

constexpr int kThreads = 256;
constexpr uint16_t kMasked = 0xFFFF;
constexpr uint32_t kMaxK = 256;

struct Scratch {
    unsigned long long* keys;  // [npow2] sort keys (value order, original index)
    double *v, *w;              // [n] sorted values / weights
    double *pw, *pwv, *pwv2;    // [n+1] prefix sums
    uint16_t* assign;           // [n] cluster of each sorted position
    float *vals, *wts, *wk;     // [n] kept values, sens weights, k-means weights (original order)
    uint32_t* kcol;             // [n] kept column of each value
};

__device__ __forceinline__ double icost(const Scratch& S, uint32_t i, uint32_t j) {  // [i, j]
    const double W = S.pw[j + 1] - S.pw[i];
    if (W <= 0.0) return 0.0;
    const double A = S.pwv[j + 1] - S.pwv[i];
    const double Q = S.pwv2[j + 1] - S.pwv2[i];
    const double c = Q - A * A / W;
    return c > 0.0 ? c : 0.0;  // std::max(0.0, c)
}

__device__ double imean(const Scratch& S, uint32_t i, uint32_t j) {
    const double W = S.pw[j + 1] - S.pw[i];
    if (W > 0.0) return (S.pwv[j + 1] - S.pwv[i]) / W;
    double acc = 0.0;
    for (uint32_t t = i; t <= j; ++t) acc += S.v[t];
    return acc / double(j - i + 1);
}

// float -> key whose unsigned order is the float order, with -0 == +0
__device__ __forceinline__ uint32_t fkey(float f) {
    uint32_t u = __float_as_uint(f);
    if ((u & 0x7fffffffu) == 0) u = 0;
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

// nearest centroid in a sorted table, ties to the lower index (nuq.cpp:43-52)
__device__ uint32_t nearest(const float* c, uint32_t k, float v) {
    uint32_t lo = 0, hi = k;  // lower_bound: first c[i] >= v
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (c[mid] < v) lo = mid + 1;
        else hi = mid;
    }
    if (lo == 0) return 0;
    if (lo == k) return k - 1;
    const double dl = double(v) - double(c[lo - 1]);
    const double dh = double(c[lo]) - double(v);
    return dl <= dh ? lo - 1 : lo;
}

__device__ void sort_small(float* a, uint32_t k) {  // thread 0: ascending
    for (uint32_t i = 1; i < k; ++i) {
        const float x = a[i];
        uint32_t j = i;
        while (j > 0 && x < a[j - 1]) {
            a[j] = a[j - 1];
            --j;
        }
        a[j] = x;
    }
}

struct Shared {
    float cent[kMaxK];
    float next[kMaxK];
    uint32_t counts[kMaxK];
    double num[kMaxK], den[kMaxK], plain[kMaxK];
    uint32_t ivf[kMaxK], ivs[kMaxK];
    double red_d[kThreads / 32];
    uint32_t red_i[kThreads / 32];
    uint32_t n, flag, changed, moved;
    double total;
    float tail;
};

// warp 0: the reference's sequential record scan over m in [m0, m1):
// accept m when cost(m) < R - eps, R := cost(m).  Exact (same comparisons,
// same order of acceptances).
template <class F>
__device__ void chain_scan(uint32_t m0, uint32_t m1, double& R, uint32_t& best, double eps, F cost) {
    const uint32_t lane = threadIdx.x & 31;
    for (uint32_t base = m0; base < m1; base += 32) {
        const uint32_t m = base + lane;
        const double c = m < m1 ? cost(m) : 0.0;
        uint32_t start = 0;
        while (true) {
            const bool ok = m < m1 && lane >= start && c < R - eps;
            const uint32_t msk = __ballot_sync(0xffffffffu, ok);
            if (!msk) break;
            const uint32_t f = __ffs(msk) - 1;
            R = __shfl_sync(0xffffffffu, c, f);
            best = base + f;
            start = f + 1;
        }
    }
}

// one assignment pass + empty-cluster repair (nuq.cpp:154-183)
__device__ void assign_and_repair(const Scratch& S, Shared& sh, uint32_t k) {
    const uint32_t n = sh.n, tid = threadIdx.x;
    for (uint32_t j = tid; j < k; j += kThreads) sh.counts[j] = 0;
    __syncthreads();
    for (uint32_t i = tid; i < n; i += kThreads) {
        const uint32_t a = nearest(sh.cent, k, float(S.v[i]));
        S.assign[i] = uint16_t(a);
        atomicAdd(&sh.counts[a], 1u);
    }
    __syncthreads();
    for (uint32_t j = 0; j < k; ++j) {
        if (sh.counts[j] != 0) continue;  // uniform across the block
        // best = first maximum of w*d^2 over stealable positions (strict >, init -1)
        double best = -1.0;
        uint32_t bi = n;
        for (uint32_t i = tid; i < n; i += kThreads) {
            const uint32_t a = S.assign[i];
            if (sh.counts[a] < 2) continue;
            const double d = S.v[i] - double(sh.cent[a]);
            const double sc = S.w[i] * d * d;
            if (sc > best) {
                best = sc;
                bi = i;
            }
        }
        for (int o = 16; o; o >>= 1) {
            const double ob = __shfl_down_sync(0xffffffffu, best, o);
            const uint32_t oi = __shfl_down_sync(0xffffffffu, bi, o);
            if (ob > best || (ob == best && oi < bi)) {
                best = ob;
                bi = oi;
            }
        }
        if ((tid & 31) == 0) {
            sh.red_d[tid >> 5] = best;
            sh.red_i[tid >> 5] = bi;
        }
        __syncthreads();
        if (tid == 0) {
            double b = sh.red_d[0];
            uint32_t i0 = sh.red_i[0];
            for (int q = 1; q < kThreads / 32; ++q)
                if (sh.red_d[q] > b || (sh.red_d[q] == b && sh.red_i[q] < i0)) {
                    b = sh.red_d[q];
                    i0 = sh.red_i[q];
                }
            sh.flag = i0;
            if (i0 < n && b > -1.0) {
                sh.counts[S.assign[i0]]--;
                S.assign[i0] = uint16_t(j);
                sh.counts[j] = 1;
                sh.cent[j] = float(S.v[i0]);
            } else {
                sh.flag = n;
            }
        }
        __syncthreads();
        if (sh.flag == n) break;  // nothing stealable
    }
    __syncthreads();
}

__device__ void intervals(const Scratch& S, Shared& sh, uint32_t k);

// Lloyd until the relative centroid movement is under tol (nuq.cpp:187-225)
__device__ uint32_t lloyd(const Scratch& S, Shared& sh, uint32_t k, uint32_t max_iters, double tol) {
    const uint32_t n = sh.n, tid = threadIdx.x;
    uint32_t iters = 0;
    while (iters < max_iters) {
        assign_and_repair(S, sh, k);
        ++iters;
        // per-cluster sums in position order: thread j owns cluster j and
        // scans its members' span [first, last]
        intervals(S, sh, k);
        for (uint32_t j = tid; j < k; j += kThreads) {
            double nu = 0.0, de = 0.0, pl = 0.0;
            const uint32_t i1 = sh.counts[j] ? sh.ivs[j] + 1 : 0;
            for (uint32_t i = sh.ivf[j]; i < i1; ++i) {
                if (S.assign[i] != j) continue;
                nu += S.w[i] * S.v[i];
                de += S.w[i];
                pl += S.v[i];
            }
            sh.num[j] = nu;
            sh.den[j] = de;
            sh.plain[j] = pl;
        }
        __syncthreads();
        if (tid == 0) {
            double mv = 0.0, mg = 0.0;
            for (uint32_t j = 0; j < k; ++j) {
                float nx;
                if (sh.counts[j] == 0) nx = sh.cent[j];
                else if (sh.den[j] > 0.0) nx = float(sh.num[j] / sh.den[j]);
                else nx = float(sh.plain[j] / double(sh.counts[j]));
                sh.next[j] = nx;
                const double dm = fabs(double(nx) - double(sh.cent[j]));
                const double am = fabs(double(sh.cent[j]));
                mv = dm > mv ? dm : mv;
                mg = am > mg ? am : mg;
            }
            sort_small(sh.next, k);
            for (uint32_t j = 0; j < k; ++j) sh.cent[j] = sh.next[j];
            sh.flag = (mv / (mg > 1e-30 ? mg : 1e-30) < tol) ? 1u : 0u;
        }
        __syncthreads();
        if (sh.flag) break;
    }
    assign_and_repair(S, sh, k);
    return iters;
}

// first/last position of every cluster (nuq.cpp:228-241); needs assign final
__device__ void intervals(const Scratch& S, Shared& sh, uint32_t k) {
    const uint32_t n = sh.n, tid = threadIdx.x;
    for (uint32_t j = tid; j < k; j += kThreads) {
        sh.ivf[j] = 0xffffffffu;
        sh.ivs[j] = 0;
    }
    __syncthreads();
    for (uint32_t i = tid; i < n; i += kThreads) {
        const uint32_t a = S.assign[i];
        atomicMin(&sh.ivf[a], i);
        atomicMax(&sh.ivs[a], i);
    }
    __syncthreads();
    for (uint32_t j = tid; j < k; j += kThreads)
        if (sh.ivf[j] == 0xffffffffu) sh.ivf[j] = 0;  // unseen: {0, 0}
    __syncthreads();
}

// block-wide minimum of cost(m) over m in [m0, m1) (+inf if empty)
template <class F>
__device__ double block_min(Shared& sh, uint32_t m0, uint32_t m1, F cost) {
    const uint32_t tid = threadIdx.x;
    double v = __longlong_as_double(0x7ff0000000000000ll);
    for (uint32_t m = m0 + tid; m < m1; m += kThreads) {
        const double c = cost(m);
        v = c < v ? c : v;
    }
    for (int o = 16; o; o >>= 1) {
        const double t = __shfl_xor_sync(0xffffffffu, v, o);
        v = t < v ? t : v;
    }
    __syncthreads();
    if ((tid & 31) == 0) sh.red_d[tid >> 5] = v;
    __syncthreads();
    double r = sh.red_d[0];
    for (int q = 1; q < kThreads / 32; ++q) r = sh.red_d[q] < r ? sh.red_d[q] : r;
    return r;
}

// exact boundary re-optimisation (nuq.cpp:246-327); returns true if changed.
// Whole block: a scan range (a pairwise cut, or one row m1 of the joint
// three-cluster cut) is first reduced to its minimum in parallel; only a
// range whose minimum beats the running record by the margin -- i.e. one
// where the reference accepts at least one cut -- is replayed exactly by
// warp 0's chain scan.  Rows m1 are evaluated kThreads/32 at a time (one per
// warp) and consumed in order, so the break on `left >= best` is the
// reference's.
__device__ bool boundary_refine(const Scratch& S, Shared& sh, uint32_t k) {
    if (k < 2) return false;
    intervals(S, sh, k);
    for (uint32_t j = 0; j < k; ++j)
        if (sh.counts[j] == 0) return false;
    constexpr uint32_t NW = kThreads / 32;
    const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    bool any = false;
    for (int sweep = 0; sweep < 32; ++sweep) {
        bool changed = false;
        for (uint32_t c = 0; c + 1 < k; ++c) {  // pairwise cuts
            const uint32_t s = sh.ivf[c], e = sh.ivs[c + 1], cur = sh.ivs[c];
            const double cc = icost(S, s, cur) + icost(S, cur + 1, e);
            const double eps = 1e-12 * (1.0 + cc);
            auto cost = [&](uint32_t m) { return icost(S, s, m) + icost(S, m + 1, e); };
            const double mn = block_min(sh, s, e, cost);
            uint32_t bm = cur;
            if (mn < cc - eps) {
                if (warp == 0) {
                    double best = cc;
                    chain_scan(s, e, best, bm, eps, cost);
                    if (lane == 0) sh.flag = bm;
                }
                __syncthreads();
                bm = sh.flag;
            }
            if (bm != cur) {
                __syncthreads();
                if (tid == 0) {
                    sh.ivs[c] = bm;
                    sh.ivf[c + 1] = bm + 1;
                }
                changed = true;
            }
            __syncthreads();
        }
        for (uint32_t c = 0; c + 2 < k; ++c) {  // joint cuts over three clusters
            const uint32_t s = sh.ivf[c], e = sh.ivs[c + 2];
            const uint32_t c1 = sh.ivs[c], c2 = sh.ivs[c + 1];
            const double cc = icost(S, s, c1) + icost(S, c1 + 1, c2) + icost(S, c2 + 1, e);
            const double eps = 1e-12 * (1.0 + cc);
            double R = cc;  // warp 0 owns the record; others read sh.total
            uint32_t b1 = c1, b2 = c2;
            for (uint32_t base = s;; base += NW) {
                // warp q: row m1 = base + q -> its left cost and row minimum
                const uint32_t m1 = base + warp;
                double left = __longlong_as_double(0x7ff0000000000000ll), mn = left;
                if (m1 + 1 < e) {
                    left = icost(S, s, m1);
                    for (uint32_t m2 = m1 + 1 + lane; m2 < e; m2 += 32) {
                        const double v = left + icost(S, m1 + 1, m2) + icost(S, m2 + 1, e);
                        mn = v < mn ? v : mn;
                    }
                    for (int o = 16; o; o >>= 1) {
                        const double t = __shfl_xor_sync(0xffffffffu, mn, o);
                        mn = t < mn ? t : mn;
                    }
                }
                if (lane == 0) {
                    sh.num[warp] = left;
                    sh.den[warp] = mn;
                }
                __syncthreads();
                if (warp == 0) {
                    uint32_t done = 0;
                    for (uint32_t q = 0; q < NW; ++q) {
                        const uint32_t r1 = base + q;
                        if (r1 + 1 >= e) {
                            done = 1;
                            break;
                        }
                        const double lq = sh.num[q];
                        if (lq >= R) {
                            done = 1;
                            break;
                        }
                        if (sh.den[q] < R - eps) {
                            uint32_t bm = 0xffffffffu;
                            chain_scan(r1 + 1, e, R, bm, eps, [&](uint32_t m2) {
                                return lq + icost(S, r1 + 1, m2) + icost(S, m2 + 1, e);
                            });
                            if (bm != 0xffffffffu) {
                                b1 = r1;
                                b2 = bm;
                            }
                        }
                    }
                    if (lane == 0) sh.flag = done;
                }
                __syncthreads();
                const bool done = sh.flag != 0;
                __syncthreads();
                if (done) break;
            }
            if (warp == 0 && lane == 0) {
                sh.red_i[0] = b1;
                sh.red_i[1] = b2;
            }
            __syncthreads();
            b1 = sh.red_i[0];
            b2 = sh.red_i[1];
            if (b1 != c1 || b2 != c2) {
                __syncthreads();
                if (tid == 0) {
                    sh.ivs[c] = b1;
                    sh.ivf[c + 1] = b1 + 1;
                    sh.ivs[c + 1] = b2;
                    sh.ivf[c + 2] = b2 + 1;
                }
                changed = true;
            }
            __syncthreads();
        }
        if (!changed) break;
        any = true;
    }
    if (!any) return false;
    // rebuild centroids, counts, assignment from the refined intervals
    for (uint32_t c = tid; c < k; c += kThreads) {
        sh.cent[c] = float(imean(S, sh.ivf[c], sh.ivs[c]));
        sh.counts[c] = sh.ivs[c] - sh.ivf[c] + 1;
    }
    __syncthreads();
    for (uint32_t c = 0; c < k; ++c)
        for (uint32_t i = sh.ivf[c] + tid; i <= sh.ivs[c]; i += kThreads) S.assign[i] = uint16_t(c);
    __syncthreads();
    return true;
}

// merge the cheapest adjacent pair + split the costliest cluster when that
// strictly lowers the objective (nuq.cpp:331-408)
__device__ bool merge_split(const Scratch& S, Shared& sh, uint32_t k) {
    if (k < 2) return false;
    intervals(S, sh, k);
    for (uint32_t j = 0; j < k; ++j)
        if (sh.counts[j] == 0) return false;
    const uint32_t tid = threadIdx.x, lane = tid & 31;
    if (tid < 32) {
        double tg[3] = {-1.0, -1.0, -1.0};
        uint32_t tc[3] = {0, 0, 0}, tcut[3] = {0, 0, 0};
        for (uint32_t c = 0; c < k; ++c) {
            const uint32_t s = sh.ivf[c], e = sh.ivs[c];
            if (s == e) continue;
            const double whole = icost(S, s, e);
            // first maximum of the gain over cuts m in [s, e), init (-1, cut 0)
            double g = -1.0;
            uint32_t gm = 0xffffffffu;
            for (uint32_t m = s + lane; m < e; m += 32) {
                const double v = whole - icost(S, s, m) - icost(S, m + 1, e);
                if (v > g) {
                    g = v;
                    gm = m;
                }
            }
            for (int o = 16; o; o >>= 1) {
                const double og = __shfl_xor_sync(0xffffffffu, g, o);
                const uint32_t om = __shfl_xor_sync(0xffffffffu, gm, o);
                if (og > g || (og == g && om < gm)) {
                    g = og;
                    gm = om;
                }
            }
            const double cg = gm == 0xffffffffu ? -1.0 : g;
            const uint32_t cut = gm == 0xffffffffu ? 0u : gm;
            for (int t = 0; t < 3; ++t) {
                if (cg > tg[t]) {
                    for (int u = 2; u > t; --u) {
                        tg[u] = tg[u - 1];
                        tc[u] = tc[u - 1];
                        tcut[u] = tcut[u - 1];
                    }
                    tg[t] = cg;
                    tc[t] = c;
                    tcut[t] = cut;
                    break;
                }
            }
        }
        uint32_t mc = k, sc = k, sat = 0;
        if (tg[0] > 0.0) {
            double bd = 0.0;
            for (uint32_t c = 0; c + 1 < k; ++c) {
                const double rise = icost(S, sh.ivf[c], sh.ivs[c + 1]) - icost(S, sh.ivf[c], sh.ivs[c]) -
                                    icost(S, sh.ivf[c + 1], sh.ivs[c + 1]);
                for (int t = 0; t < 3; ++t) {
                    if (tg[t] <= 0.0 || tc[t] == c || tc[t] == c + 1) continue;
                    const double delta = tg[t] - rise;
                    const double margin = 1e-12 * (1.0 + fabs(tg[t]));
                    if (delta > bd + margin) {
                        bd = delta;
                        mc = c;
                        sc = tc[t];
                        sat = tcut[t];
                    }
                    break;
                }
            }
        }
        if (tid == 0) {
            sh.moved = mc != k ? 1u : 0u;
            if (mc != k) {
                uint32_t q = 0;
                for (uint32_t c = 0; c < k; ++c) {
                    if (c == mc) {
                        sh.next[q++] = float(imean(S, sh.ivf[c], sh.ivs[c + 1]));
                        ++c;
                    } else if (c == sc) {
                        sh.next[q++] = float(imean(S, sh.ivf[c], sat));
                        sh.next[q++] = float(imean(S, sat + 1, sh.ivs[c]));
                    } else {
                        sh.next[q++] = sh.cent[c];
                    }
                }
                sort_small(sh.next, k);
                for (uint32_t c = 0; c < k; ++c) sh.cent[c] = sh.next[c];
            }
        }
    }
    __syncthreads();
    return sh.moved != 0;
}

// block-wide bitonic sort of keys[0, npow2) in global scratch
__device__ void bitonic(unsigned long long* a, uint32_t np) {
    for (uint32_t size = 2; size <= np; size <<= 1) {
        for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
            for (uint32_t t = threadIdx.x; t < np / 2; t += kThreads) {
                const uint32_t lo = 2 * t - (t & (stride - 1));
                const uint32_t hi = lo + stride;
                const bool up = (lo & size) == 0;
                const unsigned long long x = a[lo], y = a[hi];
                if ((x > y) == up) {
                    a[lo] = y;
                    a[hi] = x;
                }
            }
            __syncthreads();
        }
    }
}

}  // namespace

__global__ void __launch_bounds__(kThreads) kmeans_groups(QuantParams P) {
    __shared__ Shared sh;
    const uint32_t tid = threadIdx.x;
    const uint32_t gcols = P.cols / P.groups_per_row;
    const uint32_t k = 1u << P.bits;
    const size_t np = P.npow2;
    Scratch S;
    {
        uint8_t* base = P.scratch + size_t(blockIdx.x) * P.scratch_stride;
        auto take = [&](size_t bytes) {
            uint8_t* r = base;
            base += (bytes + 255) & ~size_t(255);
            return r;
        };
        S.keys = reinterpret_cast<unsigned long long*>(take(np * 8));
        S.v = reinterpret_cast<double*>(take(size_t(gcols) * 8));
        S.w = reinterpret_cast<double*>(take(size_t(gcols) * 8));
        S.pw = reinterpret_cast<double*>(take(size_t(gcols + 1) * 8));
        S.pwv = reinterpret_cast<double*>(take(size_t(gcols + 1) * 8));
        S.pwv2 = reinterpret_cast<double*>(take(size_t(gcols + 1) * 8));
        if (P.smem_prefix) {  // the interval-cost tables in shared memory
            extern __shared__ double dsm[];
            S.pw = dsm;
            S.pwv = dsm + (gcols + 1);
            S.pwv2 = dsm + 2 * size_t(gcols + 1);
        }
        S.assign = reinterpret_cast<uint16_t*>(take(size_t(gcols) * 2));
        S.vals = reinterpret_cast<float*>(take(size_t(gcols) * 4));
        S.wts = reinterpret_cast<float*>(take(size_t(gcols) * 4));
        S.wk = reinterpret_cast<float*>(take(size_t(gcols) * 4));
        S.kcol = reinterpret_cast<uint32_t*>(take(size_t(gcols) * 4));
    }
    const uint32_t n_groups = P.rows * P.groups_per_row;
    for (uint32_t g = blockIdx.x; g < n_groups; g += gridDim.x) {
        const uint32_t row = g / P.groups_per_row, c0 = (g % P.groups_per_row) * gcols;
        const size_t rbase = size_t(row) * P.cols;
        // ---- kept positions in column order (mask), block-wide compaction
        if (tid == 0) {
            uint32_t n = 0;
            for (uint32_t c = c0; c < c0 + gcols; ++c) {
                const size_t idx = rbase + c;
                if (P.mask && P.mask[idx]) {
                    P.assign[idx] = kMasked;
                    continue;
                }
                S.vals[n] = P.w[idx];
                S.wts[n] = P.sens[idx];
                S.kcol[n] = c;
                ++n;
            }
            sh.n = n;
        }
        __syncthreads();
        const uint32_t n = sh.n;
        float* cb = P.centroids + size_t(g) * k;
        if (n == 0) {
            if (tid == 0) {
                P.group_failed[g] = 1;
                P.group_obj[g] = 0.0;
                P.group_mse[g] = 0.0;
            }
            __syncthreads();
            continue;
        }
        if (P.method == 2) {
            // ---- round-to-nearest uniform levels (nuq.cpp:609-640)
            if (tid == 0) {
                float lo = S.vals[0], hi = S.vals[0];
                for (uint32_t i = 0; i < n; ++i) {
                    lo = S.vals[i] < lo ? S.vals[i] : lo;  // std::min(lo, x)
                    hi = hi < S.vals[i] ? S.vals[i] : hi;  // std::max(hi, x)
                }
                sh.total = (double(hi) - double(lo)) / double(k - 1);
                for (uint32_t j = 0; j < k; ++j) sh.cent[j] = float(double(lo) + sh.total * j);
                sh.cent[k - 1] = hi;
                sh.tail = lo;
            }
            __syncthreads();
            const double step = sh.total;
            for (uint32_t i = tid; i < n; i += kThreads) {
                uint32_t idx = 0;
                if (step > 0.0) {
                    const double t = (double(S.vals[i]) - double(sh.tail)) / step;
                    idx = uint32_t(floor(t + 0.5));
                    idx = idx < k - 1 ? idx : k - 1;
                }
                S.assign[i] = uint16_t(idx);  // original order here
            }
            __syncthreads();
        } else {
            // ---- weighted_kmeans_1d (nuq.cpp:411-502)
            if (tid == 0) {
                double tw = 0.0;
                bool bad = false;
                for (uint32_t i = 0; i < n; ++i) {
                    const float x = P.method == 1 ? 1.0f : S.wts[i];
                    if (!(x >= 0.0f) || !isfinite(x)) bad = true;
                    tw += double(x);
                }
                if (bad) P.group_failed[g] = 2;  // kmeans: negative / non-finite weight
                const bool uniform = tw == 0.0;
                for (uint32_t i = 0; i < n; ++i)
                    S.wk[i] = (uniform || P.method == 1) ? 1.0f : S.wts[i];
            }
            // sort keys: value order, then original index (= stable_sort)
            for (uint32_t i = tid; i < np; i += kThreads)
                S.keys[i] = i < n ? ((unsigned long long)fkey(S.vals[i]) << 32) | i : ~0ull;
            __syncthreads();
            bitonic(S.keys, uint32_t(np));
            for (uint32_t i = tid; i < n; i += kThreads) {
                const uint32_t o = uint32_t(S.keys[i]);
                S.v[i] = double(S.vals[o]);
                S.w[i] = double(S.wk[o]);
            }
            __syncthreads();
            if (tid == 0) {
                // distinct values <= k: exact clustering (centroids = the values)
                uint32_t nd = 0;
                for (uint32_t i = 0; i < n && nd <= k; ++i)
                    if (i == 0 || float(S.v[i]) != float(S.v[i - 1])) {
                        if (nd < k) sh.cent[nd] = float(S.v[i]);
                        ++nd;
                    }
                sh.flag = nd <= k ? nd : 0u;
                if (nd <= k)
                    for (uint32_t j = nd; j < k; ++j) sh.cent[j] = sh.cent[nd - 1];
            }
            __syncthreads();
            if (sh.flag) {
                const uint32_t nd = sh.flag;
                for (uint32_t i = tid; i < n; i += kThreads) {
                    const float x = S.vals[i];
                    uint32_t lo = 0, hi = nd;
                    while (lo < hi) {
                        const uint32_t mid = (lo + hi) >> 1;
                        if (sh.cent[mid] < x) lo = mid + 1;
                        else hi = mid;
                    }
                    S.assign[i] = uint16_t(lo);  // original order
                }
                __syncthreads();
            } else {
                if (tid == 0) {
                    // prefix sums in sorted order (make_sorted_problem)
                    S.pw[0] = S.pwv[0] = S.pwv2[0] = 0.0;
                    for (uint32_t i = 0; i < n; ++i) {
                        S.pw[i + 1] = S.pw[i] + S.w[i];
                        S.pwv[i + 1] = S.pwv[i] + S.w[i] * S.v[i];
                        S.pwv2[i + 1] = S.pwv2[i] + S.w[i] * S.v[i] * S.v[i];
                    }
                    // weighted quantile init (nuq.cpp:65-89): total in original order
                    double total = 0.0;
                    for (uint32_t i = 0; i < n; ++i) total += double(S.wk[i]);
                    uint32_t pos = 0;
                    double cum = S.w[0];
                    for (uint32_t j = 0; j < k; ++j) {
                        const double target = (double(j) + 0.5) / double(k) * total;
                        while (cum < target && pos + 1 < n) {
                            ++pos;
                            cum += S.w[pos];
                        }
                        sh.cent[j] = float(S.v[pos]);
                    }
                    sort_small(sh.cent, k);
                }
                __syncthreads();
                uint32_t budget = P.max_iters;
                long long t0 = clock64(), tl = 0, tr = 0, tm = 0;
                const uint32_t used = lloyd(S, sh, k, budget, P.tol);
                uint32_t rounds = 0, iters = used;
                tl += clock64() - t0;
                budget -= used < budget ? used : budget;
                for (int round = 0; round < 64 && budget > 0; ++round) {
                    t0 = clock64();
                    const bool refined = boundary_refine(S, sh, k);
                    tr += clock64() - t0;
                    t0 = clock64();
                    const bool moved = merge_split(S, sh, k);
                    tm += clock64() - t0;
                    if (!refined && !moved) break;
                    t0 = clock64();
                    const uint32_t it = lloyd(S, sh, k, budget, P.tol);
                    tl += clock64() - t0;
                    ++rounds;
                    iters += it;
                    budget -= it < budget ? it : budget;
                }
                if (P.prof && tid == 0) {  // dev: per-group cycle profile
                    unsigned long long* q = P.prof + size_t(g) * 6;
                    q[0] = tl;
                    q[1] = tr;
                    q[2] = tm;
                    q[3] = rounds;
                    q[4] = iters;
                }
                // back to the original order
                for (uint32_t i = tid; i < n; i += kThreads) {
                    const uint32_t o = uint32_t(S.keys[i]);
                    S.keys[i] = (unsigned long long)S.assign[i] | ((unsigned long long)o << 32);
                }
                __syncthreads();
                for (uint32_t i = tid; i < n; i += kThreads) {
                    const unsigned long long q = S.keys[i];
                    S.assign[uint32_t(q >> 32)] = uint16_t(q & 0xffffu);
                }
                __syncthreads();
            }
        }
        // ---- outputs + the group's objectives in original order (nuq.cpp:752-765)
        for (uint32_t j = tid; j < k; j += kThreads) cb[j] = sh.cent[j];
        for (uint32_t i = tid; i < n; i += kThreads) P.assign[rbase + S.kcol[i]] = S.assign[i];
        if (tid == 0) {
            double obj = 0.0, mse = 0.0;
            for (uint32_t i = 0; i < n; ++i) {
                const double d = double(S.vals[i]) - double(sh.cent[S.assign[i]]);
                obj += double(S.wts[i]) * d * d;
                mse += d * d;
            }
            P.group_obj[g] = obj;
            P.group_mse[g] = mse;
        }
        __syncthreads();
    }
}

cudaError_t launch_kmeans(const QuantParams& p, uint32_t grid, cudaStream_t st) {
    const size_t smem = p.smem_prefix ? kmeans_smem_bytes(p.cols / p.groups_per_row) : 0;
    if (smem) {
        const cudaError_t e = cudaFuncSetAttribute(
            kmeans_groups, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        if (e != cudaSuccess) return e;
    }
    kmeans_groups<<<grid, kThreads, smem, st>>>(p);
    return cudaGetLastError();
}

size_t kmeans_smem_bytes(uint32_t gcols) { return size_t(gcols + 1) * 3 * 8; }

size_t kmeans_scratch_stride(uint32_t gcols, size_t npow2) {
    auto r = [](size_t b) { return (b + 255) & ~size_t(255); };
    return r(npow2 * 8) + 2 * r(size_t(gcols) * 8) + 3 * r(size_t(gcols + 1) * 8) +
           r(size_t(gcols) * 2) + 4 * r(size_t(gcols) * 4);
}

}  // namespace sqz
