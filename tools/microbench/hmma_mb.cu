// Decode microbenchmark for the tensor-core (mma.sync m16n8k16) LUT-GEMV
// inner loop on sm_100a: PRMT byte-plane lookups build the fp16 A fragments,
// HMMA accumulates in fp32.  Operands come from shared memory (no HBM), so
// the number is the decode ceiling in weights/clk/SM.
//
// Tile = 4 rows; A rows m = 4*blk + i hold row i on column chunk blk (block-
// diagonal trick), B column n = blk holds x on that chunk, so one HMMA covers
// 4 rows x 64 columns = 256 weights and the row granularity is 4.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2306_07629_b200/csrc/tile.cuh"

#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s @%d: %s\n",#x,__LINE__,cudaGetErrorString(e)); return 1;}}while(0)

__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t s){uint32_t r; asm("prmt.b32 %0,%1,%2,%3;":"=r"(r):"r"(a),"r"(b),"r"(s)); return r;}
__device__ __forceinline__ uint32_t mulhi(uint32_t a, uint32_t b){uint32_t r; asm("mul.hi.u32 %0,%1,%2;":"=r"(r):"r"(a),"r"(b)); return r;}
__device__ __forceinline__ uint32_t madhi(uint32_t a, uint32_t b, uint32_t c){uint32_t r; asm("mad.hi.u32 %0,%1,%2,%3;":"=r"(r):"r"(a),"r"(b),"r"(c)); return r;}
__device__ __forceinline__ void hmma(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0, uint32_t b1){
  asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3},{%4,%5,%6,%7},{%8,%9},{%0,%1,%2,%3};"
    :"+f"(d[0]),"+f"(d[1]),"+f"(d[2]),"+f"(d[3]):"r"(a0),"r"(a1),"r"(a2),"r"(a3),"r"(b0),"r"(b1));
}
// high 16 bits -> low 16 bits on the FMA pipe: fp16 multiply by 1.0 of the
// upper half (selector halves 0x0xxx..0x7777 are finite fp16, so exact)
__device__ __forceinline__ uint32_t hi16(uint32_t a){uint32_t r; asm("{.reg .b16 l,h,o,one; mov.b16 one, 0x3C00; mov.b32 {l,h}, %1; mul.rn.f16 o, h, one; mov.b32 %0, {o,o};}":"=r"(r):"r"(a)); return r;}
struct Clk { unsigned long long c0,c1,t0,t1; };
__device__ __forceinline__ unsigned long long gtimer(){unsigned long long t; asm volatile("mov.u64 %0, %globaltimer;":"=l"(t)); return t;}

struct P8 { uint32_t l0,l1,h0,h1; };

// quad lookup: 4 indices in the low 4 nibbles of s -> 2 fp16x2 words
__device__ __forceinline__ void q4(uint32_t s, const P8& P, uint32_t& p01, uint32_t& p23){
  const uint32_t lo = prmt(P.l0,P.l1,s), hi = prmt(P.h0,P.h1,s);
  p01 = prmt(lo,hi,0x5140); p23 = prmt(lo,hi,0x7362);
}

// one span (32 columns of this thread's row): 3 words -> 4 HMMAs
template<int SHIFT_IMAD>
__device__ __forceinline__ void span3(uint32_t w0, uint32_t w1, uint32_t w2, const P8& P, const uint4& xa, const uint4& xb,
                                      float (&d)[4], uint32_t k16, uint32_t k29, uint32_t k30, uint32_t k31){
  const uint32_t m0 = w0 & 0x77777777u, m1 = w1 & 0x77777777u, m2 = w2 & 0x77777777u;
  uint32_t t;
  if (SHIFT_IMAD >= 2) {
    t = ((w0 >> 3) & 0x11111111u) | ((w1 >> 2) & 0x22222222u) | ((w2 >> 1) & 0x44444444u);
    if (SHIFT_IMAD == 3) { const uint32_t e0 = w0 & 0x88888888u, e1 = w1 & 0x88888888u, e2 = w2 & 0x88888888u;
      t = madhi(e0, k29, madhi(e1, k30, mulhi(e2, k31))); }
  } else if (SHIFT_IMAD) {
    const uint32_t e0 = w0 & 0x88888888u, e1 = w1 & 0x88888888u, e2 = w2 & 0x88888888u;
    t = madhi(e0, k29, madhi(e1, k30, mulhi(e2, k31)));
  } else {
    t = ((w0 >> 3) & 0x11111111u) | ((w1 >> 2) & 0x22222222u) | ((w2 >> 1) & 0x44444444u);
  }
  // quads: A (a0/a2) cols 4j..4j+3 from m0 (j=0,1), m1 (j=2,3); B (a1/a3) cols 16+4j.. from m2, t
  uint32_t sA[4], sB[4];
  sA[0] = m0; sA[2] = m1; sB[0] = m2; sB[2] = t;
  if (SHIFT_IMAD >= 2) { sA[1] = hi16(m0); sA[3] = hi16(m1); sB[1] = hi16(m2); sB[3] = hi16(t); }
  else if (SHIFT_IMAD) { sA[1] = mulhi(m0,k16); sA[3] = mulhi(m1,k16); sB[1] = mulhi(m2,k16); sB[3] = mulhi(t,k16); }
  else { sA[1] = m0 >> 16; sA[3] = m1 >> 16; sB[1] = m2 >> 16; sB[3] = t >> 16; }
  const uint32_t xs[8] = {xa.x, xa.y, xa.z, xa.w, xb.x, xb.y, xb.z, xb.w};
  #pragma unroll
  for (int j = 0; j < 4; ++j) {
    uint32_t a0,a2,a1,a3;
    q4(sA[j], P, a0, a2);
    q4(sB[j], P, a1, a3);
    hmma(d, a0, a1, a2, a3, xs[2*j], xs[2*j+1]);
  }
}

// 4-bit: 16-entry LUT, 4 words per 32 columns
struct P16 { P8 a, b; };
__device__ __forceinline__ void q4_16(uint32_t s, uint32_t pk, const P16& P, uint32_t& p01, uint32_t& p23){
  const uint32_t loA = prmt(P.a.l0,P.a.l1,s), loB = prmt(P.b.l0,P.b.l1,s);
  const uint32_t hiA = prmt(P.a.h0,P.a.h1,s), hiB = prmt(P.b.h0,P.b.h1,s);
  const uint32_t lo = prmt(loA,loB,pk), hi = prmt(hiA,hiB,pk);
  p01 = prmt(lo,hi,0x5140); p23 = prmt(lo,hi,0x7362);
}
__device__ __forceinline__ void span4(const uint4& w, const P16& P, const uint4& xa, const uint4& xb, float (&d)[4]){
  const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
  const uint32_t xs[8] = {xa.x, xa.y, xa.z, xa.w, xb.x, xb.y, xb.z, xb.w};
  uint32_t sl[4], pk[4];
  #pragma unroll
  for (int q = 0; q < 4; ++q) { sl[q] = ws[q] & 0x77777777u; pk[q] = ((ws[q] >> 1) & 0x44444444u) | 0x32103210u; }
  #pragma unroll
  for (int j = 0; j < 4; ++j) {
    // A quad j: cols 4j.. -> word j/2 half j&1 ; B quad j: cols 16+4j -> word 2+j/2
    const int wa = j >> 1, wb = 2 + (j >> 1), hsh = (j & 1) * 16;
    uint32_t a0,a2,a1,a3;
    q4_16(sl[wa] >> hsh, pk[wa] >> hsh, P, a0, a2);
    q4_16(sl[wb] >> hsh, pk[wb] >> hsh, P, a1, a3);
    hmma(d, a0, a1, a2, a3, xs[2*j], xs[2*j+1]);
  }
}

#define NSPAN 8   // spans resident in smem per warp (cycled)
// VAR 0: 3-bit SHF shifts; 1: 3-bit IMAD.HI shifts; 2: 4-bit
template<int VAR, int RT, int XCF = 0>
__global__ void __launch_bounds__(768) k_hmma(int niter, float* out, Clk* clk, uint32_t seed, uint32_t k16, uint32_t k29, uint32_t k30, uint32_t k31, int idle = 0){
  extern __shared__ uint32_t sm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // idle "role" warps (the stack kernel's publisher/loader/finisher/CSR
  // warps): wait on an mbarrier that never completes until the decode warps
  // are done (mbar_wait's suspend-hint try_wait loop)
  __shared__ __align__(8) unsigned long long ibar;
  __shared__ int idone;
  if (threadIdx.x == 0) { idone = 0; asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"((uint32_t)__cvta_generic_to_shared(&ibar))); }
  __syncthreads();

  const int WPS = VAR == 2 ? 4 : 3;
  (void)WPS;              // words per lane per span per tile
  uint32_t* pk = sm + warp * (NSPAN * RT * WPS * 32);
  uint32_t* sx = sm + (blockDim.x / 32 - idle) * (NSPAN * RT * WPS * 32);   // x: NSPAN * 4 groups * 32 halves
  const int nw = blockDim.x / 32;
  for (int i = lane; warp < int(blockDim.x / 32) - idle && i < NSPAN * RT * WPS * 32; i += 32) { uint32_t h = (i * 2654435761u) ^ seed ^ warp; pk[i] = h; }
  for (int i = threadIdx.x; i < NSPAN * 128; i += blockDim.x) sx[i] = 0x3c003800u ^ (i & 0x00ff00ff);
  __syncthreads();
  if (warp >= int(blockDim.x / 32) - idle) {
    const uint32_t a = (uint32_t)__cvta_generic_to_shared(&ibar);
    while (*(volatile int*)&idone < int(blockDim.x / 32) - idle) {
      uint32_t done;
      asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n selp.u32 %0, 1, 0, p;\n}" : "=r"(done) : "r"(a), "r"(0u), "r"(1000000u) : "memory");
    }
    return;
  }
  (void)nw;
  const uint32_t g = lane >> 2, t = lane & 3, n = g & 3;
  P8 P[RT]; P16 Q[RT];
  #pragma unroll
  for (int r = 0; r < RT; ++r) {
    P[r] = P8{sx[lane + r], sx[lane + 40], sx[lane + 50 + r], sx[lane + 60]};
    Q[r] = P16{P[r], P8{sx[lane + 70], sx[lane + 80 + r], sx[lane + 90], sx[lane + 95]}};
  }
  float d[RT][4], d2[RT][4];
  #pragma unroll
  for (int r = 0; r < RT; ++r) d[r][0] = d[r][1] = d[r][2] = d[r][3] = d2[r][0] = d2[r][1] = d2[r][2] = d2[r][3] = 0.f;
  Clk c; if (threadIdx.x==0){ c.c0 = clock64(); c.t0 = gtimer(); }
  #pragma unroll 1
  for (int it = 0; it < niter; ++it) {
    const int s = it & (NSPAN - 1);
    // x halves of this lane's B column: group G(n&1, t), half (n>>1)
    const uint4* xp = reinterpret_cast<const uint4*>(sx + s * 128);
    const uint32_t xo = XCF ? (4 * n + t) : (((n & 1) * 4 + t) * 4 + (n >> 1) * 2);
    const uint4 xa = xp[xo], xb = xp[xo + (XCF ? 16 : 1)];
    #pragma unroll
    for (int r = 0; r < RT; ++r) {
      const uint32_t* wp = pk + (s * RT + r) * WPS * 32 + lane;
      if (VAR == 2) {
        const uint4 w = make_uint4(wp[0], wp[32], wp[64], wp[96]);
        span4(w, Q[r], xa, xb, d[r]);
      } else if (VAR == 5) {   // the product's span3_mma (dual accumulators)
        sqz::Planes8 PP{P[r].l0, P[r].l1, P[r].h0, P[r].h1};
        sqz::span3_mma(wp[0], wp[32], wp[64], PP, xa, xb, d[r], d2[r]);
      } else if (VAR == 7 || VAR == 8) {   // the stack kernel's span-pair loop: 2 units / iter
        sqz::Planes8 PP{P[r].l0, P[r].l1, P[r].h0, P[r].h1};
        const int s2 = (s + 1) & (NSPAN - 1);
        const uint32_t* wq = pk + (s2 * RT + r) * WPS * 32 + lane;
        const uint4* xq = reinterpret_cast<const uint4*>(sx + s2 * 128);
        const uint4 xa2 = xq[xo], xb2 = xq[xo + (XCF ? 16 : 1)];
        if (VAR == 7) {
          sqz::span3_mma_one(wp[0], wp[32], wp[64], PP, xa, xb, d[r]);
          sqz::span3_mma_one(wq[0], wq[32], wq[64], PP, xa2, xb2, d2[r]);
        } else {
          sqz::span3_mma(wp[0], wp[32], wp[64], PP, xa, xb, d[r], d2[r]);
          sqz::span3_mma(wq[0], wq[32], wq[64], PP, xa2, xb2, d[r], d2[r]);
        }
      } else if (VAR == 6) {   // + IMAD.HI spare-index gather
        sqz::Planes8 PP{P[r].l0, P[r].l1, P[r].h0, P[r].h1};
        sqz::span3_mma<true>(wp[0], wp[32], wp[64], PP, xa, xb, d[r], d2[r], sqz::ShiftK{k29, k30, k31});
      } else if (VAR == 3) {
        span3<2>(wp[0], wp[32], wp[64], P[r], xa, xb, d[r], k16, k29, k30, k31);
      } else if (VAR == 4) {
        span3<3>(wp[0], wp[32], wp[64], P[r], xa, xb, d[r], k16, k29, k30, k31);
      } else if (VAR == 1) {
        span3<1>(wp[0], wp[32], wp[64], P[r], xa, xb, d[r], k16, k29, k30, k31);
      } else {
        span3<0>(wp[0], wp[32], wp[64], P[r], xa, xb, d[r], k16, k29, k30, k31);
      }
    }
  }
  if (threadIdx.x==0){ c.c1 = clock64(); c.t1 = gtimer(); if (blockIdx.x==0) *clk = c; }
  if (lane == 0) atomicAdd(&idone, 1);
  float a = 0.f;
  #pragma unroll
  for (int r = 0; r < RT; ++r) a += d[r][0] + d[r][1] + d[r][2] + d[r][3] + d2[r][0] + d2[r][3];
  out[blockIdx.x*blockDim.x + threadIdx.x] = a;
}

int main(){
  int dev=0; cudaDeviceProp pr; CK(cudaGetDeviceProperties(&pr, dev));
  const int nsm = pr.multiProcessorCount;
  printf("device %s SMs %d\n", pr.name, nsm);
  float* out; CK(cudaMalloc(&out, size_t(nsm)*4*1024*sizeof(float)));
  Clk* clk; CK(cudaMalloc(&clk, sizeof(Clk)));
  auto run = [&](auto kern, const char* name, int var, int rt, int warps, int ctas, int idle = 0) -> int {
    const int wps = var == 2 ? 4 : 3;
    size_t smem = size_t(warps) * NSPAN * rt * wps * 32 * 4 + NSPAN * 128 * 4;
    if (smem * ctas > 227 * 1024) { printf("%-34s warps %2d ctas %d: smem too big\n", name, warps, ctas); return 0; }
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const int grid = nsm * ctas, niter = 20000;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    kern<<<grid, (warps+idle)*32, smem>>>(100, out, clk, 1, 1u<<16, 1u<<29, 1u<<30, 1u<<31, idle); CK(cudaDeviceSynchronize());
    cudaEventRecord(e0); kern<<<grid, (warps+idle)*32, smem>>>(niter, out, clk, 2, 1u<<16, 1u<<29, 1u<<30, 1u<<31, idle); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    Clk h; cudaMemcpy(&h, clk, sizeof(Clk), cudaMemcpyDeviceToHost);
    const double ghz = double(h.c1-h.c0)/double(h.t1-h.t0);
    const double weights = double(grid) * warps * niter * rt * 1024.0 * (var >= 7 ? 2 : 1);   // 4 rows x 256 cols per span per tile
    const double wpc = weights / (ms*1e-3) / (ghz*1e9) / nsm;
    const double bpw = var == 2 ? 0.5 : 0.375;
    printf("%-34s warps %2d ctas %d: %.3f ms %.2f GHz  %.1f w/clk/SM  => %.0f GB/s equiv (at 1.965 GHz: %.0f)\n", name, warps, ctas, ms, ghz, wpc,
           weights/(ms*1e-3)*bpw/1e9, wpc*nsm*1.965e9*bpw/1e9);
    return 0;
  };
  for (int warps : {8, 12, 16}) {
    run(k_hmma<5,1,1>, "3b product RT1 xcf", 5, 1, warps, 1);
    run(k_hmma<6,1,1>, "3b product+imad RT1 xcf", 6, 1, warps, 1);
    run(k_hmma<5,2,1>, "3b product RT2 xcf", 5, 2, warps, 1);
    run(k_hmma<6,2,1>, "3b product+imad RT2 xcf", 6, 2, warps, 1);
    run(k_hmma<7,1,1>, "3b stack span-pair (one acc/unit)", 7, 1, warps, 1);
    run(k_hmma<7,1,1>, "3b span-pair + 7 idle role warps", 7, 1, warps, 1, 7);
    run(k_hmma<8,1,1>, "3b span-pair dual acc", 8, 1, warps, 1);

  }
  return 0;
}
