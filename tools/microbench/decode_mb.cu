// Decode-strategy microbenchmark for the LUT-GEMV inner loop on sm_100a.
// Measures weights/clk/SM for candidate dequant+FMA sequences with operands
// staged in shared memory (no HBM traffic), plus a pure HBM read-stream test.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <cuda_fp16.h>

#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s @%d: %s\n",#x,__LINE__,cudaGetErrorString(e)); return 1;}}while(0)

__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t s){uint32_t r; asm("prmt.b32 %0,%1,%2,%3;":"=r"(r):"r"(a),"r"(b),"r"(s)); return r;}
__device__ __forceinline__ float fhl(uint32_t w, uint32_t x, float c){float d; asm("fma.rn.f32.f16 %0,%1,%2,%3;":"=f"(d):"h"((unsigned short)(w&0xffff)),"h"((unsigned short)(x&0xffff)),"f"(c)); return d;}
__device__ __forceinline__ float fhh(uint32_t w, uint32_t x, float c){float d; asm("fma.rn.f32.f16 %0,%1,%2,%3;":"=f"(d):"h"((unsigned short)(w>>16)),"h"((unsigned short)(x>>16)),"f"(c)); return d;}

struct Clk { unsigned long long c0,c1,t0,t1; };
__device__ __forceinline__ unsigned long long gtimer(){unsigned long long t; asm volatile("mov.u64 %0, %globaltimer;":"=l"(t)); return t;}

#define NBUF 8
// shared: packed words [NBUF][32 lanes] uint4 per warp-slot; x: [NBUF*4] uint4 (broadcast)
template<int VAR>
__global__ void __launch_bounds__(256) k_decode(int niter, float* out, Clk* clk, uint32_t seed){
  extern __shared__ uint4 sm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint4* spk = sm + warp * NBUF * 32;           // per-warp packed words
  uint4* sx  = sm + 8 * NBUF * 32;              // x (shared by all warps)
  uint32_t* tab = (uint32_t*)(sx + NBUF*4) + warp * 64 * 32; // pair tables (VAR 2)
  for (int i = threadIdx.x; i < 8*NBUF*32; i += blockDim.x) { uint32_t h = (i*2654435761u) ^ seed; sm[i] = make_uint4(h, h*3u+1, h*7u+5, h*13u+11); }
  for (int i = threadIdx.x; i < NBUF*4; i += blockDim.x) { sx[i] = make_uint4(0x3c003c00u ^ (i&0x03ff03ff), 0x3800b800u, 0x3c00bc00u, 0x34003400u); }
  if (VAR == 2) for (int i = lane; i < 64*32; i += 32) tab[i] = 0x3c003800u ^ (i * 0x00010001u & 0x00ff00ffu);
  __syncthreads();
  uint32_t L0 = 0x03020100u ^ lane, L1 = 0x07060504u, H0 = 0x3c3a3836u, H1 = 0xbcbab8b6u;
  uint32_t L2 = 0x0b0a0908u, L3 = 0x0f0e0d0cu, H2 = 0x34322a28u, H3 = 0xb4b2aaa8u;
  float a0=0.f,a1=0.f,a2=0.f,a3=0.f;
  const uint32_t lane4 = lane * 4;
  const uint32_t k3210 = 0x32103210u;
  Clk c; if (threadIdx.x==0){ c.c0 = clock64(); c.t0 = gtimer(); }
  #pragma unroll 1
  for (int it = 0; it < niter; ++it) {
    const int b = it & (NBUF-1);
    uint4 w = spk[b*32 + lane];
    if (VAR == 0) { // nibble selectors (bits already clean): 32 weights from 4 words
      uint32_t ws[4] = {w.x, w.y, w.z, w.w};
      #pragma unroll
      for (int q = 0; q < 4; ++q) {
        uint4 xv = sx[b*4 + q];
        uint32_t s0 = ws[q], s1 = ws[q] >> 16;
        uint32_t lo0 = prmt(L0,L1,s0), hi0 = prmt(H0,H1,s0), lo1 = prmt(L0,L1,s1), hi1 = prmt(H0,H1,s1);
        uint32_t h0 = prmt(lo0,hi0,0x5140), h1 = prmt(lo0,hi0,0x7362), h2 = prmt(lo1,hi1,0x5140), h3 = prmt(lo1,hi1,0x7362);
        a0 = fhl(h0,xv.x,a0); a1 = fhh(h0,xv.x,a1); a2 = fhl(h1,xv.y,a2); a3 = fhh(h1,xv.y,a3);
        a0 = fhl(h2,xv.z,a0); a1 = fhh(h2,xv.z,a1); a2 = fhl(h3,xv.w,a2); a3 = fhh(h3,xv.w,a3);
      }
    } else if (VAR == 1) { // true 3-bit: 3 words -> 32 indices (24 nibble-aligned + 8 from spare bit-3s)
      uint32_t m0 = w.x & 0x77777777u, m1 = w.y & 0x77777777u, m2 = w.z & 0x77777777u;
      uint32_t t = ((w.x >> 3) & 0x11111111u) | ((w.y >> 2) & 0x22222222u) | ((w.z >> 1) & 0x44444444u);
      uint32_t ws[4] = {m0, m1, m2, t};
      #pragma unroll
      for (int q = 0; q < 4; ++q) {
        uint4 xv = sx[b*4 + q];
        uint32_t s0 = ws[q], s1 = ws[q] >> 16;
        uint32_t lo0 = prmt(L0,L1,s0), hi0 = prmt(H0,H1,s0), lo1 = prmt(L0,L1,s1), hi1 = prmt(H0,H1,s1);
        uint32_t h0 = prmt(lo0,hi0,0x5140), h1 = prmt(lo0,hi0,0x7362), h2 = prmt(lo1,hi1,0x5140), h3 = prmt(lo1,hi1,0x7362);
        a0 = fhl(h0,xv.x,a0); a1 = fhh(h0,xv.x,a1); a2 = fhl(h1,xv.y,a2); a3 = fhh(h1,xv.y,a3);
        a0 = fhl(h2,xv.z,a0); a1 = fhh(h2,xv.z,a1); a2 = fhl(h3,xv.w,a2); a3 = fhh(h3,xv.w,a3);
      }
    } else if (VAR == 2) { // LDS lane-private pair table: 16 pairs from 3 words (5 per word + 1 assembled)
      uint32_t ws[3] = {w.x, w.y, w.z};
      #pragma unroll
      for (int q = 0; q < 3; ++q) {
        #pragma unroll
        for (int p = 0; p < 5; ++p) {
          uint32_t v = (p == 1) ? ws[q] : ((6*p) > 7 ? (ws[q] >> (6*p-7)) : (ws[q] << (7-6*p)));
          uint32_t addr = (v & 0x1F80u) | lane4;
          uint32_t pr = tab[addr >> 2];
          uint4 xv = sx[b*4 + ((q*5+p)>>2)];
          uint32_t xx = ((q*5+p)&3)==0 ? xv.x : ((q*5+p)&3)==1 ? xv.y : ((q*5+p)&3)==2 ? xv.z : xv.w;
          a0 = fhl(pr, xx, a0); a1 = fhh(pr, xx, a1);
        }
      }
      uint32_t v = ((ws[0] >> 30) | ((ws[1] >> 28) & 0xc) | ((ws[2] >> 26) & 0x30)) << 7;
      uint32_t pr = tab[((v & 0x1F80u) | lane4) >> 2];
      uint4 xv = sx[b*4 + 3];
      a2 = fhl(pr, xv.w, a2); a3 = fhh(pr, xv.w, a3);
    } else if (VAR == 3) { // PRMT planes + HADD2.F32 + FFMA2 (x as fp32 pairs)
      uint32_t ws[4] = {w.x, w.y, w.z, w.w};
      const float4* sxf = (const float4*)sx;
      float2 acc0 = make_float2(a0,a1), acc1 = make_float2(a2,a3);
      #pragma unroll
      for (int q = 0; q < 4; ++q) {
        uint32_t s0 = ws[q], s1 = ws[q] >> 16;
        uint32_t lo0 = prmt(L0,L1,s0), hi0 = prmt(H0,H1,s0), lo1 = prmt(L0,L1,s1), hi1 = prmt(H0,H1,s1);
        uint32_t hh[4] = {prmt(lo0,hi0,0x5140), prmt(lo0,hi0,0x7362), prmt(lo1,hi1,0x5140), prmt(lo1,hi1,0x7362)};
        #pragma unroll
        for (int j = 0; j < 4; ++j) {
          float2 wf = __half22float2(*reinterpret_cast<__half2*>(&hh[j]));
          float2 xf = *reinterpret_cast<const float2*>(reinterpret_cast<const float*>(sxf) + ((b*16 + q*4 + j)*2 & (NBUF*16-1)));
          unsigned long long r;
          float2& acc = (j & 1) ? acc1 : acc0;
          asm("fma.rn.f32x2 %0,%1,%2,%3;":"=l"(r):"l"(*(unsigned long long*)&wf),"l"(*(unsigned long long*)&xf),"l"(*(unsigned long long*)&acc));
          acc = *(float2*)&r;
        }
      }
      a0 = acc0.x; a1 = acc0.y; a2 = acc1.x; a3 = acc1.y;
    } else if (VAR == 4) { // 4-bit: 16-entry LUT, nibble idx with bit3 -> two half-table PRMTs + combine
      uint32_t ws[4] = {w.x, w.y, w.z, w.w};
      #pragma unroll
      for (int q = 0; q < 4; ++q) {
        uint4 xv = sx[b*4 + q];
        uint32_t sl = ws[q] & 0x77777777u;
        uint32_t c2 = ((ws[q] >> 1) & 0x44444444u) | k3210;
        #pragma unroll
        for (int h = 0; h < 2; ++h) {
          uint32_t s = h ? (sl >> 16) : sl;
          uint32_t cs = h ? (c2 >> 16) : c2;
          uint32_t loA = prmt(L0,L1,s), loB = prmt(L2,L3,s), hiA = prmt(H0,H1,s), hiB = prmt(H2,H3,s);
          uint32_t lo = prmt(loA,loB,cs), hi = prmt(hiA,hiB,cs);
          uint32_t h0 = prmt(lo,hi,0x5140), h1 = prmt(lo,hi,0x7362);
          uint32_t x0 = h ? xv.z : xv.x, x1 = h ? xv.w : xv.y;
          a0 = fhl(h0,x0,a0); a1 = fhh(h0,x0,a1); a2 = fhl(h1,x1,a2); a3 = fhh(h1,x1,a3);
        }
      }
    }
  }
  if (threadIdx.x==0){ c.c1 = clock64(); c.t1 = gtimer(); if (blockIdx.x==0) *clk = c; }
  out[blockIdx.x*blockDim.x + threadIdx.x] = a0+a1+a2+a3;
}

__device__ __forceinline__ uint4 ldg_nc(const uint4* p){uint4 r; asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3},[%4];":"=r"(r.x),"=r"(r.y),"=r"(r.z),"=r"(r.w):"l"(p)); return r;}
template<int U>
__global__ void k_stream(const uint4* __restrict__ p, size_t n, uint32_t* out){
  uint32_t acc = 0;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + (U-1)*stride < n; i += U*stride) {
    uint4 v[U];
    #pragma unroll
    for (int u = 0; u < U; ++u) v[u] = ldg_nc(p + i + u*stride);
    #pragma unroll
    for (int u = 0; u < U; ++u) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
  }
  if (acc == 0x12345678u) out[0] = acc;
}

int main(){
  int dev=0; cudaDeviceProp pr; CK(cudaGetDeviceProperties(&pr, dev));
  printf("device %s SMs %d smemPerSM %zu smemOptin %zu L2 %d\n", pr.name, pr.multiProcessorCount, pr.sharedMemPerMultiprocessor, pr.sharedMemPerBlockOptin, pr.l2CacheSize);
  const int nsm = pr.multiProcessorCount;
  float* out; CK(cudaMalloc(&out, 148*64*256*sizeof(float)));
  Clk* clk; CK(cudaMalloc(&clk, sizeof(Clk)));
  size_t smem_base = (8*NBUF*32 + NBUF*4)*16, smem_tab = 8*64*32*4;
  const char* names[5] = {"A nibble-PRMT+FHFMA","B 3bit-PRMT+FHFMA","C LDS-pairtable+FHFMA","D PRMT+cvt+FFMA2","E 4bit16-PRMT+FHFMA"};
  auto run = [&](auto kern, int var, int ctas_per_sm) -> int {
    size_t smem = smem_base + (var==2 ? smem_tab : 0);
    if (smem*ctas_per_sm > 225000) return 0;
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int grid = nsm * ctas_per_sm, niter = 40000;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    kern<<<grid,256,smem>>>(100, out, clk, 1); CK(cudaDeviceSynchronize());
    cudaEventRecord(e0); kern<<<grid,256,smem>>>(niter, out, clk, 2); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    Clk h; cudaMemcpy(&h, clk, sizeof(Clk), cudaMemcpyDeviceToHost);
    double ghz = double(h.c1-h.c0)/double(h.t1-h.t0);
    double weights = double(grid)*256*niter*32.0;
    double wpc = weights / (ms*1e-3) / (ghz*1e9) / nsm;
    printf("%-26s ctas/SM %d: %.3f ms  clk %.3f GHz  %.1f weights/clk/SM  => 3bit-equiv %.0f GB/s, 4bit-equiv %.0f GB/s\n", names[var], ctas_per_sm, ms, ghz, wpc,
           weights/(ms*1e-3)*0.375/1e9, weights/(ms*1e-3)*0.5/1e9);
    return 0;
  };
  for (int occ : {1, 2, 4}) {
    run(k_decode<0>, 0, occ); run(k_decode<1>, 1, occ); run(k_decode<2>, 2, occ); run(k_decode<3>, 3, occ); run(k_decode<4>, 4, occ);
  }
  // HBM stream
  size_t bytes = size_t(4) << 30; uint4* buf; CK(cudaMalloc(&buf, bytes)); CK(cudaMemset(buf, 1, bytes));
  uint32_t* o32; CK(cudaMalloc(&o32, 64));
  for (int cps : {2, 4, 8}) for (int U : {2, 4, 8}) {
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    auto launch = [&](){ if (U==2) k_stream<2><<<nsm*cps,256>>>(buf, bytes/16, o32); else if (U==4) k_stream<4><<<nsm*cps,256>>>(buf, bytes/16, o32); else k_stream<8><<<nsm*cps,256>>>(buf, bytes/16, o32); };
    launch(); CK(cudaDeviceSynchronize());
    float best = 1e9;
    for (int r = 0; r < 5; ++r) { cudaEventRecord(e0); launch(); cudaEventRecord(e1); cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms,e0,e1); if (ms<best) best=ms; }
    printf("stream ctas/SM %d unroll %d: %.3f ms  %.0f GB/s\n", cps, U, best, bytes/(best*1e-3)/1e9);
  }
  return 0;
}
