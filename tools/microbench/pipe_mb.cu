// Per-instruction throughput probe (lane-ops / clk / SM) on sm_100a.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <cuda_fp16.h>
__device__ __forceinline__ unsigned long long gtimer(){unsigned long long t; asm volatile("mov.u64 %0, %globaltimer;":"=l"(t)); return t;}
__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t s){uint32_t r; asm volatile("prmt.b32 %0,%1,%2,%3;":"=r"(r):"r"(a),"r"(b),"r"(s)); return r;}
struct Clk { unsigned long long c0,c1,t0,t1; };
template<int OP>
__global__ void __launch_bounds__(256) k(int n, uint32_t seed, uint32_t* out, Clk* clk){
  uint32_t r[8]; float f[8]; 
  for (int i=0;i<8;++i){ r[i]=seed*(i+1)+threadIdx.x; f[i]=__int_as_float(0x3f800000u + (r[i]&0xffff)); }
  uint32_t c1 = seed ^ 0x5140, c2 = seed*3u+0x7362;
  float4 acc[2] = {make_float4(0,0,0,0), make_float4(0,0,0,0)};
  Clk c; if (threadIdx.x==0){ c.c0=clock64(); c.t0=gtimer(); }
  #pragma unroll 1
  for (int it=0; it<n; ++it){
    #pragma unroll
    for (int u=0; u<4; ++u){
      #pragma unroll
      for (int i=0;i<8;++i){
        if (OP==0) { asm volatile("fma.rn.f32 %0,%0,%1,%2;":"+f"(f[i]):"f"(f[(i+1)&7]),"f"(f[(i+3)&7])); }
        else if (OP==1) { unsigned long long a = ((unsigned long long)__float_as_uint(f[i])<<32)|__float_as_uint(f[(i+1)&7]); unsigned long long b=((unsigned long long)r[i]<<32)|r[(i+2)&7];
                          asm volatile("fma.rn.f32x2 %0,%0,%1,%0;":"+l"(a):"l"(b)); f[i]=__uint_as_float((uint32_t)a); f[(i+1)&7]=__uint_as_float((uint32_t)(a>>32)); }
        else if (OP==2) { asm volatile("fma.rn.f32.f16 %0,%1,%2,%0;":"+f"(f[i]):"h"((unsigned short)r[i]),"h"((unsigned short)(r[(i+1)&7]>>16))); }
        else if (OP==3) { asm volatile("fma.rn.f16x2 %0,%0,%1,%2;":"+r"(r[i]):"r"(r[(i+1)&7]),"r"(r[(i+3)&7])); }
        else if (OP==4) { float t; asm volatile("cvt.f32.f16 %0,%1;":"=f"(t):"h"((unsigned short)r[i])); f[i]+=0.f; r[i]^=__float_as_uint(t); }
        else if (OP==5) { r[i] = prmt(r[i], r[(i+1)&7], c1 + i); }
        else if (OP==6) { asm volatile("lop3.b32 %0,%0,%1,%2,0x96;":"+r"(r[i]):"r"(r[(i+1)&7]),"r"(c2)); }
        else if (OP==7) { asm volatile("mad.lo.u32 %0,%0,%1,%2;":"+r"(r[i]):"r"(r[(i+1)&7]),"r"(c2)); }
        else if (OP==8) { if (i < 2) { // HMMA m16n8k16 f32 acc: 2 independent accumulators
            float4& a = acc[i];
            asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3},{%4,%5,%6,%7},{%8,%9},{%0,%1,%2,%3};"
              :"+f"(a.x),"+f"(a.y),"+f"(a.z),"+f"(a.w):"r"(r[0]),"r"(r[1]),"r"(r[2]),"r"(r[3]),"r"(r[4]),"r"(r[5])); } }
        else if (OP==9) { asm volatile("fma.rn.f32 %0,%0,%1,0f3F800000;":"+f"(f[i]):"f"(f[(i+1)&7])); }
        else if (OP==10) { asm volatile("shf.r.wrap.b32 %0,%0,%1,%2;":"+r"(r[i]):"r"(r[(i+1)&7]),"r"(c2)); }
        else if (OP==12) { asm volatile("mul.hi.u32 %0,%0,%1;":"+r"(r[i]):"r"(c2)); }
        else if (OP==13) { asm volatile("{.reg .b16 l,h,o,one; mov.b16 one, 0x3C00; mov.b32 {l,h}, %0; mul.rn.f16 o, h, one; mov.b32 %0, {o,l};}":"+r"(r[i])); }
        else if (OP==14) { asm volatile("mad.hi.u32 %0,%0,%1,%2;":"+r"(r[i]):"r"(c2),"r"(r[(i+1)&7])); }
        else if (OP==11) { asm volatile("add.u32 %0,%0,%1;":"+r"(r[i]):"r"(r[(i+1)&7])); }
      }
    }
  }
  if (threadIdx.x==0){ c.c1=clock64(); c.t1=gtimer(); if(blockIdx.x==0)*clk=c; }
  uint32_t s=0; for(int i=0;i<8;++i) s^=r[i]^__float_as_uint(f[i]); s^=__float_as_uint(acc[0].x+acc[1].y+acc[0].z+acc[1].w);
  out[blockIdx.x*blockDim.x+threadIdx.x]=s;
}
int main(){
  uint32_t* out; cudaMalloc(&out, 148*8*256*4); Clk* clk; cudaMalloc(&clk,sizeof(Clk));
  const char* names[15]={"FFMA 3reg","FFMA2","FHFMA f32.f16","HFMA2 f16x2","cvt.f32.f16","PRMT","LOP3","IMAD","HMMA m16n8k16 (per-instr)","FFMA imm","SHF","IADD","IMAD.HI (mul.hi)","HMUL hi->lo","IMAD.HI+add"};
  auto run=[&](auto kern, int op){
    int grid=148*4, n=4000; kern<<<grid,256>>>(10,1,out,clk); cudaDeviceSynchronize();
    cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0); kern<<<grid,256>>>(n,2,out,clk); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms,e0,e1); Clk h; cudaMemcpy(&h,clk,sizeof(h),cudaMemcpyDeviceToHost);
    double ghz=double(h.c1-h.c0)/double(h.t1-h.t0);
    double ops=double(grid)*256*n*32*(op==8?0.25:1.0);
    printf("%-26s %.3f ms  %.2f GHz  %.1f lane-ops/clk/SM (%.2f warp-instr/clk/SM)\n",names[op],ms,ghz,ops/(ms*1e-3)/(ghz*1e9)/148, ops/32/(ms*1e-3)/(ghz*1e9)/148);
  };
  run(k<0>,0);run(k<1>,1);run(k<2>,2);run(k<3>,3);run(k<4>,4);run(k<5>,5);run(k<6>,6);run(k<7>,7);run(k<8>,8);run(k<9>,9);run(k<10>,10);run(k<11>,11);run(k<12>,12);run(k<13>,13);run(k<14>,14);
  return 0;
}
