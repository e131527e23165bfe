// M1 micro-benchmarks (design calibration, not product code): FP32 FMA issue rate with taps in
// registers / kernel-param constant bank / immediates / packed f32x2, grid-barrier latency,
// block-reduction latency, HBM copy and L2 read bandwidth.
#include <cstdio>
#include <cuda_runtime.h>
#include <cooperative_groups.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s at %d\n",cudaGetErrorString(e),__LINE__);return 1;}}while(0)
struct Taps { float w[32]; };
constexpr int NACC = 8, ITERS = 4096;
__global__ void ffma_reg(float* out, const float* win, float seed) {
  float w[16]; for (int i=0;i<16;i++) w[i]=win[i];
  float a[NACC]; for (int i=0;i<NACC;i++) a[i]=seed*(threadIdx.x+i);
  float x[NACC]; for (int i=0;i<NACC;i++) x[i]=seed+i;
  for (int it=0; it<ITERS; it++) {
    #pragma unroll
    for (int t=0;t<16;t++) {
      #pragma unroll
      for (int i=0;i<NACC;i++) a[i]=fmaf(x[i], w[t], a[i]);
    }
  }
  float s=0; for (int i=0;i<NACC;i++) s+=a[i]; out[blockIdx.x*blockDim.x+threadIdx.x]=s;
}
__global__ void ffma_param(float* out, Taps tp, float seed) {
  float a[NACC]; for (int i=0;i<NACC;i++) a[i]=seed*(threadIdx.x+i);
  float x[NACC]; for (int i=0;i<NACC;i++) x[i]=seed+i;
  for (int it=0; it<ITERS; it++) {
    #pragma unroll
    for (int t=0;t<16;t++) {
      #pragma unroll
      for (int i=0;i<NACC;i++) a[i]=fmaf(x[i], tp.w[t], a[i]);
    }
  }
  float s=0; for (int i=0;i<NACC;i++) s+=a[i]; out[blockIdx.x*blockDim.x+threadIdx.x]=s;
}
__global__ void ffma_imm(float* out, float seed) {
  float a[NACC]; for (int i=0;i<NACC;i++) a[i]=seed*(threadIdx.x+i);
  float x[NACC]; for (int i=0;i<NACC;i++) x[i]=seed+i;
  for (int it=0; it<ITERS; it++) {
    #pragma unroll
    for (int t=0;t<16;t++) {
      const float w = 0.5f + 0.03125f*t;
      #pragma unroll
      for (int i=0;i<NACC;i++) a[i]=fmaf(x[i], w, a[i]);
    }
  }
  float s=0; for (int i=0;i<NACC;i++) s+=a[i]; out[blockIdx.x*blockDim.x+threadIdx.x]=s;
}
// FIR-like: window values change every tap (a[i] += w[t]*x[i+t]) with param taps
__global__ void fir_param(float* out, Taps tp, float seed) {
  float x[NACC+16]; for (int i=0;i<NACC+16;i++) x[i]=seed+i*threadIdx.x;
  float a[NACC]; for (int i=0;i<NACC;i++) a[i]=0.f;
  for (int it=0; it<ITERS; it++) {
    #pragma unroll
    for (int t=0;t<16;t++) {
      #pragma unroll
      for (int i=0;i<NACC;i++) a[i]=fmaf(x[i+t], tp.w[t], a[i]);
    }
    #pragma unroll
    for (int i=0;i<NACC+16;i++) x[i]=x[i]*0.999f;   // keep it live
  }
  float s=0; for (int i=0;i<NACC;i++) s+=a[i]; out[blockIdx.x*blockDim.x+threadIdx.x]=s;
}
__device__ __forceinline__ unsigned long long pk(float lo, float hi){ unsigned long long r; asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(lo), "f"(hi)); return r; }
__device__ __forceinline__ void upk(unsigned long long v, float& lo, float& hi){ asm("mov.b64 {%0,%1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v)); }
__global__ void ffma2_param(float* out, Taps tp, float seed) {
  unsigned long long a[NACC/2], x[NACC/2];
  for (int i=0;i<NACC/2;i++){ a[i]=pk(seed*threadIdx.x, seed*i); x[i]=pk(seed+i, seed-i); }
  for (int it=0; it<ITERS; it++) {
    #pragma unroll
    for (int t=0;t<16;t++) {
      unsigned long long w2 = pk(tp.w[t], tp.w[t]);
      #pragma unroll
      for (int i=0;i<NACC/2;i++) asm volatile("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(a[i]) : "l"(x[i]), "l"(w2));
    }
  }
  float s=0; for (int i=0;i<NACC/2;i++){ float lo,hi; upk(a[i],lo,hi); s+=lo+hi; } out[blockIdx.x*blockDim.x+threadIdx.x]=s;
}
// grid barrier latency: sense-reversing barrier on a global counter
__device__ unsigned int g_count; __device__ volatile unsigned int g_gen;
__device__ __forceinline__ void grid_barrier(unsigned int nblocks) {
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned int gen = g_gen;
    __threadfence();
    unsigned int arrived = atomicAdd(&g_count, 1);
    if (arrived == nblocks - 1) { g_count = 0; __threadfence(); g_gen = gen + 1; }
    else { while (g_gen == gen) { } }
    __threadfence();
  }
  __syncthreads();
}
__global__ void barrier_bench(int n, long long* cycles) {
  long long t0 = clock64();
  for (int i=0;i<n;i++) grid_barrier(gridDim.x);
  if (blockIdx.x==0 && threadIdx.x==0) *cycles = clock64()-t0;
}
__global__ void coop_bench(int n) { auto g = cooperative_groups::this_grid(); for (int i=0;i<n;i++) g.sync(); }
__global__ void blockred_bench(int n, double* out) {
  __shared__ double s[32]; double v = threadIdx.x;
  for (int i=0;i<n;i++) {
    double r = v; for (int o=16;o>0;o>>=1) r += __shfl_xor_sync(0xffffffff, r, o);
    if ((threadIdx.x&31)==0) s[threadIdx.x>>5]=r; __syncthreads();
    if (threadIdx.x<32) { r = threadIdx.x < blockDim.x/32 ? s[threadIdx.x] : 0; for (int o=16;o>0;o>>=1) r += __shfl_xor_sync(0xffffffff, r, o); if(threadIdx.x==0) s[0]=r; }
    __syncthreads(); v = s[0]*1e-9 + threadIdx.x; __syncthreads();
  }
  if (threadIdx.x==0) out[blockIdx.x]=v;
}
__global__ void copy4(const float4* __restrict__ a, float4* __restrict__ b, size_t n) {
  for (size_t i = blockIdx.x*(size_t)blockDim.x+threadIdx.x; i<n; i += (size_t)gridDim.x*blockDim.x) b[i]=a[i];
}
__global__ void read4(const float4* __restrict__ a, size_t n, float* out) {
  float4 s = make_float4(0,0,0,0);
  for (size_t i = blockIdx.x*(size_t)blockDim.x+threadIdx.x; i<n; i += (size_t)gridDim.x*blockDim.x) { float4 v=a[i]; s.x+=v.x; s.y+=v.y; s.z+=v.z; s.w+=v.w; }
  if (s.x+s.y+s.z+s.w == 1234.5f) out[0]=s.x;
}
int main() {
  int dev=0; cudaDeviceProp pr; CK(cudaGetDeviceProperties(&pr, dev));
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  printf("device %s SMs %d L2 %d MB smemPerBlockOptin %zu clock %d kHz\n", pr.name, pr.multiProcessorCount, pr.l2CacheSize>>20, pr.sharedMemPerBlockOptin, clk);
  int S = pr.multiProcessorCount;
  float* out; CK(cudaMalloc(&out, 64<<20)); float* win; CK(cudaMalloc(&win, 1024)); CK(cudaMemset(win,0,1024));
  Taps tp; for (int i=0;i<32;i++) tp.w[i]=0.5f+0.01f*i;
  cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1); float ms;
  for (int bs : {256, 512}) for (int bps : {2, 4, 8}) {
    int grid = S*bps; if (bs*bps > 2048) continue;
    double fmas = (double)grid*bs*ITERS*16*NACC;
    for (int v=0; v<5; v++) {
      for (int rep=0; rep<2; rep++) {
        cudaEventRecord(e0);
        if (v==0) ffma_reg<<<grid,bs>>>(out, win, 1.0001f);
        if (v==1) ffma_param<<<grid,bs>>>(out, tp, 1.0001f);
        if (v==2) ffma_imm<<<grid,bs>>>(out, 1.0001f);
        if (v==3) fir_param<<<grid,bs>>>(out, tp, 1.0001f);
        if (v==4) ffma2_param<<<grid,bs>>>(out, tp, 1.0001f);
        cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms,e0,e1);
      }
      const char* nm[]={"ffma_reg","ffma_param","ffma_imm","fir_param","ffma2_param"};
      printf("%-12s bs=%d blk/SM=%d: %.3f ms  %.2f TFMA/s  (%.1f FMA/clk/SM @%d MHz)\n", nm[v], bs, bps, ms, fmas/ms/1e9, fmas/(ms*1e-3)/S/(clk*1e3), clk/1000);
    }
  }
  long long* cyc; CK(cudaMalloc(&cyc, 8));
  for (int bs : {128, 1024}) {
    int n=2000; void* args[]={&n,&cyc};
    for (int rep=0;rep<2;rep++){ cudaEventRecord(e0); CK(cudaLaunchCooperativeKernel((void*)barrier_bench, S, bs, args, 0, 0)); cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); }
    cudaEventElapsedTime(&ms,e0,e1); printf("custom grid barrier (grid=%d, bs=%d): %.3f us/barrier\n", S, bs, ms*1e3/n);
    void* args2[]={&n};
    for (int rep=0;rep<2;rep++){ cudaEventRecord(e0); CK(cudaLaunchCooperativeKernel((void*)coop_bench, S, bs, args2, 0, 0)); cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); }
    cudaEventElapsedTime(&ms,e0,e1); printf("cg grid.sync (grid=%d, bs=%d): %.3f us/sync\n", S, bs, ms*1e3/n);
  }
  double* dout; CK(cudaMalloc(&dout, 8*1024));
  for (int bs : {256, 1024}) { int n=20000; for(int rep=0;rep<2;rep++){ cudaEventRecord(e0); blockred_bench<<<S,bs>>>(n, dout); cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); } cudaEventElapsedTime(&ms,e0,e1); printf("block fp64 reduce+2 syncs (bs=%d): %.1f ns/iter\n", bs, ms*1e6/n); }
  // empty kernel launch latency
  for (int rep=0;rep<3;rep++){ cudaEventRecord(e0); for(int i=0;i<1000;i++) blockred_bench<<<1,32>>>(0,dout); cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); } cudaEventElapsedTime(&ms,e0,e1); printf("back-to-back tiny launches: %.2f us/launch\n", ms);
  size_t bytes = 2ull<<30; float4 *a,*b; CK(cudaMalloc(&a, bytes)); CK(cudaMalloc(&b, bytes)); CK(cudaMemset(a,0,bytes));
  size_t n4 = bytes/16;
  for (int rep=0;rep<3;rep++){ cudaEventRecord(e0); copy4<<<S*8,512>>>(a,b,n4); cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); }
  cudaEventElapsedTime(&ms,e0,e1); printf("copy 2 GiB float4: %.1f GB/s (r+w)\n", 2.0*bytes/ms/1e6);
  for (int rep=0;rep<3;rep++){ cudaEventRecord(e0); read4<<<S*8,512>>>(a,n4,out); cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); }
  cudaEventElapsedTime(&ms,e0,e1); printf("read 2 GiB float4: %.1f GB/s\n", 1.0*bytes/ms/1e6);
  size_t l2b = 48ull<<20; size_t l2n = l2b/16;
  for (int rep=0;rep<5;rep++){ cudaEventRecord(e0); for(int k=0;k<20;k++) read4<<<S*8,512>>>(a,l2n,out); cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); }
  cudaEventElapsedTime(&ms,e0,e1); printf("read 48 MiB x20 (L2-resident): %.1f GB/s\n", 20.0*l2b/ms/1e6);
  return 0;
}
