// FP32 FFMA / FFMA2 throughput microbenchmark for sm_100a (B200).
// Measures the FP32 roofline denominator used by bench.py (MEASURED_PEAKS.json
// has no FP32 entry).  Each variant runs a full grid (k CTAs per SM) of
// independent accumulator chains; reports FMA/clk/SM and TFLOP/s (2 flop/FMA).
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s @%d\n",cudaGetErrorString(e),__LINE__); return 1;}}while(0)

__device__ __forceinline__ unsigned long long f2u(float2 v){ return *reinterpret_cast<unsigned long long*>(&v); }
__device__ __forceinline__ float2 u2f(unsigned long long v){ return *reinterpret_cast<float2*>(&v); }
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c){
  unsigned long long d;
  asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(f2u(a)), "l"(f2u(b)), "l"(f2u(c)));
  return u2f(d);
}

// (1) outer-product FFMA: acc[q] += w[q] * r ; r reused across 32 consecutive FFMAs
template<int R>
__global__ void k_outer(float* out, const float* in, int iters){
  float acc[R], w[R];
  #pragma unroll
  for(int q=0;q<R;q++){ acc[q]=0.f; w[q]=in[(threadIdx.x+q)&1023]; }
  float r = in[threadIdx.x & 511];
  for(int it=0; it<iters; ++it){
    #pragma unroll
    for(int q=0;q<R;q++) acc[q] = fmaf(w[q], r, acc[q]);
    r = r * 0.999f;            // 1 extra op per R FMAs
  }
  float s=0.f;
  #pragma unroll
  for(int q=0;q<R;q++) s+=acc[q];
  out[blockIdx.x*blockDim.x+threadIdx.x]=s;
}

// (2) FFMA2 outer product with scalar-broadcast b: acc2[q] += w2[q] * (r,r)
template<int R2>
__global__ void k_outer2(float* out, const float* in, int iters){
  float2 acc[R2], w[R2];
  #pragma unroll
  for(int q=0;q<R2;q++){ acc[q]=make_float2(0.f,0.f); w[q]=make_float2(in[(threadIdx.x+2*q)&1023], in[(threadIdx.x+2*q+1)&1023]); }
  float r = in[threadIdx.x & 511];
  for(int it=0; it<iters; ++it){
    float2 rb = make_float2(r,r);
    #pragma unroll
    for(int q=0;q<R2;q++) acc[q] = ffma2(w[q], rb, acc[q]);
    r = r * 0.999f;
  }
  float s=0.f;
  #pragma unroll
  for(int q=0;q<R2;q++) s+=acc[q].x+acc[q].y;
  out[blockIdx.x*blockDim.x+threadIdx.x]=s;
}

// (3) FFMA2 outer product + one LDS per 2 FFMA2 (is the spare issue slot free?)
template<int R2>
__global__ void k_outer2_lds(float* out, const float* in, int iters){
  __shared__ float sm[2048];
  for(int i=threadIdx.x;i<2048;i+=blockDim.x) sm[i]=in[i&1023];
  __syncthreads();
  float2 acc[R2], w[R2];
  #pragma unroll
  for(int q=0;q<R2;q++){ acc[q]=make_float2(0.f,0.f); w[q]=make_float2(in[(threadIdx.x+2*q)&1023], in[(threadIdx.x+2*q+1)&1023]); }
  int p = threadIdx.x & 31;
  for(int it=0; it<iters; ++it){
    #pragma unroll
    for(int q=0;q<R2;q++){
      float r = sm[(p + q*32) & 2047];
      acc[q] = ffma2(w[q], make_float2(r,r), acc[q]);
    }
    p = (p + 7) & 2047;
  }
  float s=0.f;
  #pragma unroll
  for(int q=0;q<R2;q++) s+=acc[q].x+acc[q].y;
  out[blockIdx.x*blockDim.x+threadIdx.x]=s;
}

// (4) FFMA no reuse: independent chains, all three operands distinct per instr
template<int R>
__global__ void k_noreuse(float* out, const float* in, int iters){
  float acc[R], a[R], b[R];
  #pragma unroll
  for(int q=0;q<R;q++){ acc[q]=0.f; a[q]=in[(threadIdx.x+q)&1023]; b[q]=in[(threadIdx.x+3*q)&1023]; }
  for(int it=0; it<iters; ++it){
    #pragma unroll
    for(int q=0;q<R;q++) acc[q] = fmaf(a[q], b[q], acc[q]);
    #pragma unroll
    for(int q=0;q<R;q++) a[q] = fmaf(b[(q+1)%R], acc[q], a[q]);   // keep it honest
  }
  float s=0.f;
  #pragma unroll
  for(int q=0;q<R;q++) s+=acc[q]+a[q];
  out[blockIdx.x*blockDim.x+threadIdx.x]=s;
}

template<typename K>
int run(const char* name, K kern, int blocks, int threads, int iters, double fma_per_thread_iter, float* d_out, float* d_in){
  cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  kern<<<blocks,threads>>>(d_out,d_in,iters/10); CK(cudaDeviceSynchronize());
  float best=1e30f;
  for(int rep=0;rep<5;rep++){
    cudaEventRecord(e0); kern<<<blocks,threads>>>(d_out,d_in,iters); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms,e0,e1); if(ms<best) best=ms;
  }
  double fmas = (double)blocks*threads*iters*fma_per_thread_iter;
  int dev; cudaGetDevice(&dev); int clk_khz; cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  double tflops = 2.0*fmas/(best*1e-3)/1e12;
  printf("{\"variant\":\"%s\",\"blocks\":%d,\"threads\":%d,\"ms\":%.4f,\"tflops\":%.2f,\"fma_per_clk_per_sm_at_maxclk\":%.1f}\n",
         name, blocks, threads, best, tflops, fmas/(best*1e-3)/(clk_khz*1e3)/sms);
  return 0;
}

int main(){
  float *d_out,*d_in; CK(cudaMalloc(&d_out, 148*8*1024*sizeof(float))); CK(cudaMalloc(&d_in, 4096*sizeof(float)));
  float h[4096]; for(int i=0;i<4096;i++) h[i]=1.0f+1e-4f*(i%97); CK(cudaMemcpy(d_in,h,sizeof(h),cudaMemcpyHostToDevice));
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("{\"sms\":%d,\"clock_khz\":%d,\"spec_fp32_tflops_at_max\":%.2f}\n", sms, clk, sms*128.0*2*clk*1e3/1e12);
  const int it=20000;
  for (int occ : {2,4,8}) {
    run("ffma_outer_R32",  k_outer<32>,   sms*occ, 256, it, 32, d_out, d_in);
    run("ffma2_outer_R16", k_outer2<16>,  sms*occ, 256, it, 32, d_out, d_in);
    run("ffma2_outer_lds", k_outer2_lds<16>, sms*occ, 256, it/2, 32, d_out, d_in);
    run("ffma_noreuse_R16", k_noreuse<16>, sms*occ, 256, it/2, 32, d_out, d_in);
  }
  return 0;
}
