// Clean dot-form vs outer-form FFMA throughput (no loop-carried latency chains).
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned long long f2u(float2 v){ return *reinterpret_cast<unsigned long long*>(&v); }
__device__ __forceinline__ float2 u2f(unsigned long long v){ return *reinterpret_cast<float2*>(&v); }
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c){
  unsigned long long d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(f2u(a)), "l"(f2u(b)), "l"(f2u(c)));
  return u2f(d);
}
constexpr int R=32, W=64;
template<int S, int CH> __device__ __forceinline__ float dot_s(const float (&w)[W], const float (&x)[R]){
  float p[CH];
  #pragma unroll
  for(int c=0;c<CH;c++) p[c]=0.f;
  #pragma unroll
  for(int q=0;q<R;q++) p[q%CH]=fmaf(w[S+q],x[q],p[q%CH]);
  float s=0; 
  #pragma unroll
  for(int c=0;c<CH;c++) s+=p[c];
  return s;
}
template<int S, int CH> __device__ __forceinline__ float dot_p(const float2 (&w)[W/2], const float2 (&x)[R/2]){
  float2 p[CH];
  #pragma unroll
  for(int c=0;c<CH;c++) p[c]=make_float2(0.f,0.f);
  #pragma unroll
  for(int q=0;q<R/2;q++) p[q%CH]=ffma2(w[S+q],x[q],p[q%CH]);
  float s=0;
  #pragma unroll
  for(int c=0;c<CH;c++) s+=p[c].x+p[c].y;
  return s;
}
template<int CH> __global__ void k_dot(float* out, const float* in, int iters){
  float w[W], x[R];
  #pragma unroll
  for(int k=0;k<W;k++) w[k]=in[(threadIdx.x+k)&1023];
  #pragma unroll
  for(int k=0;k<R;k++) x[k]=in[(threadIdx.x*3+k)&1023];
  float tot=0;
  for(int it=0;it<iters;it++){
    tot += dot_s<0,CH>(w,x); tot += dot_s<3,CH>(w,x); tot += dot_s<5,CH>(w,x); tot += dot_s<8,CH>(w,x);
    tot += dot_s<13,CH>(w,x); tot += dot_s<17,CH>(w,x); tot += dot_s<22,CH>(w,x); tot += dot_s<30,CH>(w,x);
    #pragma unroll
    for(int k=0;k<4;k++) x[k]*=1.0000001f;
  }
  out[blockIdx.x*blockDim.x+threadIdx.x]=tot;
}
template<int CH> __global__ void k_dot2(float* out, const float* in, int iters){
  float2 w[W/2], x[R/2];
  #pragma unroll
  for(int k=0;k<W/2;k++) w[k]=make_float2(in[(threadIdx.x+2*k)&1023],in[(threadIdx.x+2*k+1)&1023]);
  #pragma unroll
  for(int k=0;k<R/2;k++) x[k]=make_float2(in[(threadIdx.x*3+2*k)&1023],in[(threadIdx.x*3+2*k+1)&1023]);
  float tot=0;
  for(int it=0;it<iters;it++){
    tot += dot_p<0,CH>(w,x); tot += dot_p<2,CH>(w,x); tot += dot_p<3,CH>(w,x); tot += dot_p<5,CH>(w,x);
    tot += dot_p<7,CH>(w,x); tot += dot_p<9,CH>(w,x); tot += dot_p<11,CH>(w,x); tot += dot_p<15,CH>(w,x);
    #pragma unroll
    for(int k=0;k<2;k++) x[k].x*=1.0000001f;
  }
  out[blockIdx.x*blockDim.x+threadIdx.x]=tot;
}
__global__ void k_outer(float* out, const float* in, int iters){
  float w[W], acc[R];
  #pragma unroll
  for(int k=0;k<W;k++) w[k]=in[(threadIdx.x+k)&1023];
  #pragma unroll
  for(int q=0;q<R;q++) acc[q]=0;
  float r=in[threadIdx.x&511];
  for(int it=0;it<iters;it++){
    #pragma unroll
    for(int s=0;s<8;s++){
      #pragma unroll
      for(int q=0;q<R;q++) acc[q]=fmaf(w[q+3*s],r,acc[q]);
      r*=0.9999f;
    }
  }
  float t=0;
  #pragma unroll
  for(int q=0;q<R;q++) t+=acc[q];
  out[blockIdx.x*blockDim.x+threadIdx.x]=t;
}
template<typename K> void run(const char* name, K k, int blocks, int threads, int iters, float* o, float* in){
  cudaEvent_t a,b; cudaEventCreate(&a); cudaEventCreate(&b);
  k<<<blocks,threads>>>(o,in,10); cudaDeviceSynchronize();
  float best=1e9;
  for(int r=0;r<5;r++){ cudaEventRecord(a); k<<<blocks,threads>>>(o,in,iters); cudaEventRecord(b); cudaEventSynchronize(b); float ms; cudaEventElapsedTime(&ms,a,b); if(ms<best) best=ms; }
  double fma=(double)blocks*threads*iters*8*32;
  printf("%-16s blocks %5d thr %d  %.2f TFLOP/s\n", name, blocks, threads, 2*fma/(best*1e-3)/1e12);
}
int main(){
  float *o,*in; cudaMalloc(&o,148*16*256*4); cudaMalloc(&in,4096*4);
  float h[4096]; for(int i=0;i<4096;i++) h[i]=1e-3f*(i%97); cudaMemcpy(in,h,sizeof(h),cudaMemcpyHostToDevice);
  for(int occ: {4,8}){
    run("outer", k_outer, 148*occ, 128, 4000, o, in);
    run("dot_ffma_4ch", k_dot<4>, 148*occ, 128, 4000, o, in);
    run("dot_ffma_8ch", k_dot<8>, 148*occ, 128, 4000, o, in);
    run("dot_ffma2_2ch", k_dot2<2>, 148*occ, 128, 4000, o, in);
    run("dot_ffma2_4ch", k_dot2<4>, 148*occ, 128, 4000, o, in);
  }
}
