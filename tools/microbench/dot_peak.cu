// Dot-product-form FFMA throughput (residual kernel shape): per "row", a
// 64-term dot of a register window (dynamic offset via switch) with 64
// register-resident inputs.  Compares scalar FFMA chains vs FFMA2 pairs.
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
constexpr int R=64, D=8;
template<int CH>
__device__ __forceinline__ float dot_s(const float (&w)[R+D], const float (&u)[R], int o_static_base){
  float p[CH];
  #pragma unroll
  for(int c=0;c<CH;c++) p[c]=0.f;
  #pragma unroll
  for(int q=0;q<R;q++) p[q%CH] = fmaf(w[o_static_base+q], u[q], p[q%CH]);
  float s=0.f;
  #pragma unroll
  for(int c=0;c<CH;c++) s+=p[c];
  return s;
}
template<int CH>
__global__ void k_dot(float* out, const float* in, const int* offs, int rows){
  float w[R+D], u[R];
  #pragma unroll
  for(int k=0;k<R+D;k++) w[k]=in[(threadIdx.x+k)&1023];
  #pragma unroll
  for(int k=0;k<R;k++) u[k]=in[(threadIdx.x*3+k)&1023];
  float tot=0.f;
  for(int t=0;t<rows;t++){
    int o = offs[t&255];
    float s;
    switch(o){
      case 0: s=dot_s<CH>(w,u,0); break;
      case 1: s=dot_s<CH>(w,u,1); break;
      case 2: s=dot_s<CH>(w,u,2); break;
      case 3: s=dot_s<CH>(w,u,3); break;
      case 4: s=dot_s<CH>(w,u,4); break;
      case 5: s=dot_s<CH>(w,u,5); break;
      case 6: s=dot_s<CH>(w,u,6); break;
      default: s=dot_s<CH>(w,u,7); break;
    }
    tot += s;
    #pragma unroll
    for(int c=0;c<CH;c++) u[c] = u[c]*1.0000001f;
  }
  out[blockIdx.x*blockDim.x+threadIdx.x]=tot;
}
// FFMA2 pairs: (pe,po) += (w[k],w[k+1]) * (u[q],u[q+1]); two window copies (even/odd aligned)
template<int CH>
__device__ __forceinline__ float dot_p(const float2 (&we)[(R+D)/2], const float2 (&wo)[(R+D)/2], const float2 (&u)[R/2], int o){
  float2 p[CH];
  #pragma unroll
  for(int c=0;c<CH;c++) p[c]=make_float2(0.f,0.f);
  if ((o&1)==0){
    #pragma unroll
    for(int q=0;q<R/2;q++) p[q%CH] = ffma2(we[o/2+q], u[q], p[q%CH]);
  } else {
    #pragma unroll
    for(int q=0;q<R/2;q++) p[q%CH] = ffma2(wo[o/2+q], u[q], p[q%CH]);
  }
  float s=0.f;
  #pragma unroll
  for(int c=0;c<CH;c++) s+=p[c].x+p[c].y;
  return s;
}
template<int CH>
__global__ void k_dot2(float* out, const float* in, const int* offs, int rows){
  float2 we[(R+D)/2], wo[(R+D)/2], u[R/2];
  #pragma unroll
  for(int k=0;k<(R+D)/2;k++){ we[k]=make_float2(in[(threadIdx.x+2*k)&1023],in[(threadIdx.x+2*k+1)&1023]); wo[k]=make_float2(in[(threadIdx.x+2*k+1)&1023],in[(threadIdx.x+2*k+2)&1023]); }
  #pragma unroll
  for(int k=0;k<R/2;k++) u[k]=make_float2(in[(threadIdx.x*3+2*k)&1023],in[(threadIdx.x*3+2*k+1)&1023]);
  float tot=0.f;
  for(int t=0;t<rows;t++){
    int o = offs[t&255];
    float s;
    switch(o){
      case 0: s=dot_p<CH>(we,wo,u,0); break;
      case 1: s=dot_p<CH>(we,wo,u,1); break;
      case 2: s=dot_p<CH>(we,wo,u,2); break;
      case 3: s=dot_p<CH>(we,wo,u,3); break;
      case 4: s=dot_p<CH>(we,wo,u,4); break;
      case 5: s=dot_p<CH>(we,wo,u,5); break;
      case 6: s=dot_p<CH>(we,wo,u,6); break;
      default: s=dot_p<CH>(we,wo,u,7); break;
    }
    tot += s;
    #pragma unroll
    for(int c=0;c<CH;c++) u[c].x = u[c].x*1.0000001f;
  }
  out[blockIdx.x*blockDim.x+threadIdx.x]=tot;
}
template<typename K>
int run(const char* name, K kern, int blocks, int threads, int rows, double fma_per_row, float* d_out, float* d_in, int* d_offs){
  cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  kern<<<blocks,threads>>>(d_out,d_in,d_offs,rows/10); CK(cudaDeviceSynchronize());
  float best=1e30f;
  for(int rep=0;rep<5;rep++){
    cudaEventRecord(e0); kern<<<blocks,threads>>>(d_out,d_in,d_offs,rows); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms,e0,e1); if(ms<best) best=ms;
  }
  double fmas=(double)blocks*threads*rows*fma_per_row;
  printf("{\"variant\":\"%s\",\"blocks\":%d,\"threads\":%d,\"ms\":%.4f,\"tflops\":%.2f}\n",name,blocks,threads,best,2*fmas/(best*1e-3)/1e12);
  return 0;
}
int main(){
  float *d_out,*d_in; int* d_offs;
  CK(cudaMalloc(&d_out,148*16*256*4)); CK(cudaMalloc(&d_in,4096*4)); CK(cudaMalloc(&d_offs,256*4));
  float h[4096]; for(int i=0;i<4096;i++) h[i]=1e-3f*(i%97);
  int ho[256]; unsigned s=12345; for(int i=0;i<256;i++){ s=s*1664525u+1013904223u; ho[i]=(s>>16)&7; }
  cudaMemcpy(d_in,h,sizeof(h),cudaMemcpyHostToDevice); cudaMemcpy(d_offs,ho,sizeof(ho),cudaMemcpyHostToDevice);
  int sms=148;
  for(int occ: {2,4}){
    run("dot_ffma_4ch", k_dot<4>, sms*occ, 128, 20000, R, d_out,d_in,d_offs);
    run("dot_ffma_8ch", k_dot<8>, sms*occ, 128, 20000, R, d_out,d_in,d_offs);
    run("dot_ffma2_2ch", k_dot2<2>, sms*occ, 128, 20000, R, d_out,d_in,d_offs);
    run("dot_ffma2_4ch", k_dot2<4>, sms*occ, 128, 20000, R, d_out,d_in,d_offs);
  }
}
