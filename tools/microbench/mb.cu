// Appendix-C microbenchmarks: HBM copy, RED.F64 throughput, DFMA rate.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s @%d\n",cudaGetErrorString(e),__LINE__); return 1;}}while(0)

__global__ void copy2(const double2* __restrict__ a, double2* __restrict__ b, size_t n){
  size_t i = blockIdx.x*(size_t)blockDim.x + threadIdx.x, s = (size_t)gridDim.x*blockDim.x;
  for(; i<n; i+=s) b[i]=a[i];
}
__global__ void fill_idx(uint32_t* idx, size_t n, uint32_t mod, uint32_t mode){
  size_t i = blockIdx.x*(size_t)blockDim.x + threadIdx.x; if(i>=n) return;
  uint64_t z = i*0x9E3779B97F4A7C15ull; z=(z^(z>>30))*0xBF58476D1CE4E5B9ull; z=(z^(z>>27))*0x94D049BB133111EBull; z^=z>>31;
  if(mode==0) idx[i] = (uint32_t)(z % mod);                 // uniform random over mod
  else if(mode==1) idx[i] = (uint32_t)((i/16)*16/6 % mod + (z%64)); // local window (~Kuhn-like)
  else idx[i] = (uint32_t)(i % mod);                        // sequential
}
__global__ void red_f64(const uint32_t* __restrict__ idx, double* __restrict__ t, size_t n){
  size_t i = blockIdx.x*(size_t)blockDim.x + threadIdx.x, s=(size_t)gridDim.x*blockDim.x;
  for(; i<n; i+=s) atomicAdd(t+idx[i], 1.0);
}
__global__ void dfma(double* out, int iters){
  double a=threadIdx.x*1e-3, b=1.0000001, c=1e-9, d=a+1, e=a+2, f=a+3, g=a+4, h=a+5, k=a+6,l=a+7;
  for(int i=0;i<iters;i++){ a=fma(a,b,c); d=fma(d,b,c); e=fma(e,b,c); f=fma(f,b,c); g=fma(g,b,c); h=fma(h,b,c); k=fma(k,b,c); l=fma(l,b,c);}
  if(a+d+e+f+g+h+k+l==0.123) out[0]=a;
}
int main(){
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p,0));
  printf("{\"name\":\"%s\",\"sms\":%d,\"l2_bytes\":%d,\"smem_optin\":%zu,\"clock_khz\":%d}\n",p.name,p.multiProcessorCount,p.l2CacheSize,p.sharedMemPerBlockOptin,p.clockRate);
  cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1); float ms;
  size_t nbytes = 1ull<<30; double2 *a,*b; CK(cudaMalloc(&a,nbytes)); CK(cudaMalloc(&b,nbytes));
  cudaMemset(a,0,nbytes); cudaMemset(b,0,nbytes);
  size_t n2 = nbytes/16; float best=1e9;
  for(int r=0;r<10;r++){ cudaEventRecord(e0); copy2<<<148*8,512>>>(a,b,n2); cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms,e0,e1); if(ms<best)best=ms;}
  printf("{\"bench\":\"copy_double2\",\"GBps\":%.1f}\n", 2.0*nbytes/best/1e6);
  size_t nops = 1ull<<27; uint32_t* idx; CK(cudaMalloc(&idx,nops*4)); double* t; CK(cudaMalloc(&t, (1ull<<30)));
  uint32_t mods[3] = {1u<<22 /*32MB*/, 1u<<26 /*512MB*/, 1u<<27};
  for(int mode=0; mode<3; mode++) for(int mi=0; mi<2; mi++){
    fill_idx<<<(nops+255)/256,256>>>(idx,nops,mods[mi],mode); CK(cudaDeviceSynchronize());
    best=1e9;
    for(int r=0;r<5;r++){ cudaEventRecord(e0); red_f64<<<148*16,256>>>(idx,t,nops); cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms,e0,e1); if(ms<best)best=ms;}
    printf("{\"bench\":\"red_f64\",\"mode\":%d,\"target_MB\":%u,\"Gatomic_per_s\":%.1f}\n", mode, mods[mi]*8/1000000, nops/best/1e6);
  }
  CK(cudaGetLastError());
  int iters=1<<16; best=1e9;
  for(int r=0;r<3;r++){ cudaEventRecord(e0); dfma<<<148*8,256>>>(t,iters); cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms,e0,e1); if(ms<best)best=ms;}
  printf("{\"bench\":\"dfma\",\"TFLOPs\":%.2f}\n", 2.0*8*iters*148.0*8*256/best/1e9);
  CK(cudaDeviceSynchronize());
  return 0;
}
