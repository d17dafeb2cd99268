// Probe: global atomic / scatter throughput for random cell ids (N1 design).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t hash(uint64_t x){x+=0x9E3779B97F4A7C15ull;x=(x^(x>>30))*0xBF58476D1CE4E5B9ull;x=(x^(x>>27))*0x94D049BB133111EBull;return (uint32_t)(x^(x>>31));}
__global__ void gen(uint32_t* cell, int64_t n, uint32_t ncell, int sorted){int64_t i=blockIdx.x*(int64_t)blockDim.x+threadIdx.x; for(;i<n;i+=(int64_t)gridDim.x*blockDim.x) cell[i]= sorted? (uint32_t)(i*ncell/n) : hash(i)%ncell;}
__global__ void red(const uint32_t* __restrict__ cell, int64_t n, uint32_t* cnt){int64_t i=blockIdx.x*(int64_t)blockDim.x+threadIdx.x; for(;i<n;i+=(int64_t)gridDim.x*blockDim.x) atomicAdd(cnt+cell[i],1u);}
__global__ void atom(const uint32_t* __restrict__ cell, int64_t n, uint32_t* cur, uint32_t* out){int64_t i=blockIdx.x*(int64_t)blockDim.x+threadIdx.x; for(;i<n;i+=(int64_t)gridDim.x*blockDim.x){uint32_t c=cell[i]; uint32_t s=atomicAdd(cur+c,1u); out[s]=(uint32_t)i;}}
__global__ void atom4(const uint32_t* __restrict__ cell, int64_t n, uint32_t* cur, uint32_t* out){
  int64_t i=(blockIdx.x*(int64_t)blockDim.x+threadIdx.x)*4; int64_t st=(int64_t)gridDim.x*blockDim.x*4;
  for(;i<n;i+=st){uint4 c=*(const uint4*)(cell+i); uint32_t s0=atomicAdd(cur+c.x,1u),s1=atomicAdd(cur+c.y,1u),s2=atomicAdd(cur+c.z,1u),s3=atomicAdd(cur+c.w,1u); out[s0]=i;out[s1]=i+1;out[s2]=i+2;out[s3]=i+3;}}
__global__ void copyk(const uint32_t* __restrict__ a, int64_t n, uint32_t* b){int64_t i=blockIdx.x*(int64_t)blockDim.x+threadIdx.x; for(;i<n;i+=(int64_t)gridDim.x*blockDim.x) b[i]=a[i]+1;}
__global__ void init_cur(uint32_t* cur, uint32_t ncell, int64_t n){uint32_t c=blockIdx.x*blockDim.x+threadIdx.x; if(c<ncell) cur[c]=(uint32_t)((int64_t)c*n/ncell);}
int main(){
  int64_t n=500000000; uint32_t ncell=262144;
  uint32_t *cell,*cnt,*out; cudaMalloc(&cell,n*4); cudaMalloc(&out,n*4); cudaMalloc(&cnt,ncell*4);
  cudaEvent_t a,b; cudaEventCreate(&a); cudaEventCreate(&b); float ms;
  int G=148*8, B=256;
  for(int sorted=0;sorted<2;sorted++){
    gen<<<G,B>>>(cell,n,ncell,sorted); cudaDeviceSynchronize();
    for(int rep=0;rep<2;rep++){
    cudaMemset(cnt,0,ncell*4);
    cudaEventRecord(a); red<<<G,B>>>(cell,n,cnt); cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms,a,b);
    printf("sorted=%d RED      %.3f ms  %.1f Gop/s\n",sorted,ms,n/ms/1e6);
    init_cur<<<(ncell+255)/256,256>>>(cnt,ncell,n);
    cudaEventRecord(a); atom<<<G,B>>>(cell,n,cnt,out); cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms,a,b);
    printf("sorted=%d ATOM+st  %.3f ms  %.1f Gop/s\n",sorted,ms,n/ms/1e6);
    init_cur<<<(ncell+255)/256,256>>>(cnt,ncell,n);
    cudaEventRecord(a); atom4<<<G,B>>>(cell,n,cnt,out); cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms,a,b);
    printf("sorted=%d ATOM4+st %.3f ms  %.1f Gop/s\n",sorted,ms,n/ms/1e6);
    cudaEventRecord(a); copyk<<<G,B>>>(cell,n,out); cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms,a,b);
    printf("copy u32 %.3f ms  %.1f GB/s\n",ms,n*8/ms/1e6);
    }
  }
  printf("err=%s\n",cudaGetErrorString(cudaGetLastError()));
}
