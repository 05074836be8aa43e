// Probe of the B200 memory system under random 16-byte row gathers (the p = 16 union's
// access pattern): every thread loads rows at hashed positions inside a working set of W MB.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o l2_gather_probe tools/l2_gather_probe.cu
//   ./l2_gather_probe <mode 0: ld.global.nc, 1: + L2::evict_last policy> [fetch-granularity limit]
// Run under `ncu --metrics dram__bytes_read.sum,lts__t_sectors_srcunit_tex_op_read.sum,...`
// for the per-row DRAM bytes and the L2 hit rate (profiles/r1c_l2_gather_probe.md).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint64_t mix(uint64_t z){z=(z^(z>>30))*0xBF58476D1CE4E5B9ull;z=(z^(z>>27))*0x94D049BB133111EBull;return z^(z>>31);}
__device__ __forceinline__ uint4 ldp(const uint4*p,uint64_t pol,int mode){uint4 r;
 if(mode==1) asm volatile("ld.global.nc.L2::cache_hint.v4.u32 {%0,%1,%2,%3},[%4],%5;":"=r"(r.x),"=r"(r.y),"=r"(r.z),"=r"(r.w):"l"(p),"l"(pol));
 else asm volatile("ld.global.nc.v4.u32 {%0,%1,%2,%3},[%4];":"=r"(r.x),"=r"(r.y),"=r"(r.z),"=r"(r.w):"l"(p));
 return r;}
__global__ void k(const uint4* a, uint64_t rows, int64_t iters, uint32_t* out, int mode, uint64_t salt){
  uint64_t pol; asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;":"=l"(pol));
  uint64_t t=blockIdx.x*(uint64_t)blockDim.x+threadIdx.x; uint32_t acc=0;
  for(int64_t i=0;i<iters;i+=8){ uint4 r[8];
#pragma unroll
    for(int u=0;u<8;u++){ uint64_t h=mix(t*1000003ull+i+u+salt); r[u]=ldp(a+(h%rows),pol,mode);}
#pragma unroll
    for(int u=0;u<8;u++) acc^=r[u].x^r[u].w;}
  if(acc==0x12345678) out[0]=acc;}
int main(int argc,char**argv){
  size_t tot=(size_t)1<<30; uint4* a; cudaMalloc(&a,tot); cudaMemset(a,1,tot); uint32_t*o; cudaMalloc(&o,4);
  int mode=argc>1?atoi(argv[1]):0;
  if(argc>2){ cudaError_t e=cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity,(size_t)atoi(argv[2])); printf("setlimit %s\n",cudaGetErrorString(e));}
  { size_t v=0; cudaError_t e=cudaDeviceGetLimit(&v,cudaLimitMaxL2FetchGranularity); printf("fetch granularity limit %zu (%s)\n",v,cudaGetErrorString(e)); }
  int blocks=148*8, th=256; int64_t iters=512; 
  cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int ws[]={8,16,24,32,48,64,80,96,112,128,160,256,1024};
  for(int w: ws){ uint64_t rows=((uint64_t)w<<20)/16;
    k<<<blocks,th>>>(a,rows,iters,o,mode,1); cudaDeviceSynchronize();
    cudaEventRecord(e0); for(int r=0;r<3;r++) k<<<blocks,th>>>(a,rows,iters,o,mode,r+7); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms,e0,e1); double loads=3.0*blocks*th*iters;
    printf("mode %d W %5d MB: %.3f ms/launch, %.2f G rows/s\n",mode,w,ms/3,loads/(ms*1e-3)/1e9);}
  return 0;}
