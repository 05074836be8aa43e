// Probe for the propagation-blocking design of config 5's cold arcs: what do 16-byte
// record writes cost on B200 when they land (0) sequentially, (1) at random slots, (2) in
// bin-append order (records dealt to K bins of RB slots, each bin filled in order as the
// sweep advances -- the scatter phase's pattern), and (3) a random 16-byte gather (the
// pull's cold-row pattern) for comparison.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/pb_probe tools/pb_probe.cu
//   /tmp/pb_probe [log2 records (30)] [log2 bin size (12)]
// Run under ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t bij(uint64_t i, uint64_t mask) {
  // bijection on [0, mask] (power-of-two range): odd multiply + xorshift, twice
  i = (i * 0x9E3779B97F4A7C15ull) & mask;
  i ^= i >> 7;
  i = (i * 0xBF58476D1CE4E5B9ull) & mask;
  i ^= i >> 11;
  return i & mask;
}

__global__ void k_seq(const uint4 *__restrict__ src, uint4 *__restrict__ dst, uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
}
__global__ void k_scatter(const uint4 *__restrict__ src, uint4 *__restrict__ dst, uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    dst[bij(i, n - 1)] = src[i];
}
__global__ void k_binned(const uint4 *__restrict__ src, uint4 *__restrict__ dst, uint64_t n,
                         int log_rb) {
  const uint64_t K = n >> log_rb;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t r = i & (K - 1), q = i / K;
    dst[(bij(r, K - 1) << log_rb) + q] = src[i];
  }
}
__global__ void k_gather(const uint4 *__restrict__ src, uint4 *__restrict__ dst, uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    dst[i] = __ldg(src + bij(i, n - 1));
}

// random gather with different load flavours (mode: 0 ld.global.nc, 1 ld.global.cs,
// 2 ld.global.lu, 3 ld.global.cv, 4 ld.global.nc.L2::cache_hint evict_first,
// 5 ld.global.nc.L1::no_allocate.L2::64B (prefetch-size hint), 6 ld.volatile.global,
// 7 two 8-byte loads)
template <int MODE>
__device__ __forceinline__ uint4 ldm(const uint4 *p, uint64_t pol) {
  uint4 r;
  if (MODE == 0) asm volatile("ld.global.nc.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  if (MODE == 1) asm volatile("ld.global.cs.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  if (MODE == 2) asm volatile("ld.global.lu.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  if (MODE == 3) asm volatile("ld.global.cv.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  if (MODE == 4) asm volatile("ld.global.nc.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p), "l"(pol));
  if (MODE == 5) asm volatile("ld.global.nc.L1::no_allocate.L2::64B.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  if (MODE == 6) asm volatile("ld.global.nc.L2::64B.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  if (MODE == 7) asm volatile("ld.global.L2::64B.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  if (MODE == 8) asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  if (MODE == 9) asm volatile("ld.global.nc.L2::128B.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  if (MODE == 10) asm volatile("ld.global.nc.L2::cache_hint.L2::64B.v4.u32 {%0,%1,%2,%3}, [%4], %5;" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p), "l"(pol));
  if (MODE == 11) asm volatile("ld.global.L1::evict_first.L2::64B.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
template <int MODE>
__global__ void k_gather_m(const uint4 *__restrict__ src, uint4 *__restrict__ dst, uint64_t n) {
  uint64_t pol;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  uint32_t acc = 0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint4 r = ldm<MODE>(src + bij(i, n - 1), pol);
    acc ^= r.x ^ r.y ^ r.z ^ r.w;
  }
  if (acc == 0x1234567u) dst[0].x = acc;
}

int main(int argc, char **argv) {
  const int lg = argc > 1 ? atoi(argv[1]) : 30;
  const int lrb = argc > 2 ? atoi(argv[2]) : 12;
  const uint64_t n = 1ull << lg;
  uint4 *a, *b;
  if (cudaMalloc(&a, n * 16) != cudaSuccess || cudaMalloc(&b, n * 16) != cudaSuccess) {
    printf("alloc failed\n");
    return 1;
  }
  cudaMemset(a, 1, n * 16);
  cudaMemset(b, 0, n * 16);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int grid = 148 * 8, th = 256;
  const char *names[4] = {"seq", "scatter", "binned", "gather"};
  for (int mode = (argc > 3 ? 4 : 0); mode < 4; mode++) {
    for (int rep = 0; rep < 3; rep++) {
      cudaEventRecord(e0);
      if (mode == 0) k_seq<<<grid, th>>>(a, b, n);
      if (mode == 1) k_scatter<<<grid, th>>>(a, b, n);
      if (mode == 2) k_binned<<<grid, th>>>(a, b, n, lrb);
      if (mode == 3) k_gather<<<grid, th>>>(a, b, n);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (rep == 2)
        printf("%-8s records 2^%d (%.1f GB each way), bin 2^%d: %.3f ms, %.1f G records/s, "
               "%.0f GB/s (read+write)\n", names[mode], lg, n * 16 / 1e9, lrb, ms,
               n / (ms * 1e-3) / 1e9, 2.0 * n * 16 / (ms * 1e-3) / 1e9);
    }
  }
  for (int mode = 0; mode < 12; mode++) {
    if (mode >= 1 && mode <= 4) continue;
    for (int rep = 0; rep < 2; rep++) {
      cudaEventRecord(e0);
      switch (mode) {
        case 0: k_gather_m<0><<<grid, th>>>(a, b, n); break;
        case 1: k_gather_m<1><<<grid, th>>>(a, b, n); break;
        case 2: k_gather_m<2><<<grid, th>>>(a, b, n); break;
        case 3: k_gather_m<3><<<grid, th>>>(a, b, n); break;
        case 4: k_gather_m<4><<<grid, th>>>(a, b, n); break;
        case 5: k_gather_m<5><<<grid, th>>>(a, b, n); break;
        case 6: k_gather_m<6><<<grid, th>>>(a, b, n); break;
        case 7: k_gather_m<7><<<grid, th>>>(a, b, n); break;
        case 8: k_gather_m<8><<<grid, th>>>(a, b, n); break;
        case 9: k_gather_m<9><<<grid, th>>>(a, b, n); break;
        case 10: k_gather_m<10><<<grid, th>>>(a, b, n); break;
        case 11: k_gather_m<11><<<grid, th>>>(a, b, n); break;
      }
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (rep == 1)
        printf("gather-only mode %d: %.3f ms, %.1f G rows/s\n", mode, ms, n / (ms * 1e-3) / 1e9);
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
