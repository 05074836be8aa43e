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
  for (int mode = 0; mode < 4; mode++) {
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
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
