// Probe for a push formulation of config 5's cold arcs: what does a 16-byte vector
// reduction (red.global.max.noftz.v4.bf16x2 -> REDG.E.MAX.BF16x8: 8 u16 lanes, each a
// byte-max carrier) cost on B200 against a random 16-byte load,
// when the target region is L2-resident (16-96 MB) or not (4 GB)?
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/red_probe tools/red_probe.cu
//   /tmp/red_probe [log2 ops (30)]
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t bij(uint64_t i, uint64_t mask) {
  i = (i * 0x9E3779B97F4A7C15ull) & mask;
  i ^= i >> 7;
  i = (i * 0xBF58476D1CE4E5B9ull) & mask;
  i ^= i >> 11;
  return i & mask;
}
__device__ __forceinline__ void red_max8(uint4 *p, uint4 v) {
  asm volatile("red.global.max.noftz.v4.bf16x2 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v.x),
               "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}
// n ops; op i reads src[i] (sequential stream) and hits dst[bij(i) & region_mask]
__global__ void k_red(const uint4 *__restrict__ src, uint4 *dst, uint64_t n, uint64_t rmask) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    uint4 v = __ldg(src + (i & ((1ull << 26) - 1)));
    red_max8(dst + (bij(i, n - 1) & rmask), v);
  }
}
// same, two reds per op (a 16-byte row pushed as its raw and its shifted-by-8 words)
__global__ void k_red2(const uint4 *__restrict__ src, uint4 *dst, uint64_t n, uint64_t rmask) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    uint4 v = __ldg(src + (i & ((1ull << 26) - 1)));
    uint4 *q = dst + 2 * (bij(i, n - 1) & rmask);
    red_max8(q, v);
    red_max8(q + 1, make_uint4(v.x << 8, v.y << 8, v.z << 8, v.w << 8));
  }
}
__global__ void k_gather(const uint4 *__restrict__ src, uint4 *__restrict__ out, uint64_t n,
                         uint64_t rmask) {
  uint32_t acc = 0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    uint4 r = __ldg(src + (bij(i, n - 1) & rmask));
    acc ^= r.x ^ r.y ^ r.z ^ r.w;
  }
  if (acc == 0x1234567u) out[0].x = acc;
}

int main(int argc, char **argv) {
  const int lg = argc > 1 ? atoi(argv[1]) : 30;
  const uint64_t n = 1ull << lg;
  const uint64_t big = 1ull << 28;              // 4 GB of 16-byte rows
  uint4 *a, *b, *s;
  if (cudaMalloc(&a, big * 16) != cudaSuccess || cudaMalloc(&b, 2 * big * 16) != cudaSuccess ||
      cudaMalloc(&s, (1ull << 26) * 16) != cudaSuccess) {
    printf("alloc failed\n");
    return 1;
  }
  cudaMemset(a, 1, big * 16);
  cudaMemset(b, 0, 2 * big * 16);
  cudaMemset(s, 3, (1ull << 26) * 16);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const int grid = nsm * 8, th = 256;
  const int lregion[] = {20, 21, 22, 23, 28};   // rows: 16 MB, 32 MB, 64 MB, 128 MB, 4 GB
  for (int kind = 0; kind < 3; kind++) {
    for (int ri = 0; ri < 5; ri++) {
      const uint64_t rmask = (1ull << lregion[ri]) - 1;
      float best = 1e30f;
      for (int rep = 0; rep < 3; rep++) {
        cudaEventRecord(e0);
        if (kind == 0) k_gather<<<grid, th>>>(a, b, n, rmask);
        if (kind == 1) k_red<<<grid, th>>>(s, b, n, rmask);
        if (kind == 2) k_red2<<<grid, th>>>(s, b, n, rmask);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        best = ms < best ? ms : best;
      }
      const char *nm[3] = {"gather16", "red16", "red16x2"};
      printf("%-8s region %6.0f MB (x%d): %8.3f ms  %6.1f G ops/s\n", nm[kind],
             (double)((rmask + 1) * 16) / 1e6, kind == 2 ? 2 : 1, best,
             n / (best * 1e-3) / 1e9);
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
