// Probe for a source-segmented pull of config 5's cold arcs: the cold
// source rows are cut into segments that fit the L2; one pass per segment walks that
// segment's arcs in ascending destination order, gathers the source row (an L2 hit) and
// read-modify-writes the destination's 16-byte row in a 4 GB array.  The destinations a
// pass touches are sparse (density 1/D) but ascending, so consecutive accesses share DRAM
// pages: does that lift the ~37 G/s random-access rate?
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/seg_probe tools/seg_probe.cu
//   /tmp/seg_probe
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t mix(uint64_t i) {
  i *= 0x9E3779B97F4A7C15ull;
  i ^= i >> 29;
  i *= 0xBF58476D1CE4E5B9ull;
  i ^= i >> 32;
  return (uint32_t)i;
}
// mode bit 0: gather a source row from the L2-resident segment; bit 1: write the
// destination back; bit 2: stream 8 bytes of ids per record.  One record per aligned
// group of D destinations (D a power of two), picked by a hash.  Thread t of the grid
// handles groups t, t + T, ... inside its CTA's contiguous slice of the groups.
template <int MODE>
__global__ void k_pass(uint4 *dst, const uint4 *__restrict__ seg, const uint2 *__restrict__ ids,
                       uint64_t groups, int lgD, uint64_t segmask, uint32_t seed) {
  const uint64_t per = (groups + gridDim.x - 1) / gridDim.x;
  const uint64_t g0 = blockIdx.x * per, g1 = min(groups, g0 + per);
  uint32_t acc = 0;
  for (uint64_t g = g0 + threadIdx.x; g < g1; g += blockDim.x) {
    const uint32_t h = mix(g ^ ((uint64_t)seed << 40));
    uint64_t d = (g << lgD) + (h & ((1u << lgD) - 1));
    uint4 v = make_uint4(h, h, h, h);
    if (MODE & 4) {
      const uint2 id = __ldcs(ids + g);
      v.x ^= id.x ^ id.y;
    }
    if (MODE & 1) {
      const uint4 s = __ldg(seg + (mix(g + seed) & segmask));
      v.x ^= s.x; v.y ^= s.y; v.z ^= s.z; v.w ^= s.w;
    }
    uint4 o;
    asm volatile("ld.global.L1::no_allocate.L2::64B.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(o.x), "=r"(o.y), "=r"(o.z), "=r"(o.w) : "l"(dst + d));
    uint4 m = make_uint4(__vmaxu4(o.x, v.x), __vmaxu4(o.y, v.y), __vmaxu4(o.z, v.z), __vmaxu4(o.w, v.w));
    if (MODE & 2) dst[d] = m;
    else acc ^= m.x ^ m.y ^ m.z ^ m.w;
  }
  if (!(MODE & 2) && acc == 0x1234567u) dst[0].x = acc;
}
// the wall to beat: random 16-byte reads of the 4 GB array
__global__ void k_random(const uint4 *__restrict__ src, uint4 *out, uint64_t n, uint64_t mask) {
  uint32_t acc = 0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    uint4 o;
    const uint64_t d = ((uint64_t)mix(i) << 4 ^ mix(i + n)) & mask;
    asm volatile("ld.global.L1::no_allocate.L2::64B.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(o.x), "=r"(o.y), "=r"(o.z), "=r"(o.w) : "l"(src + d));
    acc ^= o.x ^ o.y ^ o.z ^ o.w;
  }
  if (acc == 0x1234567u) out[0].x = acc;
}

int main() {
  const uint64_t big = 1ull << 28;   // 4 GB of 16-byte rows
  const uint64_t segrows = 1ull << 22;   // 64 MB segment
  uint4 *a, *s;
  uint2 *ids;
  if (cudaMalloc(&a, big * 16) != cudaSuccess || cudaMalloc(&s, segrows * 16) != cudaSuccess ||
      cudaMalloc(&ids, (big >> 2) * 8) != cudaSuccess) {
    printf("alloc failed\n");
    return 1;
  }
  cudaMemset(a, 1, big * 16);
  cudaMemset(s, 3, segrows * 16);
  cudaMemset(ids, 5, (big >> 2) * 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const int th = 256;
  {
    const uint64_t n = 1ull << 28;
    k_random<<<nsm * 8, th>>>(a, a, n, big - 1);
    cudaEventRecord(e0);
    k_random<<<nsm * 8, th>>>(a, a, n, big - 1);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("random 16-byte reads of 4 GB: %.2f ms for 2^28, %.1f G/s\n", ms, n / ms * 1e-6);
  }
  const int lgDs[] = {2, 3, 4, 5, 6};
  const int gridmul[] = {2, 8, 32};
  for (int gm = 0; gm < 3; gm++)
    for (int di = 0; di < 5; di++) {
      const int lgD = lgDs[di];
      const uint64_t groups = big >> lgD;
      const int passes = 1 << (lgD > 2 ? lgD - 2 : 0);   // 2^26 records per measurement
      const int grid = nsm * gridmul[gm];
      float t[6];
      for (int mode = 0; mode < 6; mode++) {
        float best = 1e30f;
        for (int rep = 0; rep < 2; rep++) {
          cudaEventRecord(e0);
          for (int p = 0; p < passes; p++) {
            const uint32_t seed = 17 * p + 3;
            switch (mode) {
              case 0: k_pass<0><<<grid, th>>>(a, s, ids, groups, lgD, segrows - 1, seed); break;
              case 1: k_pass<2><<<grid, th>>>(a, s, ids, groups, lgD, segrows - 1, seed); break;
              case 2: k_pass<3><<<grid, th>>>(a, s, ids, groups, lgD, segrows - 1, seed); break;
              case 3: k_pass<7><<<grid, th>>>(a, s, ids, groups, lgD, segrows - 1, seed); break;
              case 4: k_pass<5><<<grid, th>>>(a, s, ids, groups, lgD, segrows - 1, seed); break;
              case 5: k_pass<1><<<grid, th>>>(a, s, ids, groups, lgD, segrows - 1, seed); break;
            }
          }
          cudaEventRecord(e1);
          cudaEventSynchronize(e1);
          float ms;
          cudaEventElapsedTime(&ms, e0, e1);
          if (ms < best) best = ms;
        }
        t[mode] = best;
      }
      const double recs = (double)groups * passes;
      printf("grid %4d density 1/%-2d passes %2d: read %.1f  read+write %.1f  +L2 gather %.1f  "
             "+ids %.1f  | no write: gather+ids %.1f  gather %.1f  G records/s\n",
             grid, 1 << lgD, passes, recs / t[0] * 1e-6, recs / t[1] * 1e-6, recs / t[2] * 1e-6,
             recs / t[3] * 1e-6, recs / t[4] * 1e-6, recs / t[5] * 1e-6);
      if (cudaGetLastError() != cudaSuccess) { printf("launch error\n"); return 1; }
    }
  return 0;
}
