// Probe: can a gather use the whole 126 MB L2 of a B200 if every SM only reads rows whose
// home L2 slice is on its own die?  (profiles/r1c_l2_gather_probe.md: a gather issued by
// every SM keeps a copy of far-die lines in the near die, so ~64 MB are usable.)
//  A. SM -> die and 2 KB chunk -> die from the latency of atomics (they execute at the
//     home slice: ~30 cycles more from the far die), min over repeats.
//  B. random 16-byte gathers over W MB: every SM anywhere vs. every SM on its own die's
//     chunks (rejection sampling on a shared-memory bitmap).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/die_probe tools/die_probe.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

constexpr int kMaxSm = 256;
__device__ __forceinline__ uint32_t smid() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t mix(uint64_t i) {
  i *= 0x9E3779B97F4A7C15ull;
  i ^= i >> 29;
  i *= 0xBF58476D1CE4E5B9ull;
  i ^= i >> 32;
  return (uint32_t)i;
}
__device__ __forceinline__ uint32_t timed_atomic(uint32_t *p, int reps) {
  __shared__ uint32_t sink_word[32];
  const uint32_t sink = (uint32_t)__cvta_generic_to_shared(sink_word + (threadIdx.x & 31));
  uint32_t best = 0xffffffffu;
  for (int r = 0; r < reps; r++) {
    long long t0, t1;
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(t0) :: "memory");
    const uint32_t v = atomicOr(p, 0u);
    asm volatile("st.volatile.shared.u32 [%0], %1;" :: "r"(sink), "r"(v) : "memory");
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(t1) :: "memory");
    const uint32_t d = (uint32_t)(t1 - t0);
    best = d < best ? d : best;
  }
  return best;
}
// A1: one CTA per SM (the first to claim it) times K test chunks (stride `stride` chunks).
__global__ void k_sm_probe(uint32_t *buf, int K, int64_t stride_words, int *claimed, uint32_t *lat) {
  __shared__ int mine;
  const uint32_t sm = smid();
  if (threadIdx.x == 0) mine = atomicCAS(claimed + sm, 0, 1) == 0;
  __syncthreads();
  if (!mine || threadIdx.x != 0) return;
  for (int k = 0; k < K; k++) lat[sm * K + k] = timed_atomic(buf + k * stride_words, 8);
}
// A2: chunk map.  sm_die[sm] in {0, 1}; CTAs of die d time every chunk (dealt by a per-die
// counter) -> lat2[d * chunks + c].
__global__ void k_chunk_probe(uint32_t *buf, int64_t chunks, const int *sm_die, unsigned int *next,
                              uint32_t *lat2) {
  const int d = sm_die[smid()];
  if (threadIdx.x != 0 || d < 0) return;
  for (;;) {
    const int64_t c0 = (int64_t)atomicAdd(next + d, 16u);
    if (c0 >= chunks) break;
    for (int64_t c = c0; c < c0 + 16 && c < chunks; c++)
      lat2[d * chunks + c] = timed_atomic(buf + c * 512 + 8 * (c & 31), 4);
  }
}
// B: random 16-byte gathers over rows [0, rows); mode 1: only rows on the SM's own die.
__global__ void k_gather(const uint4 *__restrict__ src, uint64_t rows, const uint32_t *__restrict__ home_bits,
                         int64_t chunks, const int *sm_die, int mode, int per_thread, uint32_t *out) {
  extern __shared__ uint32_t bm[];
  for (int64_t i = threadIdx.x; i < (chunks + 31) / 32; i += blockDim.x) bm[i] = home_bits[i];
  __syncthreads();
  const uint32_t d = (uint32_t)sm_die[smid()];
  uint64_t ctr = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) * 977;
  uint32_t acc = 0;
  for (int i = 0; i < per_thread; i += 8) {
    uint64_t r[8];
#pragma unroll
    for (int u = 0; u < 8; u++) {
      for (int tries = 0;; tries++) {
        const uint64_t h = __umulhi(mix(ctr), (uint32_t)rows);
        ctr++;
        const uint64_t c = h >> 7;
        if (!mode || d > 1u || tries > 64 || ((bm[c >> 5] >> (c & 31)) & 1u) == d) { r[u] = h; break; }
      }
    }
    uint4 v[8];
#pragma unroll
    for (int u = 0; u < 8; u++)
      asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                   : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w) : "l"(src + r[u]));
#pragma unroll
    for (int u = 0; u < 8; u++) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
  }
  if (acc == 0x1234567u) out[0] = acc;
}

// B2: the real access pattern -- stream 4-byte ids, gather 16-byte rows.  ids[d] holds
// random rows of die d's chunks (d = 2: any chunk); a CTA reads slice blockIdx.x of the
// list of its SM's die (mode 1) or of list 2 (mode 0).
__global__ void k_make_ids(uint32_t *ids, uint64_t n, uint64_t rows, const uint32_t *__restrict__ home_bits) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < 3 * n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t d = (uint32_t)(i / n);
    uint64_t ctr = i * 64;
    uint32_t h;
    for (int tries = 0;; tries++) {
      h = __umulhi(mix(ctr++), (uint32_t)rows);
      const uint32_t c = h >> 7;
      if (d > 1u || tries > 60 || ((home_bits[c >> 5] >> (c & 31)) & 1u) == d) break;
    }
    ids[i] = h;
  }
}
__global__ void __launch_bounds__(256, 4) k_gather_ids(const uint4 *__restrict__ src, const uint32_t *__restrict__ ids, uint64_t n,
                             const int *sm_die, int mode, uint32_t *out) {
  const uint32_t d = mode ? (uint32_t)sm_die[smid()] : 2u;
  const uint64_t per = n / gridDim.x;
  const uint32_t *my = ids + (d > 2u ? 2u : d) * n + blockIdx.x * per;
  uint32_t acc = 0;
  for (uint64_t i = threadIdx.x; i + 7 * 256 < per; i += 8 * 256) {
    uint32_t r[8];
#pragma unroll
    for (int u = 0; u < 8; u++) r[u] = __ldcs(my + i + u * 256);
    uint4 v[8];
#pragma unroll
    for (int u = 0; u < 8; u++)
      asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                   : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w) : "l"(src + r[u]));
#pragma unroll
    for (int u = 0; u < 8; u++) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
  }
  if (acc == 0x1234567u) out[0] = acc;
}

int main() {
  setvbuf(stdout, nullptr, _IONBF, 0);
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const size_t bytes = 256ull << 20;
  const int64_t chunks = bytes >> 11;
  uint32_t *buf, *lat, *lat2, *home_bits, *out;
  int *claimed, *sm_die;
  unsigned int *next;
  cudaMalloc(&buf, bytes);
  cudaMemset(buf, 1, bytes);
  const int K = 256;
  cudaMalloc(&lat, kMaxSm * K * 4);
  cudaMemset(lat, 0, kMaxSm * K * 4);
  cudaMalloc(&claimed, kMaxSm * 4);
  cudaMemset(claimed, 0, kMaxSm * 4);
  cudaMalloc(&sm_die, kMaxSm * 4);
  cudaMalloc(&lat2, 2 * chunks * 4);
  cudaMalloc(&home_bits, (chunks + 31) / 32 * 4);
  cudaMalloc(&next, 8);
  cudaMalloc(&out, 64);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  // A1
  cudaEventRecord(e0);
  k_sm_probe<<<nsm * 16, 32>>>(buf, K, (64 << 10) / 4 + 512 + 8, claimed, lat);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float msA1;
  cudaEventElapsedTime(&msA1, e0, e1);
  std::vector<uint32_t> hl(kMaxSm * K);
  std::vector<int> hc(kMaxSm);
  cudaMemcpy(hl.data(), lat, hl.size() * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(hc.data(), claimed, kMaxSm * 4, cudaMemcpyDeviceToHost);
  int ref = -1;
  for (int s = 0; s < kMaxSm; s++) if (hc[s]) { ref = s; break; }
  std::vector<int> die(kMaxSm, -1);
  int cnt[2] = {0, 0};
  double min_abs = 1e9;
  for (int s = 0; s < kMaxSm; s++) {
    if (!hc[s]) continue;
    double ma = 0, mb = 0;
    for (int k = 0; k < K; k++) { ma += hl[ref * K + k]; mb += hl[s * K + k]; }
    ma /= K; mb /= K;
    double cov = 0, va = 0, vb = 0;
    for (int k = 0; k < K; k++) {
      const double a = hl[ref * K + k] - ma, b = hl[s * K + k] - mb;
      cov += a * b; va += a * a; vb += b * b;
    }
    const double corr = cov / std::sqrt(va * vb + 1e-9);
    die[s] = corr > 0 ? 0 : 1;
    cnt[die[s]]++;
    min_abs = std::min(min_abs, std::fabs(corr));
  }
  {
    std::vector<uint32_t> v(hl.begin() + ref * K, hl.begin() + ref * K + K);
    std::sort(v.begin(), v.end());
    printf("A1 %.2f ms: SM %d latencies min %u p25 %u median %u p75 %u max %u; dies %d / %d SMs, min |corr| %.2f\n",
           msA1, ref, v[0], v[K / 4], v[K / 2], v[3 * K / 4], v[K - 1], cnt[0], cnt[1], min_abs);
  }
  cudaMemcpy(sm_die, die.data(), kMaxSm * 4, cudaMemcpyHostToDevice);
  // A2
  cudaMemset(next, 0, 8);
  cudaEventRecord(e0);
  k_chunk_probe<<<nsm * 4, 32>>>(buf, chunks, sm_die, next, lat2);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float msA2;
  cudaEventElapsedTime(&msA2, e0, e1);
  std::vector<uint32_t> h2(2 * chunks);
  cudaMemcpy(h2.data(), lat2, h2.size() * 4, cudaMemcpyDeviceToHost);
  std::vector<uint32_t> bits((chunks + 31) / 32, 0);
  int64_t ones = 0, weak = 0;
  double gap = 0;
  for (int64_t c = 0; c < chunks; c++) {
    const int d0 = (int)h2[c], d1 = (int)h2[chunks + c];
    if (d1 < d0) { bits[c >> 5] |= 1u << (c & 31); ones++; }
    if (std::abs(d0 - d1) < 10) weak++;
    gap += std::abs(d0 - d1);
  }
  printf("A2 %.2f ms: %lld chunks, %.1f%% on die 1, mean |gap| %.1f cycles, %lld with |gap| < 10\n", msA2,
         (long long)chunks, 100.0 * ones / chunks, gap / chunks, (long long)weak);
  int runs = 0;   // run-length of home die over consecutive chunks
  for (int64_t c = 1; c < chunks; c++) runs += ((bits[c >> 5] >> (c & 31)) & 1) != ((bits[(c - 1) >> 5] >> ((c - 1) & 31)) & 1);
  printf("   die changes between consecutive 2 KB chunks: %d of %lld\n", runs, (long long)chunks - 1);
  cudaMemcpy(home_bits, bits.data(), bits.size() * 4, cudaMemcpyHostToDevice);
  // B
  const int mbs[] = {32, 48, 64, 80, 96, 112, 128, 160, 192, 256};
  const size_t smem = (chunks + 31) / 32 * 4;
  cudaFuncSetAttribute(k_gather, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  for (int mi = 0; mi < 10; mi++) {
    const uint64_t rows = ((uint64_t)mbs[mi] << 20) / 16;
    const int64_t ch = rows >> 7;
    float t[2];
    for (int mode = 0; mode < 2; mode++) {
      float best = 1e30f;
      for (int rep = 0; rep < 3; rep++) {
        cudaEventRecord(e0);
        k_gather<<<nsm * 4, 256, smem>>>((const uint4 *)buf, rows, home_bits, ch, sm_die, mode, 2048, out);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (rep > 0 && ms < best) best = ms;
      }
      t[mode] = best;
    }
    const double n = (double)nsm * 4 * 256 * 2048;
    printf("W %3d MB: any die %.1f G rows/s, own die %.1f G rows/s\n", mbs[mi], n / t[0] * 1e-6, n / t[1] * 1e-6);
  }
  {
    const uint64_t n = 1ull << 27;
    uint32_t *ids;
    if (cudaMalloc(&ids, 3 * n * 4) != cudaSuccess) { printf("ids alloc failed\n"); return 1; }
    for (int mi = 0; mi < 10; mi++) {
      const uint64_t rows = ((uint64_t)mbs[mi] << 20) / 16;
      k_make_ids<<<nsm * 8, 256>>>(ids, n, rows, home_bits);
      float t[2];
      for (int mode = 0; mode < 2; mode++) {
        float best = 1e30f;
        for (int rep = 0; rep < 3; rep++) {
          cudaEventRecord(e0);
          k_gather_ids<<<nsm * 4, 256>>>((const uint4 *)buf, ids, n, sm_die, mode, out);
          cudaEventRecord(e1);
          cudaEventSynchronize(e1);
          float ms;
          cudaEventElapsedTime(&ms, e0, e1);
          if (rep > 0 && ms < best) best = ms;
        }
        t[mode] = best;
      }
      printf("streamed ids, W %3d MB: any die %.1f G rows/s, own die %.1f G rows/s\n", mbs[mi], n / t[0] * 1e-6, n / t[1] * 1e-6);
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
