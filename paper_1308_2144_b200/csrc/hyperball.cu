// hyperball.cu -- sm_100a kernels of the HyperBall hot path and their C-ABI
// (include/hyperball_b200.h).
//
// Reference algorithm: /root/reference/pkg/src/hyperball/_kernels.py:15-114 (estimate,
// scatter_max, hll_union_range), hll.py:70-158 (hash, register values),
// centrality.py:132-150 (accumulate).  DESIGN.md explains the data layout, the work
// decomposition and the roofline of each kernel.
//
// Bit-exactness rules:
//   * sum_j 2^-M[j] is computed as the exact integer sum_j 2^(31-M[j]) times 2^-31 when
//     every register is <= 31 (always true at register_width 5); otherwise by the
//     reference's own ascending-j fp64 sum.  Both equal the reference's sequential sum.
//   * the linear-counting value comes from a host-built table (math.log).
//   * the accumulate uses explicitly rounded fp64 ops (__dmul_rn/__ddiv_rn/__dadd_rn);
//     the translation unit is also built with -fmad=false.
//   * registers are < 128 (rho_max = 65 - b <= 61), so the 7-bit-safe SIMD byte max below
//     is exact.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <type_traits>
#include <algorithm>
#include <cmath>
#include <vector>
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_segmented_sort.cuh>
#include <cub/device/device_select.cuh>
#include <cub/iterator/transform_input_iterator.cuh>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include "../../include/hyperball_b200.h"

#define HB_MIN_B 4
#define HB_MAX_B 12

namespace {

thread_local char g_err[512] = "";

int set_err(const char *what, cudaError_t e) {
  snprintf(g_err, sizeof(g_err), "%s: %s", what, cudaGetErrorString(e));
  return (int)e;
}
int set_err_msg(const char *msg) {
  snprintf(g_err, sizeof(g_err), "%s", msg);
  return -1;
}
int check_launch(const char *what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_err(what, e);
  return 0;
}

// ------------------------------------------------------------------ checked build
// HB_CHECKED=1 (make checked -> libhyperball_b200_checked.so) compiles bounds checks into
// the union kernels: every successor id, CSR position, row index, shared-memory slot and
// work-item index is tested against the sizes of the step (set per call), and a violation
// prints the site and traps.  compute-sanitizer is not available on the GPU pool, so this
// build -- run over tools/sanitize_workload.py -- is the out-of-bounds evidence
// (profiles/r2_checked_build.md).
struct CheckDims {
  int64_t rows;    // register rows addressable (cur / nxt)
  int64_t m;       // successor ids in succ
  int64_t items;   // heavy work items (partial rows)
};
#ifdef HB_CHECKED
__device__ CheckDims g_chk;
#define HB_CHK(cond, what)                                                                   \
  do {                                                                                      \
    if (g_chk.rows > 0 && !(cond)) {                                                        \
      printf("HB_CHECKED violation: %s (%s:%d) block %d thread %d\n", what, __FILE__,       \
             __LINE__, (int)blockIdx.x, (int)threadIdx.x);                                  \
      __trap();                                                                             \
    }                                                                                       \
  } while (0)
#else
#define HB_CHK(cond, what) do { } while (0)
#endif
int set_check_dims(int64_t rows, int64_t m, int64_t items, cudaStream_t s) {
#ifdef HB_CHECKED
  const CheckDims d{rows, m, items};
  cudaError_t e = cudaMemcpyToSymbolAsync(g_chk, &d, sizeof(d), 0, cudaMemcpyHostToDevice, s);
  if (e != cudaSuccess) return set_err("checked build: dims", e);
#else
  (void)rows; (void)m; (void)items; (void)s;
#endif
  return 0;
}

// ------------------------------------------------------------------ row geometry
template <int LOGP>
struct Geo {
  static constexpr int P = 1 << LOGP;
  static constexpr int CH = P / 16;               // 16-byte chunks per row
  // lanes cooperating on one row: one 16-byte chunk per lane for p <= 32, two above
  // (p = 64 / 128 / 256 -> 2 / 4 / 8 lanes: more nodes per warp round amortise the
  // per-round work; measured on configs 2-4), at most 32
#ifndef HB_G_P64
#define HB_G_P64 2
#endif
#ifndef HB_G_P128
#define HB_G_P128 4
#endif
#ifndef HB_G_P256
#define HB_G_P256 8
#endif
  static constexpr int G = LOGP == 6 ? HB_G_P64 : (LOGP == 7 ? HB_G_P128 : (LOGP == 8 ? HB_G_P256 :
                           (CH <= 2 ? CH : (CH / 2 < 32 ? CH / 2 : 32))));
  static constexpr int CPL = CH / G;              // chunks per lane
  static constexpr int NPW = 32 / G;              // rows handled side by side per warp
};

// Work-item size for heavy nodes: 16 row loads per lane (16 * NPW arcs), at least 64.
template <int LOGP>
constexpr int64_t item_arcs_t() {
  return 16 * Geo<LOGP>::NPW > 64 ? 16 * Geo<LOGP>::NPW : 64;
}
int64_t item_arcs_for(int b) {
  switch (b) {
    case 4: return item_arcs_t<4>();   case 5: return item_arcs_t<5>();
    case 6: return item_arcs_t<6>();   case 7: return item_arcs_t<7>();
    case 8: return item_arcs_t<8>();   case 9: return item_arcs_t<9>();
    case 10: return item_arcs_t<10>(); case 11: return item_arcs_t<11>();
    case 12: return item_arcs_t<12>();
  }
  return 64;
}
constexpr int64_t kLightMaxDeg = 64;

// ------------------------------------------------------------------ small helpers
__device__ __forceinline__ uint32_t prmt_sign(uint32_t d) {
  uint32_t m;
  // byte i of m = 0xFF if bit 7 of byte i of d is set, else 0x00 (prmt sign-replicate)
  asm("prmt.b32 %0, %1, 0, 0xba98;" : "=r"(m) : "r"(d));
  return m;
}
// Per-byte unsigned max of a and b, exact when every byte is < 128.
__device__ __forceinline__ uint32_t bmax(uint32_t a, uint32_t b) {
  uint32_t d = (a | 0x80808080u) - b;  // bit 7 of byte i set  <=>  a_i >= b_i
  uint32_t m = prmt_sign(d);
  return (a & m) | (b & ~m);
}
__device__ __forceinline__ uint4 bmax4(uint4 a, uint4 b) {
  return make_uint4(bmax(a.x, b.x), bmax(a.y, b.y), bmax(a.z, b.z), bmax(a.w, b.w));
}
template <int U, int CPL>
__device__ __forceinline__ void tree_merge(uint4 (&acc)[CPL], uint4 (&r)[U][CPL]) {
#pragma unroll
  for (int span = 1; span < U; span <<= 1)
#pragma unroll
    for (int u = 0; u + span < U; u += 2 * span)
#pragma unroll
      for (int c = 0; c < CPL; c++) r[u][c] = bmax4(r[u][c], r[u + span][c]);
#pragma unroll
  for (int c = 0; c < CPL; c++) acc[c] = bmax4(acc[c], r[0][c]);
}

// Per-byte max accumulator on the 16x2 integer max unit (VIMNMX.U16x2, one ALU-pipe op).
// The max of two u16 lanes always carries the larger high byte, whatever the low bytes,
// so `hi` accumulates the raw words (odd bytes valid) and `lo` the words shifted up by 8
// (even bytes valid; the shift is an IMAD on the FMA pipe).  3 instructions per merged word
// with 2 on the ALU pipe, against 4 (3 ALU) for bmax; exact for any byte values.
__device__ __forceinline__ uint32_t vmax16(uint32_t a, uint32_t b) {
  uint32_t r;
  asm("max.u16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
  return r;
}
template <int CPL>
struct MaxAcc {
  uint4 hi[CPL], lo[CPL];
  __device__ __forceinline__ void init() {
#pragma unroll
    for (int c = 0; c < CPL; c++) hi[c] = lo[c] = make_uint4(0, 0, 0, 0);
  }
  __device__ __forceinline__ void add(int c, uint4 r) {
    hi[c].x = vmax16(hi[c].x, r.x); lo[c].x = vmax16(lo[c].x, r.x << 8);
    hi[c].y = vmax16(hi[c].y, r.y); lo[c].y = vmax16(lo[c].y, r.y << 8);
    hi[c].z = vmax16(hi[c].z, r.z); lo[c].z = vmax16(lo[c].z, r.z << 8);
    hi[c].w = vmax16(hi[c].w, r.w); lo[c].w = vmax16(lo[c].w, r.w << 8);
  }
  // two rows at once: ptxas fuses max(acc, max(a, b)) into one 3-input VIMNMX3.U16x2
  __device__ __forceinline__ void add2(int c, uint4 a, uint4 b) {
    hi[c].x = vmax16(hi[c].x, vmax16(a.x, b.x)); lo[c].x = vmax16(lo[c].x, vmax16(a.x << 8, b.x << 8));
    hi[c].y = vmax16(hi[c].y, vmax16(a.y, b.y)); lo[c].y = vmax16(lo[c].y, vmax16(a.y << 8, b.y << 8));
    hi[c].z = vmax16(hi[c].z, vmax16(a.z, b.z)); lo[c].z = vmax16(lo[c].z, vmax16(a.z << 8, b.z << 8));
    hi[c].w = vmax16(hi[c].w, vmax16(a.w, b.w)); lo[c].w = vmax16(lo[c].w, vmax16(a.w << 8, b.w << 8));
  }
  // byte 2k+1 from hi, byte 2k from lo's byte 2k+1
  __device__ __forceinline__ static uint32_t join(uint32_t h, uint32_t l) {
    uint32_t r;
    asm("prmt.b32 %0, %1, %2, 0x3715;" : "=r"(r) : "r"(h), "r"(l));
    return r;
  }
  __device__ __forceinline__ uint4 get(int c) const {
    return make_uint4(join(hi[c].x, lo[c].x), join(hi[c].y, lo[c].y),
                      join(hi[c].z, lo[c].z), join(hi[c].w, lo[c].w));
  }
};
// The SWAR alternative with the same interface (one register set, 4 ops per word).
template <int CPL>
struct BmaxAcc {
  uint4 a[CPL];
  __device__ __forceinline__ void init() {
#pragma unroll
    for (int c = 0; c < CPL; c++) a[c] = make_uint4(0, 0, 0, 0);
  }
  __device__ __forceinline__ void add(int c, uint4 r) { a[c] = bmax4(a[c], r); }
  __device__ __forceinline__ void add2(int c, uint4 x, uint4 y) { add(c, x); add(c, y); }
  __device__ __forceinline__ uint4 get(int c) const { return a[c]; }
};
// VIMNMX accumulation from p = 128 up (ALU-bound loops); below, the loops are latency-bound
// and the second register set costs more than the saved ALU ops (measured, configs 3, 5s).
// Padded (unconditional) loads from p = 64 up; at p = 16 / 32 the extra L1 wavefronts of
// padded slots cost more than the predicates.
#ifndef HB_VMAX_MIN_LOGP
#define HB_VMAX_MIN_LOGP 7
#endif
#ifndef HB_PAD_MIN_LOGP
#define HB_PAD_MIN_LOGP 6
#endif
template <int LOGP>
using RowAcc = typename std::conditional<(LOGP >= HB_VMAX_MIN_LOGP), MaxAcc<Geo<LOGP>::CPL>,
                                         BmaxAcc<Geo<LOGP>::CPL>>::type;

// Source-row chunk load with 32-bit index arithmetic (one IMAD + one IMAD.WIDE.U32 per
// address): rows * chunks-per-row < 2^32 for every array the C-ABI accepts.
__device__ __forceinline__ uint4 ld_chunk(const uint4 *__restrict__ cur4, int32_t w, uint32_t ch,
                                          uint32_t k) {
  return __ldg(cur4 + ((uint32_t)w * ch + k));
}
// Small rows (p <= 2^HB_L2_64B_MAX_LOGP bytes): the L2 fetches 64 bytes instead of its
// default 128 on a miss (`.L2::64B`, SASS LDG...LTC64B).  A random 16-byte row that misses
// L2 otherwise pulls a whole 128-byte line from HBM (profiles/r1c_l2_gather_probe.md);
// tools/pb_probe.cu measured 68.6 instead of 136.8 GB of DRAM reads for 2^30 random
// 16-byte rows, same time; config 5 32.85 -> 32.4 ms, p = 64 (config 3) slightly slower.
#ifndef HB_L2_64B_MAX_LOGP
#define HB_L2_64B_MAX_LOGP 5
#endif
__device__ __forceinline__ uint4 ld_nc_64b(const uint4 *p) {
  uint4 r;
  asm("ld.global.nc.L2::64B.v4.u32 {%0, %1, %2, %3}, [%4];"
      : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
template <int LOGP>
__device__ __forceinline__ uint4 ld_row_chunk(const uint4 *__restrict__ cur4, int32_t w,
                                              uint32_t ch, uint32_t k) {
  if constexpr (LOGP <= HB_L2_64B_MAX_LOGP) return ld_nc_64b(cur4 + ((uint32_t)w * ch + k));
  else return ld_chunk(cur4, w, ch, k);
}

// L2 eviction priorities for the DRAM-bound small-p kernels (p <= 32, degree order): one
// uniform range policy over cur -- rows in the hot head (the most-read rows, first
// hb_union_step hot_lim rows) evict_last, the rest evict_first, so the random cold
// gather stops pushing the hot rows out of L2.  Config 5: 35.9 -> 34.0 ms per dense step
// at a 64 MB head (16-192 MB swept; HB_HINT_MB).  A per-lane choice between two policies
// costs more than it saves (the policy lives in the load's uniform descriptor).
#ifndef HB_HINT_MAX_LOGP
#define HB_HINT_MAX_LOGP 5
#endif
__device__ __forceinline__ uint4 ld_pol(const uint4 *p, uint64_t pol) {
  uint4 r;
  asm("ld.global.nc.L2::cache_hint.v4.u32 {%0, %1, %2, %3}, [%4], %5;"
      : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
      : "l"(p), "l"(pol));
  return r;
}
// [base, base + hot) evict_last, [base + hot, base + total) evict_first.
__device__ __forceinline__ uint64_t range_policy(const void *base, uint32_t hot, uint32_t total) {
  uint64_t pol;
  asm("createpolicy.range.global.L2::evict_last.L2::evict_first.b64 %0, [%1], %2, %3;"
      : "=l"(pol) : "l"(base), "r"(hot), "r"(total));
  return pol;
}
__device__ __forceinline__ uint4 ld_chunk_hint(const uint4 *__restrict__ cur4, int32_t w,
                                               uint32_t ch, uint32_t k, uint64_t pol) {
  return ld_pol(cur4 + ((uint32_t)w * ch + k), pol);
}
__device__ __forceinline__ uint4 ld_pol_64b(const uint4 *p, uint64_t pol) {
  uint4 r;
  asm("ld.global.nc.L2::cache_hint.L2::64B.v4.u32 {%0, %1, %2, %3}, [%4], %5;"
      : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
      : "l"(p), "l"(pol));
  return r;
}
// Same without L1 allocation, for register arrays far larger than L2 (config 5): a random
// row fetched into L1 is rarely read again by the same SM before the misses behind it
// evict it, and the hubs it would displace stay in L2 anyway (config 5: 30.6 -> 30.0 ms;
// config 5s, a 268 MB array, loses with it: 1.57 -> 1.75 ms -- hence the size switch).
__device__ __forceinline__ uint4 ld_pol_64b_na(const uint4 *p, uint64_t pol) {
  uint4 r;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.L2::64B.v4.u32 {%0, %1, %2, %3}, [%4], %5;"
      : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
      : "l"(p), "l"(pol));
  return r;
}
#ifndef HB_L1NA_MIN_MB
#define HB_L1NA_MIN_MB 1024            // register arrays from this size gather without L1
#endif
template <int LOGP, bool L1NA = false>
__device__ __forceinline__ uint4 ld_row_chunk_hint(const uint4 *__restrict__ cur4, int32_t w,
                                                   uint32_t ch, uint32_t k, uint64_t pol) {
  if constexpr (LOGP <= HB_L2_64B_MAX_LOGP) {
    if constexpr (L1NA) return ld_pol_64b_na(cur4 + ((uint32_t)w * ch + k), pol);
    return ld_pol_64b(cur4 + ((uint32_t)w * ch + k), pol);
  }
  else return ld_chunk_hint(cur4, w, ch, k, pol);
}

__device__ __forceinline__ uint4 ldg4(const uint8_t *p) {
  return __ldg(reinterpret_cast<const uint4 *>(p));
}
// Streamed CSR ids: read once per step, never reused -- keep them out of L1 and first in
// line for L2 eviction so they do not push hot register rows out.
__device__ __forceinline__ uint64_t evict_first_policy() {
  uint64_t pol;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ int32_t ld_stream_id(const int32_t *p) {
  int32_t v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.s32 %0, [%1], %2;"
               : "=r"(v) : "l"(p), "l"(evict_first_policy()));
  return v;
}
__device__ __forceinline__ int4 ld_stream_ids4(const int4 *p) {
  int4 v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.s32 {%0, %1, %2, %3}, [%4], %5;"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p), "l"(evict_first_policy()));
  return v;
}
__device__ __forceinline__ bool test_bit(const uint32_t *bm, int64_t v) {
  return (__ldg(bm + (v >> 5)) >> (v & 31)) & 1u;
}
__device__ __forceinline__ uint4 shfl_xor4(uint4 a, int off) {
  a.x = __shfl_xor_sync(0xffffffffu, a.x, off);
  a.y = __shfl_xor_sync(0xffffffffu, a.y, off);
  a.z = __shfl_xor_sync(0xffffffffu, a.z, off);
  a.w = __shfl_xor_sync(0xffffffffu, a.w, off);
  return a;
}
__device__ __forceinline__ bool neq4(uint4 a, uint4 b) {
  return ((a.x ^ b.x) | (a.y ^ b.y) | (a.z ^ b.z) | (a.w ^ b.w)) != 0u;
}
__device__ __forceinline__ bool nz4(uint4 a) { return (a.x | a.y | a.z | a.w) != 0u; }

// splitmix64 finaliser (hll.py:70-76)
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
// hll.py:79-88
__device__ __forceinline__ uint64_t hash_item(uint64_t item, uint64_t replica, uint64_t seed) {
  uint64_t key = mix64(replica + mix64(seed));
  return mix64(item + key);
}
// 2^-r as an exact double (POW2NEG, hll.py:33), r <= 255
__device__ __forceinline__ double pow2neg(uint32_t r) {
  return __hiloint2double((int)((1023u - r) << 20), 0);
}

// Per-word contribution to the exact register sum: sum over bytes of 2^(31-M) (M <= 31),
// zero count, running max.
__device__ __forceinline__ void acc_word(uint32_t w, uint64_t &S, int &zeros, uint32_t &mx) {
#pragma unroll
  for (int i = 0; i < 4; i++) {
    uint32_t m = (w >> (8 * i)) & 0xffu;
    zeros += (m == 0u);
    mx = m > mx ? m : mx;
    S += (m <= 31u) ? (uint64_t)(1u << (31u - m)) : 0ull;
  }
}

// Fused discounted-gain sums (centrality.py:26-101,149-150): up to kMaxDisc arrays
// disc[k * disc_stride + v] += (bit k of disc_div) ? delta / t : disc_scale[k] * delta.
constexpr int kMaxDisc = 8;

struct EstConst {
  double alpha_p2, lc_cut;
  const double *lc;  // lc_table[0..p]
  double *disc;      // [n_disc, disc_stride] or nullptr
  int64_t disc_stride;
  int n_disc, disc_div;
  double disc_scale[kMaxDisc];
};

// Raw estimate from the (exact) register sum, with the linear-counting switch
// (_kernels.py:31-33).
__device__ __forceinline__ double finish_estimate(double s, int zeros, const EstConst &ec) {
  double e = __ddiv_rn(ec.alpha_p2, s);
  if (e <= ec.lc_cut && zeros > 0) e = __ldg(ec.lc + zeros);
  return e;
}

// Whole-row estimate by one thread (seed / estimate_rows kernels).
template <int P>
__device__ double estimate_row_thread(const uint8_t *row, const EstConst &ec) {
  uint64_t S = 0;
  int zeros = 0;
  uint32_t mx = 0;
  for (int c = 0; c < P / 16; c++) {
    uint4 q = *reinterpret_cast<const uint4 *>(row + 16 * c);
    acc_word(q.x, S, zeros, mx);
    acc_word(q.y, S, zeros, mx);
    acc_word(q.z, S, zeros, mx);
    acc_word(q.w, S, zeros, mx);
  }
  double s;
  if (mx <= 31u) {
    s = (double)S * 0x1p-31;
  } else {  // reference order: ascending-j fp64 sum (_kernels.py:25-30)
    s = 0.0;
    for (int j = 0; j < P; j++) s = __dadd_rn(s, pow2neg(row[j]));
  }
  return finish_estimate(s, zeros, ec);
}

// Fused push (multi-GPU): every row a rank writes into its own nxt
// buffer (the lazy-write set chg_prev | chg_now) is also stored straight into the nxt
// replica of every peer over NVLink, and its change bit OR-ed into every peer's chg_now,
// so no separate all-gather runs after the union.  Pointers are peer device addresses
// (symmetric-memory / IPC mappings); n == 0 disables.
constexpr int kMaxPeers = 7;
struct Peers {
  int n;
  int pstride;   // 0: rows go unpacked into the peers' nxt; > 0: 5-bit packed into their
                 // inbox (nxt[q] = the inbox of this step), this many bytes per row
  uint8_t *nxt[kMaxPeers];
  uint32_t *chg[kMaxPeers];
};

// Packed push rows (register_width <= 5, every register < 32): each 16-register chunk ci
// of a row travels as 80 bits -- its low 64 at byte 8 ci (two 32-bit words), its high 16
// at byte 8 (p = 16, 12-byte stride) or 8 CH + 2 ci (p >= 32, 10 CH-byte stride).
__host__ __device__ constexpr int push_stride(int ch) { return ch == 1 ? 12 : 10 * ch; }
__host__ __device__ constexpr int push_hi_off(int ch, int ci) { return ch == 1 ? 8 : 8 * ch + 2 * ci; }
// 4 registers (bytes < 32) -> 20 bits, and back
__device__ __forceinline__ uint32_t gather5(uint32_t w) {
  return (w & 0x1Fu) | ((w >> 3) & 0x3E0u) | ((w >> 6) & 0x7C00u) | ((w >> 9) & 0xF8000u);
}
__device__ __forceinline__ uint32_t spread5(uint32_t x) {
  const uint32_t e = (x & 0x7C1Fu) * 0x41u;      // fields 0, 2 -> bytes 0, 2
  const uint32_t o = (x & 0xF83E0u) * 0x208u;    // fields 1, 3 -> bytes 1, 3
  return (e & 0x001F001Fu) | (o & 0x1F001F00u);
}
__device__ __forceinline__ void pack_chunk5(uint4 q, uint32_t &l0, uint32_t &l1, uint32_t &h) {
  const uint32_t g0 = gather5(q.x), g1 = gather5(q.y), g2 = gather5(q.z), g3 = gather5(q.w);
  l0 = g0 | (g1 << 20);
  l1 = (g1 >> 12) | (g2 << 8) | (g3 << 28);
  h = g3 >> 4;
}
__device__ __forceinline__ uint4 unpack_chunk5(uint32_t l0, uint32_t l1, uint32_t h) {
  return make_uint4(spread5(l0), spread5(__funnelshift_r(l0, l1, 20)), spread5(l1 >> 8),
                    spread5(__funnelshift_r(l1, h, 28)));
}

// numpy.maximum(x, 0.0) (centrality.py:134)
__device__ __forceinline__ double np_max0(double x) { return (x >= 0.0 || x != x) ? x : 0.0; }

// ------------------------------------------------------------------ shared epilogue
// Scalar tail of the epilogue for one changed node (one lane): the estimate from the
// register sum s (or, when some register is > 31, the reference's ascending-j fp64 sum
// over the stored row), then the accumulate (centrality.py:132-150).
template <int P>
__device__ __forceinline__ void node_scalar(int64_t v, double s, uint32_t zeros, bool seq,
                                            const uint8_t *nrow, double *__restrict__ est,
                                            double *__restrict__ sum_dist,
                                            double *__restrict__ sum_recip, const EstConst &ec,
                                            double tf, const double *pre_vals) {
  if (seq) {  // reference order: ascending-j fp64 sum (_kernels.py:25-30)
    s = 0.0;
    for (int j = 0; j < P; j++) s = __dadd_rn(s, pow2neg(nrow[j]));
  }
  const double e = finish_estimate(s, (int)zeros, ec);
  const double old = pre_vals ? pre_vals[0] : est[v];
  est[v] = e;
  const double d = np_max0(__dsub_rn(e, old));
  if (sum_dist)
    sum_dist[v] = __dadd_rn(pre_vals ? pre_vals[1] : sum_dist[v], __dmul_rn(tf, d));
  if (sum_recip)
    sum_recip[v] = __dadd_rn(pre_vals ? pre_vals[2] : sum_recip[v], __ddiv_rn(d, tf));
  // Runtime-indexed on purpose: ec.disc_scale[k] makes ptxas keep the estimator
  // constants in a (L1-resident) local copy instead of registers, which the load
  // pipeline of the union loops needs more (measured: a statically unrolled loop or a
  // __constant__ copy costs 8-9% on config 4).
  for (int k = 0; k < ec.n_disc; k++) {
    double *q = ec.disc + k * ec.disc_stride + v;
    const double c = ((ec.disc_div >> k) & 1) ? __ddiv_rn(d, tf) : __dmul_rn(ec.disc_scale[k], d);
    *q = __dadd_rn(*q, c);
  }
}

// Group of G lanes finishing node v, vector part: merge own row, change test, lazy write
// (+ push); then, when any group of the warp changed, the group's register sum s (all
// lanes of the group), zero count and the > 31 flag.  acc holds the max over merged
// sources.  Warp-uniform: EVERY lane of the warp calls it (groups with nothing to do pass
// doit = false), so all collectives use the full mask and no group's divergence
// serialises the others.  Returns the group's changed flag; *any_changed = the warp's.
template <int LOGP, bool PUSH>
__device__ __forceinline__ bool finish_rows(const Peers &peers, bool doit, int64_t v,
                                            const uint4 (&acc)[Geo<LOGP>::CPL],
                                            const uint4 (&pre)[Geo<LOGP>::CPL], bool have_pre,
                                            bool self_chg, int grp, int gl,
                                            const uint8_t *__restrict__ cur,
                                            uint8_t *__restrict__ nxt, bool &any_changed,
                                            double &s, uint32_t &zeros, bool &seq) {
  using Gm = Geo<LOGP>;
  constexpr unsigned kLow = Gm::G == 32 ? 0xffffffffu : ((1u << (Gm::G & 31)) - 1u);
  const uint8_t *crow = cur + (size_t)v * Gm::P;
  uint8_t *nrow = nxt + (size_t)v * Gm::P;
  uint4 nw[Gm::CPL];
  bool diff = false;
#pragma unroll
  for (int c = 0; c < Gm::CPL; c++) {
    uint4 self = pre[c];
    if (doit && !have_pre) self = ldg4(crow + 16 * (c * Gm::G + gl));
    nw[c] = bmax4(acc[c], self);
    diff |= neq4(nw[c], self);
  }
  const unsigned bal = __ballot_sync(0xffffffffu, doit && diff);
  const bool changed = ((bal >> (grp * Gm::G)) & kLow) != 0u;
  if (doit && (changed || self_chg)) {
#pragma unroll
    for (int c = 0; c < Gm::CPL; c++)
      *reinterpret_cast<uint4 *>(nrow + 16 * (c * Gm::G + gl)) = nw[c];
    if constexpr (PUSH) {
      if (peers.pstride == 0) {
        for (int q = 0; q < peers.n; q++) {
          uint8_t *prow = peers.nxt[q] + (size_t)v * Gm::P;
#pragma unroll
          for (int c = 0; c < Gm::CPL; c++)
            *reinterpret_cast<uint4 *>(prow + 16 * (c * Gm::G + gl)) = nw[c];
        }
      } else if (changed) {   // 5-bit packed into the peers' inboxes, changed rows only:
                              // a receiver refreshes the lazy-only rows from its own cur
#pragma unroll
        for (int c = 0; c < Gm::CPL; c++) {
          const int ci = c * Gm::G + gl;
          uint32_t l0, l1, h;
          pack_chunk5(nw[c], l0, l1, h);
          for (int q = 0; q < peers.n; q++) {
            uint8_t *prow = peers.nxt[q] + (size_t)v * push_stride(Gm::CH);
            *reinterpret_cast<uint32_t *>(prow + 8 * ci) = l0;
            *reinterpret_cast<uint32_t *>(prow + 8 * ci + 4) = l1;
            *reinterpret_cast<uint16_t *>(prow + push_hi_off(Gm::CH, ci)) = (uint16_t)h;
          }
        }
      }
    }
  }
  any_changed = bal != 0u;
  s = 0.0;
  zeros = 0;
  seq = false;
  if (bal == 0u) return changed;   // warp-uniform
  {
    // sum_j 2^-M[j] as exact fp64 partial sums (every M <= 31 here: at most 36 significant
    // bits, so any summation order gives the reference's sequential result), zero count by
    // SWAR, and an OR of all bytes to detect registers > 31 (sequential fallback).
    // Integer form: 2^(31-M) for every byte by one wrapping funnel shift of 2^31 (the
    // shift count's low 5 bits are M whenever M <= 31; larger registers take the
    // sequential path below), summed in 64 bits (< 2^37), scaled once: exact.
    uint64_t S = 0;
    uint32_t big = 0;
#pragma unroll
    for (int c = 0; c < Gm::CPL; c++) {
      const uint32_t ws[4] = {nw[c].x, nw[c].y, nw[c].z, nw[c].w};
#pragma unroll
      for (int q = 0; q < 4; q++) {
        const uint32_t w = ws[q];
        zeros += __popc(~(((w & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | w) & 0x80808080u);
        big |= w;
        const uint32_t t0 = __funnelshift_r(0x80000000u, 0u, w);
        const uint32_t t1 = __funnelshift_r(0x80000000u, 0u, w >> 8);
        const uint32_t t2 = __funnelshift_r(0x80000000u, 0u, w >> 16);
        const uint32_t t3 = __funnelshift_r(0x80000000u, 0u, w >> 24);
        S += ((uint64_t)t0 + t1) + ((uint64_t)t2 + t3);
      }
    }
    s = __dmul_rn(__ull2double_rn(S), 0x1p-31);
#pragma unroll
    for (int off = 1; off < Gm::G; off <<= 1) {   // xor partners stay inside the group
      s = __dadd_rn(s, __shfl_xor_sync(0xffffffffu, s, off));
      zeros += __shfl_xor_sync(0xffffffffu, zeros, off);
      big |= __shfl_xor_sync(0xffffffffu, big, off);
    }
    seq = (big & 0xE0E0E0E0u) != 0u;   // some register > 31
  }
  return changed;
}

// The whole epilogue for one node per group (heavy nodes, and the light kernel at p <= 32
// where every lane already owns a node): finish_rows, then the scalar tail on the
// group's first lane.  Returns the group's changed flag.
template <int LOGP, bool PUSH>
__device__ __forceinline__ bool finish_node(const Peers &peers, bool doit, int64_t v,
                                            const uint4 (&acc)[Geo<LOGP>::CPL],
                                            const uint4 (&pre)[Geo<LOGP>::CPL], bool have_pre,
                                            bool self_chg, int grp, int gl,
                                            const uint8_t *__restrict__ cur,
                                            uint8_t *__restrict__ nxt, double *__restrict__ est,
                                            double *__restrict__ sum_dist,
                                            double *__restrict__ sum_recip, const EstConst &ec,
                                            double tf, const double *pre_vals = nullptr) {
  using Gm = Geo<LOGP>;
  bool any;
  double s;
  uint32_t zeros;
  bool seq;
  const bool changed = finish_rows<LOGP, PUSH>(peers, doit, v, acc, pre, have_pre, self_chg,
                                               grp, gl, cur, nxt, any, s, zeros, seq);
  if (any) {   // warp-uniform
    if (__any_sync(0xffffffffu, changed && seq)) __syncwarp();  // stored rows visible
    if (changed && gl == 0)
      node_scalar<Gm::P>(v, s, zeros, seq, nxt + (size_t)v * Gm::P, est, sum_dist, sum_recip,
                         ec, tf, pre_vals);
  }
  return changed;
}

#ifndef HB_TMA_DIRECT
#define HB_TMA_DIRECT 1               // TMA light kernel, dense batches: ids straight to the issuing lanes
#endif
#ifndef HB_L1_NEXT_IDS
#define HB_L1_NEXT_IDS 2               // lines of the next round's ids prefetched into L1
#endif
#ifndef HB_L1_OWN_ROW
#define HB_L1_OWN_ROW 1
#endif
#ifndef HB_SELF_LATE
#define HB_SELF_LATE 1                // TMA light kernel: own row read in the epilogue
#endif
#ifndef HB_DEFER_TAIL
#define HB_DEFER_TAIL 1               // light kernel: deferred scalar epilogue
#endif
#ifndef HB_DEFER_MIN_LOGP
#define HB_DEFER_MIN_LOGP 8
#endif
#ifndef HB_DEFER_PRELOAD
#define HB_DEFER_PRELOAD 1
#endif
// Deferred scalar epilogue of the light kernel for G > 1 (p >= 64): a warp round finishes
// NPW = 32 / G nodes, and the scalar tail (two fp64 divisions, the estimate / sums
// read-modify-write, the discounts) would run on NPW lanes only.  Instead each round's
// (s, zeros, flags) move by shuffle to the lane that owns the node's slot in its aligned
// block of 32 ids (lane = v & 31); once the warp leaves the block, all 32 lanes run the
// tail at once (coalesced 256-byte estimate / sum accesses).  Rows were stored by the
// round, so the > 31 fallback re-reads them after a __syncwarp.
struct DeferredTail {
  int64_t blk = -1;      // block of 32 ids (v >> 5) the pending slots belong to
  double s = 0.0;
  uint32_t zeros = 0;
  uint32_t flags = 0;    // bit 0 pending, bit 1 some register > 31
  double pv[3];          // HB_DEFER_PRELOAD: the block's old estimate / sums, loaded on entry
  template <int P>
  __device__ __forceinline__ void flush(const uint8_t *__restrict__ nxt,
                                        double *__restrict__ est, double *__restrict__ sum_dist,
                                        double *__restrict__ sum_recip, const EstConst &ec,
                                        double tf) {
    if (__any_sync(0xffffffffu, flags & 1u)) {   // warp-uniform
      if (__any_sync(0xffffffffu, flags & 2u)) __syncwarp();
      if (flags & 1u) {
        const int64_t v = (blk << 5) + (threadIdx.x & 31);
        node_scalar<P>(v, s, zeros, (flags & 2u) != 0u, nxt + (size_t)v * P, est, sum_dist,
                       sum_recip, ec, tf, HB_DEFER_PRELOAD ? pv : nullptr);
      }
    }
    flags = 0;
  }
  // enter block b: its lanes' old values start loading now, consumed at the flush
  __device__ __forceinline__ void enter(int64_t b, int64_t lo, int64_t hi,
                                        const double *__restrict__ est,
                                        const double *__restrict__ sum_dist,
                                        const double *__restrict__ sum_recip) {
    blk = b;
    if (HB_DEFER_PRELOAD) {
      const int64_t v = (b << 5) + (threadIdx.x & 31);
      const bool in = v >= lo && v < hi;
      pv[0] = in ? est[v] : 0.0;
      pv[1] = in && sum_dist ? sum_dist[v] : 0.0;
      pv[2] = in && sum_recip ? sum_recip[v] : 0.0;
    }
  }
  // round results of the NPW groups of G lanes (group g = node base + g) -> slot lanes
  template <int G, int NPW>
  __device__ __forceinline__ void take(int64_t base, bool changed, double rs, uint32_t rz,
                                       bool rseq) {
    const int lane = threadIdx.x & 31;
    const int first = (int)(base & 31);
    const int g = lane - first;
    const bool mine = g >= 0 && g < NPW;
    const int src = (mine ? g : 0) * G;
    const uint32_t f = (changed ? 1u : 0u) | (rseq ? 2u : 0u);
    const double ts = __shfl_sync(0xffffffffu, rs, src);
    const uint32_t tz = __shfl_sync(0xffffffffu, rz, src);
    const uint32_t tf = __shfl_sync(0xffffffffu, f, src);
    if (mine && (tf & 1u)) {
      s = ts;
      zeros = tz;
      flags = tf;
    }
  }
};

// Batched runs (run_multi): a row of cur holds R = 2^LOGR independent runs' registers side
// by side (p1 = P / R bytes each, run r at bytes [r*p1, (r+1)*p1)).  The union is the same
// byte-wise max over the wide row; this epilogue then does per run what finish_node does
// per row: change test, estimate, accumulate -- est / sums are [R, stride] (run r at
// + r * stride) and run r's change bit goes to ra.chg[r * ra.words + v/32].  The row is
// written iff any run changed or the row changed last iteration (lazy double buffer over
// the OR of the runs' flags, which also drives the source skip).  A run's CPR = p1/16
// chunks sit on CPR consecutive lanes of one chunk slot (CPR <= G for every p1 >= 16 and
// P <= 256), so its partial sums reduce by xor-shuffles inside that lane block.
struct RunArgs {
  uint32_t *chg;      // [R, words] per-run change bitmaps
  int64_t words;
  int64_t stride;     // est / sum_dist / sum_recip run stride (>= n)
};

template <int LOGP, int LOGR>
__device__ __forceinline__ bool finish_runs(bool doit, int64_t v,
                                            const uint4 (&acc)[Geo<LOGP>::CPL],
                                            const uint4 (&pre)[Geo<LOGP>::CPL], bool have_pre,
                                            bool self_chg, int gl,
                                            const uint8_t *__restrict__ cur,
                                            uint8_t *__restrict__ nxt, double *__restrict__ est,
                                            double *__restrict__ sum_dist,
                                            double *__restrict__ sum_recip, const EstConst &ec,
                                            double tf, const RunArgs &ra) {
  using Gm = Geo<LOGP>;
  constexpr int P1 = Gm::P >> LOGR;
  constexpr int CPR = P1 / 16;
  static_assert(CPR >= 1 && CPR <= Gm::G && Gm::G % CPR == 0, "run chunks must share a lane block");
  const uint8_t *crow = cur + (size_t)v * Gm::P;
  uint8_t *nrow = nxt + (size_t)v * Gm::P;
  uint4 nw[Gm::CPL];
  unsigned my_runs = 0;
#pragma unroll
  for (int c = 0; c < Gm::CPL; c++) {
    uint4 self = pre[c];
    if (doit && !have_pre) self = ldg4(crow + 16 * (c * Gm::G + gl));
    nw[c] = bmax4(acc[c], self);
    if (doit && neq4(nw[c], self)) my_runs |= 1u << ((c * Gm::G + gl) / CPR);
  }
  unsigned runs = my_runs;
#pragma unroll
  for (int off = 1; off < Gm::G; off <<= 1) runs |= __shfl_xor_sync(0xffffffffu, runs, off);
  const bool changed = runs != 0u;
  if (doit && (changed || self_chg)) {
#pragma unroll
    for (int c = 0; c < Gm::CPL; c++)
      *reinterpret_cast<uint4 *>(nrow + 16 * (c * Gm::G + gl)) = nw[c];
  }
  if (__any_sync(0xffffffffu, changed)) {   // warp-uniform
    double s[Gm::CPL];
    uint32_t zeros[Gm::CPL], big[Gm::CPL];
#pragma unroll
    for (int c = 0; c < Gm::CPL; c++) {
      double s4[4] = {0.0, 0.0, 0.0, 0.0};
      const uint32_t ws[4] = {nw[c].x, nw[c].y, nw[c].z, nw[c].w};
      zeros[c] = 0;
      big[c] = 0;
#pragma unroll
      for (int q = 0; q < 4; q++) {
        const uint32_t w = ws[q];
        zeros[c] += __popc(~(((w & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | w) & 0x80808080u);
        big[c] |= w;
#pragma unroll
        for (int i = 0; i < 4; i++) {
          const uint32_t m = (w >> (8 * i)) & 0xffu;
          s4[i] = __dadd_rn(s4[i], __hiloint2double((int)(0x3FF00000u - (m << 20)), 0));
        }
      }
      s[c] = __dadd_rn(__dadd_rn(s4[0], s4[1]), __dadd_rn(s4[2], s4[3]));
#pragma unroll
      for (int off = 1; off < CPR; off <<= 1) {   // inside the run's lane block
        s[c] = __dadd_rn(s[c], __shfl_xor_sync(0xffffffffu, s[c], off));
        zeros[c] += __shfl_xor_sync(0xffffffffu, zeros[c], off);
        big[c] |= __shfl_xor_sync(0xffffffffu, big[c], off);
      }
    }
    bool need_seq = false;
#pragma unroll
    for (int c = 0; c < Gm::CPL; c++) {
      const int r = (c * Gm::G + gl) / CPR;
      need_seq |= ((runs >> r) & 1u) && (big[c] & 0xE0E0E0E0u) != 0u;
    }
    if (__any_sync(0xffffffffu, need_seq)) __syncwarp();   // stored rows visible
    if (gl % CPR == 0) {
#pragma unroll
      for (int c = 0; c < Gm::CPL; c++) {
        const int r = (c * Gm::G + gl) / CPR;
        if (!((runs >> r) & 1u)) continue;
        double sr = s[c];
        if ((big[c] & 0xE0E0E0E0u) != 0u) {   // reference order: ascending-j fp64 sum
          sr = 0.0;
          for (int j = 0; j < P1; j++) sr = __dadd_rn(sr, pow2neg(nrow[r * P1 + j]));
        }
        const double e = finish_estimate(sr, (int)zeros[c], ec);
        const int64_t at = (int64_t)r * ra.stride + v;
        const double old = est[at];
        est[at] = e;
        const double d = np_max0(__dsub_rn(e, old));
        if (sum_dist) sum_dist[at] = __dadd_rn(sum_dist[at], __dmul_rn(tf, d));
        if (sum_recip) sum_recip[at] = __dadd_rn(sum_recip[at], __ddiv_rn(d, tf));
        for (int k = 0; k < ec.n_disc; k++) {   // run r's discounts: [R, n_disc, stride]
          double *q = ec.disc + ((int64_t)r * ec.n_disc + k) * ec.disc_stride + v;
          const double cc = ((ec.disc_div >> k) & 1) ? __ddiv_rn(d, tf)
                                                     : __dmul_rn(ec.disc_scale[k], d);
          *q = __dadd_rn(*q, cc);
        }
        atomicOr(ra.chg + r * ra.words + (v >> 5), 1u << (v & 31));
      }
    }
  }
  return changed;
}

// Block-wide sum of two per-thread counters, one atomicAdd per block and counter.
__device__ __forceinline__ void block_add2(uint32_t a, uint32_t b, unsigned long long *out_a,
                                           unsigned long long *out_b) {
  __shared__ uint32_t red[2][32];
  uint32_t wa = __reduce_add_sync(0xffffffffu, a);
  uint32_t wb = __reduce_add_sync(0xffffffffu, b);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) { red[0][wid] = wa; red[1][wid] = wb; }
  __syncthreads();
  if (wid == 0) {
    const bool in = lane < (int)(blockDim.x >> 5);
    uint32_t x = __reduce_add_sync(0xffffffffu, in ? red[0][lane] : 0u);
    uint32_t y = __reduce_add_sync(0xffffffffu, in ? red[1][lane] : 0u);
    if (lane == 0) {
      if (x && out_a) atomicAdd(out_a, (unsigned long long)x);
      if (y && out_b) atomicAdd(out_b, (unsigned long long)y);
    }
  }
}

// ------------------------------------------------------------------ kernels
constexpr int kThreads = 256;

// Batch geometry of the union kernels.
//   light: a group of G lanes owns one node; per batch it loads NB = max(G, 8) successor
//          ids (J per lane, coalesced within the group), compacts the ids whose source
//          changed into shared memory, then every lane issues U independent 16-byte row
//          loads (its chunk of U different source rows) before merging -- while the next
//          batch's ids are already in flight.
//   heavy: the whole warp loads 32*J ids of one work item per batch, compacts them, and
//          its NPW slots of G lanes take every NPW-th compacted id, U rows in flight each.
// TMA row gather for the light kernel at p = 256 (HB_TMA_P256): 4 register rows per
// cp.async.bulk.tensor...tile::gather4 into a per-warp shared buffer, completion on an
// mbarrier; lanes read their chunks back with LDS.  No row-load registers, no address math.
#ifndef HB_TMA_P256
#define HB_TMA_P256 1
#endif
#ifndef HB_TMA_MINB
#define HB_TMA_MINB 3                 // 80 registers without the loads in flight: 3 CTAs / SM
#endif
#ifndef HB_TMA_P128
#define HB_TMA_P128 0
#endif
#ifndef HB_TMA_P64
#define HB_TMA_P64 0
#endif
#ifndef HB_TMA_MINB64
#define HB_TMA_MINB64 4
#endif
#ifndef HB_TMA_MINB128
#define HB_TMA_MINB128 4
#endif
template <int LOGP, int LOGR, bool HINT>
__host__ __device__ constexpr bool kTma() {
  return ((HB_TMA_P256 && LOGP == 8) || (HB_TMA_P128 && LOGP == 7) || (HB_TMA_P64 && LOGP == 6)) &&
         LOGR == 0 && !HINT;
}
__device__ __forceinline__ void tma_gather4(uint32_t dst, const CUtensorMap *tm, int32_t r0,
                                            int32_t r1, int32_t r2, int32_t r3, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(dst), "l"(tm), "r"(0), "r"(r0), "r"(r1),
      "r"(r2), "r"(r3), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t phase) {
  uint32_t done = 0;
  while (!done)
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared.b64 p, [%1], %2; "
                 "selp.u32 %0, 1, 0, p; }" : "=r"(done) : "r"(bar), "r"(phase) : "memory");
}

template <int LOGP>
struct Batch {
  using Gm = Geo<LOGP>;
  // 16-byte row loads in flight per lane and resident CTAs per SM of the light kernel,
  // per p (swept on configs 3, 4, 5s: more registers per thread pay at p = 64 / 256)
#ifndef HB_LOADS_P16
#define HB_LOADS_P16 8
#endif
#ifndef HB_MINB_P16
#define HB_MINB_P16 4
#endif
#ifndef HB_LOADS_P64
#define HB_LOADS_P64 8
#endif
#ifndef HB_MINB_P64
#define HB_MINB_P64 3
#endif
#ifndef HB_LOADS_P256
#define HB_LOADS_P256 16
#endif
#ifndef HB_MINB_P256
#define HB_MINB_P256 2
#endif
#ifndef HB_LOADS_P128
#define HB_LOADS_P128 8
#endif
#ifndef HB_MINB_P128
#define HB_MINB_P128 3
#endif
  static constexpr int LOADS = LOGP == 8 ? HB_LOADS_P256 : (LOGP == 6 ? HB_LOADS_P64 :
                               (LOGP <= 5 ? HB_LOADS_P16 : (LOGP == 7 ? HB_LOADS_P128 : 8)));
  static constexpr int MINB = LOGP >= 10 ? 2 : (LOGP == 8 ? (HB_TMA_P256 ? HB_TMA_MINB : HB_MINB_P256) : (LOGP == 6 ? (HB_TMA_P64 ? HB_TMA_MINB64 : HB_MINB_P64) :
                              (LOGP == 7 ? (HB_TMA_P128 ? HB_TMA_MINB128 : HB_MINB_P128) : HB_MINB_P16)));
  static constexpr int U = Gm::CPL >= LOADS ? 1 : LOADS / Gm::CPL;  // rows in flight per lane
  static constexpr int NB = Gm::G > 8 ? Gm::G : 8;            // light: ids per group batch
  static constexpr int J = NB / Gm::G;                        // light: ids loaded per lane
  static constexpr int WARP_IDS = Gm::NPW * NB;               // light: smem ids per warp
  static constexpr int HJ = (U * Gm::NPW) / 32 > 0 ? (U * Gm::NPW) / 32 : 1;  // heavy: ids/lane
  static constexpr int HEAVY_IDS = 32 * HJ;                   // heavy: smem ids per warp
};

// L2 prefetch of [p, p + bytes) with the async bulk-copy unit (no registers, no wait).
// Rounded out to 16-byte granules; every buffer here is a torch allocation (>= 512-byte
// aligned and padded), so the rounded range stays inside the allocation.
__device__ __forceinline__ void l2_prefetch(const void *p, int64_t bytes) {
  if (bytes <= 0) return;
  const uintptr_t a0 = reinterpret_cast<uintptr_t>(p) & ~(uintptr_t)15;
  const uintptr_t a1 = (reinterpret_cast<uintptr_t>(p) + (uintptr_t)bytes + 15) & ~(uintptr_t)15;
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a0), "r"((uint32_t)(a1 - a0))
               : "memory");
}

#ifndef HB_DENSE_COPY
#define HB_DENSE_COPY 1
#endif
constexpr bool kDenseCopy = HB_DENSE_COPY != 0;   // dense batches skip the id compaction
#ifndef HB_LOOK_ROUNDS
#define HB_LOOK_ROUNDS 4
#endif
#ifndef HB_CHUNK_BIG
#define HB_CHUNK_BIG 8
#endif
#ifndef HB_CHUNK_SMALL
#define HB_CHUNK_SMALL 4
#endif
constexpr int kLookRounds = HB_LOOK_ROUNDS;   // L2 prefetch distance of the light kernel, in warp rounds
// warp rounds per grid-stride chunk of the light kernel (resident warps x chunk nodes is
// the id window the GPU sweeps): 8 for p >= 256 (16 before the chunk tickets; with them
// config 4 takes 7.17 ms at 16, 7.06 ms at 8, 7.43 ms at 32), 4 below (configs 2, 3, 5s:
// 2 and 8 are within noise or slower)
template <int LOGP>
__host__ __device__ constexpr int chunk_rounds() { return LOGP >= 8 ? HB_CHUNK_BIG : HB_CHUNK_SMALL; }

// Light nodes (in-degree <= max_deg): one group of G lanes per node, NPW nodes per warp
// round.  Each warp owns one contiguous node range, balanced over the grid by arcs +
// nodes, so its offsets, ids, own rows and estimates are sequential streams: one lane
// prefetches them into L2 kLookRounds rounds ahead, leaving the random source-row
// gather as the only exposed memory latency of a round.
// _kernels.py:67-114 restated with the source-skip rule.
template <int LOGP, bool PUSH, int LOGR = 0, bool HINT = false, bool L1NA = false>
__global__ void __launch_bounds__(kThreads, Batch<LOGP>::MINB)
k_light(const int64_t *__restrict__ offsets, const int32_t *__restrict__ succ,
        const uint8_t *__restrict__ cur, uint8_t *__restrict__ nxt,
        const uint32_t *__restrict__ chg_prev, uint32_t *__restrict__ chg_now,
        double *__restrict__ est, double *__restrict__ sum_dist, double *__restrict__ sum_recip,
        EstConst ec, int64_t lo, int64_t hi, int64_t max_deg, int dense, double tf,
        unsigned long long *__restrict__ nch_out, unsigned long long *__restrict__ merged_out,
        const uint32_t *__restrict__ active, Peers peers, RunArgs ra, int64_t hot_lim,
        unsigned int *__restrict__ ticket, const __grid_constant__ CUtensorMap tmap) {
  static_assert(LOGR == 0 || !PUSH, "batched runs are single-device");
  constexpr bool kHint = HINT;
  uint64_t pol = 0;
  if (kHint) pol = range_policy(cur, (uint32_t)((uint64_t)hot_lim << LOGP), 0xFFFFFFF0u);
  using Gm = Geo<LOGP>;
  using B = Batch<LOGP>;
  __shared__ int32_t sids[kThreads / 32][B::WARP_IDS];
  const int lane = threadIdx.x & 31;
  const int gl = lane % Gm::G;
  const int grp = lane / Gm::G;
  const unsigned lowmask = Gm::G == 32 ? 0xffffffffu : ((1u << (Gm::G & 31)) - 1u);
  const unsigned gmask = lowmask << (grp * Gm::G);
  const unsigned below = (1u << gl) - 1u;
  int32_t *my_ids = &sids[threadIdx.x >> 5][grp * B::NB];
  const uint4 *cur4 = reinterpret_cast<const uint4 *>(cur);
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  uint32_t my_nch = 0, my_merged = 0;
  uint32_t tma_buf = 0, tma_bar = 0, tma_phase = 0;
  if constexpr (kTma<LOGP, LOGR, HINT>()) {
    extern __shared__ __align__(1024) uint8_t tma_smem[];
    __shared__ __align__(8) uint64_t tma_bars[kThreads / 32];
    const int wl = threadIdx.x >> 5;
    tma_buf = (uint32_t)__cvta_generic_to_shared(tma_smem) + wl * (Gm::NPW * B::U * Gm::P);
    tma_bar = (uint32_t)__cvta_generic_to_shared(&tma_bars[wl]);
    if (lane == 0) {
      asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(tma_bar));
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
  }

  // Node chunks of kChunkRounds warp rounds, dealt to warps grid-stride: at any moment the
  // resident warps sweep one contiguous window of the id space (L2 reuse of shared
  // sources, e.g. config 4's +-1024 locality), while inside a chunk the offsets, ids,
  // own rows and estimates are sequential streams that lane 0 prefetches into L2
  // kLookRounds rounds ahead -- leaving the random source-row gather as the only exposed
  // memory latency of a round.  Rounds are NPW-aligned so a round's change bits share one
  // bitmap word.
  const int64_t lo_al = (lo / Gm::NPW) * Gm::NPW;
  constexpr int64_t CN = (int64_t)chunk_rounds<LOGP>() * Gm::NPW;
  constexpr bool kDefer = LOGR == 0 && Gm::G > 1 && HB_DEFER_TAIL && LOGP >= HB_DEFER_MIN_LOGP;
  DeferredTail dt;
  const int64_t nchunks = (hi - lo_al + CN - 1) / CN;
  // Chunks are dealt grid-stride, or -- with a ticket counter (zeroed by the launcher) --
  // in the order the warps ask for them: the sweep stays one contiguous window of the id
  // space, and a warp whose chunks ran long (more arcs, more DRAM misses) simply takes
  // fewer of them.  The next ticket is drawn at the start of a chunk, so the atomic's
  // round trip hides behind the chunk's work.  (Several chunks per draw only lengthen the
  // tail: config 2 0.38 -> 0.45 / 0.59 / 0.84 ms at 2 / 4 / 8 chunks per draw.)
  // (32-bit draws: chunks + one overshoot per warp stay far below 2^32)
  auto draw = [&]() -> uint32_t {
    return lane == 0 ? atomicAdd(ticket, 1u) : 0u;
  };
  uint32_t drawn = ticket ? draw() : 0u;
  int64_t chunk = ticket ? (int64_t)__shfl_sync(0xffffffffu, drawn, 0) : warp;
  for (; chunk < nchunks;) {
  if (ticket) drawn = draw();
  const int64_t vb = lo_al + chunk * CN;
  const int64_t ve = vb + CN < hi ? vb + CN : hi;
  // prefetch of the per-round streams, kLookRounds rounds per batch: own rows, estimates,
  // sums and successor ids of rounds [pb, pe).  Ids need offsets, which lane 0 loads one
  // round before issuing their prefetch (offsets of the chunk are prefetched first).
  auto stream_prefetch = [&](int64_t pb, int64_t pe) {
    l2_prefetch(cur + (size_t)pb * Gm::P, (pe - pb) * Gm::P);
    l2_prefetch(est + pb, (pe - pb) * 8);
    if (sum_dist) l2_prefetch(sum_dist + pb, (pe - pb) * 8);
    if (sum_recip) l2_prefetch(sum_recip + pb, (pe - pb) * 8);
  };
  int64_t pf_a0 = -1, pf_a1 = -1;
  if (lane == 0 && !active) {
    l2_prefetch(offsets + vb, (ve - vb + 1) * 8);
    const int64_t pe = vb + (int64_t)kLookRounds * Gm::NPW < ve ? vb + (int64_t)kLookRounds * Gm::NPW : ve;
    stream_prefetch(vb, pe);
    const int64_t a0 = __ldg(offsets + vb), a1 = __ldg(offsets + pe);
    l2_prefetch(succ + a0, (a1 - a0) * 4);
  }
  for (int64_t base = vb; base < ve; base += Gm::NPW) {
    // frontier mode: only nodes with a changed in-neighbour (or a changed own row) work
    const bool act_v = !active || ((base + grp < ve) && test_bit(active, base + grp));
    if (active && !__any_sync(0xffffffffu, act_v)) continue;
    if constexpr (kDefer) {
      if ((base >> 5) != dt.blk) {                // left the block: run its scalar tails
        dt.flush<Gm::P>(nxt, est, sum_dist, sum_recip, ec, tf);
        dt.enter(base >> 5, lo, hi, est, sum_dist, sum_recip);
      }
    }
    if (lane == 0 && !active) {
      if (pf_a0 >= 0) {                        // ids of the batch announced last round
        l2_prefetch(succ + pf_a0, (pf_a1 - pf_a0) * 4);
        pf_a0 = -1;
      }
      const int64_t rnd = (base - vb) / Gm::NPW;
      const int64_t pb = base + (int64_t)kLookRounds * Gm::NPW;
      if (rnd % kLookRounds == 0 && pb < ve) {
        const int64_t pe = pb + (int64_t)kLookRounds * Gm::NPW < ve
                               ? pb + (int64_t)kLookRounds * Gm::NPW : ve;
        stream_prefetch(pb, pe);
        pf_a0 = __ldg(offsets + pb);           // consumed next round
        pf_a1 = __ldg(offsets + pe);
      }
    }
    const int64_t v = base + grp;
    bool valid = (v >= lo) && (v < ve) && act_v;
    int64_t beg = 0, end = 0;
    if (valid) {
      beg = __ldg(offsets + v);
      end = __ldg(offsets + v + 1);
      HB_CHK(v >= 0 && v < g_chk.rows && 0 <= beg && beg <= end && end <= g_chk.m,
             "k_light row / offsets");
      if constexpr (HB_L1_NEXT_IDS && kTma<LOGP, LOGR, HINT>()) {
        // the last group's row end is where the next round's ids start: pull their first
        // lines into L1 now, so the next round's first gathers need not wait on L2
        if (grp == Gm::NPW - 1 && gl == 0 && v + 1 < ve) {
          const int32_t *nx = succ + end;
#pragma unroll
          for (int q = 0; q < HB_L1_NEXT_IDS; q++)
            asm volatile("prefetch.global.L1 [%0];" ::"l"(nx + 32 * q));
        }
      }
      if constexpr (HB_L1_OWN_ROW && kTma<LOGP, LOGR, HINT>()) {
        // own row, read in the epilogue (HB_SELF_LATE): into L1 now
        if (gl < Gm::P / 128)
          asm volatile("prefetch.global.L1 [%0];" ::"l"(cur + (size_t)v * Gm::P + 128 * gl));
      }
      if (end - beg > max_deg) {               // heavy: handled by the item path
        valid = false;
        end = beg;
      }
    }
    const bool self_chg = valid && test_bit(chg_prev, v);
    bool pre;                                   // own row certainly needed: load early
    if (dense) pre = valid;                     // (no wait on the bitmap word)
    else pre = self_chg;
    if (kTma<LOGP, LOGR, HINT>() && HB_SELF_LATE) pre = false;   // own row read at the end
    uint4 self[Gm::CPL], acc[Gm::CPL];
#pragma unroll
    for (int c = 0; c < Gm::CPL; c++) {
      acc[c] = make_uint4(0, 0, 0, 0);
      self[c] = pre ? ldg4(cur + (size_t)v * Gm::P + 16 * (c * Gm::G + gl)) : acc[c];
    }
    // own row: part of the union anyway, so it pads the group's unused load slots (and is
    // L1-hot); groups past the range use row lo
    const int32_t fb = (int32_t)(v < ve ? v : lo);
    RowAcc<LOGP> macc;
    macc.init();
    double vals[3] = {0.0, 0.0, 0.0};
    if (LOGR == 0 && !kDefer && pre && gl == 0) {
      vals[0] = est[v];
      if (sum_dist) vals[1] = sum_dist[v];
      if (sum_recip) vals[2] = sum_recip[v];
    }
    int32_t idr[B::J];
#pragma unroll
    for (int j = 0; j < B::J; j++) {
      const int64_t k = beg + j * Gm::G + gl;
      idr[j] = (k < end) ? __ldg(succ + k) : -1;
      HB_CHK(idr[j] < g_chk.rows, "k_light successor id");
    }
    HB_CHK(fb >= 0 && fb < g_chk.rows, "k_light fallback row");
    // batches of NB ids per group; the loop runs the warp's longest node so that every
    // ballot / shuffle below is full-warp (no per-group serialisation)
    const int trips = (int)((end - beg + B::NB - 1) / B::NB);
    const int wtrips = __reduce_max_sync(0xffffffffu, (unsigned)trips);
    int total = 0;
    constexpr bool kDirect = kTma<LOGP, LOGR, HINT>() && HB_TMA_DIRECT;
    if constexpr (kDirect) {
      if (dense) {   // warp-uniform
        // Dense batches need no compaction, so the ids skip shared memory: lane q <
        // NPW * GPG owns gather4 number h = q % GPG of group g = q / GPG in every batch
        // (slots [4h, 4h + 4) of the group's U), loads those 4 ids itself one batch
        // ahead, pads past the node's end with the group's own row, and issues the gather.
        static_assert(B::U == B::NB && B::U % 4 == 0 && Gm::NPW * (B::U / 4) <= 32,
                      "direct TMA layout");
        constexpr int GPG = B::U / 4;
        const int g = (lane / GPG) & (Gm::NPW - 1), h = lane % GPG;
        const bool iss_lane = lane < Gm::NPW * GPG;
        const int64_t beg_g = __shfl_sync(0xffffffffu, beg, g * Gm::G);
        const int64_t end_g = __shfl_sync(0xffffffffu, end, g * Gm::G);
        const int32_t fbg = (int32_t)(base + g < ve ? base + g : lo);
        int32_t nid[4];
        auto load_ids = [&](int64_t k0) {
#pragma unroll
          for (int k = 0; k < 4; k++) {
            const int64_t kk = k0 + 4 * h + k;
            nid[k] = (iss_lane && kk < end_g) ? __ldg(succ + kk) : fbg;
            HB_CHK(nid[k] >= 0 && nid[k] < g_chk.rows, "k_light direct TMA row");
          }
        };
        load_ids(beg_g);
        for (int it = 0; it < wtrips; it++) {
          const bool issue = iss_lane && 4 * h < end_g - (beg_g + (int64_t)it * B::U);
          const uint32_t ngat = __popc(__ballot_sync(0xffffffffu, issue));
          if (lane == 0)
            asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(tma_bar),
                         "r"(ngat * 4 * Gm::P) : "memory");
          __syncwarp();
          if (issue) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            tma_gather4(tma_buf + (g * B::U + 4 * h) * Gm::P, &tmap, nid[0], nid[1], nid[2],
                        nid[3], tma_bar);
          }
          load_ids(beg_g + (int64_t)(it + 1) * B::U);   // next batch, in flight meanwhile
          mbar_wait(tma_bar, tma_phase);
          tma_phase ^= 1u;
          const int64_t left = end - (beg + (int64_t)it * B::U);
          const int cnt = left <= 0 ? 0 : (left < B::U ? (int)left : B::U);
          const uint4 *rows = reinterpret_cast<const uint4 *>(
              __cvta_shared_to_generic(tma_buf + grp * B::U * Gm::P));
#pragma unroll
          for (int hh = 0; hh < GPG; hh++) {
            if (4 * hh < cnt) {
#pragma unroll
              for (int u = 4 * hh; u < 4 * hh + 4; u += 2)
#pragma unroll
                for (int c = 0; c < Gm::CPL; c++)
                  macc.add2(c, rows[u * Gm::CH + c * Gm::G + gl],
                            rows[(u + 1) * Gm::CH + c * Gm::G + gl]);
            }
          }
          total += cnt;
          __syncwarp();                          // every lane done before the next gather
        }
      }
    }
    for (int it = 0; it < ((kDirect && dense) ? 0 : wtrips); it++) {
      const int64_t kb = beg + (int64_t)it * B::NB;
      int cnt = 0;
      if (kDenseCopy && dense) {
        // every source merged: the batch's valid ids are the prefix of its NB slots
#pragma unroll
        for (int j = 0; j < B::J; j++) my_ids[j * Gm::G + gl] = idr[j];
        const int64_t left = end - kb;
        cnt = left <= 0 ? 0 : (left < B::NB ? (int)left : B::NB);
      } else {
#pragma unroll
        for (int j = 0; j < B::J; j++) {
          const bool act = idr[j] >= 0 && (dense || test_bit(chg_prev, idr[j]));
          const unsigned bal = (__ballot_sync(0xffffffffu, act) >> (grp * Gm::G)) & lowmask;
          HB_CHK(!act || cnt + __popc(bal & below) < B::NB, "k_light shared id slot");
          if (act) my_ids[cnt + __popc(bal & below)] = idr[j];
          cnt += __popc(bal);
        }
      }
#pragma unroll
      for (int j = 0; j < B::J; j++) {                // next batch's ids, in flight meanwhile
        const int64_t k = kb + B::NB + j * Gm::G + gl;
        idr[j] = (k < end) ? __ldg(succ + k) : -1;
        HB_CHK(idr[j] < g_chk.rows, "k_light successor id (next batch)");
      }
      __syncwarp();
      const int cmax = __reduce_max_sync(0xffffffffu, (unsigned)cnt);
      for (int i = 0; i < cmax; i += B::U) {
        if constexpr (kTma<LOGP, LOGR, HINT>()) {
          static_assert(B::U % 4 == 0 && Gm::NPW * (B::U / 4) <= 32, "TMA gather layout");
          constexpr int GPG = B::U / 4;              // gather4 issues per lane group
          // lane q < NPW * GPG: group g = q / GPG loads rows [4h, 4h + 4), h = q % GPG, of
          // its batch slots, padded with that group's own row (a no-op merge)
          const int cg = __shfl_sync(0xffffffffu, cnt, ((lane / GPG) & (Gm::NPW - 1)) * Gm::G);
          // only groups of 4 slots holding at least one id are fetched (a batch's last
          // slots are often empty); their rows are not merged either
          const bool issue = lane < Gm::NPW * GPG && 4 * (lane % GPG) < cg - i;
          const uint32_t ngat = __popc(__ballot_sync(0xffffffffu, issue));
          if (lane == 0)
            asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(tma_bar),
                         "r"(ngat * 4 * Gm::P) : "memory");
          __syncwarp();
          if (issue) {
            const int g = lane / GPG, h = lane % GPG;
            const int64_t vg = base + g;
            const int32_t fbg = (int32_t)(vg < ve ? vg : lo);
            const int32_t *gids = &sids[threadIdx.x >> 5][g * B::NB];
            int32_t r[4];
#pragma unroll
            for (int k = 0; k < 4; k++) r[k] = (i + 4 * h + k < cg) ? gids[i + 4 * h + k] : fbg;
#pragma unroll
            for (int k = 0; k < 4; k++) HB_CHK(r[k] >= 0 && r[k] < g_chk.rows, "k_light TMA row");
            HB_CHK(cg <= B::NB && (g * B::U + 4 * h + 4) <= Gm::NPW * B::U, "k_light TMA slot");
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            tma_gather4(tma_buf + (g * B::U + 4 * h) * Gm::P, &tmap, r[0], r[1], r[2], r[3],
                        tma_bar);
          }
          mbar_wait(tma_bar, tma_phase);
          tma_phase ^= 1u;
          const uint4 *rows = reinterpret_cast<const uint4 *>(
              __cvta_shared_to_generic(tma_buf + grp * B::U * Gm::P));
#pragma unroll
          for (int h = 0; h < GPG; h++) {
            if (4 * h < cnt - i) {
#pragma unroll
              for (int u = 4 * h; u < 4 * h + 4; u += 2)
#pragma unroll
                for (int c = 0; c < Gm::CPL; c++)
                  macc.add2(c, rows[u * Gm::CH + c * Gm::G + gl],
                            rows[(u + 1) * Gm::CH + c * Gm::G + gl]);
            }
          }
          __syncwarp();                          // every lane done before the next gather
          continue;
        }
        // from p = 64 up, slots past the group's count load the fallback row instead of
        // being predicated off: merging a row that is already part of the union changes
        // nothing, and the loads stay unconditional (no zero-fill, no per-slot predicates)
        uint4 r[B::U][Gm::CPL];
#pragma unroll
        for (int u = 0; u < B::U; u++) {
          const bool ok = i + u < cnt;
          HB_CHK(!ok || i + u < B::NB, "k_light shared id read");
          const int32_t w = ok ? my_ids[i + u] : fb;
          HB_CHK(w >= 0 && w < g_chk.rows, "k_light source row");
#pragma unroll
          for (int c = 0; c < Gm::CPL; c++)
            r[u][c] = (LOGP >= HB_PAD_MIN_LOGP || ok)
                          ? (kHint ? ld_row_chunk_hint<LOGP, L1NA>(cur4, w, Gm::CH, c * Gm::G + gl, pol)
                                   : ld_row_chunk<LOGP>(cur4, w, Gm::CH, c * Gm::G + gl))
                          : make_uint4(0, 0, 0, 0);
        }
        // sequential accumulate: a pairwise tree (shorter chains) measured 20% slower on
        // config 4 (more live registers at 127/thread)
#pragma unroll
        for (int u = 0; u + 1 < B::U; u += 2)
#pragma unroll
          for (int c = 0; c < Gm::CPL; c++) macc.add2(c, r[u][c], r[u + 1][c]);
        if constexpr (B::U % 2 == 1) {
#pragma unroll
          for (int c = 0; c < Gm::CPL; c++) macc.add(c, r[B::U - 1][c]);
        }
      }
      total += cnt;
      __syncwarp();
    }
#pragma unroll
    for (int c = 0; c < Gm::CPL; c++) acc[c] = macc.get(c);
    my_merged += (gl == 0) ? (uint32_t)total : 0u;
    bool changed;
    if constexpr (kDefer) {
      bool any, seq;
      double rs;
      uint32_t rz;
      changed = finish_rows<LOGP, PUSH>(peers, valid && (total > 0 || self_chg), v, acc, self,
                                        pre, self_chg, grp, gl, cur, nxt, any, rs, rz, seq);
      if (any) dt.take<Gm::G, Gm::NPW>(base, changed, rs, rz, seq);
    } else if constexpr (LOGR == 0)
      changed = finish_node<LOGP, PUSH>(peers, valid && (total > 0 || self_chg), v, acc, self,
                                        pre, self_chg, grp, gl, cur, nxt, est, sum_dist,
                                        sum_recip, ec, tf, pre ? vals : nullptr);
    else
      changed = finish_runs<LOGP, LOGR>(valid && (total > 0 || self_chg), v, acc, self, pre,
                                        self_chg, gl, cur, nxt, est, sum_dist, sum_recip, ec,
                                        tf, ra);
    // Warp-level aggregation of the NPW change bits (they share one bitmap word).
    const unsigned bb = __ballot_sync(0xffffffffu, changed && gl == 0);
    if (lane == 0 && bb) {
      uint32_t m = 0;
#pragma unroll
      for (int g = 0; g < Gm::NPW; g++) m |= ((bb >> (g * Gm::G)) & 1u) << g;
      atomicOr(chg_now + (base >> 5), m << (base & 31));
      if constexpr (PUSH)
        for (int q = 0; q < peers.n; q++) atomicOr(peers.chg[q] + (base >> 5), m << (base & 31));
      my_nch += __popc(m);
    }
  }
  chunk = ticket ? (int64_t)__shfl_sync(0xffffffffu, drawn, 0) : chunk + nwarps;
  }  // chunk
  if constexpr (kDefer) dt.flush<Gm::P>(nxt, est, sum_dist, sum_recip, ec, tf);
  if constexpr (PUSH) __threadfence_system();   // remote rows/bits before the barrier
  block_add2(my_nch, my_merged, nch_out, merged_out);
}

#ifndef HB_SHORT_ROUNDS
#define HB_SHORT_ROUNDS 0   // measured: config 5 28.3 -> 28.4 ms (more instructions, not fewer)
#endif
template <int LOGP>
__host__ __device__ constexpr bool kShortRounds() {
  return HB_SHORT_ROUNDS && LOGP < HB_PAD_MIN_LOGP && Batch<LOGP>::U % 2 == 0;
}
// Heavy nodes, phase 1: one warp per work item (a slice of one node's arcs) leaves the
// max over the slice's changed sources as a partial row.
//
// DIE (die-affine items): a B200 is two dies, each with half of the L2;
// a line read by SMs of both dies is kept in both halves, so a gather every SM issues can
// use ~64 MB of the 126 MB.  The hot head of the register array is copied into a fixed
// buffer (`head`, die_rows rows) at the start of the step; with the home die of each of
// its 2 KB chunks known (hb_die_map), hb_die_partition has reordered the ids of every item
// once per graph -- first the sources whose head row lives on die 0, then those of die 1,
// the cold rows filling both halves evenly, item_split[i] of the former.  Pass d of item i merges its half and is drawn from queue d (ticket word 1 + d)
// by the warps of die d's SMs (g_sm_die), which take the other queue's leftovers at the
// end.  Each die then caches only its own half of the head: ~2x the hot rows stay on chip
// (tools/die_probe.cu: 265 G rows/s up to 96 MB, against 64 MB).  Pass d of item i leaves
// partial row 2 i + d.  The result does not depend on the maps.
// Opt-in (HB_DIE=1).  On config 5 it does not pay: the step's DRAM reads fall 71 -> 64 GB,
// but the 15.5 M items average 242 arcs, so two passes each double the fixed per-item work
// (8.3 -> 14.7 G warp instructions, issue 35% -> 56%): 20.5 -> 22.8 ms.
__device__ int8_t g_sm_die[256];
__device__ __forceinline__ uint32_t sm_id() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return r;
}
template <int LOGP, bool HINT = false, bool L1NA = false, bool DIE = false>
__global__ void __launch_bounds__(kThreads, (LOGP >= 10 ? 2 : 4))
k_heavy_partial(const int64_t *__restrict__ offsets, const int32_t *__restrict__ succ,
                const uint8_t *__restrict__ cur, const uint32_t *__restrict__ chg_prev,
                const int32_t *__restrict__ item_node, const int64_t *__restrict__ item_beg,
                int64_t n_items, int64_t item_arcs, int dense, uint8_t *__restrict__ partial,
                unsigned long long *__restrict__ merged_out, const uint32_t *__restrict__ active,
                int64_t hot_lim, unsigned int *__restrict__ ticket, int draw_items,
                const int32_t *__restrict__ item_split = nullptr,
                const uint8_t *__restrict__ head = nullptr, int64_t die_rows = 0) {
  constexpr bool kHint = HINT;
  uint64_t pol = 0;
  // DIE: the head copy is the evict_last range (cold rows, read from cur, lie outside it)
  if (kHint) pol = range_policy(DIE ? head : cur, (uint32_t)((uint64_t)hot_lim << LOGP), 0xFFFFFFF0u);
  using Gm = Geo<LOGP>;
  using B = Batch<LOGP>;
  __shared__ int32_t sids[kThreads / 32][B::HEAVY_IDS];
  uint32_t cls = 0;                             // DIE: the pass (source die) being merged
  if constexpr (DIE) {
    cls = (uint32_t)g_sm_die[sm_id() & 255u] & 1u;
    ticket += cls;
  }
  bool stolen = false;
  const uint4 *head4 = reinterpret_cast<const uint4 *>(head);
  const int lane = threadIdx.x & 31;
  const int gl = lane % Gm::G;
  const int slot = lane / Gm::G;
  const unsigned below = (1u << lane) - 1u;
  int32_t *wids = sids[threadIdx.x >> 5];
  const uint4 *cur4 = reinterpret_cast<const uint4 *>(cur);
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  uint32_t my_merged = 0;
  // Items are dealt grid-stride, or -- with a ticket counter (not in frontier mode) -- in
  // runs of draw_items consecutive items in the order the warps ask for them (the next
  // run is drawn when a run starts), as in k_light: no tail at the end of the launch.
  auto draw = [&]() -> uint32_t {
    return lane == 0 ? atomicAdd(ticket, 1u) : 0u;
  };
  uint32_t drawn = 0;
  int64_t it = warp, run_end = 0;
  if (ticket) {
    drawn = draw();
    it = (int64_t)__shfl_sync(0xffffffffu, drawn, 0) * draw_items;
    run_end = it + draw_items;
    drawn = draw();
  }
  for (;; it += ticket ? 1 : nwarps) {
    if (ticket && it >= run_end) {
      it = (int64_t)__shfl_sync(0xffffffffu, drawn, 0) * draw_items;
      run_end = it + draw_items;
      if (it < n_items) drawn = draw();
    }
    if constexpr (DIE) {
      if (it >= n_items && !stolen) {           // own queue empty: the other die's leftovers
        stolen = true;
        ticket += cls ? -1 : 1;
        cls ^= 1u;
        drawn = draw();
        it = (int64_t)__shfl_sync(0xffffffffu, drawn, 0) * draw_items;
        run_end = it + draw_items;
        if (it < n_items) drawn = draw();
      }
    }
    if (it >= n_items) break;
    if (active) {
      // frontier mode: most items are inactive -- the lanes test the warp's next 32
      // items (it, it + nwarps, ...) at once and the warp jumps to the first active one
      for (;;) {
        const int64_t c = it + (int64_t)lane * nwarps;
        const bool a = c < n_items && test_bit(active, __ldg(item_node + c));
        const unsigned bal = __ballot_sync(0xffffffffu, a);
        if (bal) {
          it += (int64_t)(__ffs(bal) - 1) * nwarps;
          break;
        }
        it += 32 * nwarps;
        if (it >= n_items) break;
      }
      if (it >= n_items) break;
    }
    const int64_t v = __ldg(item_node + it);
    HB_CHK(it < g_chk.items && v >= 0 && v < g_chk.rows, "k_heavy_partial item / node");
    if (active && !test_bit(active, v)) continue;   // warp-uniform: one node per item
    int64_t beg = __ldg(item_beg + it);
    int64_t end = __ldg(offsets + v + 1);
    if (end > beg + item_arcs) end = beg + item_arcs;
    HB_CHK(0 <= beg && beg <= end && end <= g_chk.m, "k_heavy_partial arc range");
    if constexpr (DIE) {
      const int64_t sp = beg + __ldg(item_split + it);
      HB_CHK(beg <= sp && sp <= end, "k_heavy_partial item split");
      if (cls == 0) end = sp; else beg = sp;
    }
    uint4 acc[Gm::CPL];
    RowAcc<LOGP> macc;
    macc.init();
    int32_t idr[B::HJ];
#pragma unroll
    for (int j = 0; j < B::HJ; j++) {
      const int64_t k = beg + j * 32 + lane;
      idr[j] = (k < end) ? ld_stream_id(succ + k) : -1;
      HB_CHK(idr[j] < g_chk.rows, "k_heavy_partial successor id");
    }
    for (int64_t kb = beg; kb < end; kb += B::HEAVY_IDS) {
      int cnt = 0;
      if (kDenseCopy && dense) {            // valid ids are the prefix of the batch
#pragma unroll
        for (int j = 0; j < B::HJ; j++) wids[j * 32 + lane] = idr[j];
        const int64_t left = end - kb;
        cnt = left < B::HEAVY_IDS ? (int)left : B::HEAVY_IDS;
      } else {
#pragma unroll
        for (int j = 0; j < B::HJ; j++) {
          const bool act = idr[j] >= 0 && (dense || test_bit(chg_prev, idr[j]));
          const unsigned bal = __ballot_sync(0xffffffffu, act);
          if (act) wids[cnt + __popc(bal & below)] = idr[j];
          cnt += __popc(bal);
        }
      }
#pragma unroll
      for (int j = 0; j < B::HJ; j++) {
        const int64_t k = kb + B::HEAVY_IDS + j * 32 + lane;
        idr[j] = (k < end) ? ld_stream_id(succ + k) : -1;
      }
      __syncwarp();
      for (int i = slot; i < cnt; i += Gm::NPW * B::U) {
        // slots past cnt re-load the batch's first row (already merged: no effect), from
        // p = 64 up; predicated off below
        uint4 r[B::U][Gm::CPL];
        // rows of this round that exist (warp-uniform): short items -- half of them at
        // p = 16 -- skip the pairs of row loads and merges past their last id
        const int need = kShortRounds<LOGP>() ? (cnt - (i - slot) + Gm::NPW - 1) / Gm::NPW : B::U;
#pragma unroll
        for (int u = 0; u < B::U; u++) {
          if (kShortRounds<LOGP>() && (u & ~1) >= need) {
#pragma unroll
            for (int c = 0; c < Gm::CPL; c++) r[u][c] = make_uint4(0, 0, 0, 0);
            continue;
          }
          const int e = i + u * Gm::NPW;
          const bool ok = e < cnt;
          HB_CHK(!ok || e < B::HEAVY_IDS, "k_heavy_partial shared id read");
          const int32_t w = wids[ok ? e : 0];
          HB_CHK(w >= 0 && w < g_chk.rows, "k_heavy_partial source row");
          const uint4 *src4 = DIE && w < die_rows ? head4 : cur4;   // hot rows: the head copy
#pragma unroll
          for (int c = 0; c < Gm::CPL; c++)
            r[u][c] = (LOGP >= HB_PAD_MIN_LOGP || ok)
                          ? (kHint ? ld_row_chunk_hint<LOGP, L1NA>(src4, w, Gm::CH, c * Gm::G + gl, pol)
                                   : ld_row_chunk<LOGP>(src4, w, Gm::CH, c * Gm::G + gl))
                          : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int u = 0; u + 1 < B::U; u += 2) {
          if (kShortRounds<LOGP>() && u >= need) continue;
#pragma unroll
          for (int c = 0; c < Gm::CPL; c++) macc.add2(c, r[u][c], r[u + 1][c]);
        }
        if constexpr (B::U % 2 == 1) {
#pragma unroll
          for (int c = 0; c < Gm::CPL; c++) macc.add(c, r[B::U - 1][c]);
        }
      }
      my_merged += (lane == 0) ? (uint32_t)cnt : 0u;
      __syncwarp();
    }
#pragma unroll
    for (int c = 0; c < Gm::CPL; c++) acc[c] = macc.get(c);
#pragma unroll
    for (int off = Gm::G; off < 32; off <<= 1)
#pragma unroll
      for (int c = 0; c < Gm::CPL; c++) acc[c] = bmax4(acc[c], shfl_xor4(acc[c], off));
    if (slot == 0) {
#pragma unroll
      for (int c = 0; c < Gm::CPL; c++)
        *reinterpret_cast<uint4 *>(partial + (size_t)(DIE ? 2 * it + cls : it) * Gm::P +
                                   16 * (c * Gm::G + gl)) = acc[c];
    }
  }
  block_add2(my_merged, 0u, merged_out, nullptr);
}

// Heavy nodes, phase 2: merge each heavy node's partial rows and run the shared epilogue.
// order[o0, o1) lists heavy indices j.  mega == 0: one lane group per node (nodes with few
// items); mega != 0: one warp per node, its NPW slots striding over the items (hubs with
// hundreds of items), merged by a shuffle tree.  Partial loads are unrolled 4-deep.
template <int LOGP, bool PUSH, int LOGR = 0>
__global__ void __launch_bounds__(kThreads)
k_heavy_finish(const int32_t *__restrict__ heavy_nodes, const int32_t *__restrict__ item_first,
               const int32_t *__restrict__ order, int64_t o0, int64_t o1, int mega,
               const uint8_t *__restrict__ partial,
               const uint8_t *__restrict__ cur, uint8_t *__restrict__ nxt,
               const uint32_t *__restrict__ chg_prev, uint32_t *__restrict__ chg_now,
               double *__restrict__ est, double *__restrict__ sum_dist,
               double *__restrict__ sum_recip, EstConst ec, double tf,
               unsigned long long *__restrict__ nch_out, const uint32_t *__restrict__ active,
               Peers peers, RunArgs ra, int pshift = 0) {
  // pshift = 1: die-affine items, two partial rows per item (k_heavy_partial<.., DIE>)
  using Gm = Geo<LOGP>;
  constexpr int UF = 4;
  const int lane = threadIdx.x & 31;
  const int gl = lane % Gm::G;
  const int grp = lane / Gm::G;
  const unsigned lowmask = Gm::G == 32 ? 0xffffffffu : ((1u << (Gm::G & 31)) - 1u);
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int per_warp = mega ? 1 : Gm::NPW;
  uint32_t my_nch = 0;
  for (int64_t base = o0 + warp * per_warp; base < o1; base += nwarps * per_warp) {
    const int64_t e = mega ? base : base + grp;
    const bool valid = e < o1;
    const int64_t j = valid ? __ldg(order + e) : 0;
    const int64_t v = valid ? __ldg(heavy_nodes + j) : 0;
    int i0 = valid ? __ldg(item_first + j) : 0, i1 = valid ? __ldg(item_first + j + 1) : 0;
    HB_CHK(!valid || (v >= 0 && v < g_chk.rows && 0 <= i0 && i0 <= i1 && i1 <= g_chk.items),
           "k_heavy_finish node / items");
    i0 <<= pshift;
    i1 <<= pshift;
    const int first = mega ? i0 + grp : i0, stride = mega ? Gm::NPW : 1;
    uint4 acc[Gm::CPL];
#pragma unroll
    for (int c = 0; c < Gm::CPL; c++) acc[c] = make_uint4(0, 0, 0, 0);
    for (int i = first; i < i1; i += stride * UF) {
      uint4 r[UF][Gm::CPL];
#pragma unroll
      for (int u = 0; u < UF; u++) {
        const int ii = i + u * stride;
#pragma unroll
        for (int c = 0; c < Gm::CPL; c++)
          r[u][c] = ii < i1 ? ldg4(partial + (size_t)ii * Gm::P + 16 * (c * Gm::G + gl))
                            : make_uint4(0, 0, 0, 0);
      }
#pragma unroll
      for (int u = 0; u < UF; u++)
#pragma unroll
        for (int c = 0; c < Gm::CPL; c++) acc[c] = bmax4(acc[c], r[u][c]);
    }
    if (mega) {
#pragma unroll
      for (int off = Gm::G; off < 32; off <<= 1)
#pragma unroll
        for (int c = 0; c < Gm::CPL; c++) acc[c] = bmax4(acc[c], shfl_xor4(acc[c], off));
    }
    const bool owner = valid && (!mega || grp == 0) && (!active || test_bit(active, v));
    bool any = false;
#pragma unroll
    for (int c = 0; c < Gm::CPL; c++) any |= nz4(acc[c]);
    any = ((__ballot_sync(0xffffffffu, any) >> (grp * Gm::G)) & lowmask) != 0u;
    const bool self_chg = owner && test_bit(chg_prev, v);
    bool changed;
    if constexpr (LOGR == 0)
      changed = finish_node<LOGP, PUSH>(peers, owner && (any || self_chg), v, acc, acc, false,
                                        self_chg, grp, gl, cur, nxt, est, sum_dist, sum_recip,
                                        ec, tf);
    else
      changed = finish_runs<LOGP, LOGR>(owner && (any || self_chg), v, acc, acc, false,
                                        self_chg, gl, cur, nxt, est, sum_dist, sum_recip, ec,
                                        tf, ra);
    if (changed && gl == 0) {
      atomicOr(chg_now + (v >> 5), 1u << (v & 31));
      if constexpr (PUSH)
        for (int q = 0; q < peers.n; q++) atomicOr(peers.chg[q] + (v >> 5), 1u << (v & 31));
      my_nch++;
    }
  }
  if constexpr (PUSH) __threadfence_system();
  block_add2(my_nch, 0u, nch_out, nullptr);
}

// Seed (engine.py:153-162): zero the row, scatter-max every replica item, estimate.
template <int LOGP>
__global__ void __launch_bounds__(kThreads)
k_seed(uint8_t *__restrict__ regs, double *__restrict__ est, int64_t n,
       const int32_t *__restrict__ perm, const int64_t *__restrict__ weights, int width,
       uint64_t seed, EstConst ec) {
  using Gm = Geo<LOGP>;
  const int b = LOGP;
  const int sat = (1 << width) - 1;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t orig = perm ? (uint64_t)__ldg(perm + i) : (uint64_t)i;
    uint8_t *row = regs + (size_t)i * Gm::P;
    for (int c = 0; c < Gm::CH; c++)
      reinterpret_cast<uint4 *>(row)[c] = make_uint4(0, 0, 0, 0);
    const int64_t w = weights ? __ldg(weights + orig) : 1;
    for (int64_t r = 1; r <= w; r++) {
      const uint64_t h = hash_item(orig, (uint64_t)r, seed);
      const uint32_t idx = (uint32_t)(h & (uint64_t)(Gm::P - 1));
      const uint64_t rest = h >> b;
      const int bitlen = rest ? 64 - __clzll((long long)rest) : 0;
      int rho = (64 - b + 1) - bitlen;  // hll.py:138-141,156
      if (rho > sat) rho = sat;
      if ((uint8_t)rho > row[idx]) row[idx] = (uint8_t)rho;
    }
    est[i] = estimate_row_thread<Gm::P>(row, ec);
  }
}

template <int LOGP>
__global__ void __launch_bounds__(kThreads)
k_estimate_rows(const uint8_t *__restrict__ regs, int64_t lo, int64_t hi, EstConst ec,
                double *__restrict__ out) {
  using Gm = Geo<LOGP>;
  for (int64_t v = lo + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < hi;
       v += (int64_t)gridDim.x * blockDim.x)
    out[v] = estimate_row_thread<Gm::P>(regs + (size_t)v * Gm::P, ec);
}

// ---- multi-GPU exchange --------------------------------------
// Pack the rows of [lo, hi) whose chg_now bit is set: ids_out[k] = v, rows_out[k] = nxt[v].
// One warp per bitmap word; positions by one atomicAdd per word (order is irrelevant:
// receivers scatter by id).
// 5-bit exchange format (register_width <= 5: every register fits 5 bits): 32 registers
// -> 5 words, a p-register row -> packed_row_bytes(p) bytes (p = 16: 12 bytes, p = 256:
// 160) -- 37.5% fewer NVLink bytes than the byte rows for p >= 32.
__host__ __device__ __forceinline__ int packed_row_bytes(int p) { return ((p * 5 + 31) / 32) * 4; }

__device__ __forceinline__ void pack_row5(const uint8_t *__restrict__ row, int p,
                                          uint32_t *__restrict__ out) {
  for (int g = 0; g < p; g += 32) {
    uint32_t w[5] = {0, 0, 0, 0, 0};
    const int cnt = p - g < 32 ? p - g : 32;
#pragma unroll
    for (int h = 0; h < 2; h++) {
      if (h * 16 >= cnt) break;
      const uint4 q = __ldg(reinterpret_cast<const uint4 *>(row + g + 16 * h));
      const uint32_t qs[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
      for (int i = 0; i < 16; i++) {
        const int r = 16 * h + i, bit = 5 * r;
        const uint32_t val = (qs[i >> 2] >> (8 * (i & 3))) & 31u;
        w[bit >> 5] |= val << (bit & 31);
        if ((bit & 31) > 27) w[(bit >> 5) + 1] |= val >> (32 - (bit & 31));
      }
    }
    const int words = (cnt * 5 + 31) / 32;
    for (int i = 0; i < words; i++) out[(g / 32) * 5 + i] = w[i];
  }
}

__device__ __forceinline__ void unpack_row5(const uint32_t *__restrict__ in, int p,
                                            uint8_t *__restrict__ row) {
  for (int g = 0; g < p; g += 32) {
    const int cnt = p - g < 32 ? p - g : 32;
    const int words = (cnt * 5 + 31) / 32;
    uint32_t w[6] = {0, 0, 0, 0, 0, 0};
    for (int i = 0; i < words; i++) w[i] = __ldg(in + (g / 32) * 5 + i);
#pragma unroll
    for (int h = 0; h < 2; h++) {
      if (h * 16 >= cnt) break;
      uint32_t qs[4] = {0, 0, 0, 0};
#pragma unroll
      for (int i = 0; i < 16; i++) {
        const int r = 16 * h + i, bit = 5 * r;
        uint32_t val = w[bit >> 5] >> (bit & 31);
        if ((bit & 31) > 27) val |= w[(bit >> 5) + 1] << (32 - (bit & 31));
        qs[i >> 2] |= (val & 31u) << (8 * (i & 3));
      }
      *reinterpret_cast<uint4 *>(row + g + 16 * h) = make_uint4(qs[0], qs[1], qs[2], qs[3]);
    }
  }
}

// Pack the rows of [lo, hi) whose chg_now bit is set: ids_out[k] = v, rows_out[k] = nxt[v]
// (byte rows, or 5-bit packed rows when packed != 0).  One warp per bitmap word;
// positions by one atomicAdd per word (order is irrelevant: receivers scatter by id).
__global__ void k_gather_changed(int64_t lo, int64_t hi, const uint32_t *__restrict__ bits,
                                 const uint8_t *__restrict__ src, int p, int packed,
                                 int32_t *__restrict__ ids_out, uint8_t *__restrict__ rows_out,
                                 unsigned long long *__restrict__ count) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t w0 = lo >> 5, w1 = (hi + 31) >> 5;
  const int rb = packed ? packed_row_bytes(p) : p;
  for (int64_t w = w0 + warp; w < w1; w += nwarps) {
    uint32_t m = __ldg(bits + w);
    const int64_t v0 = w << 5;
    if (v0 < lo) m &= ~0u << (lo - v0);
    if (v0 + 32 > hi) m &= (hi - v0 >= 32) ? ~0u : ((1u << (hi - v0)) - 1u);
    const int c = __popc(m);
    if (c == 0) continue;
    unsigned long long base = 0;
    if (lane == 0) base = atomicAdd(count, (unsigned long long)c);
    base = __shfl_sync(0xffffffffu, base, 0);
    if (lane < c) {
      const int bit = __fns(m, 0, lane + 1);
      const int64_t v = v0 + bit;
      ids_out[base + lane] = (int32_t)v;
      uint8_t *dst = rows_out + (size_t)(base + lane) * rb;
      if (packed) {
        pack_row5(src + (size_t)v * p, p, reinterpret_cast<uint32_t *>(dst));
      } else {
        const uint4 *s4 = reinterpret_cast<const uint4 *>(src + (size_t)v * p);
        uint4 *d4 = reinterpret_cast<uint4 *>(dst);
        for (int q = 0; q < p / 16; q++) d4[q] = __ldg(s4 + q);
      }
    }
  }
}

// Apply received rows: dst[ids[k]] = rows[k] (byte rows: thread per 16-byte chunk; 5-bit
// packed rows: thread per row) and set their change bits.
// Receiver side of the packed push, after the step's barrier, for every row v outside
// the rank's [lo, hi): changed this step (chg_now) -> unpacked from the inbox, where its
// owner stored it; changed only in the previous step (prev: a copy of chg_prev taken
// before it was cleared) -> nxt = cur (the lazy double buffer, refreshed locally: nothing
// crosses NVLink for it).  Only this rank writes its nxt, so a peer already in the next
// step (storing into the other inbox) cannot race it.  Thread per (row, chunk).
__global__ void k_unpack_inbox(int64_t n, int64_t lo, int64_t hi, int ch,
                               const uint32_t *__restrict__ chg_now,
                               const uint32_t *__restrict__ prev,
                               const uint8_t *__restrict__ inbox,
                               const uint8_t *__restrict__ cur, uint8_t *__restrict__ nxt) {
  const int stride = push_stride(ch);
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n * ch;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v = t / ch;
    const int ci = (int)(t - v * ch);
    if (v >= lo && v < hi) continue;
    const uint32_t bit = 1u << (v & 31);
    uint4 *dst = reinterpret_cast<uint4 *>(nxt + (size_t)v * 16 * ch) + ci;
    if (__ldg(chg_now + (v >> 5)) & bit) {
      const uint8_t *row = inbox + (size_t)v * stride;
      const uint32_t l0 = __ldg(reinterpret_cast<const uint32_t *>(row + 8 * ci));
      const uint32_t l1 = __ldg(reinterpret_cast<const uint32_t *>(row + 8 * ci + 4));
      const uint32_t h = __ldg(reinterpret_cast<const uint16_t *>(row + push_hi_off(ch, ci)));
      *dst = unpack_chunk5(l0, l1, h);
    } else if (__ldg(prev + (v >> 5)) & bit) {
      *dst = __ldg(reinterpret_cast<const uint4 *>(cur + (size_t)v * 16 * ch) + ci);
    }
  }
}
__global__ void k_scatter_rows(int64_t k, const int32_t *__restrict__ ids,
                               const uint8_t *__restrict__ rows, int p, int packed,
                               uint8_t *__restrict__ dst, uint32_t *__restrict__ bits) {
  if (packed) {
    const int rb = packed_row_bytes(p);
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < k;
         r += (int64_t)gridDim.x * blockDim.x) {
      const int64_t v = __ldg(ids + r);
      unpack_row5(reinterpret_cast<const uint32_t *>(rows + (size_t)r * rb), p,
                  dst + (size_t)v * p);
      if (bits) atomicOr(bits + (v >> 5), 1u << (v & 31));
    }
    return;
  }
  const int64_t chunks = p / 16;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < k * chunks;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = t / chunks, q = t % chunks;
    const int64_t v = __ldg(ids + r);
    reinterpret_cast<uint4 *>(dst + (size_t)v * p)[q] =
        __ldg(reinterpret_cast<const uint4 *>(rows + (size_t)r * p) + q);
    if (q == 0 && bits) atomicOr(bits + (v >> 5), 1u << (v & 31));
  }
}

// Lazy double buffer for rows this rank does not own: dst[v] = src[v] for every v outside
// [lo, hi) whose bit is set in `bits` (rows that changed last iteration).
__global__ void k_refresh_rows(int64_t n, int64_t lo, int64_t hi,
                               const uint32_t *__restrict__ bits,
                               const uint8_t *__restrict__ src, uint8_t *__restrict__ dst,
                               int p) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t words = (n + 31) >> 5;
  const int chunks = p / 16;
  for (int64_t w = warp; w < words; w += nwarps) {
    const int64_t v0 = w << 5;
    if (v0 >= lo && v0 + 32 <= hi) continue;          // fully owned
    uint32_t m = __ldg(bits + w);
    if (v0 + 32 > n) m &= (n - v0 >= 32) ? ~0u : ((1u << (n - v0)) - 1u);
    while (m) {
      const int bit = __ffs(m) - 1;
      m &= m - 1;
      const int64_t v = v0 + bit;
      if (v >= lo && v < hi) continue;
      for (int q = lane; q < chunks; q += 32)
        reinterpret_cast<uint4 *>(dst + (size_t)v * p)[q] =
            __ldg(reinterpret_cast<const uint4 *>(src + (size_t)v * p) + q);
    }
  }
}

// ---- exact backend ---------------------------------------------------
// The reference's validation backend (engine.py:178-213, _kernels.py:117-172): one bitset
// of n bits per node (MSB-first bytes, exactly the reference's rows), OR instead of max,
// weighted popcount instead of the HLL estimate -- the engine becomes a BFS oracle.  Rows
// are padded to a 16-byte stride rs.  One warp per node; the OR accumulates in the node's
// nxt row (each lane owns its chunks), so any row length works.
__global__ void k_exact_seed(int64_t n, int64_t rs, uint8_t *__restrict__ bits,
                             double *__restrict__ est, const int64_t *__restrict__ weights) {
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    bits[(size_t)v * rs + (v >> 3)] = (uint8_t)(0x80u >> (v & 7));
    est[v] = weights ? (double)__ldg(weights + v) : 1.0;
  }
}

__global__ void __launch_bounds__(kThreads)
k_exact_union(int64_t n, const int64_t *__restrict__ offsets, const int32_t *__restrict__ succ,
              const uint8_t *__restrict__ cur, uint8_t *__restrict__ nxt, int64_t rs,
              const uint32_t *__restrict__ chg_prev, uint32_t *__restrict__ chg_now,
              double *__restrict__ est, double *__restrict__ sum_dist,
              double *__restrict__ sum_recip, double tf, int dense,
              const int64_t *__restrict__ weights, const EstConst ec,
              unsigned long long *__restrict__ nch_out,
              unsigned long long *__restrict__ merged_out) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t chunks = rs / 16;
  uint32_t my_nch = 0, my_merged = 0;
  for (int64_t v = warp; v < n; v += nwarps) {
    const bool self_chg = test_bit(chg_prev, v);
    const int64_t b0 = __ldg(offsets + v), b1 = __ldg(offsets + v + 1);
    const uint4 *crow = reinterpret_cast<const uint4 *>(cur + (size_t)v * rs);
    uint4 *nrow = reinterpret_cast<uint4 *>(nxt + (size_t)v * rs);
    bool started = false;
    for (int64_t kb = b0; kb < b1; kb += 32) {
      const int64_t k = kb + lane;
      const int32_t id = k < b1 ? __ldg(succ + k) : -1;
      const bool act = id >= 0 && (dense || test_bit(chg_prev, id));
      unsigned mask = __ballot_sync(0xffffffffu, act);
      if (mask && !started) {           // first active source: nxt[v] = cur[v]
        for (int64_t c = lane; c < chunks; c += 32) nrow[c] = __ldg(crow + c);
        started = true;
      }
      my_merged += lane == 0 ? (uint32_t)__popc(mask) : 0u;
      while (mask) {
        const int src = __ffs(mask) - 1;
        mask &= mask - 1;
        const int32_t w = __shfl_sync(0xffffffffu, id, src);
        const uint4 *wrow = reinterpret_cast<const uint4 *>(cur + (size_t)w * rs);
        for (int64_t c = lane; c < chunks; c += 32) {
          uint4 a = nrow[c];
          const uint4 q = __ldg(wrow + c);
          a.x |= q.x; a.y |= q.y; a.z |= q.z; a.w |= q.w;
          nrow[c] = a;
        }
      }
    }
    if (!started) {
      if (self_chg)                     // lazy double buffer: refresh the recycled row
        for (int64_t c = lane; c < chunks; c += 32) nrow[c] = __ldg(crow + c);
      continue;
    }
    bool diff = false;
    unsigned long long cnt = 0;
    for (int64_t c = lane; c < chunks; c += 32) {
      const uint4 a = nrow[c], q = __ldg(crow + c);
      diff |= ((a.x ^ q.x) | (a.y ^ q.y) | (a.z ^ q.z) | (a.w ^ q.w)) != 0u;
      if (!weights) {
        cnt += __popc(a.x) + __popc(a.y) + __popc(a.z) + __popc(a.w);
      } else {
        const uint32_t ws[4] = {a.x, a.y, a.z, a.w};
        for (int q4 = 0; q4 < 4; q4++) {
          uint32_t x = ws[q4];
          while (x) {                   // byte j of the word, bit 7-k of the byte -> node
            const int bit = __ffs(x) - 1;
            x &= x - 1;
            const int64_t node = (c * 16 + q4 * 4 + (bit >> 3)) * 8 + (7 - (bit & 7));
            cnt += (unsigned long long)__ldg(weights + node);
          }
        }
      }
    }
    const bool changed = __any_sync(0xffffffffu, diff);
    if (changed) {
      for (int off = 16; off > 0; off >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, off);
      if (lane == 0) {
        const double e = (double)cnt;
        const double d = np_max0(__dsub_rn(e, est[v]));
        est[v] = e;
        if (sum_dist) sum_dist[v] = __dadd_rn(sum_dist[v], __dmul_rn(tf, d));
        if (sum_recip) sum_recip[v] = __dadd_rn(sum_recip[v], __ddiv_rn(d, tf));
        for (int k = 0; k < ec.n_disc; k++) {
          double *q = ec.disc + k * ec.disc_stride + v;
          const double c = ((ec.disc_div >> k) & 1) ? __ddiv_rn(d, tf)
                                                    : __dmul_rn(ec.disc_scale[k], d);
          *q = __dadd_rn(*q, c);
        }
        atomicOr(chg_now + (v >> 5), 1u << (v & 31));
        my_nch++;
      }
    }
  }
  block_add2(my_nch, my_merged, nch_out, merged_out);
}

// ---- frontier mode (sparse iterations) -------------------------------------------------
// active = chg_prev | out-neighbours(chg_prev) over the forward graph G: exactly the nodes
// the source-skip rule can change this iteration, plus the changed rows themselves (their
// recycled-buffer copy must be refreshed).  Warp per bitmap word of chg_prev.
__global__ void k_mark_active(int64_t n, const int64_t *__restrict__ fwd_off,
                              const int32_t *__restrict__ fwd_succ,
                              const uint32_t *__restrict__ chg_prev,
                              uint32_t *__restrict__ active) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t words = (n + 31) >> 5;
  for (int64_t wd = warp; wd < words; wd += nwarps) {
    uint32_t m = __ldg(chg_prev + wd);
    if ((wd << 5) + 32 > n) m &= (n - (wd << 5) >= 32) ? ~0u : ((1u << (n - (wd << 5))) - 1u);
    if (m == 0) continue;
    if (lane == 0) atomicOr(active + wd, m);
    while (m) {
      const int64_t w = (wd << 5) + __ffs(m) - 1;
      m &= m - 1;
      const int64_t b0 = __ldg(fwd_off + w), b1 = __ldg(fwd_off + w + 1);
      for (int64_t k = b0 + lane; k < b1; k += 32) {
        const int32_t d = __ldg(fwd_succ + k);
        atomicOr(active + (d >> 5), 1u << (d & 31));
      }
    }
  }
}

// The same frontier without a forward graph: active[v] = chg_prev[v] | any chg_prev[id],
// id in row v of G^T.  Light rows: one warp per 32 consecutive nodes; when their rows
// are short in total the warp streams the whole (contiguous) id range coalesced and a
// changed source marks its row's owner, found by a vote over the 33 row offsets held one
// per lane; otherwise it walks the light rows one by one.  Heavy rows (in-degree >
// light_max_deg) are skipped here and marked by k_mark_items over the schedule's work
// items, so every warp streams a bounded number of ids.  Every bitmap word is written by
// one warp of k_mark_pull (k_mark_items, launched after it, only ORs bits in).
// Change filter for the pull marking of nearly converged steps: a 2^18-bit hash bitmap of
// the changed nodes (a few thousand at most), copied into shared memory by every block,
// so the per-id test of a streamed successor id is a shared-memory lookup and the global
// change bitmap is read only on a filter hit.
constexpr int kFilterBits = 18;
constexpr int kFilterWords = (1 << kFilterBits) / 32;
__device__ __forceinline__ uint32_t filter_slot(int64_t v) {
  return ((uint32_t)v * 0x9E3779B1u) >> (32 - kFilterBits);
}
__global__ void k_build_filter(int64_t n, const uint32_t *__restrict__ bits,
                               uint32_t *__restrict__ filter) {
  const int64_t words = (n + 31) >> 5;
  for (int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w < words;
       w += (int64_t)gridDim.x * blockDim.x) {
    uint32_t b = __ldg(bits + w);
    while (b) {
      const int i = __ffs(b) - 1;
      b &= b - 1u;
      const uint32_t h = filter_slot((w << 5) + i);
      atomicOr(filter + (h >> 5), 1u << (h & 31));
    }
  }
}
template <bool FILT>
struct ChangeTest {
  const uint32_t *bits;
  uint32_t *sf;   // shared filter (FILT)
  __device__ __forceinline__ bool operator()(int64_t v) const {
    if constexpr (FILT) {
      const uint32_t h = filter_slot(v);
      if (!((sf[h >> 5] >> (h & 31)) & 1u)) return false;
    }
    return test_bit(bits, v);
  }
};
template <bool FILT>
__device__ __forceinline__ ChangeTest<FILT> make_change_test(const uint32_t *bits,
                                                             const uint32_t *filter) {
  ChangeTest<FILT> t{bits, nullptr};
  if constexpr (FILT) {
    extern __shared__ uint32_t dyn_filter[];
    for (int i = threadIdx.x; i < kFilterWords; i += blockDim.x) dyn_filter[i] = __ldg(filter + i);
    __syncthreads();
    t.sf = dyn_filter;
  }
  return t;
}

template <bool FILT>
__global__ void k_mark_pull(int64_t n, const int64_t *__restrict__ offsets,
                            const int32_t *__restrict__ succ,
                            const uint32_t *__restrict__ chg_prev, uint32_t *__restrict__ active,
                            int64_t light_max_deg, const uint32_t *__restrict__ filter) {
  const auto changed = make_change_test<FILT>(chg_prev, filter);
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t v0 = warp * 32; v0 < n; v0 += nwarps * 32) {
    const int64_t v = v0 + lane;
    const int64_t my_off = __ldg(offsets + (v < n ? v : n));
    const int64_t my_end = __ldg(offsets + (v + 1 < n ? v + 1 : n));
    const int64_t a0 = __shfl_sync(0xffffffffu, my_off, 0);
    const int64_t a1 = __shfl_sync(0xffffffffu, my_end, 31);
    bool mark = v < n && changed(v);
    const bool heavy = v < n && my_end - my_off > light_max_deg;
    const unsigned heavy_mask = __ballot_sync(0xffffffffu, heavy);
    if (heavy_mask == 0u && a1 - a0 <= 32 * 64) {
      constexpr int IL = 4;               // independent id loads per lane in flight
      for (int64_t kb = a0; kb < a1; kb += 32 * IL) {
        int32_t id[IL];
#pragma unroll
        for (int j = 0; j < IL; j++) {
          const int64_t k = kb + j * 32 + lane;
          id[j] = k < a1 ? __ldg(succ + k) : -1;
        }
        bool hit[IL];
#pragma unroll
        for (int j = 0; j < IL; j++) hit[j] = id[j] >= 0 && changed(id[j]);
#pragma unroll
        for (int j = 0; j < IL; j++) {
          unsigned bal = __ballot_sync(0xffffffffu, hit[j]);
          while (bal) {                   // warp-uniform
            const int64_t kk = kb + j * 32 + __ffs(bal) - 1;
            bal &= bal - 1;
            const int owner = __popc(__ballot_sync(0xffffffffu, my_off <= kk)) - 1;
            mark |= lane == owner;
          }
        }
      }
    } else {
      for (int r = 0; r < 32; r++) {      // light rows one by one (<= light_max_deg ids)
        const int64_t b0 = __shfl_sync(0xffffffffu, my_off, r);
        const int64_t b1 = __shfl_sync(0xffffffffu, my_end, r);
        if (((heavy_mask >> r) & 1u) || v0 + r >= n) continue;
        bool any = false;
        for (int64_t k = b0 + lane; k < b1; k += 32) any |= changed(__ldg(succ + k));
        if (__any_sync(0xffffffffu, any)) mark |= lane == r;
      }
    }
    const unsigned word = __ballot_sync(0xffffffffu, mark);
    if (lane == 0) active[v0 >> 5] = word;
  }
}

// Heavy rows of the pull marking: one warp per work item (<= item_arcs ids of one node).
template <bool FILT>
__global__ void k_mark_items(const int64_t *__restrict__ offsets, const int32_t *__restrict__ succ,
                             const uint32_t *__restrict__ chg_prev,
                             const int32_t *__restrict__ item_node,
                             const int64_t *__restrict__ item_beg, int64_t n_items,
                             int64_t item_arcs, uint32_t *__restrict__ active,
                             const uint32_t *__restrict__ filter) {
  const auto changed = make_change_test<FILT>(chg_prev, filter);
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t it = warp; it < n_items; it += nwarps) {
    const int64_t v = __ldg(item_node + it);
    const int64_t beg = __ldg(item_beg + it);
    int64_t end = __ldg(offsets + v + 1);
    if (end > beg + item_arcs) end = beg + item_arcs;
    bool any = false;
    constexpr int IL = 4;                 // independent id loads per lane in flight
    for (int64_t kb = beg; kb < end; kb += 32 * IL) {
      int32_t id[IL];
#pragma unroll
      for (int j = 0; j < IL; j++) {
        const int64_t k = kb + j * 32 + lane;
        id[j] = k < end ? ld_stream_id(succ + k) : -1;
      }
#pragma unroll
      for (int j = 0; j < IL; j++) any |= id[j] >= 0 && changed(id[j]);
    }
    if (__any_sync(0xffffffffu, any) && lane == 0 && !test_bit(active, v))
      atomicOr(active + (v >> 5), 1u << (v & 31));
  }
}

// Heavy rows of the pull marking when they are one contiguous row range [h0, h1) (the
// degree order's prefix): their ids [offsets[h0], offsets[h1]) are streamed flat, IL
// loads per lane in flight, and a changed source marks its row, found by binary search
// over the range's offsets (rare: only on hits).
template <bool FILT>
__global__ void k_mark_heavy_flat(const int64_t *__restrict__ offsets,
                                  const int32_t *__restrict__ succ,
                                  const uint32_t *__restrict__ chg_prev, int64_t h0, int64_t h1,
                                  uint32_t *__restrict__ active,
                                  const uint32_t *__restrict__ filter) {
  const auto changed = make_change_test<FILT>(chg_prev, filter);
  const int64_t a0 = __ldg(offsets + h0), a1 = __ldg(offsets + h1);
  auto hit = [&](int64_t k) {                // id at arc k changed: mark its row
    int64_t lo = h0, hi = h1;                // last row r with offsets[r] <= k
    while (hi - lo > 1) {
      const int64_t mid = (lo + hi) >> 1;
      if (__ldg(offsets + mid) <= k) lo = mid; else hi = mid;
    }
    if (!test_bit(active, lo)) atomicOr(active + (lo >> 5), 1u << (lo & 31));
  };
  // 16-byte id loads (4 ids each, IL in flight per thread) over the aligned body; the
  // unaligned head and tail (< 4 ids each) by the first threads
  const int64_t b0 = (a0 + 3) & ~(int64_t)3, b1 = a1 & ~(int64_t)3;
  const int64_t gt = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (gt < 8) {
    const int64_t k = gt < 4 ? a0 + gt : b1 + (gt - 4);
    if ((gt < 4 ? k < b0 && k < a1 : k < a1 && k >= b0) && changed(__ldg(succ + k))) hit(k);
  }
  if (b1 > b0) {
    constexpr int IL = 4;
    const int4 *q = reinterpret_cast<const int4 *>(succ + b0);
    const int64_t nq = (b1 - b0) >> 2;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x * IL;
    for (int64_t qb = (int64_t)blockIdx.x * blockDim.x * IL; qb < nq; qb += stride) {
      int4 v[IL];
#pragma unroll
      for (int j = 0; j < IL; j++) {
        const int64_t i = qb + (int64_t)j * blockDim.x + threadIdx.x;
        v[j] = i < nq ? ld_stream_ids4(q + i) : make_int4(-1, -1, -1, -1);
      }
#pragma unroll
      for (int j = 0; j < IL; j++) {
        const int64_t k = b0 + 4 * (qb + (int64_t)j * blockDim.x + threadIdx.x);
        if (v[j].x >= 0 && changed(v[j].x)) hit(k);
        if (v[j].y >= 0 && changed(v[j].y)) hit(k + 1);
        if (v[j].z >= 0 && changed(v[j].z)) hit(k + 2);
        if (v[j].w >= 0 && changed(v[j].w)) hit(k + 3);
      }
    }
  }
}

// Forward CSR by counting sort (row order inside a forward row is irrelevant for marking):
// count out-degrees with atomics, exclusive scan, scatter with per-source cursors.
// Warp-aggregated: lanes holding the same source (hubs on R-MAT) issue one atomic.
__global__ void k_count_src(int64_t m, const int32_t *__restrict__ succ,
                            unsigned long long *__restrict__ cnt) {
  const int lane = threadIdx.x & 31;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < m; base += stride) {
    const int64_t k = base + threadIdx.x;
    const bool ok = k < m;
    const int32_t src = ok ? __ldg(succ + k) : -1;
    const unsigned peers = __match_any_sync(0xffffffffu, src);
    if (ok && lane == __ffs(peers) - 1) atomicAdd(cnt + src, (unsigned long long)__popc(peers));
  }
}

// Sampled share of arcs whose source is flagged in `bits`: thread i tests the source of
// arc splitmix(seed + i) mod m; one atomic per block with the block's hit count.
__global__ void k_sample_flagged(int64_t m, const int32_t *__restrict__ succ,
                                 const uint32_t *__restrict__ bits, int64_t samples,
                                 uint64_t seed, unsigned long long *__restrict__ out) {
  uint32_t hits = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < samples;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = (int64_t)(mix64(seed + (uint64_t)i) % (uint64_t)m);
    const int32_t v = __ldg(succ + k);
    hits += (__ldg(bits + (v >> 5)) >> (v & 31)) & 1u;
  }
  hits = __reduce_add_sync(0xffffffffu, hits);
  __shared__ uint32_t red[kThreads / 32];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = hits;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t t = 0;
    for (int i = 0; i < (int)(blockDim.x >> 5); i++) t += red[i];
    if (t) atomicAdd(out, (unsigned long long)t);
  }
}

__global__ void k_scatter_fwd(int64_t n, const int64_t *__restrict__ off,
                              const int32_t *__restrict__ succ,
                              unsigned long long *__restrict__ cursor,
                              int32_t *__restrict__ fwd_dst) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t v = warp; v < n; v += nwarps) {
    const int64_t b0 = __ldg(off + v), b1 = __ldg(off + v + 1);
    for (int64_t kb = b0; kb < b1; kb += 32) {     // warp-uniform trip count
      const int64_t k = kb + lane;
      const bool ok = k < b1;
      const int32_t src = ok ? __ldg(succ + k) : -1;
      const unsigned peers = __match_any_sync(0xffffffffu, src);
      const int leader = __ffs(peers) - 1;
      unsigned long long pos = 0;
      if (ok && lane == leader) pos = atomicAdd(cursor + src, (unsigned long long)__popc(peers));
      pos = __shfl_sync(0xffffffffu, pos, leader);
      if (ok) fwd_dst[pos + __popc(peers & ((1u << lane) - 1u))] = (int32_t)v;
    }
  }
}

// ---- GPU graph build ---------------------------------------------
// Counter-based R-MAT arcs, bit-identical to graphgen.c's rmat_fn (same splitmix chain,
// same 32-bit quadrant thresholds), packed as (dst << 32 | src) keys of the TRANSPOSE;
// self-loops become the sentinel ~0 and are dropped after the sort.
__device__ __forceinline__ uint64_t gg_rng3(uint64_t seed, uint64_t stream, uint64_t a,
                                            uint64_t b) {
  return mix64(mix64(mix64(seed * 0x9E3779B97F4A7C15ull + stream) + a) + b);
}

__global__ void k_gen_rmat(int scale, int64_t m, uint64_t A, uint64_t AB, uint64_t ABC,
                           uint64_t seed, uint64_t *__restrict__ keys) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < m;
       k += (int64_t)gridDim.x * blockDim.x) {
    uint64_t s = 0, d = 0, r = 0;
    for (int l = 0; l < scale; l++) {
      uint64_t x;
      if ((l & 1) == 0) {
        r = gg_rng3(seed, 4, (uint64_t)k, (uint64_t)(l >> 1));
        x = r & 0xffffffffull;
      } else {
        x = r >> 32;
      }
      const int q = x < A ? 0 : (x < AB ? 1 : (x < ABC ? 2 : 3));
      s = (s << 1) | (uint64_t)(q >> 1);
      d = (d << 1) | (uint64_t)(q & 1);
    }
    keys[k] = (s == d) ? ~0ull : ((d << 32) | s);
  }
}

// CSR of the sorted unique keys [0, mu): thread per key position k in [0, mu]; the rows
// from the previous key's dst + 1 up to this key's dst all start at k (empty rows
// included); position mu closes every remaining row.  succ[k] = src of key k.
__global__ void k_keys_to_csr(int64_t n, int64_t mu, const uint64_t *__restrict__ keys,
                              int64_t *__restrict__ offsets, int32_t *__restrict__ succ) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k <= mu;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t d = k < mu ? (int64_t)(__ldg(keys + k) >> 32) : n;
    const int64_t prev = k > 0 ? (int64_t)(__ldg(keys + k - 1) >> 32) : -1;
    for (int64_t v = prev + 1; v <= d; v++) offsets[v] = k;
    if (k < mu) succ[k] = (int32_t)(__ldg(keys + k) & 0xffffffffull);
  }
}

// Out-degree laws and arc targets of the other synthetic configs, bit-identical to
// graphgen.c's out_degree / fill_fn (same counter-based draws, same double arithmetic:
// u01 is exact, the Poisson / Zipf CDF tables are built on the host by the same C code
// and uploaded, `below` is the 64x64 -> high-64 product).
enum { GG_ER = 1, GG_DISC = 3, GG_WEB = 4 };
__device__ __forceinline__ double gg_u01(uint64_t x) { return (double)(x >> 11) * 0x1.0p-53; }
__device__ __forceinline__ uint64_t gg_below(uint64_t x, uint64_t n) { return __umul64hi(x, n); }

__global__ void k_gen_degree(int kind, int64_t n, uint64_t seed, const double *__restrict__ cdf,
                             int64_t cdf_len, int64_t kmin, int64_t *__restrict__ deg) {
  for (int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; u < n;
       u += (int64_t)gridDim.x * blockDim.x) {
    const double x = gg_u01(gg_rng3(seed, 1, (uint64_t)u, 0));
    int64_t k;
    if (kind == GG_WEB) {                 // zipf_draw: first i with x < cdf[i]
      int64_t lo = 0, hi = cdf_len - 1;
      while (lo < hi) {
        const int64_t mid = (lo + hi) / 2;
        if (x < __ldg(cdf + mid)) hi = mid; else lo = mid + 1;
      }
      k = kmin + lo;
    } else {                              // poisson_draw: linear scan of the CDF
      k = 0;
      while (x >= __ldg(cdf + k)) k++;
    }
    deg[u] = k;
  }
}

// Geometric(p) block sizes of the disconnected config: block b has size = number of
// trials up to the first success of rng3(seed, 5, b, trial) < p (graphgen.c generate()).
__global__ void k_gen_block_sizes(int64_t nblocks, uint64_t seed, double geo_p,
                                  int64_t *__restrict__ size) {
  for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < nblocks;
       b += (int64_t)gridDim.x * blockDim.x) {
    int64_t k = 1;
    while (gg_u01(gg_rng3(seed, 5, (uint64_t)b, (uint64_t)k)) >= geo_p) k++;
    size[b] = k;
  }
}
// Block bounds per node: block b covers [giant + start[b], giant + start[b] + size[b]) cut
// at n (start = exclusive prefix sum of the sizes); the giant block is [0, giant).
__global__ void k_gen_block_bounds(int64_t n, int64_t giant, int64_t nblocks,
                                   const int64_t *__restrict__ start,
                                   const int64_t *__restrict__ size, int64_t *__restrict__ lo,
                                   int64_t *__restrict__ hi) {
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < giant;
       v += (int64_t)gridDim.x * blockDim.x) {
    lo[v] = 0;
    hi[v] = giant;
  }
  for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < nblocks;
       b += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p0 = giant + __ldg(start + b);
    if (p0 >= n) continue;
    int64_t p1 = p0 + __ldg(size + b);
    if (p1 > n) p1 = n;
    for (int64_t v = p0; v < p1; v++) {
      lo[v] = p0;
      hi[v] = p1;
    }
  }
}

// Arcs of source u at positions off[u]..off[u+1] as transpose keys (dst << 32 | src);
// self-loops become the sentinel ~0 (dropped by hb_keys_to_csr).  Warp per source.
__global__ void k_gen_arcs(int kind, int64_t n, uint64_t seed, const int64_t *__restrict__ off,
                           const int64_t *__restrict__ blo, const int64_t *__restrict__ bhi,
                           double p_local, int64_t window, uint64_t *__restrict__ keys) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t u = warp; u < n; u += nwarps) {
    const int64_t base = __ldg(off + u), k = __ldg(off + u + 1) - base;
    for (int64_t j = lane; j < k; j += 32) {
      const uint64_t r = gg_rng3(seed, 2, (uint64_t)u, (uint64_t)j);
      int64_t v;
      if (kind == GG_ER) {
        v = (int64_t)gg_below(r, (uint64_t)(n - 1));
        if (v >= u) v++;
      } else if (kind == GG_DISC) {
        const int64_t a = __ldg(blo + u), b = __ldg(bhi + u);
        v = a + (int64_t)gg_below(r, (uint64_t)(b - a));
      } else {
        const uint64_t r2 = gg_rng3(seed, 3, (uint64_t)u, (uint64_t)j);
        if (gg_u01(r) < p_local) {
          const int64_t o = 1 + (int64_t)gg_below(r2 >> 1, (uint64_t)window);
          v = (r2 & 1) ? u + o : u - o;
          v %= n;
          if (v < 0) v += n;
        } else {
          v = (int64_t)gg_below(r2, (uint64_t)n);
        }
      }
      keys[base + j] = (v == u) ? ~0ull : (((uint64_t)v << 32) | (uint64_t)u);
    }
  }
}

// Keys of the transpose of a CSR (forward graph G): arc (u -> v) becomes (v << 32 | u).
// Warp per row.  Sorting these keys gives the reference's transpose order exactly
// (graph.py:145-155: stable argsort by target of arcs listed by ascending source).
__global__ void k_transpose_keys(int64_t n, const int64_t *__restrict__ off,
                                 const int32_t *__restrict__ succ, uint64_t *__restrict__ keys) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t u = warp; u < n; u += nwarps) {
    const int64_t b0 = __ldg(off + u), b1 = __ldg(off + u + 1);
    for (int64_t k = b0 + lane; k < b1; k += 32)
      keys[k] = ((uint64_t)(uint32_t)__ldg(succ + k) << 32) | (uint64_t)u;
  }
}

__global__ void k_count_valid(const uint64_t *__restrict__ keys, const int64_t *num,
                              int64_t *__restrict__ out) {
  // keys sorted and unique: the sentinel, if present, is the last one
  const int64_t u = *num;
  *out = (u > 0 && keys[u - 1] == ~0ull) ? u - 1 : u;
}

// Finalizers (centrality.py:153-171), optionally gathering from internal order:
// out[o] for original id o reads internal row rank[o].  Explicitly rounded fp64 ops.
__global__ void k_finalize(int64_t n, const int32_t *__restrict__ rank,
                           const double *__restrict__ sum_dist,
                           const double *__restrict__ sum_recip,
                           const double *__restrict__ coreach, double *__restrict__ closeness,
                           double *__restrict__ harmonic, double *__restrict__ lin) {
  for (int64_t o = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; o < n;
       o += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v = rank ? (int64_t)__ldg(rank + o) : o;
    if (harmonic) harmonic[o] = __ldg(sum_recip + v);
    if (closeness || lin) {
      const double s = __ldg(sum_dist + v);
      if (closeness) closeness[o] = s > 0.0 ? __ddiv_rn(1.0, s) : 0.0;
      if (lin) {
        const double c = __ldg(coreach + v);
        lin[o] = s > 0.0 ? __ddiv_rn(__dmul_rn(c, c), s) : 1.0;
      }
    }
  }
}

// Id map lookup rank[id] for the relabel kernels: a random 4-byte read of a table of n
// entries (1 GB at config 5) that mostly misses L2; `.L2::64B` halves the DRAM line
// fetched per miss (HB_RELABEL_64B).
#ifndef HB_RELABEL_64B
#define HB_RELABEL_64B 1
#endif
__device__ __forceinline__ int32_t ld_rank(const int32_t *rank, int32_t id) {
#if HB_RELABEL_64B
  int32_t r;
  asm("ld.global.nc.L2::64B.s32 %0, [%1];" : "=r"(r) : "l"(rank + id));
  return r;
#else
  return __ldg(rank + id);
#endif
}
__global__ void k_relabel(int64_t r0, int64_t r1, const int64_t *__restrict__ old_off,
                          const int32_t *__restrict__ old_succ, const int32_t *__restrict__ perm,
                          const int32_t *__restrict__ rank, const int64_t *__restrict__ new_off,
                          int32_t *__restrict__ new_succ) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = r0 + warp; i < r1; i += nwarps) {
    const int64_t o = __ldg(perm + i);
    const int64_t b0 = __ldg(old_off + o), len = __ldg(old_off + o + 1) - b0;
    const int64_t d0 = __ldg(new_off + i);
    for (int64_t k = lane; k < len; k += 32) new_succ[d0 + k] = ld_rank(rank, __ldg(old_succ + b0 + k));
  }
}

// Scatter form of k_relabel over OLD rows [o0, o1): old row o becomes new row rank[o].
// Lets the degree relabel run on each slice of the upload as soon as it has landed.
__global__ void k_relabel_src(int64_t o0, int64_t o1, const int64_t *__restrict__ old_off,
                              const int32_t *__restrict__ old_succ,
                              const int32_t *__restrict__ rank,
                              const int64_t *__restrict__ new_off,
                              int32_t *__restrict__ new_succ) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t o = o0 + warp; o < o1; o += nwarps) {
    const int64_t b0 = __ldg(old_off + o), len = __ldg(old_off + o + 1) - b0;
    const int64_t d0 = __ldg(new_off + __ldg(rank + o));
    for (int64_t k = lane; k < len; k += 32) new_succ[d0 + k] = ld_rank(rank, __ldg(old_succ + b0 + k));
  }
}

__global__ void k_map_ids(int64_t m, const int32_t *ids, const int32_t *__restrict__ rank,
                          int32_t *out) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < m;
       k += (int64_t)gridDim.x * blockDim.x)
    out[k] = ld_rank(rank, ids[k]);
}

__global__ void k_hash(int64_t n, const uint64_t *__restrict__ items,
                       const uint64_t *__restrict__ replicas, uint64_t seed,
                       uint64_t *__restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = hash_item(items[i], replicas[i], seed);
}

// The at-rest register format (hll.py:128-132, 161-177: CounterArray.registers and the HLLA
// blob): each register's `width` low bits, most significant first, concatenated over the
// row, rows back to back (p * width / 8 bytes each).  8 registers make `width` whole
// bytes, so one thread packs / unpacks one group of 8.  `order` (may be NULL) reorders rows:
// packed row i <-> register row order[i] (the schedule's rank / perm).
__global__ void k_pack_registers(int64_t n, int p, int width, const uint8_t *__restrict__ regs,
                                 const int32_t *__restrict__ order, uint8_t *__restrict__ out) {
  const int groups = p / 8;
  const int64_t total = n * groups;
  const uint32_t mask = (1u << width) - 1u;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = i / groups;
    const int g = (int)(i - row * groups);
    const int64_t src = order ? (int64_t)__ldg(order + row) : row;
    const uint2 r = __ldg(reinterpret_cast<const uint2 *>(regs + src * p + g * 8));
    uint64_t acc = 0;
#pragma unroll
    for (int j = 0; j < 8; j++) {
      const uint32_t m = ((j < 4 ? r.x : r.y) >> (8 * (j & 3))) & mask;
      acc = (acc << width) | m;
    }
    uint8_t *o = out + row * ((int64_t)p * width / 8) + (int64_t)g * width;
    for (int k = 0; k < width; k++) o[k] = (uint8_t)(acc >> (8 * (width - 1 - k)));
  }
}

__global__ void k_unpack_registers(int64_t n, int p, int width, const uint8_t *__restrict__ in,
                                   const int32_t *__restrict__ order, uint8_t *__restrict__ regs) {
  const int groups = p / 8;
  const int64_t total = n * groups;
  const uint32_t mask = (1u << width) - 1u;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = i / groups;
    const int g = (int)(i - row * groups);
    const int64_t src = order ? (int64_t)__ldg(order + row) : row;
    const uint8_t *q = in + src * ((int64_t)p * width / 8) + (int64_t)g * width;
    uint64_t acc = 0;
    for (int k = 0; k < width; k++) acc = (acc << 8) | __ldg(q + k);
    uint32_t lo = 0, hi = 0;
#pragma unroll
    for (int j = 0; j < 8; j++) {
      const uint32_t m = (uint32_t)(acc >> (width * (7 - j))) & mask;
      if (j < 4) lo |= m << (8 * j); else hi |= m << (8 * (j - 4));
    }
    *reinterpret_cast<uint2 *>(regs + row * p + g * 8) = make_uint2(lo, hi);
  }
}

// out[r] = popcount of bitmap row r (rows of `words` uint32): per-run changed counts of a
// batched step.  One block per row.
__global__ void k_count_bits(const uint32_t *__restrict__ bits, int64_t words,
                             unsigned long long *__restrict__ out) {
  const uint32_t *row = bits + (int64_t)blockIdx.x * words;
  uint32_t c = 0;
  for (int64_t i = threadIdx.x; i < words; i += blockDim.x) c += __popc(__ldg(row + i));
  __shared__ uint32_t red[32];
  c = __reduce_add_sync(0xffffffffu, c);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x < 32) {
    uint32_t x = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0u;
    x = __reduce_add_sync(0xffffffffu, x);
    if (threadIdx.x == 0) out[blockIdx.x] = x;
  }
}

// ------------------------------------------------------------------ launch helpers
// Device-scoped state.  Every C-ABI entry point that launches work first makes the
// stream's device current (DevGuard), so a host that drives several GPUs from one thread
// may call it with any current device; everything cached below is kept per device
// ordinal (SM count, L2 set-aside, opt-in shared-memory sizes).
constexpr int kMaxDevices = 64;

// ---- L2 die maps (die-affine heavy items, see k_heavy_partial) ----------------------
// An atomic executes at the home L2 slice of its address: from an SM of the other die it
// takes ~400 cycles longer on a B200 (tools/die_probe.cu: 263-291 against 656-727 cycles),
// so the latency of atomicOr(p, 0) -- which leaves the data alone -- tells the dies apart.
__device__ __forceinline__ uint32_t timed_atomic(uint32_t *p, int reps) {
  __shared__ uint32_t sink_word[32];
  const uint32_t sink = (uint32_t)__cvta_generic_to_shared(sink_word + (threadIdx.x & 31));
  uint32_t best = 0xffffffffu;
  for (int r = 0; r < reps; r++) {
    long long t0, t1;
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(t0) :: "memory");
    const uint32_t v = atomicOr(p, 0u);
    // the store needs v: the second clock read issues after the atomic has returned
    asm volatile("st.volatile.shared.u32 [%0], %1;" :: "r"(sink), "r"(v) : "memory");
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(t1) :: "memory");
    const uint32_t d = (uint32_t)(t1 - t0);
    best = d < best ? d : best;
  }
  return best;
}
// word to probe in chunk c of the 2 KB grid over [base, base + bytes)
__device__ __forceinline__ uint32_t *probe_word(uint8_t *base, int64_t bytes, int64_t c) {
  const uintptr_t b = reinterpret_cast<uintptr_t>(base);
  uintptr_t a = ((b >> 11) + (uintptr_t)c) << 11;
  a = a < b ? ((b + 3) & ~(uintptr_t)3) : a;
  const uintptr_t lim = b + (uintptr_t)bytes - 4;
  return reinterpret_cast<uint32_t *>(a < lim ? a : (lim & ~(uintptr_t)3));
}
constexpr int kDieTest = 128;      // test chunks of the SM classification
// one warp per SM (the first CTA to claim it): latency of kDieTest spread-out chunks
__global__ void k_sm_probe(uint8_t *base, int64_t bytes, int64_t stride, int *claimed,
                           uint32_t *lat) {
  __shared__ int mine;
  const uint32_t sm = sm_id() & 255u;
  if (threadIdx.x == 0) mine = atomicCAS(claimed + sm, 0, 1) == 0;
  __syncthreads();
  if (!mine || threadIdx.x != 0) return;
  for (int k = 0; k < kDieTest; k++)
    lat[sm * kDieTest + k] = timed_atomic(probe_word(base, bytes, k * stride), 6);
}
// every chunk timed from both dies (chunks dealt 16 at a time by a counter per die)
__global__ void k_chunk_probe(uint8_t *base, int64_t bytes, int64_t chunks, unsigned int *next,
                              uint32_t *lat2) {
  const int d = g_sm_die[sm_id() & 255u] & 1;
  if (threadIdx.x != 0) return;
  for (;;) {
    const int64_t c0 = (int64_t)atomicAdd(next + d, 16u);
    if (c0 >= chunks) break;
    for (int64_t c = c0; c < c0 + 16 && c < chunks; c++)
      lat2[d * chunks + c] = timed_atomic(probe_word(base, bytes, c), 4);
  }
}
// bit c = 1 when die 1 is closer; stats: [chunks on die 1, chunks with a gap < 64 cycles]
__global__ void k_chunk_bits(const uint32_t *__restrict__ lat2, int64_t chunks,
                             uint32_t *__restrict__ bits, unsigned long long *stats) {
  const int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (w >= (chunks + 31) / 32) return;
  uint32_t m = 0;
  int ones = 0, weak = 0;
  for (int i = 0; i < 32 && w * 32 + i < chunks; i++) {
    const int64_t c = w * 32 + i;
    const int a = (int)lat2[c], b = (int)lat2[chunks + c];
    if (b < a) { m |= 1u << i; ones++; }
    weak += (a > b ? a - b : b - a) < 64;
  }
  bits[w] = m;
  atomicAdd(stats, (unsigned long long)ones);
  atomicAdd(stats + 1, (unsigned long long)weak);
}

// Reorder the ids of every heavy item by the pass that merges them (see k_heavy_partial):
// pass 0 = the sources whose head row is homed on die 0, pass 1 those of die 1; the cold
// sources (ids >= die_rows, read from DRAM wherever they live) fill pass 0 up to half of
// the item, the rest go to pass 1, so both passes are as even as the hot ids allow (a pass
// of 257 ids would cost a second, almost empty, batch of row loads).  The order inside a
// class is kept.  One warp per item (<= 512 ids); split[i] = ids of pass 0.
constexpr int kDieItemMax = 512;
__global__ void __launch_bounds__(kThreads)
k_die_partition(int64_t n_items, const int32_t *__restrict__ item_node,
                const int64_t *__restrict__ item_beg, const int64_t *__restrict__ offsets,
                int32_t *succ, int64_t item_arcs, int logp, uint32_t head_off, int64_t die_rows,
                const uint32_t *__restrict__ die_bits, int32_t *__restrict__ split) {
  __shared__ int32_t buf[kThreads / 32][3][kDieItemMax];
  const int lane = threadIdx.x & 31;
  const unsigned below = (1u << lane) - 1u;
  int32_t(*my)[kDieItemMax] = buf[threadIdx.x >> 5];
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t it = warp; it < n_items; it += nwarps) {
    const int64_t v = __ldg(item_node + it);
    const int64_t beg = __ldg(item_beg + it);
    int64_t end = __ldg(offsets + v + 1);
    if (end > beg + item_arcs) end = beg + item_arcs;
    int n[3] = {0, 0, 0};
    for (int64_t k = beg; k < end; k += 32) {
      const bool ok = k + lane < end;
      const uint32_t id = ok ? (uint32_t)succ[k + lane] : 0u;
      const uint32_t c = (head_off + (id << logp)) >> 11;
      const int cls = (int64_t)id < die_rows ? (int)((__ldg(die_bits + (c >> 5)) >> (c & 31)) & 1u) : 2;
#pragma unroll
      for (int q = 0; q < 3; q++) {
        const unsigned bq = __ballot_sync(0xffffffffu, ok && cls == q);
        if (ok && cls == q) my[q][n[q] + __popc(bq & below)] = (int32_t)id;
        n[q] += __popc(bq);
      }
    }
    __syncwarp();
    const int total = n[0] + n[1] + n[2];
    int c0 = (total + 1) / 2 - n[0];             // cold ids of pass 0
    c0 = c0 < 0 ? 0 : (c0 > n[2] ? n[2] : c0);
    const int p0 = n[0] + c0;
    for (int i = lane; i < total; i += 32) {
      int32_t id;
      if (i < n[0]) id = my[0][i];
      else if (i < p0) id = my[2][i - n[0]];
      else if (i < p0 + n[1]) id = my[1][i - p0];
      else id = my[2][c0 + (i - p0 - n[1])];
      succ[beg + i] = id;
    }
    if (lane == 0) split[it] = p0;
    __syncwarp();
  }
}

struct DevGuard {
  int prev = -1, dev = -1;
  explicit DevGuard(cudaStream_t s) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (cudaStreamGetDevice(s, &dev) != cudaSuccess) dev = prev;
    if (dev >= 0 && dev != prev) cudaSetDevice(dev);
    cudaGetLastError();
  }
  ~DevGuard() {
    if (prev >= 0 && dev != prev) cudaSetDevice(prev);
  }
};

int current_device() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) dev = 0;
  return dev;
}

// SM -> die table of the current device: 0 = not measured, 1 = g_sm_die valid, -1 = the
// device did not split into two dies: die-affine items stay off.
int g_die_state[64];
int g_die_sms[64][2];
bool sm_die_ready() { return g_die_state[current_device()] == 1; }

// Opt-in dynamic shared memory of `func` on the current device (once per device and
// kernel; the return code is checked).
int ensure_smem_attr(const void *func, int bytes, const char *what) {
  static struct { const void *f; int dev; int bytes; } done[256];
  static int n_done = 0;
  const int dev = current_device();
  for (int i = 0; i < n_done; i++)
    if (done[i].f == func && done[i].dev == dev && done[i].bytes >= bytes) return 0;
  cudaError_t e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e != cudaSuccess) return set_err(what, e);
  if (n_done < 256) done[n_done++] = {func, dev, bytes};
  return 0;
}

// Persisting-L2 window over the hot head of the register array.  In degree order the
// internal ids sort nodes by in-degree, which on the R-MAT configs is also the read
// frequency of a row (corr > 0.999): the first 3% of rows serve ~78% of all row reads
// (config 5 at 1/16 scale).  Without help those rows are evicted by the streamed ids and
// the cold rows; an access-policy window marks them persisting.  hot_rows == 0 disables.
// HB_L2_PERSIST_MB overrides the set-aside size (0 = off); hb_set_l2_persist(0) turns the
// whole mechanism off for a host application that manages the L2 set-aside itself.  The
// set-aside limit is only ever raised (a larger limit the host set is kept).
bool g_l2_persist = true;

// L2 set-aside for the persisting window of the current step, set per device when it
// changes: 64 MB for rows of p <= 32 (config 5: 32.4 -> 30.6 ms against 32 MB; 48-96 MB
// swept, >= 72 MB thrashes), 32 MB above (config 2: 0.39 -> 0.38 ms against 64 MB).  Never
// set below the limit the host application had; HB_L2_PERSIST_MB overrides.  Returns the
// window size to use (0 = off).
size_t persist_bytes(size_t want) {
  static size_t applied[kMaxDevices], host_have[kMaxDevices], max_sz[kMaxDevices];
  static bool init[kMaxDevices];
  const int dev = current_device();
  if (!init[dev]) {
    init[dev] = true;
    cudaDeviceProp prop;
    if (cudaGetDeviceProperties(&prop, dev) == cudaSuccess)
      max_sz[dev] = std::min((size_t)prop.persistingL2CacheMaxSize,
                             (size_t)prop.accessPolicyMaxWindowSize);
    if (cudaDeviceGetLimit(&host_have[dev], cudaLimitPersistingL2CacheSize) != cudaSuccess)
      host_have[dev] = 0;
    applied[dev] = host_have[dev];
    cudaGetLastError();
  }
  if (const char *e = getenv("HB_L2_PERSIST_MB")) want = (size_t)atoll(e) << 20;
  want = std::min(want, max_sz[dev]);
  if (want == 0) return 0;
  const size_t target = std::max(want, host_have[dev]);
  if (target != applied[dev]) {
    if (cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, target) != cudaSuccess) {
      cudaGetLastError();
      return std::min(want, applied[dev]);
    }
    applied[dev] = target;
  }
  return want;
}

// Bytes of the evict_last head (HB_HINT_MB, default 64); HB_PERSIST_WINDOW=0 turns the
// persisting access-policy window off.
// smallest register array that uses die-affine items (HB_DIE_MIN_MB, read per call: the
// tests lower it to reach the path on small graphs)
size_t die_min_bytes() {
  const char *e = getenv("HB_DIE_MIN_MB");
  return (size_t)(e ? atoll(e) : HB_L1NA_MIN_MB) << 20;
}
// persisting window over the head copy of the die-affine items (HB_DIE_WINDOW_MB; default:
// the step's window size)
size_t die_window_bytes(size_t win) {
  const char *e = getenv("HB_DIE_WINDOW_MB");
  return e ? (size_t)atoll(e) << 20 : win;
}
int64_t hint_bytes() {
  static int64_t b = [] {
    int64_t mb = 64;
    if (const char *e = getenv("HB_HINT_MB")) mb = atoll(e);
    return mb << 20;
  }();
  return b;
}
bool persist_window_on() {
  static bool on = [] {
    const char *e = getenv("HB_PERSIST_WINDOW");
    return !(e && atoi(e) == 0);
  }();
  return on && g_l2_persist;
}

void set_hot_window(cudaStream_t s, const void *base, size_t hot_bytes, size_t cap) {
  cudaStreamAttrValue attr;
  memset(&attr, 0, sizeof(attr));
  if (cap && hot_bytes) {
    const size_t w = hot_bytes < cap ? hot_bytes : cap;
    attr.accessPolicyWindow.base_ptr = const_cast<void *>(base);
    attr.accessPolicyWindow.num_bytes = w;
    attr.accessPolicyWindow.hitRatio = 1.0f;
    attr.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    attr.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
  }
  cudaStreamSetAttribute(s, cudaStreamAttributeAccessPolicyWindow, &attr);
  cudaGetLastError();
}

int num_sms() {
  static int per_dev[kMaxDevices];
  const int dev = current_device();
  if (per_dev[dev] == 0) {
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0)
      v = 148;
    cudaGetLastError();
    per_dev[dev] = v;
  }
  return per_dev[dev];
}
// Grid for `work_warps` warps of work: enough CTAs to fill every SM several times over,
// capped by the work; kernels grid-stride over the rest.
unsigned grid_for_warps(int64_t work_warps) {
  const int64_t per_cta = kThreads / 32;
  int64_t ctas = (work_warps + per_cta - 1) / per_cta;
  const int64_t cap = (int64_t)num_sms() * 8;  // 8 resident 256-thread CTAs per SM
  if (ctas > cap) ctas = cap;
  if (ctas < 1) ctas = 1;
  return (unsigned)ctas;
}
unsigned grid_for_threads(int64_t work) { return grid_for_warps((work + 31) / 32); }

// Grid of the light kernel: whole waves of its resident set.  The 8-CTAs-per-SM cap above
// is 2 2/3 waves of a kernel that fits 3 CTAs per SM (the TMA kernel at p = 256, the
// p = 64 / 128 kernels), so the last third of the launch ran at 2/3 occupancy (ncu: 34.0%
// warps active against 37.5% theoretical).  One wave (HB_GRID_WAVES, env override for
// sweeps) also keeps the resident warps sweeping one window of the id space in step.
#ifndef HB_GRID_WAVES
#define HB_GRID_WAVES 1
#endif
int resident_ctas(const void *func, size_t smem) {
  static struct { const void *f; int dev; size_t smem; int occ; } memo[256];
  static int n_memo = 0;
  const int dev = current_device();
  for (int i = 0; i < n_memo; i++)
    if (memo[i].f == func && memo[i].dev == dev && memo[i].smem == smem) return memo[i].occ;
  int occ = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, func, kThreads, smem) != cudaSuccess ||
      occ <= 0)
    occ = 0;
  cudaGetLastError();
  if (n_memo < 256) memo[n_memo++] = {func, dev, smem, occ};
  return occ;
}
unsigned grid_resident(const void *func, size_t smem, int64_t work_warps) {
  static const int waves = [] {
    const char *e = getenv("HB_GRID_WAVES");
    const int w = e ? atoi(e) : HB_GRID_WAVES;
    return w;
  }();
  const int occ = resident_ctas(func, smem);
  if (waves <= 0 || occ <= 0) return grid_for_warps(work_warps);
  const int64_t per_cta = kThreads / 32;
  int64_t ctas = (work_warps + per_cta - 1) / per_cta;
  const int64_t cap = (int64_t)num_sms() * occ * waves;
  if (ctas > cap) ctas = cap;
  if (ctas < 1) ctas = 1;
  return (unsigned)ctas;
}

#ifndef HB_OVERLAP_LIGHT_DEFAULT
#define HB_OVERLAP_LIGHT_DEFAULT 0   // measured on config 5: 27.3 ms back to back; side by side
                                     // 33.9 / 27.5 / 36.0 ms with 1 / 2 / 3 light CTAs per SM
#endif
#ifndef HB_TMA_L2PROMO
#define HB_TMA_L2PROMO CU_TENSOR_MAP_L2_PROMOTION_L2_256B
#endif
// 2D tensor map over the register rows ([rows, p] bytes, one row per box) for the TMA
// row gather; the driver entry point is resolved once through the runtime.
int encode_row_map(CUtensorMap *tm, const uint8_t *base, int64_t rows, int p) {
  static PFN_cuTensorMapEncodeTiled_v12000 enc = [] {
    PFN_cuTensorMapEncodeTiled_v12000 f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void **)&f, cudaEnableDefault, &q) !=
            cudaSuccess || q != cudaDriverEntryPointSuccess)
      f = nullptr;
    cudaGetLastError();
    return f;
  }();
  if (!enc) return set_err_msg("cuTensorMapEncodeTiled unavailable");
  if (rows <= 0) return set_err_msg("TMA row map: no rows");
  const cuuint64_t dims[2] = {(cuuint64_t)p, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)p};
  const cuuint32_t box[2] = {(cuuint32_t)p, 1};
  const cuuint32_t es[2] = {1, 1};
  const CUresult r = enc(tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<uint8_t *>(base), dims,
                         strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         CU_TENSOR_MAP_SWIZZLE_NONE, (CUtensorMapL2promotion)HB_TMA_L2PROMO,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : set_err_msg("cuTensorMapEncodeTiled failed");
}

// Side stream of the current device for the light kernel of an overlapped step (below):
// created on first use, non-blocking; fork / join by two events, so the caller's stream
// still orders the whole step.
struct SideStream {
  cudaStream_t st = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
  int state = 0;   // 0 = not tried, 1 = ready, -1 = unavailable
};
SideStream *side_stream() {
  static SideStream sd[kMaxDevices];
  SideStream &x = sd[current_device()];
  if (x.state == 0) {
    x.state = -1;
    if (cudaStreamCreateWithFlags(&x.st, cudaStreamNonBlocking) == cudaSuccess &&
        cudaEventCreateWithFlags(&x.fork, cudaEventDisableTiming) == cudaSuccess &&
        cudaEventCreateWithFlags(&x.join, cudaEventDisableTiming) == cudaSuccess)
      x.state = 1;
    cudaGetLastError();
  }
  return x.state == 1 ? &x : nullptr;
}
// Overlapped step (p <= 32 rows of a register array >= 1 GB, heavy items present, ticket-
// dealt): the heavy-item kernel is bound by the DRAM random-access rate of its cold rows,
// the light kernel half by streams (own rows, estimates, sums, ids) -- run side by side
// they share the SMs, HB_OVERLAP_LIGHT resident CTAs per SM for the light kernel, the rest
// for the items.  Off by default (HB_OVERLAP_LIGHT=0): the two kernels turn out to be
// bound by the same resource -- the misses of both are served at the same DRAM
// random-access rate -- so side by side they take as long as back to back.
int overlap_light_ctas() {
  const char *e = getenv("HB_OVERLAP");
  if (e && e[0] == '0') return 0;
  const char *l = getenv("HB_OVERLAP_LIGHT");
  const int v = l ? atoi(l) : HB_OVERLAP_LIGHT_DEFAULT;
  return v > 0 ? v : 0;
}

template <int LOGP, bool PUSH, int LOGR = 0>
int union_step_impl(int64_t lo, int64_t hi, const int64_t *offsets, const int32_t *succ,
                    const uint8_t *cur, uint8_t *nxt, const uint32_t *chg_prev,
                    uint32_t *chg_now, double *est, double *sum_dist, double *sum_recip,
                    double tf, EstConst ec, int dense, int64_t light_max_deg,
                    const int32_t *heavy_nodes, const int32_t *item_first, int64_t n_heavy,
                    const int32_t *finish_order, int64_t n_mega,
                    const int32_t *item_node, const int64_t *item_beg, int64_t n_items,
                    int64_t item_arcs, uint8_t *partial, unsigned long long *nch,
                    unsigned long long *merged, int64_t hot_rows, const uint32_t *active,
                    const Peers &peers, cudaStream_t s, RunArgs ra = RunArgs{nullptr, 0, 0},
                    int64_t n_rows = 0, unsigned int *ticket = nullptr,
                    uint8_t *die_head = nullptr, int64_t die_head_rows = 0,
                    const int32_t *item_split = nullptr) {
  using Gm = Geo<LOGP>;
  CUtensorMap tmap;
  memset(&tmap, 0, sizeof(tmap));
  size_t tma_smem = 0;
  if constexpr (kTma<LOGP, LOGR, false>()) {
    if (int e = encode_row_map(&tmap, cur, n_rows, Gm::P)) return e;
    tma_smem = (size_t)(kThreads / 32) * Geo<LOGP>::NPW * Batch<LOGP>::U * Gm::P;
    if (int e = ensure_smem_attr((const void *)k_light<LOGP, PUSH, LOGR, false>, (int)tma_smem,
                                 "k_light smem attribute"))
      return e;
  }
  const size_t win = hot_rows > 0 && persist_window_on()
                        ? persist_bytes((size_t)(LOGP <= HB_HINT_MAX_LOGP ? 64 : 32) << 20) : 0;
  if (win > 0) {
    cudaCtxResetPersistingL2Cache();    // lines of last iteration's buffer stop persisting
    set_hot_window(s, cur, (size_t)hot_rows * Gm::P, win);
  }
  constexpr bool kCanHint = LOGP <= HB_HINT_MAX_LOGP;
  const bool l1na = (size_t)n_rows * Gm::P >= ((size_t)HB_L1NA_MIN_MB << 20);
  // die-affine heavy items: hinted rows (p <= 32) of a register array too large for L1,
  // ticket-dealt (not in frontier mode), with the chunk map of this `cur` buffer
  const bool die = kCanHint && (size_t)n_rows * Gm::P >= die_min_bytes() && die_head &&
                   item_split && ticket && !active && n_items > 0 && hot_rows > 0 &&
                   item_arcs <= kDieItemMax && sm_die_ready();
  const int64_t die_rows = die ? std::min<int64_t>(hot_rows, die_head_rows) : 0;
  const int64_t hot_lim = hot_rows > 0 ? std::min<int64_t>(hot_rows, hint_bytes() / Gm::P) : 0;
  const bool hint = kCanHint && hot_lim > 0;
  int pshift = 0;
  // overlapped step: the light kernel on the side stream, next to the heavy items
  int lshare = 0;
  SideStream *side = nullptr;
  if constexpr (kCanHint && !PUSH && LOGR == 0) {
    if (hint && l1na && ticket && !active && n_items > 0 && hi > lo && (lshare = overlap_light_ctas()) > 0)
      side = side_stream();
  }
  if (!side) lshare = 0;
  if (side) {
    if (cudaEventRecord(side->fork, s) != cudaSuccess ||
        cudaStreamWaitEvent(side->st, side->fork, 0) != cudaSuccess)
      return set_err("hb_union_step overlap fork", cudaGetLastError());
    if (win > 0) set_hot_window(side->st, cur, (size_t)hot_rows * Gm::P, win);
  }
  cudaStream_t sl = side ? side->st : s;     // the light kernel's stream
  if (n_items > 0) {
    // ticket word 1 deals the heavy items (word 0 the light kernel's chunks), except in
    // frontier mode, whose skip-ahead probe walks the grid-stride order
    unsigned int *hticket = ticket && !active ? ticket + 1 : nullptr;
    const void *hfunc = !hint ? (const void *)k_heavy_partial<LOGP, false>
                        : (l1na ? (const void *)k_heavy_partial<LOGP, kCanHint, kCanHint>
                                : (const void *)k_heavy_partial<LOGP, kCanHint>);
    if constexpr (kCanHint) {
      if (die && hint && die_rows > 0)
        hfunc = (const void *)k_heavy_partial<LOGP, true, true, true>;
    }
    const bool die_on = kCanHint && hfunc == (const void *)k_heavy_partial<LOGP, kCanHint, kCanHint, kCanHint>;
    unsigned hgrid = hticket ? grid_resident(hfunc, 0, n_items) : grid_for_warps(n_items);
    if (side) {
      const int occ = resident_ctas(hfunc, 0);
      if (occ > lshare) hgrid = std::min<unsigned>(hgrid, (unsigned)(num_sms() * (occ - lshare)));
      else { lshare = 0; }
    }
    // items per draw: ~16 draws per resident warp, at most 8 items (config 5: 27.8 ms; 28.0 /
    // 28.2 ms at 32 / 128; 4 is 27.6 ms but the draws start to queue on config 5s; env
    // overrides for sweeps)
    static const int dpw = [] { const char *e = getenv("HB_DRAWS_PER_WARP"); return e ? atoi(e) : 16; }();
    static const int dmax = [] { const char *e = getenv("HB_DRAW_MAX"); return e ? atoi(e) : 8; }();
    const int draw_items = (int)std::max<int64_t>(
        1, std::min<int64_t>(dmax, n_items / ((int64_t)hgrid * (kThreads / 32) * dpw)));
    if constexpr (kCanHint) {
      if (die_on) {
        pshift = 1;
        // the head copy the passes gather from (fixed address: its die map is static)
        if (cudaMemcpyAsync(die_head, cur, (size_t)die_rows * Gm::P, cudaMemcpyDeviceToDevice, s) != cudaSuccess)
          return set_err("hb_union_step head copy", cudaGetLastError());
        if (win > 0) set_hot_window(s, die_head, (size_t)die_rows * Gm::P, die_window_bytes(win));
        k_heavy_partial<LOGP, true, true, true><<<hgrid, kThreads, 0, s>>>(
            offsets, succ, cur, chg_prev, item_node, item_beg, n_items, item_arcs, dense,
            partial, merged, active, die_rows, hticket, draw_items, item_split, die_head, die_rows);
        if (win > 0) set_hot_window(s, cur, (size_t)hot_rows * Gm::P, win);
      } else if (hint && l1na)
        k_heavy_partial<LOGP, true, true><<<hgrid, kThreads, 0, s>>>(
            offsets, succ, cur, chg_prev, item_node, item_beg, n_items, item_arcs, dense,
            partial, merged, active, hot_lim, hticket, draw_items);
      else if (hint)
        k_heavy_partial<LOGP, true><<<hgrid, kThreads, 0, s>>>(
            offsets, succ, cur, chg_prev, item_node, item_beg, n_items, item_arcs, dense,
            partial, merged, active, hot_lim, hticket, draw_items);
    }
    if (!hint)
      k_heavy_partial<LOGP, false><<<hgrid, kThreads, 0, s>>>(
          offsets, succ, cur, chg_prev, item_node, item_beg, n_items, item_arcs, dense,
          partial, merged, active, hot_lim, hticket, draw_items);
    if (int e = check_launch("k_heavy_partial")) return e;
  }
  if (hi > lo) {
    const int64_t warps = (hi - lo + Gm::NPW - 1) / Gm::NPW + 1;   // capped at the resident set
    if constexpr (kCanHint) {
      if (hint && l1na)
        k_light<LOGP, PUSH, LOGR, true, true><<<(side && lshare > 0) ? std::min<unsigned>(grid_resident((const void *)k_light<LOGP, PUSH, LOGR, true, true>, 0, warps), (unsigned)(num_sms() * lshare)) : grid_resident((const void *)k_light<LOGP, PUSH, LOGR, true, true>, 0, warps), kThreads, 0, sl>>>(
            offsets, succ, cur, nxt, chg_prev, chg_now, est, sum_dist, sum_recip, ec, lo, hi,
            light_max_deg, dense, tf, nch, merged, active, peers, ra, hot_lim, ticket, tmap);
      else if (hint)
        k_light<LOGP, PUSH, LOGR, true><<<grid_resident((const void *)k_light<LOGP, PUSH, LOGR, true>, 0, warps), kThreads, 0, s>>>(
            offsets, succ, cur, nxt, chg_prev, chg_now, est, sum_dist, sum_recip, ec, lo, hi,
            light_max_deg, dense, tf, nch, merged, active, peers, ra, hot_lim, ticket, tmap);
    }
    if (!hint)
      k_light<LOGP, PUSH, LOGR, false><<<grid_resident((const void *)k_light<LOGP, PUSH, LOGR, false>, tma_smem, warps), kThreads, tma_smem, s>>>(
          offsets, succ, cur, nxt, chg_prev, chg_now, est, sum_dist, sum_recip, ec, lo, hi,
          light_max_deg, dense, tf, nch, merged, active, peers, ra, hot_lim, ticket, tmap);
    if (int e = check_launch("k_light")) return e;
  }
  if (side) {
    if (win > 0) set_hot_window(side->st, nullptr, 0, 0);
    if (cudaEventRecord(side->join, side->st) != cudaSuccess ||
        cudaStreamWaitEvent(s, side->join, 0) != cudaSuccess)
      return set_err("hb_union_step overlap join", cudaGetLastError());
  }
  if (n_heavy > 0) {
    if (n_mega > 0) {
      k_heavy_finish<LOGP, PUSH, LOGR><<<grid_for_warps(n_mega), kThreads, 0, s>>>(
          heavy_nodes, item_first, finish_order, 0, n_mega, 1, partial, cur, nxt, chg_prev,
          chg_now, est, sum_dist, sum_recip, ec, tf, nch, active, peers, ra, pshift);
      if (int e = check_launch("k_heavy_finish(mega)")) return e;
    }
    if (n_heavy > n_mega)
      k_heavy_finish<LOGP, PUSH, LOGR>
          <<<grid_for_warps((n_heavy - n_mega + Gm::NPW - 1) / Gm::NPW), kThreads, 0, s>>>(
              heavy_nodes, item_first, finish_order, n_mega, n_heavy, 0, partial, cur, nxt,
              chg_prev, chg_now, est, sum_dist, sum_recip, ec, tf, nch, active, peers, ra, pshift);
    if (int e = check_launch("k_heavy_finish")) return e;
  }
  if (win > 0) set_hot_window(s, nullptr, 0, 0);
  return 0;
}

#define HB_DISPATCH(B, CALL)                 \
  switch (B) {                               \
    case 4: { constexpr int LB = 4; CALL; } break;   \
    case 5: { constexpr int LB = 5; CALL; } break;   \
    case 6: { constexpr int LB = 6; CALL; } break;   \
    case 7: { constexpr int LB = 7; CALL; } break;   \
    case 8: { constexpr int LB = 8; CALL; } break;   \
    case 9: { constexpr int LB = 9; CALL; } break;   \
    case 10: { constexpr int LB = 10; CALL; } break; \
    case 11: { constexpr int LB = 11; CALL; } break; \
    case 12: { constexpr int LB = 12; CALL; } break; \
    default: return set_err_msg("unsupported log2m (b) for this build");  \
  }

}  // namespace

// Row sort (schedule setup): ascending source ids inside every CSR row after relabelling,
// so consecutive arcs of a hub read neighbouring register rows (shared 128-byte lines at
// small p).  cub::DeviceSegmentedSort over row batches of < 2^31 arcs, ping-ponging
// between the two id buffers.
struct ShiftOff {
  int64_t base;
  __host__ __device__ __forceinline__ int operator()(const int64_t &x) const {
    return (int)(x - base);
  }
};
using OffIt = cub::TransformInputIterator<int, ShiftOff, const int64_t *>;


// ------------------------------------------------------------------ C-ABI
template <int LOGP>
static int64_t light_npw_t() { return Geo<LOGP>::NPW; }
template <int LOGP>
static int64_t light_window_t() { return (int64_t)Geo<LOGP>::NPW * chunk_rounds<LOGP>(); }

extern "C" {

const char *hb_version(void) { return "hyperball_b200 0.1 (sm_100a)"; }
const char *hb_last_error(void) { return g_err; }
int hb_min_log2m(void) { return HB_MIN_B; }
int hb_max_log2m(void) { return HB_MAX_B; }
int64_t hb_item_arcs(int b) { return item_arcs_for(b); }
int64_t hb_light_max_deg(int b) {
  if (const char *e = getenv("HB_LIGHT_MAX_DEG")) {   // sweeps
    const int64_t v = atoll(e);
    if (v > 0) return v;
  }
  // 16- / 32-register rows: one lane per node (or two) keeps 8 row loads in flight by
  // itself, and a heavy item costs ~400 warp instructions before its first row -- nodes of
  // up to 128 arcs are cheaper in the light kernel (config 5 27.7 -> 27.1 ms, config 5s
  // 1.50 -> 1.45 ms; 96-192 within 1%, 256-512 back to 27.7, 2048 29.4 ms); above, 64
  // (config 2, p = 128: 0.39 ms at 64, 0.49 at 256)
  return b <= 5 ? 2 * kLightMaxDeg : kLightMaxDeg;
}
int64_t hb_light_npw(int b) {
  switch (b) {
    case 4: return light_npw_t<4>();   case 5: return light_npw_t<5>();
    case 6: return light_npw_t<6>();   case 7: return light_npw_t<7>();
    case 8: return light_npw_t<8>();   case 9: return light_npw_t<9>();
    case 10: return light_npw_t<10>(); case 11: return light_npw_t<11>();
    case 12: return light_npw_t<12>();
  }
  return 1;
}
int64_t hb_light_window(int b) {
  switch (b) {
    case 4: return light_window_t<4>();   case 5: return light_window_t<5>();
    case 6: return light_window_t<6>();   case 7: return light_window_t<7>();
    case 8: return light_window_t<8>();   case 9: return light_window_t<9>();
    case 10: return light_window_t<10>(); case 11: return light_window_t<11>();
    case 12: return light_window_t<12>();
  }
  return 1;
}

int hb_seed(uint8_t *regs, double *est, int64_t n, int b, int register_width, uint64_t seed,
            const int32_t *perm, const int64_t *weights, const double *lc_table,
            double alpha_p2, double lc_cut, void *stream) {
  DevGuard dg_((cudaStream_t)stream);
  if (register_width < 1 || register_width > 8) return set_err_msg("hb_seed: bad register_width");
  if (n == 0) return 0;
  if (n < 0 || !regs || !est || !lc_table) return set_err_msg("hb_seed: bad arguments");
  cudaStream_t s = (cudaStream_t)stream;
  EstConst ec{alpha_p2, lc_cut, lc_table, nullptr, 0, 0, 0, {0, 0, 0, 0, 0, 0, 0, 0}};
  HB_DISPATCH(b, (k_seed<LB><<<grid_for_threads(n), kThreads, 0, s>>>(
                     regs, est, n, perm, weights, register_width, seed, ec)));
  return check_launch("k_seed");
}

int hb_estimate_rows(const uint8_t *regs, int64_t lo, int64_t hi, int b,
                     const double *lc_table, double alpha_p2, double lc_cut, double *out,
                     void *stream) {
  DevGuard dg_((cudaStream_t)stream);
  if (hi <= lo) return 0;
  if (lo < 0 || !regs || !lc_table || !out) return set_err_msg("hb_estimate_rows: bad arguments");
  cudaStream_t s = (cudaStream_t)stream;
  EstConst ec{alpha_p2, lc_cut, lc_table, nullptr, 0, 0, 0, {0, 0, 0, 0, 0, 0, 0, 0}};
  HB_DISPATCH(b, (k_estimate_rows<LB><<<grid_for_threads(hi - lo), kThreads, 0, s>>>(
                     regs, lo, hi, ec, out)));
  return check_launch("k_estimate_rows");
}

int hb_union_step_v2(const hb_step_args *a) {
  if (!a || a->struct_size < offsetof(hb_step_args, peer_packed_stride))
    return set_err_msg("hb_union_step_v2: null args or struct_size < hb_step_args_min_size()");
  const int64_t pstride =
      a->struct_size >= offsetof(hb_step_args, peer_packed_stride) + sizeof(int64_t)
          ? a->peer_packed_stride : 0;
  static const bool tickets_on = [] {          // HB_TICKETS=0: grid-stride chunks (sweeps)
    const char *e = getenv("HB_TICKETS");
    return !(e && e[0] == '0');
  }();
  uint64_t *ticket = tickets_on && a->struct_size >= offsetof(hb_step_args, ticket) + sizeof(uint64_t *)
                         ? a->ticket : nullptr;
  const bool has_die = a->struct_size >= offsetof(hb_step_args, item_split) + sizeof(void *);
  uint8_t *die_head = has_die && ticket && a->item_split && a->die_rows > 0 ? a->die_head : nullptr;
  const int64_t die_head_rows = die_head ? a->die_rows : 0;
  const int32_t *item_split = die_head ? a->item_split : nullptr;
  DevGuard dg_((cudaStream_t)a->stream);
  const int n_peers = a->n_peers, n_disc = a->n_disc;
  const int64_t n = a->n, lo = a->lo, hi = a->hi, t = a->t;
  if (n_peers < 0 || n_peers > kMaxPeers || (n_peers > 0 && (!a->peer_nxt || !a->peer_chg)))
    return set_err_msg("hb_union_step: bad peer arguments (at most 7 peers)");
  Peers peers;
  memset(&peers, 0, sizeof(peers));
  peers.n = n_peers;
  for (int q = 0; q < n_peers; q++) {
    peers.nxt[q] = a->peer_nxt[q];
    peers.chg[q] = a->peer_chg[q];
  }
  if (n_peers > 0 && pstride != 0) {
    if (pstride != push_stride((1 << a->b) / 16))
      return set_err_msg("hb_union_step: peer_packed_stride must be hb_push_row_stride(b)");
    peers.pstride = (int)pstride;
  }
  if (n_disc < 0 || n_disc > kMaxDisc || (n_disc > 0 && (!a->disc || !a->disc_scale)))
    return set_err_msg("hb_union_step: bad discount arguments (at most 8 fused)");
  if (n < 0 || lo < 0 || hi > n || lo > hi || t < 1 || !a->nch_out)
    return set_err_msg("hb_union_step: bad range / t / nch_out");
  if (n > 0 && (!a->offsets || !a->cur || !a->nxt || !a->chg_prev || !a->chg_now || !a->est ||
                !a->lc_table))
    return set_err_msg("hb_union_step: null graph / register / flag / estimate array");
  if ((a->n_items > 0 && (!a->item_node || !a->item_beg || !a->partial)) ||
      (a->n_heavy > 0 && (!a->heavy_nodes || !a->item_first || !a->finish_order || !a->partial)) ||
      a->n_mega < 0 || a->n_mega > a->n_heavy)
    return set_err_msg("hb_union_step: heavy schedule arrays missing");
  cudaStream_t s = (cudaStream_t)a->stream;
  cudaError_t e;
  if ((e = cudaMemsetAsync(a->nch_out, 0, sizeof(uint64_t), s)) != cudaSuccess)
    return set_err("hb_union_step memset nch", e);
  if (a->merged_out && (e = cudaMemsetAsync(a->merged_out, 0, sizeof(uint64_t), s)) != cudaSuccess)
    return set_err("hb_union_step memset merged", e);
  if (ticket && (e = cudaMemsetAsync(ticket, 0, sizeof(uint64_t) * (die_head ? 2 : 1), s)) != cudaSuccess)
    return set_err("hb_union_step memset ticket", e);
  if (a->clear_chg_now && n > 0) {
    if ((e = cudaMemsetAsync(a->chg_now, 0, sizeof(uint32_t) * (size_t)((n + 31) / 32), s)) !=
        cudaSuccess)
      return set_err("hb_union_step memset chg_now", e);
  }
  if (n == 0) return 0;
  // checked build: the sizes the kernels' bounds checks use (the graph's id count is not
  // known here -- offsets live on the device -- so the caller passes it; 0 = unchecked)
  if (int er = set_check_dims(a->check_rows > 0 ? a->check_rows : n,
                              a->check_m > 0 ? a->check_m : INT64_MAX, a->n_items, s))
    return er;
  EstConst ec{a->alpha_p2, a->lc_cut, a->lc_table, a->disc, a->disc_stride, n_disc, a->disc_div,
              {0, 0, 0, 0, 0, 0, 0, 0}};
  for (int k = 0; k < n_disc; k++) ec.disc_scale[k] = a->disc_scale[k];
  const double tf = (double)t;
  unsigned long long *nch = reinterpret_cast<unsigned long long *>(a->nch_out);
  unsigned long long *merged = reinterpret_cast<unsigned long long *>(a->merged_out);
  if (n_peers > 0) {
    HB_DISPATCH(a->b, return (union_step_impl<LB, true>(
                       lo, hi, a->offsets, a->succ, a->cur, a->nxt, a->chg_prev, a->chg_now,
                       a->est, a->sum_dist, a->sum_recip, tf, ec, a->dense, a->light_max_deg,
                       a->heavy_nodes, a->item_first, a->n_heavy, a->finish_order, a->n_mega,
                       a->item_node, a->item_beg, a->n_items, a->item_arcs, a->partial, nch,
                       merged, a->hot_rows, a->active, peers, s, RunArgs{nullptr, 0, 0}, n,
                       reinterpret_cast<unsigned int *>(ticket), die_head, die_head_rows, item_split)));
  }
  HB_DISPATCH(a->b, return (union_step_impl<LB, false>(
                     lo, hi, a->offsets, a->succ, a->cur, a->nxt, a->chg_prev, a->chg_now,
                     a->est, a->sum_dist, a->sum_recip, tf, ec, a->dense, a->light_max_deg,
                     a->heavy_nodes, a->item_first, a->n_heavy, a->finish_order, a->n_mega,
                     a->item_node, a->item_beg, a->n_items, a->item_arcs, a->partial, nch,
                     merged, a->hot_rows, a->active, peers, s, RunArgs{nullptr, 0, 0}, n,
                       reinterpret_cast<unsigned int *>(ticket), die_head, die_head_rows, item_split)));
  return 0;
}

int hb_union_step(int64_t n, int64_t lo, int64_t hi, const int64_t *offsets,
                  const int32_t *succ, const uint8_t *cur, uint8_t *nxt,
                  const uint32_t *chg_prev, uint32_t *chg_now, int clear_chg_now,
                  double *est, double *sum_dist, double *sum_recip, int64_t t,
                  const double *lc_table, double alpha_p2, double lc_cut, int b, int dense,
                  int64_t light_max_deg, const int32_t *heavy_nodes, const int32_t *item_first,
                  int64_t n_heavy, const int32_t *finish_order, int64_t n_mega,
                  const int32_t *item_node, const int64_t *item_beg,
                  int64_t n_items, int64_t item_arcs, uint8_t *partial, uint64_t *nch_out,
                  uint64_t *merged_out, int64_t hot_rows, double *disc, int64_t disc_stride,
                  int n_disc, const double *disc_scale, int disc_div, const uint32_t *active,
                  int n_peers, uint8_t *const *peer_nxt, uint32_t *const *peer_chg,
                  void *stream) {
  hb_step_args a;
  memset(&a, 0, sizeof(a));
  a.struct_size = sizeof(a);
  a.n = n; a.lo = lo; a.hi = hi; a.offsets = offsets; a.succ = succ;
  a.cur = cur; a.nxt = nxt; a.chg_prev = chg_prev; a.chg_now = chg_now; a.est = est;
  a.b = b; a.dense = dense; a.clear_chg_now = clear_chg_now; a.n_disc = n_disc; a.t = t;
  a.lc_table = lc_table; a.alpha_p2 = alpha_p2; a.lc_cut = lc_cut;
  a.sum_dist = sum_dist; a.sum_recip = sum_recip;
  a.disc = disc; a.disc_stride = disc_stride; a.disc_scale = disc_scale; a.disc_div = disc_div;
  a.n_peers = n_peers; a.light_max_deg = light_max_deg;
  a.heavy_nodes = heavy_nodes; a.item_first = item_first; a.n_heavy = n_heavy;
  a.finish_order = finish_order; a.n_mega = n_mega; a.item_node = item_node;
  a.item_beg = item_beg; a.n_items = n_items; a.item_arcs = item_arcs; a.partial = partial;
  a.nch_out = nch_out; a.merged_out = merged_out; a.hot_rows = hot_rows; a.active = active;
  a.peer_nxt = peer_nxt; a.peer_chg = peer_chg; a.stream = stream;
  return hb_union_step_v2(&a);
}

void hb_set_l2_persist(int enable) { g_l2_persist = enable != 0; }

// SM -> die classification of the current device (once): latency vectors of kDieTest
// chunks per SM, split by the sign of their correlation with the first SM's vector.
static int classify_sms(uint8_t *base, int64_t bytes, int64_t chunks, cudaStream_t s) {
  const int dev = current_device();
  if (g_die_state[dev] != 0) return 0;
  g_die_state[dev] = -1;
  const int64_t stride = chunks / kDieTest;
  if (stride < 3) return 0;                       // needs >= 768 KB to probe
  int *claimed = nullptr;
  uint32_t *lat = nullptr;
  if (cudaMalloc(&claimed, 256 * sizeof(int)) != cudaSuccess ||
      cudaMalloc(&lat, 256 * kDieTest * sizeof(uint32_t)) != cudaSuccess) {
    cudaFree(claimed);
    return set_err("hb_die_map: scratch", cudaGetLastError());
  }
  std::vector<uint32_t> hl(256 * kDieTest);
  std::vector<int> hc(256);
  cudaMemsetAsync(claimed, 0, 256 * sizeof(int), s);
  cudaMemsetAsync(lat, 0, 256 * kDieTest * sizeof(uint32_t), s);
  k_sm_probe<<<num_sms() * 16, 32, 0, s>>>(base, bytes, stride, claimed, lat);
  cudaMemcpyAsync(hl.data(), lat, hl.size() * 4, cudaMemcpyDeviceToHost, s);
  cudaMemcpyAsync(hc.data(), claimed, hc.size() * 4, cudaMemcpyDeviceToHost, s);
  const cudaError_t e = cudaStreamSynchronize(s);
  cudaFree(claimed);
  cudaFree(lat);
  if (e != cudaSuccess) return set_err("hb_die_map: SM probe", e);
  int ref = -1;
  for (int i = 0; i < 256; i++) if (hc[i]) { ref = i; break; }
  if (ref < 0) return 0;
  int8_t die[256];
  int cnt[2] = {0, 0};
  double min_abs = 1.0;
  for (int i = 0; i < 256; i++) {
    die[i] = (int8_t)(i & 1);                     // SMs no CTA landed on: either queue
    if (!hc[i]) continue;
    double ma = 0, mb = 0, cov = 0, va = 0, vb = 0;
    for (int k = 0; k < kDieTest; k++) { ma += hl[ref * kDieTest + k]; mb += hl[i * kDieTest + k]; }
    ma /= kDieTest; mb /= kDieTest;
    for (int k = 0; k < kDieTest; k++) {
      const double a = hl[ref * kDieTest + k] - ma, b = hl[i * kDieTest + k] - mb;
      cov += a * b; va += a * a; vb += b * b;
    }
    const double corr = cov / std::sqrt(va * vb + 1e-9);
    die[i] = corr > 0 ? 0 : 1;
    cnt[die[i]]++;
    min_abs = std::min(min_abs, std::fabs(corr));
  }
  // two dies, each with at least a quarter of the SMs, cleanly separated
  if (cnt[0] * 4 < cnt[0] + cnt[1] || cnt[1] * 4 < cnt[0] + cnt[1] || min_abs < 0.5) return 0;
  if (cudaMemcpyToSymbol(g_sm_die, die, sizeof(die)) != cudaSuccess)
    return set_err("hb_die_map: SM table", cudaGetLastError());
  g_die_sms[dev][0] = cnt[0];
  g_die_sms[dev][1] = cnt[1];
  g_die_state[dev] = 1;
  return 0;
}

int hb_die_map(void *base, int64_t bytes, uint32_t *bits_out, int64_t *stats, void *stream) {
  cudaStream_t s = (cudaStream_t)stream;
  DevGuard dg_(s);
  if (stats) stats[0] = stats[1] = stats[2] = stats[3] = 0;
  if (!base || bytes < 4096 || !bits_out || !stats) return set_err_msg("hb_die_map: bad arguments");
  // opt-in (HB_DIE=1): on config 5 the two passes per item cost more instructions than the
  // L2 hits they add save; without it the call reports "no split"
  const char *en = getenv("HB_DIE");
  if (!en || en[0] != '1') return 0;
  const int64_t chunks = (int64_t)(((reinterpret_cast<uintptr_t>(base) & 2047u) + (uint64_t)bytes + 2047u) >> 11);
  if (int e = classify_sms((uint8_t *)base, bytes, chunks, s)) return e;
  const int dev = current_device();
  if (g_die_state[dev] != 1) return 0;            // stats all zero: not available
  uint32_t *lat2 = nullptr;
  unsigned long long *scr = nullptr;              // [0] the two deal counters, [2..3] stats
  if (cudaMalloc(&lat2, 2 * chunks * sizeof(uint32_t)) != cudaSuccess ||
      cudaMalloc(&scr, 4 * sizeof(unsigned long long)) != cudaSuccess) {
    cudaFree(lat2);
    return set_err("hb_die_map: scratch", cudaGetLastError());
  }
  cudaMemsetAsync(scr, 0, 4 * sizeof(unsigned long long), s);
  k_chunk_probe<<<num_sms() * 4, 32, 0, s>>>((uint8_t *)base, bytes, chunks,
                                             reinterpret_cast<unsigned int *>(scr), lat2);
  k_chunk_bits<<<(unsigned)(((chunks + 31) / 32 + 255) / 256), 256, 0, s>>>(lat2, chunks, bits_out, scr + 2);
  unsigned long long h[2] = {0, 0};
  cudaMemcpyAsync(h, scr + 2, sizeof(h), cudaMemcpyDeviceToHost, s);
  const cudaError_t e = cudaStreamSynchronize(s);
  cudaFree(lat2);
  cudaFree(scr);
  if (e != cudaSuccess) return set_err("hb_die_map: chunk probe", e);
  stats[0] = g_die_sms[dev][0];
  stats[1] = g_die_sms[dev][1];
  stats[2] = (int64_t)h[0];
  stats[3] = (int64_t)h[1];
  return 0;
}
int hb_die_partition(int64_t n_items, const int32_t *item_node, const int64_t *item_beg,
                     const int64_t *offsets, int32_t *succ, int64_t item_arcs, int b,
                     const void *head, int64_t die_rows, const uint32_t *die_bits,
                     int32_t *item_split, void *stream) {
  cudaStream_t s = (cudaStream_t)stream;
  DevGuard dg_(s);
  if (n_items <= 0) return 0;
  if (!item_node || !item_beg || !offsets || !succ || !head || !die_bits || !item_split ||
      b < HB_MIN_B || b > HB_MAX_B || die_rows < 0 || item_arcs <= 0 || item_arcs > kDieItemMax)
    return set_err_msg("hb_die_partition: bad arguments (item_arcs <= 512)");
  k_die_partition<<<grid_for_warps(n_items), kThreads, 0, s>>>(
      n_items, item_node, item_beg, offsets, succ, item_arcs, b,
      (uint32_t)(reinterpret_cast<uintptr_t>(head) & 2047u), die_rows, die_bits, item_split);
  return check_launch("k_die_partition");
}
int64_t hb_die_map_words(const void *base, int64_t bytes) {
  const int64_t chunks = (int64_t)(((reinterpret_cast<uintptr_t>(base) & 2047u) + (uint64_t)bytes + 2047u) >> 11);
  return (chunks + 31) / 32;
}
uint64_t hb_step_args_size(void) { return sizeof(hb_step_args); }
uint64_t hb_step_args_min_size(void) { return offsetof(hb_step_args, peer_packed_stride); }

int hb_push_row_stride(int b) {
  if (b < HB_MIN_B || b > HB_MAX_B) return -1;
  return push_stride((1 << b) / 16);
}

int hb_unpack_inbox(int64_t n, int64_t lo, int64_t hi, int b, const uint32_t *chg_now,
                    const uint32_t *chg_prev_copy, const uint8_t *inbox, const uint8_t *cur,
                    uint8_t *nxt, void *stream) {
  DevGuard dg_((cudaStream_t)stream);
  if (b < HB_MIN_B || b > HB_MAX_B || n < 0 || lo < 0 || hi > n || lo > hi)
    return set_err_msg("hb_unpack_inbox: bad arguments");
  if (n == 0) return 0;
  if (!chg_now || !chg_prev_copy || !inbox || !cur || !nxt)
    return set_err_msg("hb_unpack_inbox: null array");
  const int ch = (1 << b) / 16;
  k_unpack_inbox<<<grid_for_threads(n * ch), kThreads, 0, (cudaStream_t)stream>>>(
      n, lo, hi, ch, chg_now, chg_prev_copy, inbox, cur, nxt);
  return check_launch("k_unpack_inbox");
}

int hb_union_step_runs(int64_t n, int64_t lo, int64_t hi, const int64_t *offsets,
                       const int32_t *succ, const uint8_t *cur, uint8_t *nxt,
                       const uint32_t *chg_prev, uint32_t *chg_now, uint32_t *chg_runs,
                       double *est, double *sum_dist, double *sum_recip, int64_t run_stride,
                       int64_t t, const double *lc_table, double alpha_p2, double lc_cut, int b,
                       int log2_runs, int dense, int64_t light_max_deg,
                       const int32_t *heavy_nodes, const int32_t *item_first, int64_t n_heavy,
                       const int32_t *finish_order, int64_t n_mega, const int32_t *item_node,
                       const int64_t *item_beg, int64_t n_items, int64_t item_arcs,
                       uint8_t *partial, uint64_t *nch_out, uint64_t *merged_out,
                       uint64_t *run_nch_out, int64_t hot_rows, double *disc,
                       int64_t disc_stride, int n_disc, const double *disc_scale, int disc_div,
                       const uint32_t *active, void *stream) {
  DevGuard dg_((cudaStream_t)stream);
  const int wb = b + log2_runs;
  if (log2_runs < 1 || log2_runs > 4 || b < HB_MIN_B || wb > 8)
    return set_err_msg("hb_union_step_runs: need 2..16 runs and runs * p <= 256");
  if (n < 0 || lo < 0 || hi > n || lo > hi || t < 1 || !nch_out || !chg_runs || !run_nch_out ||
      run_stride < n || (n > 0 && (!offsets || !cur || !nxt || !chg_prev || !chg_now ||
                                   !est || !lc_table)))
    return set_err_msg("hb_union_step_runs: bad arguments");
  if ((n_items > 0 && (!item_node || !item_beg || !partial)) ||
      (n_heavy > 0 && (!heavy_nodes || !item_first || !finish_order || !partial)) ||
      n_mega < 0 || n_mega > n_heavy)
    return set_err_msg("hb_union_step_runs: heavy schedule arrays missing");
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t words = (n + 31) / 32;
  const int runs = 1 << log2_runs;
  cudaError_t e;
  if ((e = cudaMemsetAsync(nch_out, 0, sizeof(uint64_t), s)) != cudaSuccess ||
      (merged_out && (e = cudaMemsetAsync(merged_out, 0, sizeof(uint64_t), s)) != cudaSuccess))
    return set_err("hb_union_step_runs memset", e);
  if (n == 0) return cudaMemsetAsync(run_nch_out, 0, sizeof(uint64_t) * runs, s) == cudaSuccess
                         ? 0 : set_err_msg("hb_union_step_runs memset");
  if ((e = cudaMemsetAsync(chg_now, 0, sizeof(uint32_t) * (size_t)words, s)) != cudaSuccess ||
      (e = cudaMemsetAsync(chg_runs, 0, sizeof(uint32_t) * (size_t)words * runs, s)) !=
          cudaSuccess)
    return set_err("hb_union_step_runs memset", e);
  if (n_disc < 0 || n_disc > kMaxDisc || (n_disc > 0 && (!disc || !disc_scale)))
    return set_err_msg("hb_union_step_runs: bad discount arguments (at most 8 fused)");
  EstConst ec{alpha_p2, lc_cut, lc_table, disc, disc_stride, n_disc, disc_div, {0, 0, 0, 0, 0, 0, 0, 0}};
  for (int k = 0; k < n_disc; k++) ec.disc_scale[k] = disc_scale[k];
  Peers peers;
  memset(&peers, 0, sizeof(peers));
  const RunArgs ra{chg_runs, words, run_stride};
  const double tf = (double)t;
  if (int er = set_check_dims(n, INT64_MAX, n_items, s)) return er;
  int rc = 0;
#define HB_RUNS_CASE(WB, LR)                                                                   \
  if (wb == WB && log2_runs == LR)                                                             \
    rc = union_step_impl<WB, false, LR>(                                                       \
        lo, hi, offsets, succ, cur, nxt, chg_prev, chg_now, est, sum_dist, sum_recip, tf, ec,  \
        dense, light_max_deg, heavy_nodes, item_first, n_heavy, finish_order, n_mega,          \
        item_node, item_beg, n_items, item_arcs, partial,                                      \
        reinterpret_cast<unsigned long long *>(nch_out),                                       \
        reinterpret_cast<unsigned long long *>(merged_out), hot_rows, active, peers, s, ra);   \
  else
#if HB_G_P64 >= 2
  HB_RUNS_CASE(6, 1)
#endif
#if HB_G_P128 >= 4
  HB_RUNS_CASE(7, 1)
#endif
#if HB_G_P128 >= 2
  HB_RUNS_CASE(7, 2)
#endif
#if HB_G_P256 >= 8
  HB_RUNS_CASE(8, 1)
#endif
#if HB_G_P256 >= 4
  HB_RUNS_CASE(8, 2)
#endif
  HB_RUNS_CASE(5, 1) HB_RUNS_CASE(6, 2)
  HB_RUNS_CASE(7, 3) HB_RUNS_CASE(8, 3) HB_RUNS_CASE(8, 4)
  return set_err_msg("hb_union_step_runs: unsupported (p, runs)");
#undef HB_RUNS_CASE
  if (rc) return rc;
  k_count_bits<<<runs, 256, 0, s>>>(chg_runs, words,
                                    reinterpret_cast<unsigned long long *>(run_nch_out));
  return check_launch("k_count_bits");
}

int hb_pack_registers(int64_t n, int b, int width, const uint8_t *regs, const int32_t *order,
                      uint8_t *out, void *stream) {
  DevGuard dg_((cudaStream_t)stream);
  if (n <= 0) return 0;
  if (b < HB_MIN_B || b > 16 || width < 1 || width > 8 || !regs || !out)
    return set_err_msg("hb_pack_registers: bad arguments");
  const int p = 1 << b;
  k_pack_registers<<<grid_for_threads(n * (p / 8)), kThreads, 0, (cudaStream_t)stream>>>(
      n, p, width, regs, order, out);
  return check_launch("k_pack_registers");
}

int hb_unpack_registers(int64_t n, int b, int width, const uint8_t *packed, const int32_t *order,
                        uint8_t *regs, void *stream) {
  DevGuard dg_((cudaStream_t)stream);
  if (n <= 0) return 0;
  if (b < HB_MIN_B || b > 16 || width < 1 || width > 8 || !packed || !regs)
    return set_err_msg("hb_unpack_registers: bad arguments");
  const int p = 1 << b;
  k_unpack_registers<<<grid_for_threads(n * (p / 8)), kThreads, 0, (cudaStream_t)stream>>>(
      n, p, width, packed, order, regs);
  return check_launch("k_unpack_registers");
}

int hb_finalize(int64_t n, const int32_t *rank, const double *sum_dist, const double *sum_recip,
                const double *coreach, double *closeness, double *harmonic, double *lin,
                void *stream) {
  DevGuard dg_((cudaStream_t)stream);
  if (n <= 0) return 0;
  if ((closeness || lin) && !sum_dist) return set_err_msg("hb_finalize: sum_dist required");
  if (harmonic && !sum_recip) return set_err_msg("hb_finalize: sum_recip required");
  if (lin && !coreach) return set_err_msg("hb_finalize: coreach required");
  k_finalize<<<grid_for_threads(n), kThreads, 0, (cudaStream_t)stream>>>(
      n, rank, sum_dist, sum_recip, coreach, closeness, harmonic, lin);
  return check_launch("k_finalize");
}

int hb_packed_row_bytes(int b) { return packed_row_bytes(1 << b); }

int hb_gather_changed(int64_t lo, int64_t hi, const uint32_t *chg_bits, const uint8_t *rows,
                      int b, int packed, int32_t *ids_out, uint8_t *rows_out,
                      uint64_t *count_out, void *stream) {
  DevGuard dg_((cudaStream_t)stream);
  cudaStream_t s = (cudaStream_t)stream;
  if (!count_out || lo < 0 || (hi > lo && (!chg_bits || !rows || !ids_out || !rows_out)) ||
      b < HB_MIN_B || b > HB_MAX_B)
    return set_err_msg("hb_gather_changed: bad arguments");
  cudaError_t e = cudaMemsetAsync(count_out, 0, sizeof(uint64_t), s);
  if (e != cudaSuccess) return set_err("hb_gather_changed memset", e);
  if (hi <= lo) return 0;
  k_gather_changed<<<grid_for_warps(((hi + 31) >> 5) - (lo >> 5)), kThreads, 0, s>>>(
      lo, hi, chg_bits, rows, 1 << b, packed, ids_out, rows_out,
      reinterpret_cast<unsigned long long *>(count_out));
  return check_launch("k_gather_changed");
}

int hb_scatter_rows(int64_t k, const int32_t *ids, const uint8_t *rows, int b, int packed,
                    uint8_t *dst, uint32_t *chg_bits, void *stream) {
  DevGuard dg_((cudaStream_t)stream);
  if (k <= 0) return 0;
  if (!ids || !rows || !dst || !chg_bits || b < HB_MIN_B || b > HB_MAX_B)
    return set_err_msg("hb_scatter_rows: bad arguments");
  k_scatter_rows<<<grid_for_threads(packed ? k : k * ((1 << b) / 16)), kThreads, 0,
                   (cudaStream_t)stream>>>(k, ids, rows, 1 << b, packed, dst, chg_bits);
  return check_launch("k_scatter_rows");
}

int hb_refresh_rows(int64_t n, int64_t lo, int64_t hi, const uint32_t *bits, const uint8_t *src,
                    uint8_t *dst, int b, void *stream) {
  DevGuard dg_((cudaStream_t)stream);
  if (n <= 0) return 0;
  if (!bits || !src || !dst || lo < 0 || hi > n || lo > hi || b < HB_MIN_B || b > HB_MAX_B)
    return set_err_msg("hb_refresh_rows: bad arguments");
  k_refresh_rows<<<grid_for_warps((n + 31) >> 5), kThreads, 0, (cudaStream_t)stream>>>(
      n, lo, hi, bits, src, dst, 1 << b);
  return check_launch("k_refresh_rows");
}

int hb_sort_rows(int64_t n, const int64_t *offsets, int64_t n_batches,
                 const int64_t *host_batch_rows, const int64_t *host_batch_arcs, int32_t *ids,
                 int32_t *alt, void *temp, uint64_t *temp_bytes, int *result_in_alt,
                 void *stream) {
  DevGuard dg_((cudaStream_t)stream);
  cudaStream_t s = (cudaStream_t)stream;
  if (!host_batch_rows || !host_batch_arcs || !temp_bytes || n_batches < 0)
    return set_err_msg("hb_sort_rows: batch arrays / temp_bytes");
  for (int64_t q = 0; q < n_batches; q++)
    if (host_batch_rows[q + 1] < host_batch_rows[q] ||
        host_batch_arcs[q + 1] - host_batch_arcs[q] >= ((int64_t)1 << 31))
      return set_err_msg("hb_sort_rows: a batch must hold < 2^31 arcs");
  size_t need = 0;
  for (int64_t q = 0; q < n_batches; q++) {       // temp size: max over batches
    const int64_t r0 = host_batch_rows[q], r1 = host_batch_rows[q + 1];
    const int64_t a0 = host_batch_arcs[q], items = host_batch_arcs[q + 1] - a0;
    if (r1 == r0) continue;
    cub::DoubleBuffer<int32_t> keys(ids + a0, alt + a0);
    OffIt beg(offsets + r0, ShiftOff{a0}), end(offsets + r0 + 1, ShiftOff{a0});
    size_t bytes = 0;
    cudaError_t e = cub::DeviceSegmentedSort::SortKeys(nullptr, bytes, keys, (int)items,
                                                       (int)(r1 - r0), beg, end, s);
    if (e != cudaSuccess) return set_err("hb_sort_rows (size)", e);
    need = bytes > need ? bytes : need;
  }
  if (!temp) {                                     // size query
    *temp_bytes = need;
    return 0;
  }
  if (*temp_bytes < need) return set_err_msg("hb_sort_rows: temp buffer too small");
  for (int64_t q = 0; q < n_batches; q++) {
    const int64_t r0 = host_batch_rows[q], r1 = host_batch_rows[q + 1];
    const int64_t a0 = host_batch_arcs[q], items = host_batch_arcs[q + 1] - a0;
    if (r1 == r0) continue;
    cub::DoubleBuffer<int32_t> keys(ids + a0, alt + a0);
    OffIt beg(offsets + r0, ShiftOff{a0}), end(offsets + r0 + 1, ShiftOff{a0});
    size_t bytes = need;
    cudaError_t e = cub::DeviceSegmentedSort::SortKeys(temp, bytes, keys, (int)items,
                                                       (int)(r1 - r0), beg, end, s);
    if (e != cudaSuccess) return set_err("hb_sort_rows", e);
    if (keys.Current() != ids + a0) {              // keep the result in `ids`
      e = cudaMemcpyAsync(ids + a0, alt + a0, sizeof(int32_t) * (size_t)items,
                          cudaMemcpyDeviceToDevice, s);
      if (e != cudaSuccess) return set_err("hb_sort_rows copy", e);
    }
  }
  if (result_in_alt) *result_in_alt = 0;
  return check_launch("hb_sort_rows");
}

int hb_exact_seed(int64_t n, int64_t row_stride, uint8_t *bits, double *est,
                  const int64_t *weights, void *stream) {
  DevGuard dg_((cudaStream_t)stream);
  if (n <= 0) return 0;
  if (row_stride % 16 || row_stride * 8 < n) return set_err_msg("hb_exact_seed: bad row_stride");
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e = cudaMemsetAsync(bits, 0, (size_t)n * (size_t)row_stride, s);
  if (e != cudaSuccess) return set_err("hb_exact_seed memset", e);
  k_exact_seed<<<grid_for_threads(n), kThreads, 0, s>>>(n, row_stride, bits, est, weights);
  return check_launch("k_exact_seed");
}

int hb_exact_union_step(int64_t n, const int64_t *offsets, const int32_t *succ,
                        const uint8_t *cur, uint8_t *nxt, int64_t row_stride,
                        const uint32_t *chg_prev, uint32_t *chg_now, double *est,
                        double *sum_dist, double *sum_recip, int64_t t, int dense,
                        const int64_t *weights, double *disc, int64_t disc_stride, int n_disc,
                        const double *disc_scale, int disc_div, uint64_t *nch_out,
                        uint64_t *merged_out, void *stream) {
  DevGuard dg_((cudaStream_t)stream);
  cudaStream_t s = (cudaStream_t)stream;
  if (n < 0 || t < 1 || !nch_out || row_stride % 16)
    return set_err_msg("hb_exact_union_step: bad arguments");
  if (n_disc < 0 || n_disc > kMaxDisc || (n_disc > 0 && (!disc || !disc_scale)))
    return set_err_msg("hb_exact_union_step: bad discount arguments (at most 8 fused)");
  EstConst ec{0.0, 0.0, nullptr, disc, disc_stride, n_disc, disc_div, {0, 0, 0, 0, 0, 0, 0, 0}};
  for (int k = 0; k < n_disc; k++) ec.disc_scale[k] = disc_scale[k];
  cudaError_t e = cudaMemsetAsync(nch_out, 0, sizeof(uint64_t), s);
  if (e == cudaSuccess && merged_out) e = cudaMemsetAsync(merged_out, 0, sizeof(uint64_t), s);
  if (e == cudaSuccess && n > 0)
    e = cudaMemsetAsync(chg_now, 0, sizeof(uint32_t) * (size_t)((n + 31) / 32), s);
  if (e != cudaSuccess) return set_err("hb_exact_union_step memset", e);
  if (n == 0) return 0;
  k_exact_union<<<grid_for_warps(n), kThreads, 0, s>>>(
      n, offsets, succ, cur, nxt, row_stride, chg_prev, chg_now, est, sum_dist, sum_recip,
      (double)t, dense, weights, ec, reinterpret_cast<unsigned long long *>(nch_out),
      reinterpret_cast<unsigned long long *>(merged_out));
  return check_launch("k_exact_union");
}

int hb_mark_active(int64_t n, const int64_t *fwd_offsets, const int32_t *fwd_succ,
                   const uint32_t *chg_prev, uint32_t *active, void *stream) {
  DevGuard dg_((cudaStream_t)stream);
  cudaStream_t s = (cudaStream_t)stream;
  if (n <= 0) return 0;
  if (!fwd_offsets || !fwd_succ || !chg_prev || !active)
    return set_err_msg("hb_mark_active: bad arguments");
  cudaError_t e = cudaMemsetAsync(active, 0, sizeof(uint32_t) * (size_t)((n + 31) / 32), s);
  if (e != cudaSuccess) return set_err("hb_mark_active memset", e);
  k_mark_active<<<grid_for_warps((n + 31) / 32), kThreads, 0, s>>>(n, fwd_offsets, fwd_succ,
                                                                   chg_prev, active);
  return check_launch("k_mark_active");
}

static int mark_pull_impl(int64_t n, const int64_t *offsets, const int32_t *succ,
                          const uint32_t *chg_prev, uint32_t *active, int64_t light_max_deg,
                          const int32_t *item_node, const int64_t *item_beg, int64_t n_items,
                          int64_t item_arcs, const uint32_t *filter, cudaStream_t s,
                          int64_t h0 = -1, int64_t h1 = -1) {
  const size_t smem = filter ? sizeof(uint32_t) * kFilterWords : 0;
  if (filter) {
    const int fb = (int)(sizeof(uint32_t) * kFilterWords);
    if (int e = ensure_smem_attr((const void *)k_mark_pull<true>, fb, "k_mark_pull smem")) return e;
    if (int e = ensure_smem_attr((const void *)k_mark_items<true>, fb, "k_mark_items smem")) return e;
    if (int e = ensure_smem_attr((const void *)k_mark_heavy_flat<true>, fb, "k_mark_heavy_flat smem"))
      return e;
    k_mark_pull<true><<<grid_for_warps((n + 31) / 32), kThreads, smem, s>>>(
        n, offsets, succ, chg_prev, active, light_max_deg, filter);
  } else {
    k_mark_pull<false><<<grid_for_warps((n + 31) / 32), kThreads, 0, s>>>(
        n, offsets, succ, chg_prev, active, light_max_deg, nullptr);
  }
  if (int e = check_launch("k_mark_pull")) return e;
  if (n_items > 0 && h0 >= 0 && h1 > h0) {     // heavy rows contiguous: flat stream
    const unsigned grid = (unsigned)num_sms() * 4;
    if (filter)
      k_mark_heavy_flat<true><<<grid, kThreads, smem, s>>>(offsets, succ, chg_prev, h0, h1,
                                                           active, filter);
    else
      k_mark_heavy_flat<false><<<grid, kThreads, 0, s>>>(offsets, succ, chg_prev, h0, h1,
                                                         active, nullptr);
    return check_launch("k_mark_heavy_flat");
  }
  if (n_items > 0) {
    if (filter)
      k_mark_items<true><<<grid_for_warps(n_items), kThreads, smem, s>>>(
          offsets, succ, chg_prev, item_node, item_beg, n_items, item_arcs, active, filter);
    else
      k_mark_items<false><<<grid_for_warps(n_items), kThreads, 0, s>>>(
          offsets, succ, chg_prev, item_node, item_beg, n_items, item_arcs, active, nullptr);
    return check_launch("k_mark_items");
  }
  return 0;
}

int hb_mark_pull(int64_t n, const int64_t *offsets, const int32_t *succ,
                 const uint32_t *chg_prev, uint32_t *active, int64_t light_max_deg,
                 const int32_t *item_node, const int64_t *item_beg, int64_t n_items,
                 int64_t item_arcs, void *stream) {
  DevGuard dg_((cudaStream_t)stream);
  if (n <= 0) return 0;
  if (!offsets || !chg_prev || !active || (n_items > 0 && (!item_node || !item_beg)))
    return set_err_msg("hb_mark_pull: bad arguments");
  return mark_pull_impl(n, offsets, succ, chg_prev, active, light_max_deg, item_node,
                        item_beg, n_items, item_arcs, nullptr, (cudaStream_t)stream);
}

int hb_mark_pull_filtered(int64_t n, const int64_t *offsets, const int32_t *succ,
                          const uint32_t *chg_prev, uint32_t *active, int64_t light_max_deg,
                          const int32_t *item_node, const int64_t *item_beg, int64_t n_items,
                          int64_t item_arcs, int64_t heavy_lo, int64_t heavy_hi,
                          uint32_t *filter, void *stream) {
  DevGuard dg_((cudaStream_t)stream);
  if (n <= 0) return 0;
  if (!offsets || !chg_prev || !active || (n_items > 0 && (!item_node || !item_beg)) ||
      (heavy_hi > heavy_lo && (heavy_lo < 0 || heavy_hi > n)))
    return set_err_msg("hb_mark_pull_filtered: bad arguments");
  cudaStream_t s = (cudaStream_t)stream;
  if (filter) {
    cudaError_t e = cudaMemsetAsync(filter, 0, sizeof(uint32_t) * kFilterWords, s);
    if (e != cudaSuccess) return set_err("hb_mark_pull_filtered memset", e);
    k_build_filter<<<grid_for_threads((n + 31) / 32), kThreads, 0, s>>>(n, chg_prev, filter);
    if (int er = check_launch("k_build_filter")) return er;
  }
  return mark_pull_impl(n, offsets, succ, chg_prev, active, light_max_deg, item_node,
                        item_beg, n_items, item_arcs, filter, s, heavy_lo, heavy_hi);
}

int64_t hb_change_filter_words(void) { return kFilterWords; }

int hb_forward_csr(int64_t n, const int64_t *offsets, const int32_t *succ, int64_t m,
                   int64_t *fwd_offsets, int64_t *cursor, int32_t *fwd_dst, void *temp,
                   uint64_t *temp_bytes, void *stream) {
  DevGuard dg_((cudaStream_t)stream);
  cudaStream_t s = (cudaStream_t)stream;
  if (!temp_bytes) return set_err_msg("hb_forward_csr: temp_bytes");
  size_t need = 0;
  cudaError_t e = cub::DeviceScan::ExclusiveSum(nullptr, need, fwd_offsets, fwd_offsets,
                                                n + 1, s);
  if (e != cudaSuccess) return set_err("hb_forward_csr scan size", e);
  if (!temp) {
    *temp_bytes = need;
    return 0;
  }
  if (n <= 0) return 0;
  e = cudaMemsetAsync(fwd_offsets, 0, sizeof(int64_t) * (size_t)(n + 1), s);
  if (e != cudaSuccess) return set_err("hb_forward_csr memset", e);
  if (m > 0)
    k_count_src<<<grid_for_threads(m), kThreads, 0, s>>>(
        m, succ, reinterpret_cast<unsigned long long *>(fwd_offsets));
  size_t bytes = *temp_bytes;
  e = cub::DeviceScan::ExclusiveSum(temp, bytes, fwd_offsets, fwd_offsets, n + 1, s);
  if (e != cudaSuccess) return set_err("hb_forward_csr scan", e);
  e = cudaMemcpyAsync(cursor, fwd_offsets, sizeof(int64_t) * (size_t)n,
                      cudaMemcpyDeviceToDevice, s);
  if (e != cudaSuccess) return set_err("hb_forward_csr cursor", e);
  k_scatter_fwd<<<grid_for_warps(n), kThreads, 0, s>>>(
      n, offsets, succ, reinterpret_cast<unsigned long long *>(cursor), fwd_dst);
  return check_launch("hb_forward_csr");
}

int hb_sample_flagged_arcs(int64_t m, const int32_t *succ, const uint32_t *bits,
                           int64_t samples, uint64_t seed, uint64_t *out, void *stream) {
  DevGuard dg_((cudaStream_t)stream);
  if (m < 0 || samples < 0 || !out || (m > 0 && samples > 0 && (!succ || !bits)))
    return set_err_msg("hb_sample_flagged_arcs: bad arguments");
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e = cudaMemsetAsync(out, 0, sizeof(uint64_t), s);
  if (e != cudaSuccess) return set_err("hb_sample_flagged_arcs memset", e);
  if (m == 0 || samples == 0) return 0;
  k_sample_flagged<<<grid_for_threads(samples), kThreads, 0, s>>>(
      m, succ, bits, samples, seed, reinterpret_cast<unsigned long long *>(out));
  return check_launch("k_sample_flagged");
}

int hb_gen_rmat_keys(int scale, int64_t m, uint64_t thr_a, uint64_t thr_ab, uint64_t thr_abc,
                     uint64_t seed, uint64_t *keys, void *stream) {
  DevGuard dg_((cudaStream_t)stream);
  if (scale < 1 || scale > 31 || m < 0) return set_err_msg("hb_gen_rmat_keys: bad scale / m");
  if (m == 0) return 0;
  k_gen_rmat<<<grid_for_threads(m), kThreads, 0, (cudaStream_t)stream>>>(scale, m, thr_a, thr_ab,
                                                                          thr_abc, seed, keys);
  return check_launch("k_gen_rmat");
}

int hb_keys_to_csr(int64_t n, int64_t m, uint64_t *keys, uint64_t *alt, void *temp,
                   uint64_t *temp_bytes, int64_t *m_out, int64_t *offsets, int32_t *succ,
                   void *stream) {
  DevGuard dg_((cudaStream_t)stream);
  cudaStream_t s = (cudaStream_t)stream;
  if (!temp_bytes) return set_err_msg("hb_keys_to_csr: temp_bytes");
  cub::DoubleBuffer<uint64_t> db(keys, alt);
  size_t b_sort = 0, b_uniq = 0;
  cudaError_t e = cub::DeviceRadixSort::SortKeys(nullptr, b_sort, db, m, 0, 64, s);
  if (e != cudaSuccess) return set_err("hb_keys_to_csr sort size", e);
  e = cub::DeviceSelect::Unique(nullptr, b_uniq, keys, alt, m_out, m, s);
  if (e != cudaSuccess) return set_err("hb_keys_to_csr unique size", e);
  const size_t need = (b_sort > b_uniq ? b_sort : b_uniq) + 64;
  if (!temp) {
    *temp_bytes = need;
    return 0;
  }
  if (*temp_bytes < need) return set_err_msg("hb_keys_to_csr: temp buffer too small");
  // temp layout: [int64 counters (64 B)] [cub scratch]
  int64_t *cnt = reinterpret_cast<int64_t *>(temp);
  void *scratch = reinterpret_cast<char *>(temp) + 64;
  size_t bytes = need - 64;
  e = cub::DeviceRadixSort::SortKeys(scratch, bytes, db, m, 0, 64, s);
  if (e != cudaSuccess) return set_err("hb_keys_to_csr sort", e);
  uint64_t *sorted = db.Current(), *other = db.Alternate();
  bytes = need - 64;
  e = cub::DeviceSelect::Unique(scratch, bytes, sorted, other, cnt, m, s);
  if (e != cudaSuccess) return set_err("hb_keys_to_csr unique", e);
  k_count_valid<<<1, 1, 0, s>>>(other, cnt, cnt + 1);
  int64_t mu = 0;
  e = cudaMemcpyAsync(&mu, cnt + 1, sizeof(int64_t), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return set_err("hb_keys_to_csr count", e);
  k_keys_to_csr<<<grid_for_threads(mu + 1), kThreads, 0, s>>>(n, mu, other, offsets, succ);
  *m_out = mu;
  return check_launch("k_keys_to_csr");
}

// ------------------------------------------------------------------ schedule setup
// Node order, relabelled offsets and heavy-node work items of schedule.py, on the device.
struct RankBounds {
  int64_t b[kMaxPeers + 2];
  int world;
};
__device__ __forceinline__ int owner_rank(const RankBounds &rb, int64_t v) {
  int r = 0;
  while (r + 1 < rb.world && v >= rb.b[r + 1]) r++;
  return r;
}
// Sort window of the `window` order: HB_WINDOW_MULT chunk windows of the light kernel
// (env override for sweeps).
#ifndef HB_WINDOW_MULT
#define HB_WINDOW_MULT 8
#endif
int64_t sort_window(int b) {
  static const int mult = [] {
    const char *e = getenv("HB_WINDOW_MULT");
    const int m = e ? atoi(e) : HB_WINDOW_MULT;
    return m > 0 ? m : 1;
  }();
  return hb_light_window(b) * mult;
}
// key per node: order 1 (degree) 0xFFFFFFFF - in-degree, so an ascending stable sort is by
// descending in-degree; order 2 (window) the same in the low 32 bits under the global index
// of the node's light-kernel chunk window (rank r, window w of its range) in the high 32
__global__ void k_order_keys(int64_t n, const int64_t *__restrict__ off, int order, int64_t win,
                             int64_t npw, RankBounds rb, uint64_t *__restrict__ keys,
                             int32_t *__restrict__ vals) {
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t dk = 0xFFFFFFFFull - (uint64_t)(__ldg(off + v + 1) - __ldg(off + v));
    uint64_t key = dk;
    if (order == 2) {
      const int r = owner_rank(rb, v);
      const int64_t lo_al = rb.b[r] / npw * npw;
      const uint64_t g = (uint64_t)r * (uint64_t)(n / win + 2) + (uint64_t)((v - lo_al) / win);
      key |= g << 32;
    }
    keys[v] = key;
    vals[v] = (int32_t)v;
  }
}
// sorted position j -> internal id (degree order dealt round-robin over the ranks: ranking
// position j goes to rank j % W, slot j / W of its range); perm, rank, permuted degrees
__global__ void k_order_finish(int64_t n, const int32_t *__restrict__ sorted, int deal,
                               RankBounds rb, const int64_t *__restrict__ off,
                               int32_t *__restrict__ perm, int32_t *__restrict__ rank,
                               int64_t *__restrict__ new_deg) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n;
       j += (int64_t)gridDim.x * blockDim.x) {
    const int32_t v = __ldg(sorted + j);
    const int64_t pos = deal ? rb.b[j % rb.world] + j / rb.world : j;
    perm[pos] = v;
    rank[v] = (int32_t)pos;
    new_deg[pos] = __ldg(off + v + 1) - __ldg(off + v);
  }
}
__global__ void k_degree_max(int64_t n, const int64_t *__restrict__ off,
                             unsigned long long *__restrict__ out) {
  int64_t mx = 0;
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x)
    mx = max(mx, __ldg(off + v + 1) - __ldg(off + v));
  mx = (int64_t)__reduce_max_sync(0xffffffffu, (unsigned)mx);
  if ((threadIdx.x & 31) == 0 && mx) atomicMax(out, (unsigned long long)mx);
}
// heavy rows of rows [lo, lo + nrows): flags and counts per row for the scans
__global__ void k_heavy_flags(int64_t nrows, const int64_t *__restrict__ row_off,
                              int64_t light_max_deg, int64_t item_arcs, int64_t mega_items,
                              int64_t *__restrict__ hflag, int64_t *__restrict__ icnt,
                              int64_t *__restrict__ mflag, unsigned long long *__restrict__ nonzero) {
  uint32_t nz = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nrows;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t d = __ldg(row_off + i + 1) - __ldg(row_off + i);
    const bool h = d > light_max_deg;
    const int64_t c = h ? (d + item_arcs - 1) / item_arcs : 0;
    hflag[i] = h;
    icnt[i] = c;
    mflag[i] = c > mega_items;
    nz += d > 0;
  }
  nz = __reduce_add_sync(0xffffffffu, nz);
  if ((threadIdx.x & 31) == 0 && nz) atomicAdd(nonzero, (unsigned long long)nz);
}
__global__ void k_heavy_fill(int64_t nrows, int64_t lo, const int64_t *__restrict__ row_off,
                             int64_t item_arcs, const int64_t *__restrict__ hflag,
                             const int64_t *__restrict__ icnt, const int64_t *__restrict__ mflag,
                             const int64_t *__restrict__ hidx, const int64_t *__restrict__ isum,
                             const int64_t *__restrict__ midx, int64_t n_heavy, int64_t n_items,
                             int64_t n_mega, int32_t *__restrict__ heavy,
                             int32_t *__restrict__ item_first, int32_t *__restrict__ item_node,
                             int64_t *__restrict__ item_beg, int32_t *__restrict__ finish_order) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nrows;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (i == 0) item_first[n_heavy] = (int32_t)n_items;
    if (!hflag[i]) continue;
    const int64_t j = hidx[i], f = isum[i], c = icnt[i], b0 = __ldg(row_off + i);
    heavy[j] = (int32_t)(lo + i);
    item_first[j] = (int32_t)f;
    for (int64_t k = 0; k < c; k++) {
      item_node[f + k] = (int32_t)(lo + i);
      item_beg[f + k] = b0 + k * item_arcs;
    }
    // mega nodes first (in heavy order), then the others
    finish_order[mflag[i] ? midx[i] : n_mega + (j - midx[i])] = (int32_t)j;
  }
}
__global__ void k_heavy_totals(int64_t nrows, const int64_t *__restrict__ hflag,
                               const int64_t *__restrict__ icnt, const int64_t *__restrict__ mflag,
                               const int64_t *__restrict__ hidx, const int64_t *__restrict__ isum,
                               const int64_t *__restrict__ midx, int64_t *__restrict__ out) {
  const int64_t l = nrows - 1;
  out[0] = nrows ? hidx[l] + hflag[l] : 0;
  out[1] = nrows ? isum[l] + icnt[l] : 0;
  out[2] = nrows ? midx[l] + mflag[l] : 0;
}

static size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

int hb_max_degree(int64_t n, const int64_t *offsets, uint64_t *scratch, int64_t *out,
                  void *stream) {
  DevGuard dg_((cudaStream_t)stream);
  cudaStream_t s = (cudaStream_t)stream;
  if (!out || !scratch || n < 0 || (n > 0 && !offsets))
    return set_err_msg("hb_max_degree: bad arguments");
  *out = 0;
  if (n == 0) return 0;
  unsigned long long *d = reinterpret_cast<unsigned long long *>(scratch);
  cudaError_t e = cudaMemsetAsync(d, 0, sizeof(*d), s);
  if (e != cudaSuccess) return set_err("hb_max_degree memset", e);
  k_degree_max<<<grid_for_threads(n), kThreads, 0, s>>>(n, offsets, d);
  unsigned long long h = 0;
  e = cudaMemcpyAsync(&h, d, sizeof(h), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return set_err("hb_max_degree", e);
  *out = (int64_t)h;
  return 0;
}

int hb_schedule_order(int64_t n, const int64_t *offsets, int order, int b, int world,
                      const int64_t *bounds, int32_t *perm, int32_t *rank,
                      int64_t *new_offsets, void *temp, uint64_t *temp_bytes, void *stream) {
  DevGuard dg_((cudaStream_t)stream);
  cudaStream_t s = (cudaStream_t)stream;
  if (!temp_bytes || (order != 1 && order != 2) || world < 1 || world > kMaxPeers + 1 ||
      b < HB_MIN_B || b > HB_MAX_B || n < 0 || n > INT32_MAX || !bounds)
    return set_err_msg("hb_schedule_order: bad arguments");
  const int end_bit = order == 1 ? 32 : 64;
  size_t b_sort = 0, b_scan = 0;
  cub::DoubleBuffer<uint64_t> dk(nullptr, nullptr);
  cub::DoubleBuffer<int32_t> dv(nullptr, nullptr);
  cudaError_t e = cub::DeviceRadixSort::SortPairs(nullptr, b_sort, dk, dv, (int)n, 0, end_bit, s);
  if (e == cudaSuccess)
    e = cub::DeviceScan::InclusiveSum(nullptr, b_scan, (int64_t *)nullptr, (int64_t *)nullptr,
                                      (int)n, s);
  if (e != cudaSuccess) return set_err("hb_schedule_order size", e);
  const size_t k8 = align256(8 * (size_t)n), v4 = align256(4 * (size_t)n);
  const size_t need = 2 * k8 + 2 * v4 + std::max(b_sort, b_scan) + 256;
  if (!temp) {
    *temp_bytes = need;
    return 0;
  }
  if (*temp_bytes < need) return set_err_msg("hb_schedule_order: temp buffer too small");
  if (n == 0) return cudaMemsetAsync(new_offsets, 0, 8, s) == cudaSuccess ? 0 : set_err_msg("memset");
  if (!offsets || !perm || !rank || !new_offsets) return set_err_msg("hb_schedule_order: null array");
  char *t = reinterpret_cast<char *>(temp);
  uint64_t *k0 = reinterpret_cast<uint64_t *>(t), *k1 = reinterpret_cast<uint64_t *>(t + k8);
  int32_t *v0 = reinterpret_cast<int32_t *>(t + 2 * k8);
  int32_t *v1 = reinterpret_cast<int32_t *>(t + 2 * k8 + v4);
  void *scratch = t + 2 * k8 + 2 * v4;
  RankBounds rb;
  memset(&rb, 0, sizeof(rb));
  rb.world = world;
  for (int r = 0; r <= world; r++) rb.b[r] = bounds[r];
  k_order_keys<<<grid_for_threads(n), kThreads, 0, s>>>(n, offsets, order, sort_window(b),
                                                        hb_light_npw(b), rb, k0, v0);
  if (int er = check_launch("k_order_keys")) return er;
  cub::DoubleBuffer<uint64_t> keys(k0, k1);
  cub::DoubleBuffer<int32_t> vals(v0, v1);
  size_t bytes = need - 2 * k8 - 2 * v4;
  e = cub::DeviceRadixSort::SortPairs(scratch, bytes, keys, vals, (int)n, 0, end_bit, s);
  if (e != cudaSuccess) return set_err("hb_schedule_order sort", e);
  int64_t *new_deg = reinterpret_cast<int64_t *>(keys.Alternate());   // free after the sort
  k_order_finish<<<grid_for_threads(n), kThreads, 0, s>>>(n, vals.Current(),
                                                          order == 1 && world > 1, rb, offsets,
                                                          perm, rank, new_deg);
  if (int er = check_launch("k_order_finish")) return er;
  if ((e = cudaMemsetAsync(new_offsets, 0, 8, s)) != cudaSuccess)
    return set_err("hb_schedule_order memset", e);
  bytes = need - 2 * k8 - 2 * v4;
  e = cub::DeviceScan::InclusiveSum(scratch, bytes, new_deg, new_offsets + 1, (int)n, s);
  if (e != cudaSuccess) return set_err("hb_schedule_order scan", e);
  return 0;
}

int hb_heavy_items(int64_t nrows, int64_t lo, const int64_t *row_offsets, int64_t light_max_deg,
                   int64_t item_arcs, int64_t mega_items, int32_t *heavy, int32_t *item_first,
                   int32_t *item_node, int64_t *item_beg, int32_t *finish_order,
                   int64_t *counts, void *temp, uint64_t *temp_bytes, void *stream) {
  DevGuard dg_((cudaStream_t)stream);
  cudaStream_t s = (cudaStream_t)stream;
  if (!temp_bytes || nrows < 0 || nrows > INT32_MAX || item_arcs < 1)
    return set_err_msg("hb_heavy_items: bad arguments");
  size_t b_scan = 0;
  cudaError_t e = cub::DeviceScan::ExclusiveSum(nullptr, b_scan, (int64_t *)nullptr,
                                                (int64_t *)nullptr, (int)std::max<int64_t>(nrows, 1), s);
  if (e != cudaSuccess) return set_err("hb_heavy_items size", e);
  const size_t a8 = align256(8 * (size_t)std::max<int64_t>(nrows, 1));
  const size_t need = 6 * a8 + 256 + b_scan;
  if (!temp) {
    *temp_bytes = need;
    return 0;
  }
  if (*temp_bytes < need) return set_err_msg("hb_heavy_items: temp buffer too small");
  if (!counts) return set_err_msg("hb_heavy_items: counts");
  char *t = reinterpret_cast<char *>(temp);
  int64_t *hflag = (int64_t *)t, *icnt = (int64_t *)(t + a8), *mflag = (int64_t *)(t + 2 * a8);
  int64_t *hidx = (int64_t *)(t + 3 * a8), *isum = (int64_t *)(t + 4 * a8), *midx = (int64_t *)(t + 5 * a8);
  int64_t *dtot = (int64_t *)(t + 6 * a8);              // n_heavy, n_items, n_mega, nonzero
  void *scratch = t + 6 * a8 + 256;
  if ((e = cudaMemsetAsync(dtot, 0, 32, s)) != cudaSuccess) return set_err("hb_heavy_items memset", e);
  if (nrows > 0) {
    if (!row_offsets) return set_err_msg("hb_heavy_items: null offsets");
    k_heavy_flags<<<grid_for_threads(nrows), kThreads, 0, s>>>(
        nrows, row_offsets, light_max_deg, item_arcs, mega_items, hflag, icnt, mflag,
        reinterpret_cast<unsigned long long *>(dtot + 3));
    size_t bytes = b_scan;
    e = cub::DeviceScan::ExclusiveSum(scratch, bytes, hflag, hidx, (int)nrows, s);
    if (e == cudaSuccess) { bytes = b_scan; e = cub::DeviceScan::ExclusiveSum(scratch, bytes, icnt, isum, (int)nrows, s); }
    if (e == cudaSuccess) { bytes = b_scan; e = cub::DeviceScan::ExclusiveSum(scratch, bytes, mflag, midx, (int)nrows, s); }
    if (e != cudaSuccess) return set_err("hb_heavy_items scan", e);
    k_heavy_totals<<<1, 1, 0, s>>>(nrows, hflag, icnt, mflag, hidx, isum, midx, dtot);
  }
  if ((e = cudaMemcpyAsync(counts, dtot, 32, cudaMemcpyDeviceToHost, s)) == cudaSuccess)
    e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return set_err("hb_heavy_items counts", e);
  if (!heavy) return 0;                                  // count phase
  if (counts[1] > INT32_MAX) return set_err_msg("hb_heavy_items: more than 2^31 work items");
  if (!item_first) return set_err_msg("hb_heavy_items: null outputs");
  if (counts[0] == 0) {
    return cudaMemsetAsync(item_first, 0, 4, s) == cudaSuccess ? 0 : set_err_msg("memset");
  }
  if (!item_node || !item_beg || !finish_order) return set_err_msg("hb_heavy_items: null outputs");
  k_heavy_fill<<<grid_for_threads(nrows), kThreads, 0, s>>>(
      nrows, lo, row_offsets, item_arcs, hflag, icnt, mflag, hidx, isum, midx, counts[0],
      counts[1], counts[2], heavy, item_first, item_node, item_beg, finish_order);
  return check_launch("k_heavy_fill");
}

int hb_gen_degrees(int kind, int64_t n, uint64_t seed, const double *cdf, int64_t cdf_len,
                   int64_t kmin, int64_t *deg, void *stream) {
  DevGuard dg_((cudaStream_t)stream);
  if (n <= 0) return 0;
  if ((kind != GG_ER && kind != GG_DISC && kind != GG_WEB) || !cdf || cdf_len < 1 || !deg)
    return set_err_msg("hb_gen_degrees: bad arguments");
  k_gen_degree<<<grid_for_threads(n), kThreads, 0, (cudaStream_t)stream>>>(kind, n, seed, cdf,
                                                                           cdf_len, kmin, deg);
  return check_launch("k_gen_degree");
}

int hb_gen_blocks(int64_t n, int64_t giant, double geo_p, uint64_t seed, int64_t *size,
                  int64_t *start, int64_t *lo, int64_t *hi, void *temp, uint64_t *temp_bytes,
                  void *stream) {
  DevGuard dg_((cudaStream_t)stream);
  cudaStream_t s = (cudaStream_t)stream;
  if (!temp_bytes) return set_err_msg("hb_gen_blocks: temp_bytes");
  const int64_t nb = n > giant ? n - giant : 0;
  size_t need = 0;
  cudaError_t e = cub::DeviceScan::ExclusiveSum(nullptr, need, size, start, nb > 0 ? nb : 1, s);
  if (e != cudaSuccess) return set_err("hb_gen_blocks scan size", e);
  if (!temp) {
    *temp_bytes = need;
    return 0;
  }
  if (n <= 0) return 0;
  if (!lo || !hi || giant < 0 || !(geo_p > 0.0) || (nb > 0 && (!size || !start)))
    return set_err_msg("hb_gen_blocks: bad arguments");
  if (nb > 0) {
    k_gen_block_sizes<<<grid_for_threads(nb), kThreads, 0, s>>>(nb, seed, geo_p, size);
    size_t bytes = *temp_bytes;
    e = cub::DeviceScan::ExclusiveSum(temp, bytes, size, start, nb, s);
    if (e != cudaSuccess) return set_err("hb_gen_blocks scan", e);
  }
  const int64_t g = giant < n ? giant : n;
  k_gen_block_bounds<<<grid_for_threads(nb > g ? nb : g), kThreads, 0, s>>>(n, g, nb, start,
                                                                             size, lo, hi);
  return check_launch("k_gen_block_bounds");
}

int hb_gen_arc_keys(int kind, int64_t n, uint64_t seed, const int64_t *offsets,
                    const int64_t *block_lo, const int64_t *block_hi, double p_local,
                    int64_t window, uint64_t *keys, void *stream) {
  DevGuard dg_((cudaStream_t)stream);
  if (n <= 0) return 0;
  if ((kind != GG_ER && kind != GG_DISC && kind != GG_WEB) || !offsets || !keys ||
      (kind == GG_DISC && (!block_lo || !block_hi)) || (kind == GG_WEB && window < 1))
    return set_err_msg("hb_gen_arc_keys: bad arguments");
  k_gen_arcs<<<grid_for_warps(n), kThreads, 0, (cudaStream_t)stream>>>(
      kind, n, seed, offsets, block_lo, block_hi, p_local, window, keys);
  return check_launch("k_gen_arcs");
}

int hb_transpose_csr(int64_t n, int64_t m, const int64_t *offsets, const int32_t *succ,
                     uint64_t *keys, uint64_t *alt, void *temp, uint64_t *temp_bytes,
                     int64_t *out_offsets, int32_t *out_succ, void *stream) {
  DevGuard dg_((cudaStream_t)stream);
  cudaStream_t s = (cudaStream_t)stream;
  if (!temp_bytes || n < 0 || m < 0) return set_err_msg("hb_transpose_csr: bad arguments");
  int bits = 1;
  while (bits < 32 && ((int64_t)1 << bits) < n) bits++;
  cub::DoubleBuffer<uint64_t> db(keys, alt);
  size_t need = 0;
  cudaError_t e = cub::DeviceRadixSort::SortKeys(nullptr, need, db, m > 0 ? m : 1, 0, 32 + bits, s);
  if (e != cudaSuccess) return set_err("hb_transpose_csr sort size", e);
  if (!temp) {
    *temp_bytes = need;
    return 0;
  }
  if (!out_offsets || (m > 0 && (!offsets || !succ || !keys || !alt || !out_succ)))
    return set_err_msg("hb_transpose_csr: bad arguments");
  if (m == 0) {
    e = cudaMemsetAsync(out_offsets, 0, sizeof(int64_t) * (size_t)(n + 1), s);
    return e == cudaSuccess ? 0 : set_err("hb_transpose_csr memset", e);
  }
  k_transpose_keys<<<grid_for_warps(n), kThreads, 0, s>>>(n, offsets, succ, keys);
  size_t bytes = *temp_bytes;
  e = cub::DeviceRadixSort::SortKeys(temp, bytes, db, m, 0, 32 + bits, s);
  if (e != cudaSuccess) return set_err("hb_transpose_csr sort", e);
  k_keys_to_csr<<<grid_for_threads(m + 1), kThreads, 0, s>>>(n, m, db.Current(), out_offsets,
                                                             out_succ);
  return check_launch("k_keys_to_csr");
}

int hb_relabel_csr(int64_t n, const int64_t *old_offsets, const int32_t *old_succ,
                   const int32_t *perm, const int32_t *rank, const int64_t *new_offsets,
                   int32_t *new_succ, void *stream) {
  DevGuard dg_((cudaStream_t)stream);
  if (n <= 0) return 0;
  if (!old_offsets || !perm || !rank || !new_offsets)   // succ arrays may be empty (NULL)
    return set_err_msg("hb_relabel_csr: bad arguments");
  k_relabel<<<grid_for_warps(n), kThreads, 0, (cudaStream_t)stream>>>(
      0, n, old_offsets, old_succ, perm, rank, new_offsets, new_succ);
  return check_launch("k_relabel");
}

int hb_relabel_csr_rows(int64_t n, int64_t r0, int64_t r1, const int64_t *old_offsets,
                        const int32_t *old_succ, const int32_t *perm, const int32_t *rank,
                        const int64_t *new_offsets, int32_t *new_succ, void *stream) {
  DevGuard dg_((cudaStream_t)stream);
  if (r0 < 0 || r1 > n || r0 > r1) return set_err_msg("hb_relabel_csr_rows: bad row range");
  if (r1 == r0) return 0;
  if (!old_offsets || !perm || !rank || !new_offsets)
    return set_err_msg("hb_relabel_csr_rows: bad arguments");
  k_relabel<<<grid_for_warps(r1 - r0), kThreads, 0, (cudaStream_t)stream>>>(
      r0, r1, old_offsets, old_succ, perm, rank, new_offsets, new_succ);
  return check_launch("k_relabel");
}

int hb_relabel_csr_src_rows(int64_t n, int64_t o0, int64_t o1, const int64_t *old_offsets,
                            const int32_t *old_succ, const int32_t *rank,
                            const int64_t *new_offsets, int32_t *new_succ, void *stream) {
  DevGuard dg_((cudaStream_t)stream);
  if (o0 < 0 || o1 > n || o0 > o1) return set_err_msg("hb_relabel_csr_src_rows: bad row range");
  if (o1 == o0) return 0;
  if (!old_offsets || !rank || !new_offsets)
    return set_err_msg("hb_relabel_csr_src_rows: bad arguments");
  k_relabel_src<<<grid_for_warps(o1 - o0), kThreads, 0, (cudaStream_t)stream>>>(
      o0, o1, old_offsets, old_succ, rank, new_offsets, new_succ);
  return check_launch("k_relabel_src");
}

int hb_map_ids(int64_t m, const int32_t *ids, const int32_t *rank, int32_t *out, void *stream) {
  DevGuard dg_((cudaStream_t)stream);
  if (m <= 0) return 0;
  if (!ids || !rank || !out) return set_err_msg("hb_map_ids: bad arguments");
  k_map_ids<<<grid_for_threads(m), kThreads, 0, (cudaStream_t)stream>>>(m, ids, rank, out);
  return check_launch("k_map_ids");
}

int hb_hash_items(int64_t n, const uint64_t *items, const uint64_t *replicas, uint64_t seed,
                  uint64_t *out, void *stream) {
  DevGuard dg_((cudaStream_t)stream);
  if (n <= 0) return 0;
  if (!items || !replicas || !out) return set_err_msg("hb_hash_items: bad arguments");
  k_hash<<<grid_for_threads(n), kThreads, 0, (cudaStream_t)stream>>>(n, items, replicas, seed,
                                                                      out);
  return check_launch("k_hash");
}

}  // extern "C"
